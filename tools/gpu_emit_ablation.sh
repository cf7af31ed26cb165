# Emit-kernel ablation (FB_SCAN_DEBUG switches; results are wrong under them) + one full ncu
# capture of the emit launch. TAG names the output files.
TAG=${TAG:-x}
mkdir -p gpurun_out
timeout 300 python tools/time_phases.py --iters 10 --env FB_SCAN_DEBUG=0,2,4,6 \
  > gpurun_out/abl_${TAG}.log 2>&1
cat gpurun_out/abl_${TAG}.log | grep emit
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_emit_win|k_scan_(tc|cnf)' \
  --launch-skip 3 --launch-count 1 -o gpurun_out/emit_${TAG} -f \
  python tools/profile_scan.py --iters 3 > gpurun_out/prof_${TAG}.log 2>&1
tail -n 2 gpurun_out/prof_${TAG}.log
