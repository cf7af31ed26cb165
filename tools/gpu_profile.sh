# One-GPU profiling pass: launch list of bench.py (kernel-filtered) + full capture of the
# CNF emit kernel. Outputs land in gpurun_out/ (scratch); summaries go to profiles/.
set -x
TAG=${TAG:-r1}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'^k_' --csv \
  --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
  > gpurun_out/b_ncu_${TAG}.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_scan_(tc|cnf)' \
  --launch-skip 3 --launch-count 1 -o gpurun_out/emit_${TAG} -f \
  python tools/profile_scan.py --iters 3 > gpurun_out/prof_${TAG}.log 2>&1
tail -n 3 gpurun_out/*_${TAG}.log
