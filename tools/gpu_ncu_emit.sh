# Full ncu capture of one emit-pass launch (the 4th k_scan_tc launch of profile_scan.py).
TAG=${TAG:-x}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_scan_(tc|cnf)' \
  --launch-skip 3 --launch-count 1 -o gpurun_out/emit_${TAG} -f \
  python tools/profile_scan.py --iters 3 > gpurun_out/prof_${TAG}.log 2>&1
tail -n 3 gpurun_out/prof_${TAG}.log
