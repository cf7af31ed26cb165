# Full ncu capture of one k_scan_cnf launch (config 2 emit pass) + launch list of a bench step.
TAG=${TAG:-x}
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_scan_cnf' \
  --launch-skip 2 --launch-count 1 -o gpurun_out/cnf_${TAG} -f \
  python tools/profile_scan.py --iters 4 > gpurun_out/prof_cnf_${TAG}.log 2>&1
tail -n 3 gpurun_out/prof_cnf_${TAG}.log
