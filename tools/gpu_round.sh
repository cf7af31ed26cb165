# Round measurement pass on one B200: GPU parity tests, smoke, bench (with CPU baseline),
# reference arm, launch list (kernel-filtered), one full ncu capture of the emit kernel.
TAG=${TAG:-r1}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu_${TAG}.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_${TAG}.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_${TAG}.json 2> gpurun_out/bench_ref_${TAG}.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'^k_' --csv \
  --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
  > gpurun_out/b_ncu_${TAG}.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_scan_cnf' \
  --launch-skip 2 --launch-count 1 -o gpurun_out/emit_${TAG} -f \
  python tools/profile_scan.py --iters 3 > gpurun_out/prof_${TAG}.log 2>&1
tail -n 2 gpurun_out/pytest_gpu_${TAG}.log gpurun_out/smoke_${TAG}.log
cat gpurun_out/bench_${TAG}.json gpurun_out/bench_ref_${TAG}.json
