mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_r2b.log 2>&1
tail -5 gpurun_out/pytest_gpu_r2b.log
timeout 300 python tools/time_b1.py --profile > gpurun_out/time_b1_r2b.log 2>&1
timeout 200 python tools/time_b1.py --reference --n 1000 > gpurun_out/time_b1_ref_r2b.log 2>&1
head -3 gpurun_out/time_b1_r2b.log; cat gpurun_out/time_b1_ref_r2b.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_r2b.json 2> gpurun_out/bench_r2b.err
cat gpurun_out/bench_r2b.json; tail -3 gpurun_out/bench_r2b.err
