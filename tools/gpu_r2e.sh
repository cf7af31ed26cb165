mkdir -p gpurun_out
timeout 300 python tools/time_phases.py --iters 20 > gpurun_out/phases_r2e.log 2>&1; tail -2 gpurun_out/phases_r2e.log
timeout 300 python tools/time_b1.py --n 2000 > gpurun_out/time_b1_r2e.log 2>&1; tail -4 gpurun_out/time_b1_r2e.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_r2e.log 2>&1; tail -6 gpurun_out/pytest_gpu_r2e.log
grep -E "passed|failed" gpurun_out/reference_suite.log | tail -3
