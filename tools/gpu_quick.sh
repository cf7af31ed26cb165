# Quick GPU check: parity tests, then per-phase timings of the config-2 workload.
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
timeout 300 python tools/time_phases.py --iters 20 > gpurun_out/phases.log 2>&1
cat gpurun_out/pytest_gpu.log gpurun_out/phases.log
