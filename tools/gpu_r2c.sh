mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_pack_gpu.py tests/test_reference_suite.py -q -x > gpurun_out/pytest_r2c.log 2>&1; tail -3 gpurun_out/pytest_r2c.log
grep -E "passed|failed" gpurun_out/reference_suite.log | tail -2
TAG=r2c bash tools/gpu_ncu_cnf.sh
bash tools/micro/i8_peak.sh 400000 > gpurun_out/i8_peak_r2c.log 2>&1; cat gpurun_out/i8_peak_r2c.log
