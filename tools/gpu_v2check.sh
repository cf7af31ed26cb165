# New emit kernel (FB_EMIT_V2=1): small-shape hang probes under the progress watchdog, the GPU
# parity suites, the ablation + one ncu capture, and a timeline trace.
export FB_EMIT_V2=1
for c in "50000 200 1" "400000 24 100" "50000 24 1" "2000000 256 5000"; do
  FB_EMIT_PROGRESS=1 timeout 60 python tools/hang_probe.py $c 2>&1 | tail -4
done
timeout 400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -x -q 2>&1 | tail -3
TAG=${TAG:-v4} bash tools/gpu_emit_ablation.sh
FB_EMIT_TRACE=1 timeout 120 python tools/hang_probe.py 10000000 256 10000 2>&1 | tail -18
