timeout 200 python tools/time_phases.py --iters 10 --env FB_EMIT_STAGES=3,2,3,3,2,3 2>&1 | grep emit
