# ad-hoc GPU job (overwritten per experiment; the committed copy is the last one run)
timeout 600 python tools/atomic_trace.py --scale 24 --hub 2048 > gpurun_out/atrace4.md 2>&1; echo at=$?; cat gpurun_out/atrace4.md
