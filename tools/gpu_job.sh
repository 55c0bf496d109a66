# ad-hoc GPU job (overwritten per experiment; the committed copy is the last one run)
python -c "import __graft_entry__ as e; e.build()" > gpurun_out/build.log 2>&1
timeout 600 python tools/e2e_breakdown.py --iters 4 --again 2>&1 | tail -9
