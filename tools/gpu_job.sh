# ad-hoc GPU job (overwritten per experiment; the committed copy is the last one run)
python -c "import __graft_entry__ as e; e.build()" > gpurun_out/build.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/rcp tools/rc_probe.cu && compute-sanitizer --tool racecheck /tmp/rcp > gpurun_out/rc_probe.log 2>&1
PR_FP64=1 timeout 600 python tools/pr_precision.py h512b >> gpurun_out/prec4.jsonl 2>> gpurun_out/prec4.err
timeout 1500 python -m pytest tests -q -m gpu -k "wraparound or stress or sanitizer or fan_in or trace" > gpurun_out/pytest4.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/pytest4.log
