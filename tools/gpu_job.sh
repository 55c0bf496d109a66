# ad-hoc GPU job (overwritten per experiment; the committed copy is the last one run)
python -c "import __graft_entry__ as e; e.build()" > gpurun_out/build.log 2>&1
timeout 120 python -c "import __graft_entry__ as e; e.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
timeout 1800 python -m pytest tests -q -m gpu --timeout 600 > gpurun_out/pytest.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1; echo bench_rc=$?; tail -c 300 gpurun_out/bench.log
timeout 900 python bench.py --impl reference --steps 5 --warmup 2 > gpurun_out/ref.log 2>&1; echo ref_rc=$?; tail -c 600 gpurun_out/ref.log
