# ad-hoc GPU job (overwritten per experiment; the committed copy is the last one run)
python -c "import __graft_entry__ as e; e.build()" > gpurun_out/build.log 2>&1
timeout 120 python -c "import __graft_entry__ as e; e.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
timeout 1800 python -m pytest tests -q -m gpu --timeout 600 > gpurun_out/pytest.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo bench_rc=$?; tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['pagerank']['kernel_ms'], d['bfs']['kernel_ms'], d['bfs']['gteps'], d['e2e']['value'], d['roofline']['frac'], d['atomic_ceiling']['frac'])"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo ncu1_rc=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_persistent -c 1 -o gpurun_out/pr_full7 -f python tools/profile_run.py --app pr --threads 1024 --fetch 128 --iters 1 > gpurun_out/ncu_pr.log 2>&1; echo ncu_rc=$?
timeout 900 python bench.py --impl reference --steps 5 --warmup 2 > gpurun_out/ref.log 2>&1; echo ref_rc=$?
