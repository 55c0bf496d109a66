# ad-hoc GPU job (overwritten per experiment; the committed copy is the last one run)
python -c "import __graft_entry__ as e; e.build()" > gpurun_out/build.log 2>&1
timeout 120 python -c "import __graft_entry__ as e; e.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
timeout 1800 python -m pytest tests -q -m gpu --timeout 600 > gpurun_out/pytest.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1; echo bench_rc=$?; tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['pagerank']['kernel_ms'], d['bfs']['kernel_ms'], d['bfs']['gteps'], d['e2e']['value'], d['roofline']['frac'])"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_persistent -c 1 -o gpurun_out/bfs_full6 -f python tools/profile_run.py --app bfs --threads 256 --fetch 128 --iters 1 > gpurun_out/ncu_bfs.log 2>&1; echo ncu_rc=$?
timeout 300 python tools/grid_latency.py --runs 2 --cells cta:256:128,cta:128:16 > gpurun_out/grid_final.md 2>&1; cat gpurun_out/grid_final.md
