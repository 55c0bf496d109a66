# ad-hoc GPU job (overwritten per experiment; the committed copy is the last one run)
python -c "import __graft_entry__ as e; e.build()" > gpurun_out/build.log 2>&1
timeout 600 python tools/e2e_breakdown.py --iters 4 2>&1 | tail -1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_tag" --csv --log-file gpurun_out/create_new.csv python tools/e2e_breakdown.py --iters 2 > /dev/null 2>&1; echo ncu=$?
timeout 1800 python -m pytest tests -q -m gpu -x --timeout 600 > gpurun_out/pytest.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo bench_rc=$?; tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['pagerank']['kernel_ms'], d['pagerank']['ms'], d['bfs']['kernel_ms'], d['bfs']['ms'], d['bfs']['gteps'], d['e2e'])"
