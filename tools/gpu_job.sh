# ad-hoc GPU job (overwritten per experiment; the committed copy is the last one run)
python -c "import __graft_entry__ as e; e.build()" > gpurun_out/build.log 2>&1
timeout 1800 python -m pytest tests -q -m gpu -x --timeout 600 > gpurun_out/pytest.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest.log
timeout 600 python tools/e2e_breakdown.py --iters 4 2>&1 | tail -1
ATOS_LIB=paper_2112_00132_b200/variants/libatos_64aa7a1.so timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_ctl.log 2>&1; tail -1 gpurun_out/bench_ctl.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('64aa7a1', d['value'], d['ms_per_step'], d['pagerank']['kernel_ms'], d['pagerank']['ms'], d['bfs']['kernel_ms'], d['bfs']['ms'], d['e2e']['value'])"
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo bench_rc=$?; tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('final', d['value'], d['ms_per_step'], d['pagerank']['kernel_ms'], d['pagerank']['ms'], d['bfs']['kernel_ms'], d['bfs']['ms'], d['e2e']['value'])"
