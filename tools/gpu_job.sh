# ad-hoc GPU job (overwritten per experiment; the committed copy is the last one run)
python -c "import __graft_entry__ as e; e.build()" > gpurun_out/build.log 2>&1
timeout 1800 python -m pytest tests -q -m gpu -x --timeout 600 > gpurun_out/pytest.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest.log
for v in old new old new; do
  if [ $v = old ]; then export ATOS_LIB=paper_2112_00132_b200/variants/libatos_old.so; else unset ATOS_LIB; fi
  echo "== $v"; timeout 600 python tools/e2e_breakdown.py 2>&1 | tail -1
done
unset ATOS_LIB
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo bench_rc=$?; tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['pagerank']['kernel_ms'], d['pagerank']['ms'], d['bfs']['kernel_ms'], d['bfs']['ms'], d['bfs']['gteps'], d['e2e']['value'])"
