# ad-hoc GPU job (overwritten per experiment; the committed copy is the last one run)
python -c "import __graft_entry__ as e; e.build()" > gpurun_out/build.log 2>&1
VD=paper_2112_00132_b200/variants
for v in hint0 slot4; do ATOS_LIB=$VD/libatos_$v.so timeout 120 python tests/harness/quick_check.py >> gpurun_out/qc.log 2>&1; echo "$v rc=$?" >> gpurun_out/qc.log; done; tail -4 gpurun_out/qc.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 300 -k "bfs" > gpurun_out/pt.log 2>&1; echo pt=$?; tail -2 gpurun_out/pt.log
for rep in 1 2 3; do
for lib in product hint0 slot4; do
  if [ $lib = product ]; then L=""; else L=$VD/libatos_$lib.so; fi
  grep -q "$lib rc=0" gpurun_out/qc.log || [ $lib = product ] || continue
  echo "== $lib rep $rep" >> gpurun_out/pop.md
  ATOS_LIB=$L timeout 200 python tests/harness/pr_variants.py --app bfs --runs 5 --no-oracle --variants '{"t256": {"cta_threads": 256}}' >> gpurun_out/pop.md 2>&1
  ATOS_LIB=$L timeout 200 python tests/harness/pr_variants.py --runs 2 --no-oracle --variants '{"pr": {"cta_threads": 1024}}' >> gpurun_out/pop.md 2>&1
done; done
for lib in product hint0 slot4; do
  if [ $lib = product ]; then L=""; else L=$VD/libatos_$lib.so; fi
  echo "== $lib grid" >> gpurun_out/pop.md
  ATOS_LIB=$L timeout 300 python tools/grid_latency.py --runs 2 --cells cta:256:128,cta:128:16 >> gpurun_out/pop.md 2>&1
done
