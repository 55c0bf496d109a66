# ad-hoc GPU job (overwritten per experiment; the committed copy is the last one run)
python -c "import __graft_entry__ as e; e.build()" > gpurun_out/build.log 2>&1
VD=paper_2112_00132_b200/variants
ATOS_LIB=$VD/libatos_nodone.so timeout 120 python tests/harness/quick_check.py > gpurun_out/qc.log 2>&1; echo "nodone rc=$?" >> gpurun_out/qc.log; tail -2 gpurun_out/qc.log
timeout 300 python -m pytest tests/test_gpu_parity.py -q -k "serial_order" > gpurun_out/pt.log 2>&1; echo pt=$?; tail -2 gpurun_out/pt.log
B='{"t256": {"cta_threads": 256}, "nofilter": {"cta_threads": 256, "bfs_filter": false}, "f64": {"cta_threads": 256, "fetch_size": 64}, "f256": {"cta_threads": 256, "fetch_size": 256}, "t512": {"cta_threads": 512}}'
for rep in 1 2 3; do
for lib in product nodone; do
  if [ $lib = product ]; then L=""; else L=$VD/libatos_$lib.so; fi
  echo "== $lib rep $rep" >> gpurun_out/bfsv.md
  ATOS_LIB=$L timeout 200 python tests/harness/pr_variants.py --app bfs --runs 5 --no-oracle --variants "$B" >> gpurun_out/bfsv.md 2>&1
done; done
ATOS_LIB=$VD/libatos_nodone.so timeout 300 python tools/grid_latency.py --runs 2 --cells cta:256:128,cta:128:16 >> gpurun_out/bfsv.md 2>&1
