# ad-hoc GPU job (overwritten per experiment; the committed copy is the last one run)
python -c "import __graft_entry__ as e; e.build()" > gpurun_out/build.log 2>&1
VD=paper_2112_00132_b200/variants
for v in ch1k ch4k bag2; do ATOS_LIB=$VD/libatos_$v.so timeout 120 python tests/harness/quick_check.py >> gpurun_out/qc.log 2>&1; echo "$v rc=$?" >> gpurun_out/qc.log; done; grep rc= gpurun_out/qc.log
for rep in 1 2 3; do
for lib in product ch1k ch4k bag2; do
  if [ $lib = product ]; then L=""; V='{"t256f128": {"cta_threads": 256}, "t256f64": {"cta_threads": 256, "fetch_size": 64}, "t512f128": {"cta_threads": 512}}'; else L=$VD/libatos_$lib.so; V='{"t256f128": {"cta_threads": 256}, "t512f128": {"cta_threads": 512}}'; fi
  grep -q "$lib rc=0" gpurun_out/qc.log || [ $lib = product ] || continue
  echo "== $lib rep $rep" >> gpurun_out/btune.md
  ATOS_LIB=$L timeout 200 python tests/harness/pr_variants.py --app bfs --runs 5 --no-oracle --variants "$V" >> gpurun_out/btune.md 2>&1
done; done
for lib in product bag2; do
  if [ $lib = product ]; then L=""; else L=$VD/libatos_$lib.so; fi
  echo "== $lib grid" >> gpurun_out/btune.md
  ATOS_LIB=$L timeout 300 python tools/grid_latency.py --runs 2 --cells cta:256:128,cta:128:16,cta:512:32 >> gpurun_out/btune.md 2>&1
done
