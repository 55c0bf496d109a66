# ad-hoc GPU job (overwritten per experiment; the committed copy is the last one run)
python -c "import __graft_entry__ as e; e.build()" > gpurun_out/build.log 2>&1
VD=paper_2112_00132_b200/variants
for v in a2n8 a2n6; do ATOS_LIB=$VD/libatos_$v.so timeout 120 python tests/harness/quick_check.py >> gpurun_out/qc.log 2>&1; echo "$v rc=$?" >> gpurun_out/qc.log; done; tail -4 gpurun_out/qc.log
for rep in 1 2; do
for lib in product a2n8 a2n6; do
  if [ $lib = product ]; then L=""; V='{"f128": {"cta_threads": 1024}, "f64": {"cta_threads": 1024, "fetch_size": 64}}'; fi
  if [ $lib = a2n8 ]; then L=$VD/libatos_$lib.so; V='{"f64": {"cta_threads": 1024, "fetch_size": 64}, "f32": {"cta_threads": 1024, "fetch_size": 32}}'; fi
  if [ $lib = a2n6 ]; then L=$VD/libatos_$lib.so; V='{"f96": {"cta_threads": 1024, "fetch_size": 96}, "f64": {"cta_threads": 1024, "fetch_size": 64}}'; fi
  grep -q "$lib rc=0" gpurun_out/qc.log || [ $lib = product ] || continue
  echo "== $lib rep $rep" >> gpurun_out/nbf.md
  ATOS_LIB=$L timeout 300 python tests/harness/pr_variants.py --runs 2 --no-oracle --variants "$V" >> gpurun_out/nbf.md 2>&1
done; done
ATOS_LIB=$VD/libatos_wprof.so timeout 300 python tests/harness/pr_variants.py --runs 1 --no-oracle --variants '{"t1024": {"cta_threads": 1024}}' > gpurun_out/wprof2.md 2>&1
ATOS_LIB=$VD/libatos_wprof.so timeout 300 python tests/harness/pr_variants.py --app bfs --runs 1 --no-oracle --variants '{"t256": {"cta_threads": 256}}' >> gpurun_out/wprof2.md 2>&1
