# ad-hoc GPU job (overwritten per experiment; the committed copy is the last one run)
python -c "import __graft_entry__ as e; e.build()" > gpurun_out/build.log 2>&1
VD=paper_2112_00132_b200/variants
timeout 120 python tests/harness/quick_check.py >> gpurun_out/qc.log 2>&1; echo "product rc=$?" >> gpurun_out/qc.log
for v in old512r1 rep4 rep1; do ATOS_LIB=$VD/libatos_$v.so timeout 120 python tests/harness/quick_check.py >> gpurun_out/qc.log 2>&1; echo "$v rc=$?" >> gpurun_out/qc.log; done; grep rc= gpurun_out/qc.log
for rep in 1 2 3; do
for lib in product old512r1 rep4 rep1; do
  if [ $lib = product ]; then L=""; else L=$VD/libatos_$lib.so; fi
  grep -q "$lib rc=0" gpurun_out/qc.log || continue
  echo "== $lib rep $rep" >> gpurun_out/ab.md
  ATOS_LIB=$L timeout 200 python tests/harness/pr_variants.py --runs 2 $( [ $rep = 1 ] || echo --no-oracle ) --variants '{"pr": {"cta_threads": 1024}}' >> gpurun_out/ab.md 2>&1
done; done
timeout 900 python -m pytest tests -q -m gpu -x --timeout 600 -k "pagerank" > gpurun_out/pytest_pr.log 2>&1; echo pt=$?; tail -2 gpurun_out/pytest_pr.log
