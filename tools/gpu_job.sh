# ad-hoc GPU job (overwritten per experiment; the committed copy is the last one run)
python -c "import __graft_entry__ as e; e.build()" > gpurun_out/build.log 2>&1
VD=paper_2112_00132_b200/variants
for v in h128 h256 h2048; do ATOS_LIB=$VD/libatos_$v.so timeout 120 python tests/harness/quick_check.py >> gpurun_out/qc.log 2>&1; echo "$v rc=$?" >> gpurun_out/qc.log; done; tail -3 gpurun_out/qc.log
for rep in 1 2; do
for lib in product h128 h256 h2048; do
  if [ $lib = product ]; then L=""; else L=$VD/libatos_$lib.so; fi
  grep -q "$lib rc=0" gpurun_out/qc.log || [ $lib = product ] || continue
  echo "== $lib rep $rep" >> gpurun_out/hdeg.md
  ATOS_LIB=$L timeout 300 python tests/harness/pr_variants.py --runs 2 $( [ $rep = 1 ] || echo --no-oracle ) --variants '{"hc16": {"cta_threads": 1024}, "hc32": {"cta_threads": 1024, "pr_hub_check": 32}}' >> gpurun_out/hdeg.md 2>&1
done; done
