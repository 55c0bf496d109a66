# ad-hoc GPU job (overwritten per experiment; the committed copy is the last one run)
python -c "import __graft_entry__ as e; e.build()" > gpurun_out/build.log 2>&1
VD=paper_2112_00132_b200/variants
for rep in 1 2; do
for lib in product h4096 h8192 h16k; do
  if [ $lib = product ]; then L=""; else L=$VD/libatos_$lib.so; fi
  echo "== $lib rep $rep" >> gpurun_out/hthr.md
  ATOS_LIB=$L timeout 200 python tests/harness/pr_variants.py --runs 2 $( [ $rep = 1 ] || echo --no-oracle ) --variants '{"pr": {"cta_threads": 1024}}' >> gpurun_out/hthr.md 2>&1
done; done
