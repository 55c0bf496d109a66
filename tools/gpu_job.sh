# ad-hoc GPU job (overwritten per experiment; the committed copy is the last one run)
python -c "import __graft_entry__ as e; e.build()" > gpurun_out/build.log 2>&1
VD=paper_2112_00132_b200/variants
timeout 120 python tools/quick_check.py >> gpurun_out/qc.log 2>&1; echo "product rc=$?" >> gpurun_out/qc.log; tail -2 gpurun_out/qc.log
for rep in 1 2 3; do
for lib in product nohubitem; do
  if [ $lib = product ]; then L=""; else L=$VD/libatos_$lib.so; fi
  echo "== $lib rep $rep" >> gpurun_out/hi.md
  ATOS_LIB=$L timeout 200 python tools/pr_variants.py --runs 2 --no-oracle --variants '{"pr": {"cta_threads": 1024}}' >> gpurun_out/hi.md 2>&1
done; done
timeout 1500 python -m pytest tests -q -m gpu -x --timeout 600 -k "pagerank or peer or color or gc" > gpurun_out/pytest.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest.log
