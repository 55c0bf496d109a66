# ad-hoc GPU job (overwritten per experiment; the committed copy is the last one run)
python -c "import __graft_entry__ as e; e.build()" > gpurun_out/build.log 2>&1
V='{"t1024": {"cta_threads": 1024}}'
for rep in 1 2; do
  echo "== old_r01 rep $rep" >> gpurun_out/regr.md
  (cd old_r01 && timeout 300 python tools/pr_variants.py --runs 3 --no-oracle --variants "$V") >> gpurun_out/regr.md 2>&1
  echo "== current rep $rep" >> gpurun_out/regr.md
  ATOS_LIB=paper_2112_00132_b200/variants/libatos_nohub.so timeout 300 python tools/pr_variants.py --runs 3 --no-oracle --variants "$V" >> gpurun_out/regr.md 2>&1
  echo "== old_r01 bfs rep $rep" >> gpurun_out/regr.md
  (cd old_r01 && timeout 300 python tools/pr_variants.py --app bfs --runs 5 --no-oracle --variants '{"t256": {"cta_threads": 256}}') >> gpurun_out/regr.md 2>&1
  echo "== current bfs rep $rep" >> gpurun_out/regr.md
  timeout 300 python tools/pr_variants.py --app bfs --runs 5 --no-oracle --variants '{"t256": {"cta_threads": 256}}' >> gpurun_out/regr.md 2>&1
done
