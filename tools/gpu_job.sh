# ad-hoc GPU job (overwritten per experiment; the committed copy is the last one run)
python -c "import __graft_entry__ as e; e.build()" > gpurun_out/build.log 2>&1
for rep in 1 2; do
  echo "== rep $rep" >> gpurun_out/hc3.md
  timeout 400 python tests/harness/pr_variants.py --runs 2 $( [ $rep = 1 ] || echo --no-oracle ) --variants '{"hc1": {"cta_threads": 1024, "pr_hub_check": 1}, "hc2": {"cta_threads": 1024, "pr_hub_check": 2}, "hc4": {"cta_threads": 1024, "pr_hub_check": 4}, "hc16": {"cta_threads": 1024}}' >> gpurun_out/hc3.md 2>&1
done
