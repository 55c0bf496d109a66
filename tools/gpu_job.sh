# ad-hoc GPU job (overwritten per experiment; the committed copy is the last one run)
python -c "import __graft_entry__ as e; e.build()" > gpurun_out/build.log 2>&1
VD=paper_2112_00132_b200/variants
for v in self; do ATOS_LIB=$VD/libatos_$v.so timeout 120 python tools/quick_check.py >> gpurun_out/qc.log 2>&1; echo "$v rc=$?" >> gpurun_out/qc.log; done
tail -3 gpurun_out/qc.log
for rep in 1 2; do
for lib in product self; do
  if [ $lib = product ]; then L=""; V='{"pr": {"cta_threads": 1024}}'; B='{"t256": {"cta_threads": 256}}'; else L=$VD/libatos_$lib.so; V='{"f16": {"cta_threads": 1024, "fetch_size": 16}, "f32": {"cta_threads": 1024, "fetch_size": 32}, "f64": {"cta_threads": 1024, "fetch_size": 64}, "t512f32": {"cta_threads": 512, "fetch_size": 32}}'; B='{"t256f32": {"cta_threads": 256, "fetch_size": 32}, "t256f128": {"cta_threads": 256, "fetch_size": 128}, "t1024f32": {"cta_threads": 1024, "fetch_size": 32}}'; fi
  grep -q "$lib rc=0" gpurun_out/qc.log || [ $lib = product ] || continue
  echo "== $lib rep $rep" >> gpurun_out/self.md
  ATOS_LIB=$L timeout 300 python tools/pr_variants.py --runs 2 --no-oracle --variants "$V" >> gpurun_out/self.md 2>&1
  ATOS_LIB=$L timeout 200 python tools/pr_variants.py --app bfs --runs 5 --no-oracle --variants "$B" >> gpurun_out/self.md 2>&1
done; done
ATOS_LIB=$VD/libatos_self.so timeout 300 python tools/grid_latency.py --runs 2 --cells cta:256:32,cta:256:8,cta:1024:8 >> gpurun_out/self.md 2>&1
