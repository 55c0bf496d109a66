# ad-hoc GPU job (overwritten per experiment; the committed copy is the last one run)
python -c "import __graft_entry__ as e; e.build()" > gpurun_out/build.log 2>&1
VD=paper_2112_00132_b200/variants
for v in noresv gcw8; do ATOS_LIB=$VD/libatos_$v.so timeout 120 python tools/quick_check.py >> gpurun_out/qc.log 2>&1; echo "$v rc=$?" >> gpurun_out/qc.log; done
timeout 120 python tools/quick_check.py >> gpurun_out/qc.log 2>&1; echo "product rc=$?" >> gpurun_out/qc.log
tail -4 gpurun_out/qc.log
for rep in 1 2; do
for lib in product noresv; do
  if [ $lib = product ]; then L=""; else L=$VD/libatos_$lib.so; fi
  echo "== $lib rep $rep" >> gpurun_out/resv.md
  ATOS_LIB=$L timeout 200 python tools/pr_variants.py --runs 2 --no-oracle --variants '{"pr": {"cta_threads": 1024}}' >> gpurun_out/resv.md 2>&1
  ATOS_LIB=$L timeout 200 python tools/pr_variants.py --app bfs --runs 5 --no-oracle --variants '{"t256": {"cta_threads": 256}}' >> gpurun_out/resv.md 2>&1
done; done
for lib in product gcw8; do
  if [ $lib = product ]; then L=""; else L=$VD/libatos_$lib.so; fi
  echo "== $lib" >> gpurun_out/gcw.md
  ATOS_LIB=$L timeout 600 python tools/gc_diag.py --scale 22 --runs 2 --cells persistent:cta:128,persistent:warp:128,discrete:cta:32,bsp:cta:32,bsp:warp:32 >> gpurun_out/gcw.md 2>&1
done
