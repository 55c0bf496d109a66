# ad-hoc GPU job (overwritten per experiment; the committed copy is the last one run)
python -c "import __graft_entry__ as e; e.build()" > gpurun_out/build.log 2>&1
VD=paper_2112_00132_b200/variants
for v in a2n8 a4n8 a3n6; do ATOS_LIB=$VD/libatos_$v.so timeout 120 python tools/quick_check.py >> gpurun_out/qc.log 2>&1; echo "$v rc=$?" >> gpurun_out/qc.log; done
V='{"t1024": {"cta_threads": 1024}, "t1024_cap28": {"cta_threads": 1024, "queue_capacity": 268435456}}'
for rep in 1 2; do
for lib in product a2n8 a4n8 a3n6 a1; do
  if [ $lib = product ]; then L=""; else L=$VD/libatos_$lib.so; fi
  grep -q "$lib rc=0" gpurun_out/qc.log || [ $lib = product ] || [ $lib = a1 ] || continue
  echo "== $lib rep $rep" >> gpurun_out/agents.md
  ATOS_LIB=$L timeout 200 python tools/pr_variants.py --runs 3 --no-oracle --variants "$V" >> gpurun_out/agents.md 2>&1
done; done
timeout 900 python -m pytest tests/test_peer.py -q -x > gpurun_out/pytest_peer.log 2>&1; echo peer_rc=$?; tail -3 gpurun_out/pytest_peer.log
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "staging or hub_sweep or floor" > gpurun_out/pytest_st.log 2>&1; echo st_rc=$?; tail -3 gpurun_out/pytest_st.log
