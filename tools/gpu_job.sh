# ad-hoc GPU job (overwritten per experiment; the committed copy is the last one run)
python -c "import __graft_entry__ as e; e.build()" > gpurun_out/build.log 2>&1
for v in old new; do
  if [ $v = old ]; then export ATOS_LIB=paper_2112_00132_b200/variants/libatos_old.so; else unset ATOS_LIB; fi
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_pr_seed|PrInitSplit" --csv --log-file gpurun_out/seed_$v.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_$v.log 2>&1; echo ncu_$v=$?
done
unset ATOS_LIB
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_pr_seed" -c 1 -o gpurun_out/seed_full python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo full=$?
