# final pass after R33 + bench value normalisation: bench, launch list, ncu full captures, C5
timeout 600 python bench.py > gpurun_out/bench17.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches17.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-color > gpurun_out/bench17_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_persistent -c 1 -o gpurun_out/pr17 -f \
  python tools/profile_run.py --app pr --iters 1 --fetch 128 --threads 1024 > gpurun_out/pr17_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_persistent -c 1 -o gpurun_out/bfs17 -f \
  python tools/profile_run.py --app bfs --iters 1 --fetch 128 --threads 256 > gpurun_out/bfs17_ncu.log 2>&1
timeout 1500 python tools/c5_single.py --jacobi-max-s 1100 --runs 3 --pr-variants '{"default": {}}' > gpurun_out/c5_v6.log 2>&1; echo rc=$? >> gpurun_out/c5_v6.log
