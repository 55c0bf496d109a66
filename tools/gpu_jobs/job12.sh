# end-of-round measurement pass: bench, launch list, ncu full captures, experiments
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests12.log 2>&1; echo tests_rc=$? >> gpurun_out/gpu_tests12.log
timeout 600 python bench.py > gpurun_out/bench12.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches12.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-color > gpurun_out/bench12_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_persistent -c 1 -o gpurun_out/pr12 -f \
  python tools/profile_run.py --app pr --iters 1 --fetch 128 --threads 512 > gpurun_out/pr12_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_persistent -c 1 -o gpurun_out/bfs12 -f \
  python tools/profile_run.py --app bfs --iters 1 --fetch 128 --threads 256 > gpurun_out/bfs12_ncu.log 2>&1
timeout 1200 python tools/experiments.py kernels grid color timeline heatmap > gpurun_out/experiments12.md 2>&1
