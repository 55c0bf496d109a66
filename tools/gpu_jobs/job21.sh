# AGENT_G=2 default: smoke, full GPU tests, bench, launch list, one ncu --set full PR capture
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke21.log 2>&1; echo smoke_rc=$? >> gpurun_out/smoke21.log
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests21.log 2>&1; echo tests_rc=$? >> gpurun_out/gpu_tests21.log
timeout 600 python bench.py > gpurun_out/bench21.log 2>&1; echo bench_rc=$? >> gpurun_out/bench21.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches21.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-color > gpurun_out/ncu_launch21.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_persistent -c 1 -o gpurun_out/pr21 \
  python tools/profile_run.py --app pr --iters 1 --fetch 128 --threads 1024 > gpurun_out/ncu_pr21.log 2>&1
