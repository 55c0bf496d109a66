# ad-hoc GPU job (overwritten per experiment; the committed copy is the last one run)
python -c "import __graft_entry__ as e; e.build()" > gpurun_out/build.log 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1; echo bench_rc=$?; tail -c 300 gpurun_out/bench.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo ncu1_rc=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_persistent -c 1 -o gpurun_out/bfs_full3 -f python tools/profile_run.py --app bfs --threads 256 --fetch 128 --iters 1 > gpurun_out/ncu_bfs.log 2>&1; echo ncu3_rc=$?
timeout 600 ncu --section PmSampling --section PmSampling_WarpStates --section LaunchStats --section Occupancy --clock-control none -k regex:k_persistent -c 1 -o gpurun_out/bfs_pm3 -f python tools/profile_run.py --app bfs --threads 256 --fetch 128 --iters 1 > gpurun_out/ncu_pm_bfs.log 2>&1; echo pm=$?
timeout 600 python tests/harness/experiments.py timeline > gpurun_out/timeline.md 2>&1; echo tl=$?
