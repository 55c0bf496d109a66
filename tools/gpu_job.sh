# ad-hoc GPU job (overwritten per experiment; the committed copy is the last one run)
python -c "import __graft_entry__ as e; e.build()" > gpurun_out/build.log 2>&1
timeout 120 python -c "import __graft_entry__ as e; e.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
timeout 1800 python -m pytest tests -q -m gpu --timeout 600 > gpurun_out/pytest.log 2>&1; echo pytest_rc=$?; tail -5 gpurun_out/pytest.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1; echo bench_rc=$?; tail -c 300 gpurun_out/bench.log
timeout 600 ncu --section PmSampling --section PmSampling_WarpStates --section LaunchStats --section Occupancy --clock-control none -k regex:k_persistent -c 1 -o gpurun_out/pr_pm -f python tools/profile_run.py --app pr --threads 1024 --fetch 128 --iters 1 > gpurun_out/ncu_pm_pr.log 2>&1; echo pm1=$?
timeout 600 ncu --section PmSampling --section PmSampling_WarpStates --section LaunchStats --section Occupancy --clock-control none -k regex:k_persistent -c 1 -o gpurun_out/bfs_pm -f python tools/profile_run.py --app bfs --threads 256 --fetch 128 --iters 1 > gpurun_out/ncu_pm_bfs.log 2>&1; echo pm2=$?
timeout 900 python tools/peer_bench.py --scale 22 --runs 3 --oracle > gpurun_out/peer.md 2>&1; echo peer=$?
