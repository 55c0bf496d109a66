# R30 compensation: gpu tests, RMAT-24 timing/accuracy with and without, C5 parity
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests6.log 2>&1; echo tests_rc=$? >> gpurun_out/gpu_tests6.log
timeout 600 python tools/pr_variants.py --app pr --variants '{"comp": {}, "nocomp": {"pr_compensate": false}, "comp_discrete": {"kernel": "discrete"}}' > gpurun_out/prvar6.log 2>&1
timeout 1500 python tools/c5_single.py --jacobi-max-s 1100 --runs 3 --pr-variants '{"comp32": {}, "nocomp32": {"pr_compensate": false}}' > gpurun_out/c5_v3.log 2>&1; echo rc=$? >> gpurun_out/c5_v3.log
