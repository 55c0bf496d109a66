# R30 fp64 seeding: gpu tests, RMAT-24 timing, C5 parity
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests7.log 2>&1; echo tests_rc=$? >> gpurun_out/gpu_tests7.log
timeout 600 python tools/pr_variants.py --app pr --variants '{"default": {}, "fp64res": {"pr_residue_fp64": true}}' > gpurun_out/prvar7.log 2>&1
timeout 1500 python tools/c5_single.py --jacobi-max-s 1100 --runs 3 --pr-variants '{"fp32": {}}' > gpurun_out/c5_v4.log 2>&1; echo rc=$? >> gpurun_out/c5_v4.log
