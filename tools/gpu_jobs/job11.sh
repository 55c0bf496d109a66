# R32 lost-add capture: full gpu tests, RMAT-24 timing, C5 parity
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests11.log 2>&1; echo tests_rc=$? >> gpurun_out/gpu_tests11.log
timeout 600 python tools/pr_variants.py --app pr --runs 4 --variants '{"lost": {}, "nolost": {"pr_lost_capture": false}, "lost_discrete": {"kernel": "discrete"}}' > gpurun_out/prvar11.log 2>&1
timeout 1500 python tools/c5_single.py --jacobi-max-s 1100 --runs 3 --pr-variants '{"lost": {}, "nolost": {"pr_lost_capture": false}}' > gpurun_out/c5_v5.log 2>&1; echo rc=$? >> gpurun_out/c5_v5.log
