# R33: PageRank without hub splitting by default; config sweep, full tests, bench
timeout 900 python tools/pr_variants.py --app pr --runs 3 --variants '{"t512f128": {}, "t512f64": {"fetch_size": 64}, "t256f64": {"cta_threads": 256, "fetch_size": 64}, "t256f128": {"cta_threads": 256}, "t1024f128": {"cta_threads": 1024}, "t512f32": {"fetch_size": 32}, "split_on": {"hub_split": 1}}' > gpurun_out/prvar15.log 2>&1
timeout 300 python tools/pr_variants.py --app bfs --no-oracle --runs 5 --variants '{"default": {}, "split_off": {"hub_split": 0}}' > gpurun_out/bfsvar15.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests15.log 2>&1; echo tests_rc=$? >> gpurun_out/gpu_tests15.log
