# agent pipelining A/B (ATOS_AGENT_PIPE 1 = default build vs 0 = variant), then full GPU tests
timeout 300 python tools/pr_variants.py --app pr --no-oracle --runs 3 --variants '{"t1024f128": {"cta_threads": 1024}, "t512f128": {}}' > gpurun_out/pr20_pipe.log 2>&1
timeout 200 python tools/pr_variants.py --app bfs --no-oracle --runs 5 --variants '{"t256f128": {}, "t512f128": {"cta_threads": 512}}' > gpurun_out/bfs20_pipe.log 2>&1
bash tools/libswap.sh paper_2112_00132_b200/variants/libatos_nopipe.so \
  timeout 300 python tools/pr_variants.py --app pr --no-oracle --runs 3 --variants '{"t1024f128": {"cta_threads": 1024}, "t512f128": {}}' > gpurun_out/pr20_nopipe.log 2>&1
bash tools/libswap.sh paper_2112_00132_b200/variants/libatos_nopipe.so \
  timeout 200 python tools/pr_variants.py --app bfs --no-oracle --runs 5 --variants '{"t256f128": {}, "t512f128": {"cta_threads": 512}}' > gpurun_out/bfs20_nopipe.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests20.log 2>&1; echo tests_rc=$? >> gpurun_out/gpu_tests20.log
