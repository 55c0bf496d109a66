# BFS / PR ring-buffer depth sweep (build-time ATOS_NBUF variants)
V='{"t256f128": {}, "t256f64": {"fetch_size": 64}, "t512f128": {"cta_threads": 512}, "t128f64": {"cta_threads": 128, "fetch_size": 64}}'
timeout 300 python tools/pr_variants.py --app bfs --no-oracle --runs 5 --variants "$V" > gpurun_out/bfs_nbuf4.log 2>&1
for v in 6 8; do
  bash tools/libswap.sh paper_2112_00132_b200/variants/libatos_nbuf$v.so \
    timeout 300 python tools/pr_variants.py --app bfs --no-oracle --runs 5 --variants "$V" > gpurun_out/bfs_nbuf$v.log 2>&1
  bash tools/libswap.sh paper_2112_00132_b200/variants/libatos_nbuf$v.so \
    timeout 300 python tools/pr_variants.py --app pr --no-oracle --runs 2 --variants '{"t512f128": {}}' > gpurun_out/pr_nbuf$v.log 2>&1
done
