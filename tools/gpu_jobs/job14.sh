# hub chunk splitting vs PageRank edge pushes / BFS time (build-time ATOS_SPLIT_DEG / ATOS_CHUNK_EDGES variants)
for v in nosplit chunk8k; do
  bash tools/libswap.sh paper_2112_00132_b200/variants/libatos_$v.so \
    timeout 600 python tools/pr_variants.py --app pr --no-oracle --runs 2 --variants '{"default": {}, "f64": {"fetch_size": 64}}' > gpurun_out/pr_$v.log 2>&1
  bash tools/libswap.sh paper_2112_00132_b200/variants/libatos_$v.so \
    timeout 300 python tools/pr_variants.py --app bfs --no-oracle --runs 5 --variants '{"default": {}}' > gpurun_out/bfs_$v.log 2>&1
done
