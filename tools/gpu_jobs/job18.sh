# PageRank (T=1024 F=128, no splitting) build-knob sweep + phase profile
V='{"t1024f128": {"cta_threads": 1024}, "t1024f192": {"cta_threads": 1024, "fetch_size": 192}}'
timeout 300 python tools/pr_variants.py --app pr --no-oracle --runs 2 --variants "$V" > gpurun_out/pr18_base.log 2>&1
for v in nbuf3 nbuf6 unroll4 unroll12; do
  bash tools/libswap.sh paper_2112_00132_b200/variants/libatos_$v.so \
    timeout 300 python tools/pr_variants.py --app pr --no-oracle --runs 2 --variants "$V" > gpurun_out/pr18_$v.log 2>&1
done
bash tools/libswap.sh paper_2112_00132_b200/variants/libatos_wprof.so \
  timeout 300 python tools/profile_run.py --app pr --iters 1 --fetch 128 --threads 1024 > gpurun_out/wprof18.log 2>&1
