# NBUF 3/5 and AGENT_G 3 against the AGENT_G=2 default (RMAT-24; alternating, 2 reps)
PRV='{"t1024f128": {"cta_threads": 1024}}'
BFV='{"t256f128": {}}'
for rep in 1 2; do
for v in base nbuf3 nbuf5 ag3; do
  if [ $v = base ]; then
    timeout 200 python tools/pr_variants.py --app pr --no-oracle --runs 3 --variants "$PRV" 2>&1 | grep '^| t' | sed "s/^/$v pr /" >> gpurun_out/job23.log
    timeout 100 python tools/pr_variants.py --app bfs --no-oracle --runs 5 --variants "$BFV" 2>&1 | grep '^| t' | sed "s/^/$v bfs /" >> gpurun_out/job23.log
  else
    bash tools/libswap.sh paper_2112_00132_b200/variants/libatos_$v.so timeout 200 python tools/pr_variants.py --app pr --no-oracle --runs 3 --variants "$PRV" 2>&1 | grep '^| t' | sed "s/^/$v pr /" >> gpurun_out/job23.log
    bash tools/libswap.sh paper_2112_00132_b200/variants/libatos_$v.so timeout 100 python tools/pr_variants.py --app bfs --no-oracle --runs 5 --variants "$BFV" 2>&1 | grep '^| t' | sed "s/^/$v bfs /" >> gpurun_out/job23.log
  fi
done
done
