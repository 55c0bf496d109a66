# AGENT_G sweep (items per agent lane per L2 round-trip phase): PageRank/BFS on RMAT-24
L=paper_2112_00132_b200/libatos.so
cp $L /tmp/base.so
for rep in 1 2 3; do
for v in base g2 g1; do
  if [ $v = base ]; then cp /tmp/base.so $L; else cp tools/libatos_$v.so $L; fi
  pf=128
  timeout 300 python bench.py --no-e2e --no-color --no-cpu-baseline --steps 3 --warmup 3 --pr-fetch $pf > /tmp/o.json 2>/tmp/e.log
  python -c "import json;d=json.loads(open('/tmp/o.json').read().strip().splitlines()[-1]);print('$v pf=$pf', 'pr_ms=%.1f'%d['pagerank']['ms'], 'pushes=%.3g'%d['pagerank']['edge_pushes'], 'bfs_ms=%.2f'%d['bfs']['ms'], 'value=%.1f'%d['value'])" >> gpurun_out/agentg.log 2>&1 || tail -3 /tmp/e.log >> gpurun_out/agentg.log
done
done
cp /tmp/base.so $L
