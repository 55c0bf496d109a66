# round-1 final-ish measurement pass: phase profile, bench, launch list, ncu full captures
timeout 300 python -m pytest tests -m gpu -x -q -k "fp64_seeding or sink" > gpurun_out/gpu_tests5.log 2>&1
set -x
for app in bfs pr; do
  thr=256; [ $app = pr ] && thr=512
  bash tools/libswap.sh paper_2112_00132_b200/variants/libatos_wprof.so \
    timeout 300 python tools/profile_run.py --app $app --iters 2 --fetch 128 --threads $thr > gpurun_out/wprof_$app.log 2>&1
done
timeout 600 python bench.py > gpurun_out/bench5.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches5.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-color > gpurun_out/bench5_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_persistent -c 1 -o gpurun_out/pr5 -f \
  python tools/profile_run.py --app pr --iters 1 --fetch 128 --threads 512 > gpurun_out/pr5_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_persistent -c 1 -o gpurun_out/bfs5 -f \
  python tools/profile_run.py --app bfs --iters 1 --fetch 128 --threads 256 > gpurun_out/bfs5_ncu.log 2>&1
