# ad-hoc GPU job (overwritten per experiment; the committed copy is the last one run)
python -c "import __graft_entry__ as e; e.build()" > gpurun_out/build.log 2>&1
timeout 600 python tools/e2e_breakdown.py --iters 8 > gpurun_out/e2e.md 2>&1; echo e2e=$?; cat gpurun_out/e2e.md
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 2 --warmup 1 --backend gloo --no-color > gpurun_out/bench2.log 2>&1; echo b2=$?; tail -c 1500 gpurun_out/bench2.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-color --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo bench_rc=$?; tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e'])"
