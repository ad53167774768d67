nvidia-smi --query-gpu=index,name --format=csv,noheader
timeout 600 python -m pytest tests/test_multigpu.py -x -q -m gpu 2>&1 | tail -5
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err; echo bench2 rc=$?
tail -3 gpurun_out/bench_n2.err
