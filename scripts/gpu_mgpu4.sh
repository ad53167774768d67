nvidia-smi --query-gpu=index,name --format=csv,noheader | wc -l
timeout 600 python -m pytest tests/test_multigpu.py -x -q -m gpu 2>&1 | tail -2
for n in 2 4; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2953$n bench.py --gpus $n --steps 5 --warmup 3 > gpurun_out/bench_n$n.json 2> gpurun_out/bench_n$n.err; echo bench$n rc=$?
done
