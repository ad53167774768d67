set -o pipefail
mkdir -p gpurun_out
python paper_2507_18748_b200/build.py > /dev/null
timeout 900 python -m pytest tests/test_multigpu.py -x -q -m gpu 2>&1 | tail -3 | tee gpurun_out/mgpu_pytest.txt
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_r2.json 2> gpurun_out/bench_r2.err; echo bench rc=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/bench_r2_n2.json 2> gpurun_out/bench_r2_n2.err; echo bench2 rc=$?
