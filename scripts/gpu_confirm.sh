set -o pipefail
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4 | tee gpurun_out/pytest_gpu.txt || exit 1
timeout 400 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_confirm.json 2> gpurun_out/bench_confirm.err; echo bench rc=$?
