set -o pipefail
mkdir -p gpurun_out
python paper_2507_18748_b200/build.py > /dev/null
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -4 | tee gpurun_out/pytest_gpu.txt || exit 1
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_main.json 2> gpurun_out/bench_main.err; echo bench rc=$?
