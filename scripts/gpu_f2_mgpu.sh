set -o pipefail
mkdir -p gpurun_out
python paper_2507_18748_b200/build.py > /dev/null
timeout 900 python -m pytest tests/test_multigpu.py -x -q -m gpu 2>&1 | tail -5 | tee gpurun_out/mgpu_pytest.txt
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_f2.json 2> gpurun_out/bench_f2.err; echo bench rc=$?
