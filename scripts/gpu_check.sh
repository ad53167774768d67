set -o pipefail
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4 || exit 1
for f in 0 2 6; do
PPIPE_DEBUG_FLAGS=$f python bench.py --config 5 --models 200 --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/exp_$f.json 2> gpurun_out/exp_$f.err
done
PPIPE_DEBUG_FLAGS=8 python bench.py --config 5 --models 200 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e 2>&1 | grep "ppipe debug" | tail -1 | tee gpurun_out/debug_line.txt
timeout 400 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench3.json 2> gpurun_out/bench3.err; echo bench rc=$?
if [ -x scripts/micro/pipes ]; then scripts/micro/pipes > gpurun_out/pipes.txt 2>&1; fi
