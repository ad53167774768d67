set -o pipefail
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 || exit 1
python scripts/e2e_probe.py 2>&1 | tail -3
timeout 400 python bench.py --steps 5 --warmup 3 > gpurun_out/bench3.json 2> gpurun_out/bench3.err; echo bench rc=$?
bash scripts/gpu_var.sh
