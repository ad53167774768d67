# GPU parity tests and one full config-5 step against the bounds-checked debug build
export PPIPE_LIB=variants/dcheck.so
timeout 1200 python -m pytest tests -m gpu -x -q -k "not nccl" 2>&1 | tail -4
timeout 600 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/dcheck_bench.json 2> gpurun_out/dcheck_bench.err; echo bench rc=$?
grep -h "PPIPE_DCHECK" gpurun_out/dcheck_bench.* | head -5
