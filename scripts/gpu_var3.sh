mkdir -p gpurun_out
: > gpurun_out/var3.txt
for v in base match base match; do
  PPIPE_LIB=variants/$v.so timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --no-sweep --no-f2 --no-pb 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', '%.4g'%d['value'], round(d['ms_per_step'],2), d['phase_ms']['score'], d['config']['frontier_points'])" >> gpurun_out/var3.txt
done
PPIPE_LIB=variants/match.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1 >> gpurun_out/var3.txt
cat gpurun_out/var3.txt
