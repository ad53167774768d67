mkdir -p gpurun_out
: > gpurun_out/var2.txt
for v in base a10 a12 b8; do
  PPIPE_LIB=variants/$v.so timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --no-sweep --no-f2 --no-pb 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', '%.4g'%d['value'], round(d['ms_per_step'],2), d['phase_ms'])" >> gpurun_out/var2.txt
done
cat gpurun_out/var2.txt
