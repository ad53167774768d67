mkdir -p gpurun_out
: > gpurun_out/e2e_var.txt
for v in c4 c6 c8 c4 c6 c8; do
  PPIPE_LIB=variants/$v.so timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-sweep --no-f2 --no-pb 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', '%.4g'%d['value'], round(d['ms_per_step'],2), 'e2e', '%.4g'%d['e2e']['value'], round(d['e2e']['ms_per_step'],2))" >> gpurun_out/e2e_var.txt
done
cat gpurun_out/e2e_var.txt
