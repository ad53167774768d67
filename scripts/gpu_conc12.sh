mkdir -p gpurun_out
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-sweep --no-f2 --no-pb"
for i in 1 2; do
  $B > gpurun_out/c12_base_$i.json 2>/dev/null; echo base $i rc=$?
  for v in conc1 conc2; do PPIPE_LIB=variants/$v.so $B > gpurun_out/c12_${v}_$i.json 2>/dev/null; echo $v $i rc=$?; done
done
for f in gpurun_out/c12_*.json; do python -c "
import json,sys;d=json.loads(open('$f').read().strip().splitlines()[-1]);print('$f',d['value'],d['ms_per_step'],d['phase_ms'],d['clocks']['sm_mhz'],d['clocks']['reasons'])"; done
for v in conc2 conc1; do
PPIPE_LIB=variants/$v.so timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/c12_pytest_$v.log 2>&1; echo "pytest $v rc=$?"
tail -1 gpurun_out/c12_pytest_$v.log
done
