set -o pipefail
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$B > gpurun_out/full_plain3.json 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:score12 -s 1 -c 1 -o gpurun_out/score12_r1 $B \
  > gpurun_out/ncu_12.log 2>&1; echo ncu rc=$?
