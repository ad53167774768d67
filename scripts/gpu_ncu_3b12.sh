set -o pipefail
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$B > gpurun_out/full_plain2.json 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:'score(3b|12)' -s 2 -c 2 -o gpurun_out/score3b12_r1 $B \
  > gpurun_out/ncu_3b12.log 2>&1; echo ncu rc=$?
