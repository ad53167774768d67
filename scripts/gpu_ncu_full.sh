# One ncu --set full capture of the three score kernels of one timed config-5 step.
set -o pipefail
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$B > gpurun_out/full_plain.json 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:score -s 3 -c 3 -o gpurun_out/score_full_r1 $B \
  > gpurun_out/ncu_full.log 2>&1; echo ncu rc=$?
