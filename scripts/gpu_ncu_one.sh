# One ncu --set full capture of one kernel (regex $K, skip $SKIP launches) of a timed config-5 step.
set -o pipefail
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-sweep"
$B > gpurun_out/ncu_plain_$TAG.json 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$K -s $SKIP -c 1 -o gpurun_out/$TAG $B \
  > gpurun_out/ncu_$TAG.log 2>&1; echo ncu rc=$?
