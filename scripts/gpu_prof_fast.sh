set -o pipefail
B="python bench.py --config 5 --models 200 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --margin 999"
$B > gpurun_out/pfast.json 2>&1 && ncu --set full --clock-control none --import-source on -k regex:score3a -s 1 -c 1 -o gpurun_out/score3a_fastonly $B > gpurun_out/ncu_fast.log 2>&1; echo ncu rc=$?
