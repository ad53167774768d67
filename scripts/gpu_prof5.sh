set -o pipefail
B5="python bench.py --config 5 --models 200 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$B5 > gpurun_out/c5m200.json 2>&1 && ncu --set full --clock-control none --import-source on -k regex:score3b -s 1 -c 1 -o gpurun_out/score3b_v12 $B5 > gpurun_out/ncu9.log 2>&1; echo ncu2 rc=$?
