set -o pipefail
B5="python bench.py --config 5 --models 200 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$B5 > gpurun_out/c5m200.json 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5m200_v10.csv $B5 > gpurun_out/ncu7.log 2>&1; echo ncu1 rc=$?
ncu --set full --clock-control none --import-source on -k regex:score3 -s 2 -c 2 -o gpurun_out/score3_c5m200_v10 $B5 > gpurun_out/ncu8.log 2>&1; echo ncu2 rc=$?
