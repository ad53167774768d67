set -o pipefail
B5="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
$B5 > gpurun_out/prof_plain.json 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5_full.csv $B5 > gpurun_out/ncu_a.log 2>&1; echo ncu1 rc=$?
B200="python bench.py --config 5 --models 200 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$B200 > gpurun_out/prof_200.json 2>&1 && ncu --set full --clock-control none --import-source on -k regex:score3 -s 2 -c 2 -o gpurun_out/score3_full_v12 $B200 > gpurun_out/ncu_b.log 2>&1; echo ncu2 rc=$?
