B5="python bench.py --config 5 --models 200 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$B5 > gpurun_out/l5.json 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5m200.csv $B5 > gpurun_out/ncu_l.log 2>&1; echo rc=$?
