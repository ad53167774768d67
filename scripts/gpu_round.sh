set -o pipefail
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4 || exit 1
timeout 400 python bench.py --steps 5 --warmup 3 > gpurun_out/bench2.json 2> gpurun_out/bench2.err; echo bench rc=$?
B4="python bench.py --config 4 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
$B4 > gpurun_out/c4.json 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv $B4 > gpurun_out/ncu1.log 2>&1; echo ncu1 rc=$?
ncu --set full --clock-control none --import-source on -k regex:score_kernel -c 1 -o gpurun_out/score_c4 $B4 > gpurun_out/ncu2.log 2>&1; echo ncu2 rc=$?
