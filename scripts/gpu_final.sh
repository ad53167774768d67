set -o pipefail
mkdir -p gpurun_out
python paper_2507_18748_b200/build.py > /dev/null
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-sweep --no-f2 --no-pb"
$B > gpurun_out/launch_plain.json 2> gpurun_out/launch_plain.err || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launches.log 2>&1; echo ncu rc=$?
ncu --set full --clock-control none --import-source on -k regex:score3a -s 0 -c 1 -o gpurun_out/score3a $B > gpurun_out/ncu_3a.log 2>&1; echo 3a rc=$?
ncu --set full --clock-control none --import-source on -k regex:score3b -s 0 -c 1 -o gpurun_out/score3b $B > gpurun_out/ncu_3b.log 2>&1; echo 3b rc=$?
ncu --set full --clock-control none --import-source on -k regex:score12 -s 0 -c 1 -o gpurun_out/score12 $B > gpurun_out/ncu_12.log 2>&1; echo 12 rc=$?
P="python scripts/pb_probe.py --config 4 --reps 1"
ncu --set full --clock-control none -k regex:pb_score3 -s 100 -c 1 -o gpurun_out/pb3 $P > gpurun_out/ncu_pb3.log 2>&1; echo pb3 rc=$?
