# F2 on config 4: launch list, then one full capture each of f2_g3 and f2_q3 (after a plain run exits 0).
set -o pipefail
mkdir -p gpurun_out
P="python scripts/f2_probe.py --config 4 --reps 1"
$P > gpurun_out/f2_plain.txt 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/f2_launches.csv $P > gpurun_out/f2_ncu_launches.log 2>&1; echo launches rc=$?
ncu --set full --clock-control none --import-source on -k regex:f2_g3 -c 1 -o gpurun_out/f2_g3 $P > gpurun_out/f2_ncu_g3.log 2>&1; echo g3 rc=$?
ncu --set full --clock-control none --import-source on -k regex:f2_q3 -c 1 -o gpurun_out/f2_q3 $P > gpurun_out/f2_ncu_q3.log 2>&1; echo q3 rc=$?
