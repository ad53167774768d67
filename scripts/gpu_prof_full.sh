set -o pipefail
B5="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$B5 > gpurun_out/pf_plain.json 2>&1 && ncu --set full --clock-control none --import-source on -k regex:score3a -s 1 -c 1 -o gpurun_out/score3a_full_cfg5 $B5 > gpurun_out/ncu_pf.log 2>&1; echo ncu rc=$?
