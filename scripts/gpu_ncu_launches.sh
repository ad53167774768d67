# ncu launch list (per-kernel durations) of the default bench command; the plain run must exit 0 first.
set -o pipefail
python bench.py --steps 2 --warmup 1 > gpurun_out/launch_plain.json 2> gpurun_out/launch_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 1 > gpurun_out/ncu_launches.log 2>&1; echo ncu rc=$?
