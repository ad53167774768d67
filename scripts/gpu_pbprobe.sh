mkdir -p gpurun_out
python paper_2507_18748_b200/build.py > /dev/null
for c in 2 3; do timeout 300 python scripts/pb_probe.py --config $c --reps 3 2>&1 | tail -2; done | tee gpurun_out/pb_probe.txt
timeout 300 python scripts/pb_probe.py --config 4 --reps 1 2>&1 | tail -2 | tee -a gpurun_out/pb_probe.txt
