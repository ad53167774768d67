set -o pipefail
mkdir -p gpurun_out
python paper_2507_18748_b200/build.py > /dev/null
timeout 900 python -m pytest tests/test_pb_gpu.py -x -q 2>&1 | tail -4 | tee gpurun_out/pb_pytest.txt || exit 1
for c in 2 3; do timeout 300 python scripts/pb_probe.py --config $c --reps 3 2>&1 | tail -1; done | tee gpurun_out/pb_probe.txt
timeout 300 python scripts/pb_probe.py --config 4 --reps 2 2>&1 | tail -1 | tee -a gpurun_out/pb_probe.txt
