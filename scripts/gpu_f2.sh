set -o pipefail
mkdir -p gpurun_out
python paper_2507_18748_b200/build.py
timeout 300 python scripts/f2_probe.py --config 4 --reps 3 2>&1 | tee gpurun_out/f2_probe.txt
timeout 900 python -m pytest tests/test_f2_gpu.py -x -q 2>&1 | tail -15 | tee gpurun_out/f2_pytest.txt
