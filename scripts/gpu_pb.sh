set -o pipefail
mkdir -p gpurun_out
python paper_2507_18748_b200/build.py > /dev/null
timeout 900 python -m pytest tests/test_pb_gpu.py -x -q 2>&1 | tail -15 | tee gpurun_out/pb_pytest.txt
