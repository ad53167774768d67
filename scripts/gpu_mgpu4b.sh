mkdir -p gpurun_out
python paper_2507_18748_b200/build.py > /dev/null
timeout 1200 python -m pytest tests/test_multigpu.py -x -q -m gpu 2>&1 | tail -3 | tee gpurun_out/mgpu4_pytest.txt
