mkdir -p gpurun_out
python paper_2507_18748_b200/build.py > /dev/null
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -25 | tee gpurun_out/quick.txt
for i in 1 2; do timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-sweep --no-f2 --no-pb 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4g'%d['value'], round(d['ms_per_step'],2), d['phase_ms']['score'])" | tee -a gpurun_out/quick.txt; done
