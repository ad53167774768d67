mkdir -p gpurun_out
python paper_2507_18748_b200/build.py > /dev/null
CUDA_LAUNCH_BLOCKING=1 python -c "
import paper_2507_18748_b200 as pp
from workloads import config1
w=config1()
try:
    f=pp.run(w, frontier=3); print('ok', f.n_points)
except Exception as e: print('ERR', e)
" 2>&1 | tail -3 | tee gpurun_out/pbdbg.txt
timeout 120 compute-sanitizer --tool memcheck python -c "
import paper_2507_18748_b200 as pp
from workloads import config1
w=config1()
f=pp.run(w, frontier=3); print('ok', f.n_points)
" 2>&1 | head -40 | tee -a gpurun_out/pbdbg.txt
