#!/bin/bash
# One parameterized runner for the GPU-box tasks (run through gpurun from the repo root):
#   gpurun --timeout 1800 -- 'bash scripts/gpu.sh tests bench launches'
# Tasks (run in the order given; each logs under gpurun_out/):
#   tests      pytest -m gpu (the driver's round-end suite) + smoke()
#   bench      default bench line (config 5, N=1)            -> gpurun_out/bench.json
#   launches   ncu launch list of the default bench command (after a plain run exits 0)
#   full       one ncu --set full capture of the score kernels of one config-5 step
#   frontier   one ncu --set full capture of the frontier-pass kernels
#   dcheck     the bounds-checked build (scripts/variants.py dcheck) over the GPU suite + one step
#   mgpu N     multi-GPU tests + an N-rank bench (box must have N GPUs)
#   golden     the full config-5 hash test against tests/golden/config5_oracle.json
set -o pipefail
mkdir -p gpurun_out
B="python bench.py"
while [ $# -gt 0 ]; do
  t=$1; shift
  case $t in
    tests)
      timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
      timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log ;;
    bench)
      timeout 900 $B > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -c 3000 gpurun_out/bench.json ;;
    launches)
      $B --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/launch_plain.json 2> gpurun_out/launch_plain.err && \
      ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv \
        $B --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1; echo "ncu launches rc=$?" ;;
    full)
      X="$B --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
      $X > gpurun_out/full_plain.json 2>&1 && \
      ncu --set full --clock-control none --import-source on -k regex:score -s 9 -c 3 -o gpurun_out/score_full $X \
        > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?" ;;
    frontier)
      X="$B --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
      $X > gpurun_out/fr_plain.json 2>&1 && \
      ncu --set full --clock-control none --import-source on -k regex:fp_ -c 12 -o gpurun_out/frontier_full $X \
        > gpurun_out/ncu_frontier.log 2>&1; echo "ncu frontier rc=$?" ;;
    dcheck)
      python scripts/variants.py dcheck:-DPPIPE_DEBUG_CHECKS > gpurun_out/dcheck_build.log 2>&1
      PPIPE_LIB=variants/dcheck.so timeout 1500 python -m pytest tests -m gpu -x -q -k "not nccl and not golden" 2>&1 | tail -4
      PPIPE_LIB=variants/dcheck.so timeout 600 $B --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/dcheck_bench.json 2> gpurun_out/dcheck_bench.err; echo "dcheck bench rc=$?"
      grep -h "PPIPE_DCHECK" gpurun_out/dcheck_bench.* | head -5 ;;
    mgpu)
      n=$1; shift
      nvidia-smi --query-gpu=index,name --format=csv,noheader | wc -l
      timeout 900 python -m pytest tests/test_multigpu.py -x -q -m gpu 2>&1 | tail -3
      timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2954$n \
        bench.py --gpus $n --steps 10 --warmup 3 > gpurun_out/bench_n$n.json 2> gpurun_out/bench_n$n.err; echo "bench n=$n rc=$?"; tail -c 2500 gpurun_out/bench_n$n.json ;;
    golden)
      timeout 900 python -m pytest tests/test_config5_golden.py -x -q -m gpu 2>&1 | tail -5 ;;
    *) echo "unknown task $t"; exit 2 ;;
  esac
done
