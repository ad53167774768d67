for f in 0 1 2 3 4 6; do
PPIPE_DEBUG_FLAGS=$f python bench.py --config 5 --models 200 --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/exp_$f.json 2> gpurun_out/exp_$f.err
done
