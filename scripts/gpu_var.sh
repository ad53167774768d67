# Time every variants/*.so on the 200-model config-5 slice (flags 0 and 6) and the full config 5.
for v in variants/*.so; do n=$(basename $v .so)
  for f in 0 6; do PPIPE_LIB=$v PPIPE_DEBUG_FLAGS=$f python bench.py --config 5 --models 200 --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/var_${n}_f$f.json 2>/dev/null; done
  if [ -n "$FULL" ]; then PPIPE_LIB=$v python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/var_${n}_full.json 2>/dev/null; fi
done
echo done
