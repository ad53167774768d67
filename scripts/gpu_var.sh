# Time every variants/*.so: 200-model config-5 slice (flags 0 and 6) unless ONLY_FULL, full config 5 if FULL/ONLY_FULL.
for v in variants/*.so; do n=$(basename $v .so)
  if [ -z "$ONLY_FULL" ]; then
  for f in 0 6; do PPIPE_LIB=$v PPIPE_DEBUG_FLAGS=$f python bench.py --config 5 --models 200 --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/var_${n}_f$f.json 2>/dev/null; done
  fi
  if [ -n "$FULL$ONLY_FULL" ]; then PPIPE_LIB=$v python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/var_${n}_full.json 2>/dev/null; fi
done
echo done
