# compute-sanitizer memcheck over small workloads (one tool per call)
TOOL=${TOOL:-memcheck}
timeout 1500 compute-sanitizer --tool $TOOL --error-exitcode 9 --print-limit 20 python scripts/sanitize_run.py > gpurun_out/sanitize_$TOOL.log 2>&1; echo sanitize rc=$?
tail -15 gpurun_out/sanitize_$TOOL.log
