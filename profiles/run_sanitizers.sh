#!/bin/bash
# compute-sanitizer over profiles/sanitize_run.py, one tool per invocation
# (run under gpurun: TOOL=memcheck|racecheck|synccheck bash profiles/run_sanitizers.sh)
TOOL=${TOOL:-memcheck}
mkdir -p gpurun_out
VEST_GRAPH=${VEST_GRAPH:-1} timeout ${SAN_TIMEOUT:-1500} compute-sanitizer --tool "$TOOL" --print-limit 50 \
  --log-file "gpurun_out/sanitize_${TOOL}.log" python profiles/sanitize_run.py > "gpurun_out/sanitize_${TOOL}.out" 2>&1
echo "sanitizer $TOOL rc=$?"
tail -3 "gpurun_out/sanitize_${TOOL}.log"
