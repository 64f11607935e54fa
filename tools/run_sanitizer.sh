#!/bin/bash
# One compute-sanitizer tool per gpurun call (B200_PROFILING.md): TOOL=memcheck|racecheck|synccheck|initcheck
TOOL=${TOOL:-memcheck}
python tools/sanitize_cases.py > gpurun_out/san_plain_$TOOL.log 2>&1 || { echo "plain run failed"; cat gpurun_out/san_plain_$TOOL.log; exit 1; }
EXTRA=""
[ "$TOOL" = "memcheck" ] && EXTRA="--leak-check full"
timeout 1500 compute-sanitizer --tool $TOOL $EXTRA --target-processes all --print-limit 200 \
  python tools/sanitize_cases.py > gpurun_out/sanitizer_$TOOL.log 2>&1
echo "exit=$?" >> gpurun_out/sanitizer_$TOOL.log
tail -25 gpurun_out/sanitizer_$TOOL.log
