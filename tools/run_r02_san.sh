#!/bin/bash
# compute-sanitizer over every round kernel (tools/sanitize_run.py), one tool per call
set -u
mkdir -p gpurun_out
TOOL=${1:-racecheck}
python tools/sanitize_run.py > gpurun_out/san_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
if [ "$TOOL" = racecheck ]; then
  timeout 2400 compute-sanitizer --tool racecheck --racecheck-report all python tools/sanitize_run.py > gpurun_out/san_racecheck.log 2>&1
else
  timeout 2400 compute-sanitizer --tool $TOOL python tools/sanitize_run.py > gpurun_out/san_$TOOL.log 2>&1
fi
echo "$TOOL rc=$?"
tail -5 gpurun_out/san_$TOOL.log
