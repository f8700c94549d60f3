#!/bin/bash
# compute-sanitizer over smoke-size calls, one tool per invocation (memcheck, racecheck, synccheck, initcheck)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool $tool --error-exitcode 99 --print-limit 50 \
    python tools/sanitize_calls.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_$tool.log
done
