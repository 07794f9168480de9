#!/bin/bash
# compute-sanitizer memcheck and racecheck over tools/sanitize_probe.py (GPU box)
mkdir -p gpurun_out
for tool in memcheck racecheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 --error-exitcode 9 \
      python tools/sanitize_probe.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_$tool.log
done
