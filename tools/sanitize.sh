#!/bin/bash
# compute-sanitizer over tools/sanitize_probe.py; logs in gpurun_out/sanitizer_<tool>.txt
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 7 --print-limit 50 \
     python tools/sanitize_probe.py > gpurun_out/sanitizer_$tool.txt 2>&1
  echo "$tool rc=$?" | tee -a gpurun_out/sanitizer_$tool.txt
done
