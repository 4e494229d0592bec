#!/bin/bash
# kernel-knob sweep on one GPU: tools/sweep.sh "ENV=.. ENV=.." "ENV=.." ...
mkdir -p gpurun_out
for cfg in "$@"; do
  env $cfg timeout 300 python tools/kernel_sweep.py 300 2>&1 | tail -1 | tee -a gpurun_out/sweep.jsonl
done
