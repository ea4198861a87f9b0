#!/bin/bash
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  N=6 timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_probe.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitize_$tool.log
done
