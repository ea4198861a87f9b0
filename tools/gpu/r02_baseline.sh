#!/bin/bash
# Round-2 first GPU call: GPU tests, a short bench, ncu of the default key switch.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-extras --no-cpu > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'key_switch_tc|ks_reduce' -c 4 \
  -o gpurun_out/ncu_ks -f python bench.py --steps 1 --warmup 3 --no-extras --no-cpu > gpurun_out/ncu_ks.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_ks.log
