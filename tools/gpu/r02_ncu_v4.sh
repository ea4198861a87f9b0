#!/bin/bash
mkdir -p gpurun_out
N_NAND=1184 VARIANTS=6085 KS_VARIANTS=0 timeout 300 python tools/variant_sweep.py > gpurun_out/v4_plain.log 2>&1
N_NAND=1184 VARIANTS=6085 KS_VARIANTS=0 timeout 900 ncu --set full --import-source on --clock-control none \
  -k regex:blind_rotate_kernel_v4 -c 1 -o gpurun_out/ncu_v4_src -f python tools/variant_sweep.py > gpurun_out/ncu_v4.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_v4.log
