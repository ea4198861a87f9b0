#!/bin/bash
# Phase breakdown of the v4 kernel (instrumented build).
mkdir -p gpurun_out
rm -rf paper_2101_03403_b200/_build
CVM_NVCC_EXTRA=-DCVM_PHASE_PROF python paper_2101_03403_b200/build.py > gpurun_out/phbuild.log 2>&1
N_NAND=1184 timeout 300 python tools/v4_phases.py > gpurun_out/v4phases.log 2>&1
N_NAND=148 timeout 300 python tools/v4_phases.py >> gpurun_out/v4phases.log 2>&1
echo "rc=$?" >> gpurun_out/v4phases.log
