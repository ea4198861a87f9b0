#!/bin/bash
# Phase breakdown of the pair kernel (instrumented build, then restore the product build).
mkdir -p gpurun_out
rm -rf paper_2101_03403_b200/_build
CVM_NVCC_EXTRA="-DCVM_PHASE_PROF $PH_EXTRA" python paper_2101_03403_b200/build.py > gpurun_out/phbuild.log 2>&1
for n in ${PH_N:-1 26 74}; do N_NAND=$n timeout 300 python tools/pair_phases.py; done > gpurun_out/phases.log 2>&1
echo "rc=$?" >> gpurun_out/phases.log
