#!/bin/bash
mkdir -p gpurun_out
rm -rf paper_2101_03403_b200/_build
CVM_NVCC_EXTRA=-DCVM_PHASE_PROF python paper_2101_03403_b200/build.py > gpurun_out/phbuild.log 2>&1
for vw in "6085 1184" "6045 592" "6025 296" "6015 148"; do set -- $vw; VARIANT=$1 N_NAND=$2 timeout 300 python tools/v4_phases.py; done > gpurun_out/v4phases_w.log 2>&1
echo "rc=$?" >> gpurun_out/v4phases_w.log
