#!/bin/bash
# A/B of a compile-time v4 option: AB_FLAG=-DX=0 vs the default build, alternating.
mkdir -p gpurun_out
: > gpurun_out/ab.log
for round in 1 2; do
  for flags in "" "$AB_FLAG"; do
    rm -f paper_2101_03403_b200/_build/blind_rotate_v4.cu.o
    CVM_NVCC_EXTRA="$flags" python paper_2101_03403_b200/build.py >> gpurun_out/ab_build.log 2>&1 || exit 1
    echo "flags=[$flags]" >> gpurun_out/ab.log
    N_NAND=${N_NAND:-4736} VARIANTS=6085,6085 KS_VARIANTS=9 timeout 180 python tools/variant_sweep.py 2>&1 | grep "^6085" >> gpurun_out/ab.log
  done
done
