#!/bin/bash
# A/B of builds of the library (AB_LIBS = space-separated .so paths; TREE =
# the tree's own build), alternating AB_ROUNDS times over AB_CASES (N:variant).
mkdir -p gpurun_out
: > gpurun_out/ablib.log
for round in $(seq ${AB_ROUNDS:-2}); do
  for lib in ${AB_LIBS}; do
    [ "$lib" = TREE ] && lib=""
    echo "lib=[$lib]" >> gpurun_out/ablib.log
    for nv in ${AB_CASES:-74:96 4736:6085}; do
      n=${nv%%:*}; v=${nv##*:}
      CVM_LIB_PATH="$lib" N_NAND=$n VARIANTS=$v,$v KS_VARIANTS=9 timeout 180 python tools/variant_sweep.py 2>&1 | grep "^$v " | tail -1 | sed "s/^/N=$n /" | cut -c1-60 >> gpurun_out/ablib.log
    done
  done
done
