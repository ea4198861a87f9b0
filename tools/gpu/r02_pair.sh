#!/bin/bash
# Pair-kernel experiment: build, parity + determinism, latency sweep, phase breakdown.
mkdir -p gpurun_out
python paper_2101_03403_b200/build.py > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x \
  -k "variants_bit_identical or deterministic or random_circuits or nand_level" > gpurun_out/pair_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pair_tests.log
for n in 1 26 74; do N_NAND=$n VARIANTS=96 KS_VARIANTS=9 timeout 300 python tools/variant_sweep.py; done \
  > gpurun_out/pair_sweep.log 2>&1
bash tools/gpu/pair_phases.sh
