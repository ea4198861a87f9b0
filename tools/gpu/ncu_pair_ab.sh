#!/bin/bash
# Warp-state stall breakdown of the pair kernel for two library builds (NCU_LIBS).
mkdir -p gpurun_out
for lib in $NCU_LIBS; do
  tag=$(basename $lib .so)
  CVM_LIB_PATH="$lib" N_NAND=74 VARIANTS=96 KS_VARIANTS=9 timeout 600 ncu --clock-control none -k regex:blind_rotate_pair -c 1 \
    --section WarpStateStats --section SchedulerStats --metrics l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,smsp__inst_executed.sum,gpu__time_duration.sum \
    --print-units base python tools/variant_sweep.py > gpurun_out/ncu_pair_$tag.log 2>&1
done
