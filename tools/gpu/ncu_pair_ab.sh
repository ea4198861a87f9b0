mkdir -p gpurun_out
for lib in "" "paper_2101_03403_b200/_lib_ab/libcvm_head.so"; do
CVM_LIB_PATH="$lib" N_NAND=74 VARIANTS=96 KS_VARIANTS=9 timeout 600 ncu --clock-control none -k regex:blind_rotate_pair -c 1 --metrics l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum,gpu__time_duration.sum python tools/variant_sweep.py > gpurun_out/ncu_pair_$([ -z "$lib" ] && echo new || echo head).log 2>&1
done
