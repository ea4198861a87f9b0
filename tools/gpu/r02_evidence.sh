#!/bin/bash
# Round-2 evidence on the HEAD build: launch list + per-launch DRAM traffic of
# the bench command, ncu --set full of the v4 kernel (bench), the default key
# switch (split-K tcgen05 + ks_reduce) and the pair kernel on a 74-gate level.
mkdir -p gpurun_out
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --print-units base --csv --log-file gpurun_out/traffic.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu --no-extras > gpurun_out/traffic_run.log 2>&1
echo "traffic rc=$?" >> gpurun_out/traffic_run.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:blind_rotate_kernel_v4 -c 1 \
  -o gpurun_out/r02_ncu_v4 -f python bench.py --steps 1 --warmup 1 --no-cpu --no-extras > gpurun_out/ncu_v4.log 2>&1
echo "v4 rc=$?" >> gpurun_out/ncu_v4.log
N_NAND=74 VARIANTS=96 KS_VARIANTS=9 timeout 900 ncu --set full --import-source on --clock-control none \
  -k regex:'key_switch_tc|ks_reduce|blind_rotate_pair' -c 6 -o gpurun_out/r02_ncu_narrow -f \
  python tools/variant_sweep.py > gpurun_out/ncu_narrow.log 2>&1
echo "narrow rc=$?" >> gpurun_out/ncu_narrow.log
N_NAND=7104 VARIANTS=6085 KS_VARIANTS=9 timeout 900 ncu --set full --clock-control none \
  -k regex:'key_switch_tc' -c 2 -o gpurun_out/r02_ncu_ks_wide -f \
  python tools/variant_sweep.py > gpurun_out/ncu_ks_wide.log 2>&1
echo "kswide rc=$?" >> gpurun_out/ncu_ks_wide.log
