#!/bin/bash
# Driver-equivalent round-end commands on the HEAD build.
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
s=$(date +%s.%N); timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_final.log 2>&1; echo "bench rc=$? wall=$(echo "$(date +%s.%N) - $s" | bc)" >> gpurun_out/bench_final.log
s=$(date +%s.%N); timeout 1200 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_ref_final.log 2>&1; echo "ref rc=$? wall=$(echo "$(date +%s.%N) - $s" | bc)" >> gpurun_out/bench_ref_final.log
