#!/bin/bash
# Full validation: GPU tests, default bench (with CPU baseline and the other
# configs), the reference arm, smoke, and a timing breakdown of cvm_dag_batch.
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1200 python bench.py > gpurun_out/bench_full.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_full.log
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref.log
CVM_DAG_TIMING=1 timeout 300 python - > gpurun_out/dag_timing.log 2>&1 <<'PY'
import sys, numpy as np
sys.path.insert(0, "integration"); sys.path.insert(0, ".")
import refshim, paper_2101_03403_b200 as P
ks = P.KeySet(1); ctx = P.Context(0); ctx.upload_keyset(ks)
d = refshim.record_fu("add", 16)
rng = np.random.default_rng(0)
lwe = np.concatenate([ks.encrypt_words(rng.integers(0, 65536, 256), 16, 1),
                      ks.encrypt_words(rng.integers(0, 65536, 256), 16, 2)], axis=1)
for _ in range(3):
    P.dag_batch(ctx, d, lwe)
PY
