#!/bin/bash
# Round-2 cost tables (reference CostTable grammar) on the HEAD kernels, and a
# launch list of the config-5 program (narrow levels).
mkdir -p gpurun_out/costs
timeout 900 python tools/cost_table.py gpurun_out/costs > gpurun_out/costs.log 2>&1; echo "rc=$?" >> gpurun_out/costs.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --print-units base --csv \
  --log-file gpurun_out/c5_launches.csv python - > gpurun_out/c5_run.log 2>&1 <<'PY'
import json, sys, numpy as np
sys.path.insert(0, "integration"); sys.path.insert(0, ".")
import refshim, paper_2101_03403_b200 as P
ks = P.KeySet(1); ctx = P.Context(0); ctx.upload_keyset(ks)
meta = json.load(open("tests/golden/programs.json"))[0]
dag = refshim.record_program([tuple(i) for i in meta["insns"]], len(meta["mem"]))
out, st = P.dag_batch(ctx, dag, ks.encrypt_words(meta["mem"], 16, 5).reshape(1, -1, 631))
print(st)
PY
echo "rc=$?" >> gpurun_out/c5_run.log
