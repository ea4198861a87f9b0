"""Debug helper: first node where the GPU and the oracle disagree on a random DAG."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]
import oracle as O  # noqa: E402
import paper_2101_03403_b200 as P  # noqa: E402
from paper_2101_03403_b200.api import GATE_KINDS  # noqa: E402

TR = ["NAND", "AND", "OR", "XOR", "XNOR", "NOR", "ANDNY", "ANDYN", "ORNY", "ORYN"]
ks = P.KeySet(20260808)
k = ks.export()
ok = O.CloudKeys(k["bk"], k["ksk"], O.MODE_NTT)
ctx = P.Context(0)
ctx.upload_keyset(ks)
for seed in (1, 2, 3):
    rng = np.random.default_rng(seed)
    bits = rng.integers(0, 2, 8).astype(np.uint8)
    cins = ks.encrypt(bits, 300 + seed)
    bk = P.Backend(ctx, ks)
    hs = list(bk.import_lwe(cins))
    kinds = TR + ["MUX", "NOT", "COPY", "CONSTANT"]
    for _ in range(40):
        kk = kinds[rng.integers(len(kinds))]
        pick = lambda: int(hs[rng.integers(len(hs))])  # noqa: E731
        if kk == "MUX":
            h = bk.mux_gate(pick(), pick(), pick())
        elif kk in ("NOT", "COPY"):
            h = bk.unary_gate(kk, pick())
        elif kk == "CONSTANT":
            h = bk.constant(bool(rng.integers(2)))
        else:
            h = bk.binary_gate(kk, pick(), pick())
        hs.append(h)
    nodes = bk.nodes()
    ref = O.eval_dag(ok, nodes, cins)
    got = bk.export_lwe(np.arange(1, len(nodes) + 1, dtype=np.uint64))
    bad = [i for i in range(len(nodes)) if not np.array_equal(got[i], ref[i])]
    print("seed", seed, "bad nodes", len(bad), "of", len(nodes))
    for i in bad[:4]:
        kd, inp, nd = nodes[i][:3]
        deps = list(nodes[i][3:3 + nd])
        print("  node", i + 1, GATE_KINDS[kd], "input" if inp else "", "deps", deps,
              [GATE_KINDS[nodes[d - 1][0]] for d in deps],
              "dec gpu/ref", ks.decrypt(got[i:i + 1])[0], ks.decrypt(ref[i:i + 1])[0],
              "ndiff words", int((got[i] != ref[i]).sum()))
