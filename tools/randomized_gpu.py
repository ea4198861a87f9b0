"""Evidence run: the reference tests' randomized wide-word checks at scale
(alu_add_test.cc RandomizedWide at 16 / 32 bits, AluAddSubSelect
RandomizedWidth16; the multiply / divide / shift / compare units at 16 bits,
alu_shift_mul_div_test.cc) -- seeded random operands through cvm_dag_batch on
the reference-recorded circuits, compared with the reference SimBackend
(refshim.sim_fu_batch) on the same operands.  Division by zero is included
(the reference defines it: all ones).  Summary:
profiles/r02_randomized_gpu.json.

    python tools/randomized_gpu.py [OUT.json]
"""
import json
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "integration"))
import paper_2101_03403_b200 as P  # noqa: E402
import refshim  # noqa: E402

# (op, width, instances); add_cin / addsub take a third (carry / select) bit
PLAN = [("add", 32, 8192), ("sub", 32, 8192), ("add", 16, 8192), ("add_cin", 16, 8192),
        ("addsub", 16, 8192), ("cmp", 16, 8192), ("umul", 16, 2048), ("smul", 16, 2048),
        ("udiv", 16, 2048), ("lsl", 16, 4096), ("lsr", 16, 4096), ("asr", 16, 4096),
        ("orn", 32, 8192), ("eor", 32, 8192)]
CHUNK = 4096
USES_C = {"add_cin", "addsub"}
SHIFTS = {"lsl", "lsr", "asr"}


def main():
    out_path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/randomized.json"
    ks = P.KeySet(10)
    ctx = P.Context(0)
    ctx.upload_keyset(ks)
    rng = np.random.default_rng(31337)
    res = {}
    for op, w, n in PLAN:
        dag = refshim.record_fu(op, w)
        nout = len(dag.outputs)
        a = rng.integers(0, 1 << w, n, dtype=np.uint64)
        # shift amounts are words too; keep most in range so every stage is exercised
        b = (rng.integers(0, w, n, dtype=np.uint64) if op in SHIFTS
             else rng.integers(0, 1 << w, n, dtype=np.uint64))
        if op == "udiv":
            b[::64] = 0  # divide by zero: the reference's all-ones quotient
        c = rng.integers(0, 2, n, dtype=np.uint64) if op in USES_C else None
        want, _, _ = refshim.sim_fu_batch(op, w, a, b, c)
        mism, boots, t0 = 0, 0, time.time()
        for c0 in range(0, n, CHUNK):
            parts = [ks.encrypt_words(a[c0:c0 + CHUNK], w, 40 + c0),
                     ks.encrypt_words(b[c0:c0 + CHUNK], w, 41 + c0)]
            if c is not None:
                parts.append(ks.encrypt(c[c0:c0 + CHUNK].astype(np.uint8), 42 + c0)
                             .reshape(-1, 1, 631))
            got_lwe, st = P.dag_batch(ctx, dag, np.concatenate(parts, axis=1))
            got = ks.decrypt_words(got_lwe.reshape(-1, 631), nout)
            mask = np.uint64((1 << nout) - 1) if nout < 64 else np.uint64(0xFFFFFFFFFFFFFFFF)
            mism += int(np.count_nonzero(got != (want[c0:c0 + CHUNK] & mask)))
            boots += int(st["executed_bootstraps"])
        dt = time.time() - t0
        key = f"{op}{w}"
        res[key] = {"instances": n, "output_bits": nout, "mismatches": mism,
                    "bootstraps": boots, "seconds": round(dt, 1)}
        print(key, res[key], flush=True)
    json.dump({"what": "seeded random operands through cvm_dag_batch on reference-recorded "
                       "circuits vs the reference SimBackend", "results": res},
              open(out_path, "w"), indent=1)
    return 0 if all(r["mismatches"] == 0 for r in res.values()) else 1


if __name__ == "__main__":
    sys.exit(main())
