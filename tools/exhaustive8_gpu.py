"""Evidence run: the reference's exhaustive width-8 suites (alu_exhaustive8_test.cc:
MulUnsigned, MulSigned, DivUnsigned, Bitwise, ShiftRegAllAmounts;
alu_add_test.cc: AluAdd ExhaustiveWidth8 and CarryInExhaustiveWidth8, AluSub
ExhaustiveWidth8, AluAddSubSelect ExhaustiveWidth8BothModes) through the CUDA
path.  Every operand pair is encrypted, evaluated by cvm_dag_batch on the
circuit the reference records, decrypted, and compared with the reference's
own SimBackend on the same operands (refshim.sim_fu_batch) -- no semantics are
restated here.  Too long for the test suite (~25 GPU-minutes); the summary is
committed as profiles/r02_exhaustive8_gpu.json (adder family:
profiles/r02_exhaustive8_adders_gpu.json).

    python tools/exhaustive8_gpu.py [OUT.json] [ops...]
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

W = 8
# op -> operand tuples (a, b[, c]) of the reference test
PAIRS = {
    "add": [(a, b) for a in range(256) for b in range(256)],
    "add_cin": [(a, b, c) for a in range(256) for b in range(256) for c in range(2)],
    "sub": [(a, b) for a in range(256) for b in range(256)],
    "addsub": [(a, b, c) for a in range(256) for b in range(256) for c in range(2)],
    "umul": [(a, b) for a in range(256) for b in range(256)],
    "smul": [(a, b) for a in range(256) for b in range(256)],
    "udiv": [(a, b) for a in range(256) for b in range(1, 256)],
    "and": [(a, b) for a in range(256) for b in range(256)],
    "orr": [(a, b) for a in range(256) for b in range(256)],
    "eor": [(a, b) for a in range(256) for b in range(256)],
    "orn": [(a, b) for a in range(256) for b in range(256)],
    "lsl": [(v, s) for v in range(256) for s in range(8)],
    "lsr": [(v, s) for v in range(256) for s in range(8)],
    "asr": [(v, s) for v in range(256) for s in range(8)],
}
CHUNK = 8192


def main():
    out_path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/exhaustive8.json"
    ops = sys.argv[2:] or list(PAIRS)
    ks = P.KeySet(8)
    ctx = P.Context(0)
    ctx.upload_keyset(ks)
    res = {}
    for op in ops:
        dag = refshim.record_fu(op, W)
        nout = len(dag.outputs)
        pairs = np.array(PAIRS[op], np.uint64)
        cin = pairs[:, 2] if pairs.shape[1] > 2 else None
        want, _, _ = refshim.sim_fu_batch(op, W, pairs[:, 0], pairs[:, 1], cin)
        mism, boots, t0 = 0, 0, time.time()
        for c0 in range(0, len(pairs), CHUNK):
            p = pairs[c0:c0 + CHUNK]
            a = ks.encrypt_words(p[:, 0], W, 10 + c0)
            b = ks.encrypt_words(p[:, 1], W, 11 + c0)
            parts = [a, b]
            if cin is not None:  # the carry-in / select bit follows the operands
                parts.append(ks.encrypt(p[:, 2].astype(np.uint8), 12 + c0).reshape(-1, 1, 631))
            got_lwe, st = P.dag_batch(ctx, dag, np.concatenate(parts, axis=1))
            got = ks.decrypt_words(got_lwe.reshape(-1, 631), nout)
            mask = np.uint64((1 << nout) - 1)
            mism += int(np.count_nonzero(got != (want[c0:c0 + CHUNK] & mask)))
            boots += int(st["executed_bootstraps"])
        dt = time.time() - t0
        res[op] = {"instances": len(pairs), "outputs_bits": nout, "mismatches": mism,
                   "bootstraps": boots, "seconds": round(dt, 1),
                   "bootstraps_per_s": round(boots / dt)}
        print(op, res[op], flush=True)
    doc = {"what": "exhaustive width-8 suites of alu_exhaustive8_test.cc through cvm_dag_batch "
                   "(reference-recorded circuits), compared with the reference SimBackend",
           "results": res}
    json.dump(doc, open(out_path, "w"), indent=1)
    return 0 if all(r["mismatches"] == 0 for r in res.values()) else 1


if __name__ == "__main__":
    sys.exit(main())
