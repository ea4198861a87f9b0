"""Configs 2-5 on the GPU: decrypted results equal the reference SimBackend's
golden results (tests/golden/, produced by running the reference itself)."""
import gzip
import json
import os

import numpy as np
import pytest

import paper_2101_03403_b200 as P

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")
with gzip.open(os.path.join(GOLD, "vectors.json.gz"), "rt") as fh:
    VECTORS = json.load(fh)
PROGRAMS = json.load(open(os.path.join(GOLD, "programs.json")))


def _golden(op, width, limit):
    ow = P.api.lib.cvm_fu_out_width(P.FU[op], width)
    rows = [r for r in VECTORS[op] if len(r[3]) == ow]
    return rows[:limit]


def _run_batch(keyset, ctx, op, width, rows, seed):
    a = keyset.encrypt_words([r[0] for r in rows], width, seed)
    b = keyset.encrypt_words([r[1] for r in rows], width, seed + 1)
    c = None
    if op in ("add_cin", "addsub"):
        c = keyset.encrypt(np.array([r[2] for r in rows], np.uint8), seed + 2)
    out, st = P.fu_batch(ctx, op, width, a, b, c)
    bits = keyset.decrypt(out.reshape(-1, 631)).reshape(len(rows), -1)
    return ["".join(str(x) for x in row) for row in bits], st


@pytest.mark.parametrize("op,n", [("add", 32), ("add_cin", 16), ("sub", 16), ("addsub", 16),
                                  ("cmp", 32), ("and", 16), ("orr", 16), ("eor", 16),
                                  ("orn", 16), ("lsl", 16), ("lsr", 16), ("asr", 8)])
def test_config2_3_units_16bit(op, n, keyset, ctx):
    rows = _golden(op, 16, n)
    got, st = _run_batch(keyset, ctx, op, 16, rows, 300 + P.FU[op] * 7)
    assert got == [r[3] for r in rows]
    assert st["bootstrapped"] > 0


def test_config4_mul16(keyset, ctx):
    rows = _golden("umul", 16, 8)
    got, st = _run_batch(keyset, ctx, "umul", 16, rows, 501)
    assert got == [r[3] for r in rows]
    assert st["last_flush_levels"] == 118


def test_div16_and_smul16(keyset, ctx):
    for op, seed in (("udiv", 601), ("smul", 611)):
        rows = _golden(op, 16, 4)
        got, _ = _run_batch(keyset, ctx, op, 16, rows, seed)
        assert got == [r[3] for r in rows], op


def test_config5_program_on_gpu(keyset, ctx):
    """BASELINE configs[4]: 8 encrypted 16-bit registers, 64 random
    instructions + UDIV, dataflow-scheduled across instruction fences."""
    meta = PROGRAMS[0]
    bk = P.Backend(ctx, keyset)
    mem_ct = keyset.encrypt_words(meta["mem"], 16, 701)
    mem = [bk.import_lwe(w) for w in mem_ct]
    regs, nzcv = bk.machine_run([tuple(i) for i in meta["insns"]], mem)
    # the key owner decrypts the final state: one flush, evaluating only the
    # cone of influence of the 8 registers and NZCV (dead gates skipped)
    bits = bk.decrypt_bits(np.concatenate([regs.ravel(), nzcv]))
    words = bits[:128].reshape(8, 16).astype(np.int64)
    vals = [int((w << np.arange(16)).sum()) for w in words]
    assert vals == meta["regs"]
    assert list(bits[128:]) == meta["nzcv"]
    st = bk.stats()
    assert st["flushes"] == 1  # one flush for the whole program (no branches)
    assert st["bootstrapped"] == 26038  # recorded, as the reference DAG
    assert st["executed"] == 8483       # live cone of the outputs in that DAG
    assert st["pending"] == 26038 - 8483


def _live_gates(nodes, outs):
    """Bootstrapped gates in the cone of influence of `outs` (reference DAG)."""
    mark = np.zeros(len(nodes), bool)
    stack = list(outs)
    while stack:
        i = stack.pop()
        if mark[i - 1]:
            continue
        mark[i - 1] = True
        nd = nodes[i - 1][2]
        stack.extend(int(x) for x in nodes[i - 1][3:3 + nd])
    boot = (nodes[:, 1] == 0) & (nodes[:, 0] >= 3)
    return int((boot & mark).sum())


def test_demand_driven_flush_keeps_dead_gates_pending(keyset, ctx):
    """Decrypting the low half of a MUL16 evaluates exactly the cone of those
    16 bits in the reference DAG (1,293 of 3,376 gates); asking for the high
    half afterwards evaluates the remaining live gates, same results."""
    d = np.load(os.path.join(GOLD, "dags.npz"))
    nodes, outs = d["umul_16_nodes"], d["umul_16_out"]
    lo_live = _live_gates(nodes, outs[:16])
    all_live = _live_gates(nodes, outs)
    assert lo_live == 1293
    bk = P.Backend(ctx, keyset)
    a = bk.import_lwe(keyset.encrypt_words([0xBEEF], 16, 801)[0])
    b = bk.import_lwe(keyset.encrypt_words([0x1234], 16, 802)[0])
    p = bk.fu("umul", a, b)
    assert bk.decrypt_word(p[:16]) == (0xBEEF * 0x1234) & 0xFFFF
    st = bk.stats()
    assert st["executed"] == lo_live and st["pending"] == 3376 - lo_live
    assert bk.decrypt_word(p[16:]) == (0xBEEF * 0x1234) >> 16
    st = bk.stats()
    assert st["executed"] == all_live and st["pending"] == 3376 - all_live
