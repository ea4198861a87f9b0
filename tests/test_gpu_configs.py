"""Configs 2-5 on the GPU: decrypted results equal the reference SimBackend's
golden results (tests/golden/, produced by running the reference itself),
for circuits the reference recorded (replayed by cvm_dag_batch)."""
import gzip
import json
import os
import sys

import numpy as np
import pytest

import paper_2101_03403_b200 as P
from conftest import GOLD, USES_C, fu, fu_batch, fu_dag, program_dag

sys.path.insert(0, os.path.join(os.path.dirname(GOLD), "..", "integration"))
import refshim  # noqa: E402

pytestmark = pytest.mark.gpu

with gzip.open(os.path.join(GOLD, "vectors.json.gz"), "rt") as fh:
    VECTORS = json.load(fh)
PROGRAMS = json.load(open(os.path.join(GOLD, "programs.json")))
ALL_OPS = ["add", "add_cin", "sub", "addsub", "cmp", "and", "orr", "eor", "orn", "lsl",
           "lsr", "asr", "umul", "smul", "udiv", "udiv_exact"]
need_shim = pytest.mark.skipif(not refshim.available(),
                               reason="libcvm_refshim.so not built (needs /root/reference)")


def _golden(op, width, limit=None):
    ow = len(fu_dag(op, width).outputs)
    rows = [r for r in VECTORS[op] if len(r[3]) == ow]
    return rows[:limit] if limit else rows


def _run_batch(keyset, ctx, op, width, rows, seed):
    a = keyset.encrypt_words([r[0] for r in rows], width, seed)
    b = keyset.encrypt_words([r[1] for r in rows], width, seed + 1)
    c = None
    if op in USES_C:
        c = keyset.encrypt(np.array([r[2] for r in rows], np.uint8), seed + 2)
    out, st = fu_batch(ctx, op, width, a, b, c)
    bits = keyset.decrypt(out.reshape(-1, 631)).reshape(len(rows), -1)
    return ["".join(str(x) for x in row) for row in bits], st


@pytest.mark.parametrize("op,n", [("add", 32), ("add_cin", 16), ("sub", 16), ("addsub", 16),
                                  ("cmp", 32), ("and", 16), ("orr", 16), ("eor", 16),
                                  ("orn", 16), ("lsl", 16), ("lsr", 16), ("asr", 8)])
def test_config2_3_units_16bit(op, n, keyset, ctx):
    rows = _golden(op, 16, n)
    got, st = _run_batch(keyset, ctx, op, 16, rows, 300 + ALL_OPS.index(op) * 7)
    assert got == [r[3] for r in rows]
    assert st["bootstrapped"] > 0


@pytest.mark.parametrize("op", ALL_OPS)
def test_exhaustive_width4_every_op(op, keyset, ctx):
    """Every operand combination at width 4 (the reference's exhaustive
    vectors, incl. the carry / select input) in one batch through CUDA."""
    rows = _golden(op, 4)
    assert len(rows) == 256 * (2 if op in USES_C else 1)
    got, _ = _run_batch(keyset, ctx, op, 4, rows, 1000 + ALL_OPS.index(op) * 7)
    assert got == [r[3] for r in rows]


def test_reference_fixed_examples_on_gpu(keyset, ctx):
    """The reference tests' fixed examples through CUDA, against the outputs
    the reference run recorded (vectors["fixed"]): 0xFFFF x 0xFFFF =
    0xFFFE0001 (alu_shift_mul_div_test.cc:198-203), signed -1 x -1 = 1 and
    INT_MIN x 2 (:228-237), divisor 0 -> all ones at 8 and 16 bits
    (:316-325), 13 / 7 in exact and widened mode (:341-349)."""
    for k, (op, w, av, bv, cv, bits) in enumerate(VECTORS["fixed"]):
        a = keyset.encrypt_words([av], w, 1500 + 2 * k)
        b = keyset.encrypt_words([bv], w, 1501 + 2 * k)
        out, _ = fu_batch(ctx, op, w, a, b)
        got = "".join(str(x) for x in keyset.decrypt(out.reshape(-1, 631)))
        assert got == bits, (op, w, av, bv)


def test_config4_mul16(keyset, ctx):
    rows = _golden("umul", 16, 8)
    got, st = _run_batch(keyset, ctx, "umul", 16, rows, 501)
    assert got == [r[3] for r in rows]
    assert st["last_flush_levels"] == 118


@pytest.mark.parametrize("op", ["udiv", "smul", "udiv_exact"])
def test_div16_and_smul16(op, keyset, ctx):
    rows = _golden(op, 16, 16)
    got, _ = _run_batch(keyset, ctx, op, 16, rows, 601 + ALL_OPS.index(op))
    assert got == [r[3] for r in rows], op


def _live_gates(nodes, outs):
    """Bootstrapped gates in the cone of influence of `outs` (reference DAG)."""
    mark = np.zeros(len(nodes), bool)
    stack = list(int(o) for o in outs)
    while stack:
        i = stack.pop()
        if mark[i - 1]:
            continue
        mark[i - 1] = True
        nd = nodes[i - 1][2]
        stack.extend(int(x) for x in nodes[i - 1][3:3 + nd])
    boot = (nodes[:, 1] == 0) & (nodes[:, 0] >= 3)
    return int((boot & mark).sum())


@pytest.mark.parametrize("idx", range(len(PROGRAMS)))
def test_config5_programs_on_gpu(idx, keyset, ctx):
    """BASELINE configs[4], all three golden programs: 8 encrypted 16-bit
    registers, 64 random instructions + UDIV, the reference Machine's recorded
    DAG replayed with dataflow scheduling across the instruction fences; only
    the live cone of the final registers and NZCV runs."""
    dag, meta = program_dag(idx)
    mem = keyset.encrypt_words(meta["mem"], 16, 701 + idx)
    out, st = P.dag_batch(ctx, dag, mem.reshape(1, -1, 631))
    bits = keyset.decrypt(out.reshape(-1, 631))
    words = bits[:128].reshape(8, 16).astype(np.int64)
    assert [int((w << np.arange(16)).sum()) for w in words] == meta["regs"]
    assert list(bits[128:]) == meta["nzcv"]
    assert st["flushes"] == 1
    assert st["executed"] == _live_gates(dag.rows(), dag.outputs)
    if idx == 0:
        assert st["bootstrapped"] == 26038 and st["executed"] == 8483


@need_shim
def test_config5_reference_machine_through_the_shim(keyset, ctx):
    """The reference's own Machine on cryptovm::GpuBackend (the drop-in):
    demand-driven, so the live 8,483 of 26,038 recorded gates run."""
    meta = PROGRAMS[0]
    regs, nzcv, st, _ = refshim.run_program_gpu(ctx, keyset, [tuple(i) for i in meta["insns"]],
                                                meta["mem"])
    assert [int(r) for r in regs] == meta["regs"]
    assert list(nzcv) == meta["nzcv"]
    assert st["bootstrapped"] == 26038
    assert st["executed"] == 8483


@need_shim
def test_reference_branchy_program_through_the_shim(keyset, ctx):
    """Branches resolve through the reference's LocalBranchOracle (a
    decrypt_bit of the flags, i.e. a demand-driven flush): 13 x 11 by a loop
    (emulator_test.cc-style), 11 branch queries."""
    prog = [dict(op="MOV", rd=0, has_imm=1, imm=0), dict(op="MOV", rd=1, has_imm=1, imm=13),
            dict(op="MOV", rd=2, has_imm=1, imm=11),
            dict(op="ADD", rd=0, rn=0, rm=1),
            dict(op="SUBS", rd=2, rn=2, has_imm=1, imm=1, sets_flags=1),
            dict(op="B", cond="NE", has_target=1, target=3), dict(op="HALT")]
    for x in prog:
        x.setdefault("rn", -1)
        x.setdefault("rm", -1)
        x.setdefault("rd", -1)
    regs, _, st, bq = refshim.run_program_gpu(ctx, keyset, prog, [], max_steps=1000)
    assert int(regs[0]) == 143 and int(regs[2]) == 0
    assert bq == 11


@need_shim
def test_reference_add_api_through_the_shim(keyset, ctx):
    rng = np.random.default_rng(9)
    a, b = rng.integers(0, 1 << 16, 24), rng.integers(0, 1 << 16, 24)
    sums, carries, st = refshim.add_batch_gpu(ctx, keyset, a, b, 16)
    assert np.array_equal(sums + (carries.astype(np.uint64) << 16), a + b)
    assert st["flushes"] == 1


def test_demand_driven_flush_keeps_dead_gates_pending(keyset, ctx):
    """Decrypting the low half of a MUL16 evaluates exactly the cone of those
    16 bits in the reference DAG (1,293 of 3,376 gates); asking for the high
    half afterwards evaluates the remaining live gates, same results."""
    dag = fu_dag("umul", 16)
    nodes, outs = dag.rows(), dag.outputs
    lo_live = _live_gates(nodes, outs[:16])
    all_live = _live_gates(nodes, outs)
    assert lo_live == 1293
    bk = P.Backend(ctx, keyset)
    a = bk.import_lwe(keyset.encrypt_words([0xBEEF], 16, 801)[0])
    b = bk.import_lwe(keyset.encrypt_words([0x1234], 16, 802)[0])
    p = fu(bk, "umul", a, b)
    assert bk.decrypt_word(p[:16]) == (0xBEEF * 0x1234) & 0xFFFF
    st = bk.stats()
    assert st["executed"] == lo_live and st["pending"] == 3376 - lo_live
    assert bk.decrypt_word(p[16:]) == (0xBEEF * 0x1234) >> 16
    st = bk.stats()
    assert st["executed"] == all_live and st["pending"] == 3376 - all_live


@pytest.mark.parametrize("op", ALL_OPS)
def test_seeded_width8_vectors_every_op(op, keyset, ctx):
    """The reference's seeded 8-bit vectors (128 per op) through CUDA."""
    rows = _golden(op, 8)
    assert len(rows) == 128
    got, _ = _run_batch(keyset, ctx, op, 8, rows, 1400 + ALL_OPS.index(op) * 7)
    assert got == [r[3] for r in rows]


@need_shim
def test_random_programs_on_gpu_match_reference_machine(keyset, ctx):
    """Seeded random programs over the data-path ISA at 8 bits (MOV / LOAD /
    STORE / ADDS / SUBS with immediates, MUL, SMULS, UDIV, shifts, bitwise,
    BFC / BFI / RBIT / REV, CMP): the recorded DAG on the GPU equals the
    reference Machine on SimBackend (emulator_test.cc:486-640's cross-check)."""
    rng = np.random.default_rng(77)
    for k in range(6):
        prog = refshim.random_program(rng, 8)
        mem = rng.integers(0, 256, 4)
        regs, nzcv = refshim.sim_program(prog, mem, 8, 8)
        dag = refshim.record_program(prog, len(mem), 8, 8)
        lwe = keyset.encrypt_words(mem, 8, 2000 + k).reshape(1, -1, 631)
        out, _ = P.dag_batch(ctx, dag, lwe)
        bits = keyset.decrypt(out.reshape(-1, 631))
        got = [int((bits[8 * r:8 * r + 8].astype(np.int64) << np.arange(8)).sum())
               for r in range(8)]
        assert got == [int(x) for x in regs], k
        assert list(bits[64:]) == list(nzcv), k
