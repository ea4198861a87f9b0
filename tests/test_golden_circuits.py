"""Host logic against the reference's golden fixtures (no GPU needed).

tests/golden/ was produced by running the reference implementation itself
(oracle/ref_golden.cpp linked against /root/reference/proj/core/src, script
tests/golden/make_golden.py).  These tests check that the product's C++
functional units and machine (paper_2101_03403_b200/csrc/alu.cpp,
machine.cpp), recorded through the cleartext recorder, emit exactly the
reference's gate DAG node for node and compute the reference's results.
"""
import gzip
import json
import os

import numpy as np
import pytest

import paper_2101_03403_b200 as P

GOLD = os.path.join(os.path.dirname(__file__), "golden")
DAGS = np.load(os.path.join(GOLD, "dags.npz"))
with gzip.open(os.path.join(GOLD, "vectors.json.gz"), "rt") as fh:
    VECTORS = json.load(fh)
PROGRAMS = json.load(open(os.path.join(GOLD, "programs.json")))
PROG_ARR = np.load(os.path.join(GOLD, "programs.npz"))

USES_C = {"add_cin", "addsub"}
# ops with a reference fixture; "mul_lo" (the emulator's MUL) is checked below
REF_OPS = [op for op in P.FU_OPS if op != "mul_lo"]


def _record(op, w, av=0, bv=0, cv=0):
    b = P.Backend()  # cleartext recorder
    a = b.encrypt_word(av, w)
    bb = b.encrypt_word(bv, w)
    c = b.encrypt_bit(cv) if op in USES_C else 0
    return b, b.fu(op, a, bb, c)


@pytest.mark.parametrize("w", [4, 8, 16])
@pytest.mark.parametrize("op", REF_OPS)
def test_dag_identical_to_reference(op, w):
    b, out = _record(op, w)
    gold = DAGS[f"{op}_{w}_nodes"]
    mine = b.nodes()
    assert mine.shape == gold.shape
    assert np.array_equal(mine, gold)
    assert np.array_equal(out, DAGS[f"{op}_{w}_out"])


@pytest.mark.parametrize("op", REF_OPS)
def test_vectors_match_reference(op):
    # the operand width is implied by the result length (distinct per width)
    width_of = {P.api.lib.cvm_fu_out_width(P.FU[op], wd): wd for wd in (4, 8, 16)}
    for av, bv, cv, bits in VECTORS[op]:
        w = width_of[len(bits)]
        b, out = _record(op, w, av, bv, cv)
        got = "".join(str(x) for x in b.decrypt_bits(out))
        assert got == bits, (op, w, av, bv, cv)


def test_reference_edge_examples():
    """Fixed examples the reference tests single out
    (alu_shift_mul_div_test.cc): 0xFFFF * 0xFFFF and division by zero."""
    b, out = _record("umul", 16, 0xFFFF, 0xFFFF)
    assert b.decrypt_word(out) == 0xFFFE0001
    b, out = _record("udiv", 8, 200, 0)
    assert b.decrypt_word(out) == 0xFF
    b, out = _record("udiv_exact", 4, 13, 7)  # exact-mode overflow case
    want = [v for v in VECTORS["udiv_exact"] if v[0] == 13 and v[1] == 7][0][3]
    assert "".join(str(x) for x in b.decrypt_bits(out)) == want


@pytest.mark.parametrize("meta", PROGRAMS, ids=[f"seed{m['seed']}" for m in PROGRAMS])
def test_config5_program_matches_reference(meta):
    b = P.Backend()
    mem = [b.encrypt_word(v, 16) for v in meta["mem"]]
    prog = [tuple(i) for i in meta["insns"]]
    regs, nzcv = b.machine_run(prog, mem)
    assert [b.decrypt_word(r) for r in regs] == meta["regs"]
    assert list(b.decrypt_bits(nzcv)) == meta["nzcv"]
    gold = PROG_ARR[f"p{meta['seed']}_nodes"]
    assert np.array_equal(b.nodes(), gold)


def test_level_statistics_match_survey():
    """Dataflow depths of the configs' units."""
    expect = {("add", 16): (195, 9), ("cmp", 16): (217, 14), ("lsl", 16): (64, 4),
              ("umul", 16): (3376, 118), ("udiv", 16): (4016, 208), ("and", 16): (16, 1)}
    for (op, w), (gates, levels) in expect.items():
        b, _ = _record(op, w)
        st = b.stats()
        assert st["bootstrapped"] == gates, op
        assert st["levels_run"] == levels, op


def test_input_errors_mirror_reference():
    b = P.Backend()
    with pytest.raises(P.CvmInputError):
        b.binary_gate("AND", 0, 0)  # invalid handle (sim_backend.cpp:53-57)
    h = b.constant(True)
    with pytest.raises(P.CvmInputError):
        b.binary_gate("NOT", h, h)  # not a binary gate (sim_backend.cpp:47-49)
    with pytest.raises(P.CvmInputError):
        b.unary_gate("AND", h)  # not a unary gate (sim_backend.cpp:80-83)
    with pytest.raises(P.CvmInputError):
        b.pop_region()  # unbalanced (sim_backend.cpp:140-142)
    with pytest.raises(P.CvmInputError):
        b.fu("add", np.array([h, h], np.uint64), np.array([h], np.uint64))  # width mismatch
    with pytest.raises(P.CvmInputError):
        b.fu("lsl", np.array([h] * 3, np.uint64), np.array([h] * 3, np.uint64))  # not 2^k


@pytest.mark.parametrize("w", [4, 8, 16])
def test_mul_lo_is_the_reference_umul_dag_low_half(w):
    """mul_lo records exactly the reference mul_unsigned DAG and returns its
    low half -- what Machine::execute keeps for MUL (emulator.cpp:271-285)."""
    b, out = _record("mul_lo", w)
    assert np.array_equal(b.nodes(), DAGS[f"umul_{w}_nodes"])
    assert np.array_equal(out, DAGS[f"umul_{w}_out"][:w])
    for av, bv, cv, bits in VECTORS["umul"]:
        if len(bits) != 2 * w:
            continue
        b, out = _record("mul_lo", w, av, bv)
        assert "".join(str(x) for x in b.decrypt_bits(out)) == bits[:w]
