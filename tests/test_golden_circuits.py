"""Recorded circuits against the reference's golden fixtures (no GPU needed).

The B200 library holds no copy of the reference's functional units or
emulator: the reference records them (integration/cryptovm_dag_export.cpp,
driving the unmodified alu.cpp / emulator.cpp compiled from /root/reference)
and the library replays the table (cvm_backend_replay_dag / cvm_dag_batch).
These tests check, on the cleartext recorder (SimBackend semantics):
  * the live recorder (integration/refshim.py) emits exactly the golden DAGs
    that tests/golden/make_golden.py stored from the reference run;
  * replaying a table re-creates it node for node;
  * replayed circuits compute the reference's golden results, including the
    fixed examples the reference's own tests single out.
"""
import gzip
import json
import os
import sys

import numpy as np
import pytest

import paper_2101_03403_b200 as P
from conftest import GOLD, USES_C, fu_dag, program_dag

sys.path.insert(0, os.path.join(os.path.dirname(GOLD), "..", "integration"))
import refshim  # noqa: E402

DAGS = np.load(os.path.join(GOLD, "dags.npz"))
with gzip.open(os.path.join(GOLD, "vectors.json.gz"), "rt") as fh:
    VECTORS = json.load(fh)
PROGRAMS = json.load(open(os.path.join(GOLD, "programs.json")))
REF_OPS = [op for op in refshim.FU_OPS if op != "mul_lo"]
need_shim = pytest.mark.skipif(not refshim.available(),
                               reason="libcvm_refshim.so not built (needs /root/reference)")


def _replay_clear(dag, in_bits):
    """Replay on the cleartext recorder: returns (backend, output handles)."""
    b = P.Backend()
    ins = np.array([b.encrypt_bit(int(x)) for x in in_bits], np.uint64)
    return b, b.replay_outputs(dag, ins)


def _operand_bits(op, w, av, bv, cv):
    bits = [(av >> i) & 1 for i in range(w)] + [(bv >> i) & 1 for i in range(w)]
    return bits + ([cv] if op in USES_C else [])


@need_shim
@pytest.mark.parametrize("w", [4, 8, 16])
@pytest.mark.parametrize("op", REF_OPS)
def test_recorder_emits_the_golden_dag(op, w):
    d = refshim.record_fu(op, w)
    assert np.array_equal(d.rows(), DAGS[f"{op}_{w}_nodes"])
    assert np.array_equal(d.outputs, DAGS[f"{op}_{w}_out"])


@need_shim
@pytest.mark.parametrize("w", [4, 8, 16])
def test_recorder_mul_lo_is_umul_low_half(w):
    """MUL as Machine::execute issues it (emulator.cpp:271-285): the
    mul_unsigned DAG, low half kept."""
    d = refshim.record_fu("mul_lo", w)
    assert np.array_equal(d.rows(), DAGS[f"umul_{w}_nodes"])
    assert np.array_equal(d.outputs, DAGS[f"umul_{w}_out"][:w])


@need_shim
@pytest.mark.parametrize("idx", range(len(PROGRAMS)))
def test_recorder_program_dag_is_golden(idx):
    dag, meta = program_dag(idx)
    rec = refshim.record_program([tuple(i) for i in meta["insns"]], len(meta["mem"]))
    assert np.array_equal(rec.rows(), dag.rows())
    assert np.array_equal(rec.outputs, dag.outputs)


@pytest.mark.parametrize("w", [4, 16])
@pytest.mark.parametrize("op", ["add", "cmp", "lsl", "umul", "udiv", "addsub"])
def test_replay_recreates_the_table(op, w):
    dag = fu_dag(op, w)
    b, _ = _replay_clear(dag, np.zeros(dag.n_inputs, np.uint8))
    assert np.array_equal(b.nodes(), dag.rows())


@pytest.mark.parametrize("op", REF_OPS)
def test_vectors_match_reference(op):
    """Every golden vector (exhaustive at width 4, seeded at 8 and 16)."""
    dags = {}
    for av, bv, cv, bits in VECTORS[op]:
        w = next(wd for wd in (4, 8, 16) if len(fu_dag(op, wd).outputs) == len(bits))
        dag = dags.setdefault(w, fu_dag(op, w))
        b, out = _replay_clear(dag, _operand_bits(op, w, av, bv, cv))
        assert "".join(str(x) for x in b.decrypt_bits(out)) == bits, (op, w, av, bv, cv)


def test_reference_fixed_examples():
    """The fixed examples of the reference's own tests, as the reference run
    recorded them (vectors["fixed"], tests/golden/make_golden.py FIXED):
    0xFFFF x 0xFFFF = 0xFFFE0001 (alu_shift_mul_div_test.cc:198-203), signed
    -1 x -1 and INT_MIN x 2 (:228-237), divisor 0 -> all ones (:316-325),
    13 / 7 exact-mode overflow vs widened (:341-349)."""
    fixed = VECTORS["fixed"]
    assert len(fixed) == 11
    expect = {("umul", 16, 0xFFFF, 0xFFFF): 0xFFFE0001, ("smul", 16, 0xFFFF, 0xFFFF): 1,
              ("smul", 16, 0x8000, 2): 0xFFFF0000, ("udiv", 4, 13, 7): 1}
    for op, w, av, bv, cv, bits in fixed:
        b, out = _replay_clear(fu_dag(op, w), _operand_bits(op, w, av, bv, cv))
        assert "".join(str(x) for x in b.decrypt_bits(out)) == bits, (op, w, av, bv)
        val = int(bits[::-1], 2)
        if (op, w, av, bv) in expect:
            assert val == expect[(op, w, av, bv)]
        elif op == "udiv":
            assert val == (1 << w) - 1  # divisor 0
        else:
            assert op == "udiv_exact" and val != 1  # the documented overflow


@pytest.mark.parametrize("idx", range(len(PROGRAMS)))
def test_config5_program_replay_matches_reference(idx):
    dag, meta = program_dag(idx)
    bits = [(v >> i) & 1 for v in meta["mem"] for i in range(16)]
    b, out = _replay_clear(dag, bits)
    vals = b.decrypt_bits(out)
    regs = [int((vals[16 * r:16 * r + 16].astype(np.int64) << np.arange(16)).sum())
            for r in range(8)]
    assert regs == meta["regs"]
    assert list(vals[128:]) == meta["nzcv"]


def test_level_statistics_match_survey():
    """Dataflow depths of the configs' units."""
    expect = {("add", 16): (195, 9), ("cmp", 16): (217, 14), ("lsl", 16): (64, 4),
              ("umul", 16): (3376, 118), ("udiv", 16): (4016, 208), ("and", 16): (16, 1)}
    for (op, w), (gates, levels) in expect.items():
        dag = fu_dag(op, w)
        b, _ = _replay_clear(dag, np.zeros(dag.n_inputs, np.uint8))
        st = b.stats()
        assert st["bootstrapped"] == gates == dag.bootstrapped(), op
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


def test_replay_rejects_malformed_tables():
    dag = fu_dag("add", 4)
    b = P.Backend()
    ins = np.array([b.encrypt_bit(0) for _ in range(dag.n_inputs)], np.uint64)
    with pytest.raises(P.CvmInputError):
        b.replay(dag, ins[:-1])  # input count differs from the table's
    bad = P.Dag(dag.nodes.copy(), dag.outputs)
    i = int(np.flatnonzero(bad.nodes["kind"] == P.KIND["AND"])[0])
    bad.nodes["dep"][i, 0] = i + 1  # refers to itself: not an earlier node
    with pytest.raises(P.CvmInputError):
        b.replay(bad, ins)
    bad = P.Dag(dag.nodes.copy(), dag.outputs)
    bad.nodes["ndeps"][i] = 3  # a binary gate with three operands
    with pytest.raises(P.CvmInputError):
        b.replay(bad, ins)
    bad = P.Dag(dag.nodes.copy(), dag.outputs)
    bad.nodes["kind"][i] = 14  # no such GateKind
    with pytest.raises(P.CvmInputError):
        b.replay(bad, ins)


@need_shim
def test_random_programs_replay_matches_reference_machine():
    """30 seeded random straight-line programs over the data-path ISA at 8
    bits (the shape of emulator_test.cc:486-640): the recorded DAG replayed
    on the cleartext recorder gives the reference Machine's registers and
    NZCV (Machine on SimBackend, cvmref_sim_program)."""
    rng = np.random.default_rng(4242)
    for _ in range(30):
        prog = refshim.random_program(rng, 8)
        mem = rng.integers(0, 256, 4)
        regs, nzcv = refshim.sim_program(prog, mem, 8, 8)
        dag = refshim.record_program(prog, len(mem), 8, 8)
        bits = [(int(v) >> i) & 1 for v in mem for i in range(8)]
        b, out = _replay_clear(dag, bits)
        vals = b.decrypt_bits(out)
        got = [int((vals[8 * k:8 * k + 8].astype(np.int64) << np.arange(8)).sum())
               for k in range(8)]
        assert got == [int(x) for x in regs]
        assert list(vals[64:]) == list(nzcv)
