"""Backend contract edge cases on the device path (gates.hpp:109-132 semantics,
SURVEY §8 a-2, a-5, a-7, a-16): folded free ops at export time, blob round
trips and the InputError paths, plan replay on new inputs, slab growth,
scratch-slot reuse by cvm_dag_batch, and concurrent recording."""
import threading

import numpy as np
import pytest

import paper_2101_03403_b200 as P
from conftest import fu, fu_batch
from paper_2101_03403_b200._native import CvmInputError, lib

pytestmark = pytest.mark.gpu
MU = 1 << 29


def test_export_folded_constants_negations_and_duplicates(keyset, ctx):
    bk = P.Backend(ctx, keyset)
    a = bk.encrypt_bit(1)
    c0, c1 = bk.constant(False), bk.constant(True)
    na = bk.unary_gate("NOT", a)
    cp = bk.unary_gate("COPY", na)
    g = bk.binary_gate("AND", a, c1)  # a bootstrapped gate with a constant input
    hs = [c0, c1, na, cp, a, a, g, c0]
    raw = bk.export_lwe(hs)
    assert list(keyset.decrypt(raw)) == [0, 1, 0, 0, 1, 1, 1, 0]
    # trivial samples: a = 0, b = -+1/8
    assert not raw[0, :630].any() and raw[0, 630] == (0 - MU) % 2**32
    assert not raw[1, :630].any() and raw[1, 630] == MU
    # NOT is the negation of every word; COPY aliases it; duplicates agree
    assert np.array_equal(raw[2], (0 - raw[4].astype(np.int64)) % 2**32)
    assert np.array_equal(raw[2], raw[3]) and np.array_equal(raw[4], raw[5])


def test_blob_round_trip_and_input_errors(keyset, ctx):
    bk = P.Backend(ctx, keyset)
    h = bk.binary_gate("XOR", bk.encrypt_bit(1), bk.encrypt_bit(0))
    blob = bk.export_bit(h)
    assert len(blob) == 631 * 4
    h2 = bk.import_bit(blob)
    assert bk.decrypt_bit(h2) is True
    assert bk.decrypt_bit(bk.unary_gate("NOT", h2)) is False
    with pytest.raises(CvmInputError):
        bk.import_bit(blob[:-1])              # sim_backend.cpp:124-126
    with pytest.raises(CvmInputError):
        bk.decrypt_bit(10**9)                  # invalid handle, :53-57
    with pytest.raises(CvmInputError):
        bk.binary_gate("NOT", h, h2)           # wrong kind, :47-49
    with pytest.raises(CvmInputError):
        bk.unary_gate("AND", h)                # :80-83
    with pytest.raises(CvmInputError):
        bk.pop_region()                        # unbalanced, :140-142


def test_plan_replay_on_new_inputs(keyset, ctx):
    """A captured 8-bit adder replays (CUDA graph or plain launches) on new
    ciphertexts written into its input slots."""
    rng = np.random.default_rng(5)
    bk = P.Backend(ctx, keyset)
    a = bk.import_lwe(keyset.encrypt_words(np.array([0]), 8, 1).reshape(-1, 631))
    b = bk.import_lwe(keyset.encrypt_words(np.array([0]), 8, 2).reshape(-1, 631))
    outs = fu(bk, "add", a, b)
    plan = bk.capture_plan()
    assert plan.info()["gates"] > 0
    slots_a = [bk.handle_slot(h)[0] for h in a]
    slots_b = [bk.handle_slot(h)[0] for h in b]
    for trial, graph in enumerate((True, False, True)):
        x, y = (int(v) for v in rng.integers(0, 256, 2))
        ca = keyset.encrypt_words(np.array([x]), 8, 10 + trial).reshape(-1, 631)
        cb = keyset.encrypt_words(np.array([y]), 8, 20 + trial).reshape(-1, 631)
        for i in range(8):
            ctx.upload(slots_a[i], ca[i])
            ctx.upload(slots_b[i], cb[i])
        plan.run(ctx, graph=graph)
        ctx.sync()
        got = keyset.decrypt_words(bk.export_lwe(outs), 9)[0]
        assert got == x + y, (trial, graph)


def test_submit_level_rejects_bad_levels(ctx):
    n = ctx.alloc(2)
    with pytest.raises(CvmInputError):  # NOT is not a bootstrapped kind
        ctx.submit_level([("NOT", [(n, 1, 0)], n + 1)])
    with pytest.raises(CvmInputError):  # output slot beyond capacity
        ctx.submit_level([("AND", [(n, 1, 0), (n, 1, 0)], 1 << 40)])


def test_slab_growth_preserves_contents(keyset, ctx):
    bits = np.array([1, 0, 1, 1, 0], np.uint8)
    c = keyset.encrypt(bits, 77)
    first = ctx.alloc(len(bits))
    ctx.upload(first, c)
    cap0 = lib.cvm_slots_capacity(ctx.handle)
    ctx.alloc(cap0 + 50_000)  # forces a reallocation of the slab
    assert lib.cvm_slots_capacity(ctx.handle) > cap0
    assert np.array_equal(ctx.download(first, len(bits)), c)


def test_fu_batch_reuses_its_scratch_slots(keyset, ctx):
    a = keyset.encrypt_words(np.arange(32) * 7 % 65536, 16, 3)
    b = keyset.encrypt_words(np.arange(32) * 13 % 65536, 16, 4)
    fu_batch(ctx, "add", 16, a, b)
    used = lib.cvm_slots_capacity(ctx.handle)
    for _ in range(3):
        out, st = fu_batch(ctx, "add", 16, a, b)
    assert lib.cvm_slots_capacity(ctx.handle) == used
    sums = keyset.decrypt_words(out.reshape(-1, 631), 17)
    assert np.array_equal(sums, (np.arange(32) * 7 % 65536) + (np.arange(32) * 13 % 65536))


def test_dag_batch_rejects_overflowing_batch(ctx):
    """batch x inputs x 631 must not wrap around 2^64 into a small, matching
    word count (capi.cpp cvm_dag_batch_regions)."""
    import ctypes
    from conftest import fu_dag
    dag = fu_dag("add", 16)
    batch = (1 << 64) // (dag.n_inputs * 631) + 1
    wrapped = (batch * dag.n_inputs * 631) % (1 << 64)
    outs = np.asarray(dag.outputs, np.uint64)
    buf = np.zeros(max(wrapped, 1), np.uint32)
    with pytest.raises(CvmInputError, match="batch too large"):
        P._native.check(lib.cvm_dag_batch(ctx.handle, dag.nodes.ctypes.data, dag.n_nodes,
                                          outs.ctypes.data, len(outs), ctypes.c_uint64(batch),
                                          buf.ctypes.data, wrapped, buf.ctypes.data, 0, None))


def test_concurrent_recording_threads(keyset, ctx):
    """gates.hpp:102-104: independent gates may be recorded concurrently."""
    bk = P.Backend(ctx, keyset)
    n_threads, per = 4, 12
    rng = np.random.default_rng(9)
    xs = rng.integers(0, 2, (n_threads, per, 2))
    ins = [[(bk.encrypt_bit(int(p[0])), bk.encrypt_bit(int(p[1]))) for p in row] for row in xs]
    outs = [[None] * per for _ in range(n_threads)]

    def work(k):
        for i, (ha, hb) in enumerate(ins[k]):
            outs[k][i] = bk.binary_gate("NAND", bk.binary_gate("XOR", ha, hb), ha)

    ts = [threading.Thread(target=work, args=(k,)) for k in range(n_threads)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    got = bk.decrypt_bits(np.array(outs, np.uint64).ravel()).reshape(n_threads, per)
    want = 1 - ((xs[..., 0] ^ xs[..., 1]) & xs[..., 0])
    assert np.array_equal(got, want)


def test_plan_rejects_foreign_context(keyset, ctx):
    """A plan's job tables and slots belong to the context that captured it."""
    bk = P.Backend(ctx, keyset)
    bk.binary_gate("AND", bk.encrypt_bit(1), bk.encrypt_bit(1))
    plan = bk.capture_plan()
    other = P.Context(0)
    try:
        with pytest.raises(CvmInputError):
            plan.run(other)
    finally:
        other.close()
    plan.run(ctx)  # its own context still works
    ctx.sync()


def test_region_attribution(keyset, ctx):
    """Gates carry the region path open at recording (push_region /
    pop_region, as GateDag does); executed counts follow demand-driven
    evaluation (dead gates stay unexecuted)."""
    bk = P.Backend(ctx, keyset)
    a, b = bk.encrypt_bit(1), bk.encrypt_bit(0)
    bk.push_region("adder")
    g1 = bk.binary_gate("AND", a, b)
    bk.push_region("carry")
    g2 = bk.binary_gate("OR", g1, a)
    bk.pop_region()
    bk.push_region("carry")  # the same path is interned once
    bk.binary_gate("XOR", g2, b)
    bk.pop_region()
    bk.pop_region()
    bk.binary_gate("NAND", a, b)
    r = bk.regions()
    assert r == {"": (1, 0), "adder": (1, 0), "adder/carry": (2, 0)}
    assert bk.decrypt_bit(g2) is True
    r = bk.regions()
    assert r == {"": (1, 0), "adder": (1, 1), "adder/carry": (2, 1)}


def test_evaluate_serves_bitwise_decrypts_from_host(keyset, ctx):
    """cvm_backend_evaluate flushes the cone once and keeps the values on the
    host: the reference's bit-by-bit decrypt_word (word.cpp:70-77) then runs
    with no further flush, and the cached words equal the device slots."""
    bk = P.Backend(ctx, keyset)
    a = bk.import_lwe(keyset.encrypt_words([0xBEEF], 16, 61)[0])
    b = bk.import_lwe(keyset.encrypt_words([0x1234], 16, 62)[0])
    out = fu(bk, "add", a, b)
    bk.evaluate(out)
    st0 = bk.stats()
    bits = [bk.decrypt_bit(int(h)) for h in out]
    st1 = bk.stats()
    assert st1["flushes"] == st0["flushes"] == 1
    assert sum(int(x) << i for i, x in enumerate(bits)) == 0xBEEF + 0x1234
    got = bk.export_lwe(out)  # from the cache
    for h, row in zip(out, got):
        slot, sign, const = bk.handle_slot(int(h))
        dev = ctx.download(slot, 1)[0].astype(np.int64)
        want = (sign * dev) % 2**32
        want[630] = (want[630] + const) % 2**32
        assert np.array_equal(row, want.astype(np.uint32))


def test_recorded_table_keeps_reference_regions(keyset, ctx):
    """A table recorded by the reference carries GateDag region indices and
    names; replayed on the device, every bootstrapped gate is attributed to
    its reference region path (the labels of the NVTX launch ranges)."""
    import os
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                    "integration"))
    import refshim
    if not refshim.available():
        pytest.skip("libcvm_refshim.so not built")
    dag = refshim.record_fu("add", 16)
    assert dag.regions[:2] == ["", "adder"] and "adder/sum" in dag.regions
    bk = P.Backend(ctx, keyset)
    ins = bk.import_lwe(np.concatenate([keyset.encrypt_words([7], 16, 71)[0],
                                        keyset.encrypt_words([9], 16, 72)[0]]))
    out = bk.replay_outputs(dag, ins)
    gates = (dag.nodes["input"] == 0) & (dag.nodes["kind"] >= P.KIND["NAND"])
    want = {}
    for r, n in zip(*np.unique(dag.nodes["region"][gates], return_counts=True)):
        want[dag.regions[r]] = int(n)
    got = {k: v[0] for k, v in bk.regions().items() if v[0]}
    assert got == want
    assert bk.decrypt_word(out) == 16
    assert sum(v[1] for v in bk.regions().values()) == bk.stats()["executed"]


def test_replay_rejects_bad_region_index_before_recording(keyset, ctx):
    """A region index past the table's names is an InputError raised before any
    gate of the table is recorded (backend.cpp GpuBackend::replay)."""
    from conftest import fu_dag
    dag = fu_dag("and", 4)
    nodes = dag.nodes.copy()
    gate = np.flatnonzero(nodes["input"] == 0)[0]
    nodes["region"][gate] = 5
    bad = P.Dag(nodes, dag.outputs, regions=["", "a", "b"])
    bk = P.Backend(ctx, keyset)
    ins = bk.import_lwe(keyset.encrypt_words([3, 5], 4, 9).reshape(-1, 631))
    before = len(bk.nodes())
    with pytest.raises(CvmInputError, match="region index out of range"):
        bk.replay(bad, ins)
    assert len(bk.nodes()) == before


def test_empty_and_degenerate_inputs(keyset, ctx):
    """Empty batches, levels, tables and handle lists are no-ops, and a table
    whose outputs are its inputs (no gates) returns the input ciphertexts."""
    from conftest import fu_dag
    dag = fu_dag("add", 16)
    out, st = P.dag_batch(ctx, dag, np.zeros((0, dag.n_inputs, 631), np.uint32))
    assert out.shape == (0, len(dag.outputs), 631) and st["executed"] == 0
    ctx.submit_level([])
    ctx.sync()
    bk = P.Backend(ctx, keyset)
    assert bk.export_lwe([]).shape == (0, 631)
    bk.evaluate([])
    assert len(bk.replay(P.Dag(np.zeros(0, P.DAG_DTYPE), []), [])) == 0
    # identity table: two input nodes, outputs = the inputs in swapped order
    ident = P.Dag.from_rows([[0, 1, 0, 0, 0, 0, 0], [0, 1, 0, 0, 0, 0, 0]], [2, 1])
    lwe = keyset.encrypt(np.array([1, 0]), 5)
    got, st = P.dag_batch(ctx, ident, lwe.reshape(1, 2, 631))
    assert np.array_equal(got[0], lwe[::-1]) and st["executed"] == 0
