"""GPU parity: the sm_100a path (through the C ABI) against the CPU oracle.

Raw torus32 coefficients must be bit-exact: the oracle computes every
negacyclic product exactly (NTT over 2^64-2^32+1), the GPU with an FP64 FFT
whose rounding error stays far below 1/2, so equality
of every one of the 631 words of every output ciphertext is asserted.
Decrypted bits are checked against the boolean truth tables of
sim_backend.cpp:25-51,98-106.
"""
import numpy as np
import pytest

import oracle as O
import paper_2101_03403_b200 as P
from conftest import fu, fu_batch

pytestmark = pytest.mark.gpu

MU = 1 << 29
TRUTH = {
    "NAND": lambda a, b: 1 - (a & b), "AND": lambda a, b: a & b, "OR": lambda a, b: a | b,
    "XOR": lambda a, b: a ^ b, "XNOR": lambda a, b: 1 - (a ^ b), "NOR": lambda a, b: 1 - (a | b),
    "ANDNY": lambda a, b: (1 - a) & b, "ANDYN": lambda a, b: a & (1 - b),
    "ORNY": lambda a, b: (1 - a) | b, "ORYN": lambda a, b: a | (1 - b),
}


def _bits(n, seed):
    return np.random.default_rng(seed).integers(0, 2, n).astype(np.uint8)


def test_nand_level_bit_exact(keyset, ctx, oracle_keys):
    """Config 1 shape (independent NANDs, one level) at oracle-checkable size."""
    n = 48
    a, b = _bits(n, 1), _bits(n, 2)
    ca, cb = keyset.encrypt(a, 11), keyset.encrypt(b, 12)
    base = ctx.alloc(3 * n)
    ctx.upload(base, ca)
    ctx.upload(base + n, cb)
    ctx.submit_level([("NAND", [(base + i, 1, 0), (base + n + i, 1, 0)], base + 2 * n + i)
                      for i in range(n)])
    ctx.sync()
    out = ctx.download(base + 2 * n, n)
    ref = oracle_keys.gates(np.full(n, O.NAND, np.uint8), ca, cb)
    assert np.array_equal(out, ref)
    assert np.array_equal(keyset.decrypt(out), 1 - (a & b))


@pytest.mark.parametrize("variant", [9, 96, 5247, 6085, 6035, 6015])
def test_kernel_variants_bit_identical(variant, keyset, ctx, oracle_keys):
    """Every blind-rotation kernel variant (one gate per CTA via L1, G gates per
    CTA on a bulk-copy shared-memory key ring) gives the oracle's ciphertexts,
    including a partially filled last CTA (n not a multiple of G)."""
    from paper_2101_03403_b200._native import lib, check
    n = 13
    a, b = _bits(n, 3), _bits(n, 4)
    ca, cb = keyset.encrypt(a, 13), keyset.encrypt(b, 14)
    old = lib.cvm_get_br_variant()
    check(lib.cvm_set_br_variant(variant))
    try:
        base = ctx.alloc(3 * n)
        ctx.upload(base, ca)
        ctx.upload(base + n, cb)
        ctx.submit_level([("XOR", [(base + i, 1, 0), (base + n + i, -1, 0)],
                           base + 2 * n + i) for i in range(n)])
        ctx.sync()
        out = ctx.download(base + 2 * n, n)
    finally:
        check(lib.cvm_set_br_variant(old))
    # XOR(a, NOT b) with the NOT folded into the operand's sign
    nb = (np.uint32(0) - cb).astype(np.uint32)
    ref = oracle_keys.gates(np.full(n, O.XOR, np.uint8), ca, nb)
    assert np.array_equal(out, ref)
    assert np.array_equal(keyset.decrypt(out), a ^ (1 - b))


@pytest.mark.parametrize("n", [192, 700, 1224, 1376, 1584, 1984])
def test_wide_level_planner_bit_identical(n, keyset, ctx, oracle_keys):
    """Auto selection of a wide level: full waves of the v4 warp kernel, then
    the remainder on another v4 wave with fewer warps per SM, on v3 rounds
    and/or latency rounds -- pair or wide (blind_rotate.cu; 192 alone and as
    the remainder of 1376 take three pair rounds).  The sizes hit each combination;
    the result must equal the whole level on one kernel (6085, pinned to the
    oracle by test_kernel_variants_bit_identical)."""
    from paper_2101_03403_b200._native import lib, check
    a, b = _bits(n, 40), _bits(n, 41)
    ca, cb = keyset.encrypt(a, 81), keyset.encrypt(b, 82)
    base = ctx.alloc(4 * n)
    ctx.upload(base, ca)
    ctx.upload(base + n, cb)
    gates = lambda dst: [("AND", [(base + i, 1, 0), (base + n + i, 1, 0)], dst + i)  # noqa: E731
                         for i in range(n)]
    old = lib.cvm_get_br_variant()
    try:
        check(lib.cvm_set_br_variant(0))
        ctx.submit_level(gates(base + 2 * n))
        check(lib.cvm_set_br_variant(6085))
        ctx.submit_level(gates(base + 3 * n))
        ctx.sync()
    finally:
        check(lib.cvm_set_br_variant(old))
    auto, ref = ctx.download(base + 2 * n, n), ctx.download(base + 3 * n, n)
    assert np.array_equal(auto, ref)
    assert np.array_equal(keyset.decrypt(auto), a & b)
    # not only self-consistent: a sample spread over every kernel of the
    # plan (head waves, remainder kernels) against the exact oracle
    idx = np.unique(np.concatenate([np.arange(0, n, max(1, n // 24)), [n - 1]]))
    want = oracle_keys.gates(np.full(len(idx), O.AND, np.uint8), ca[idx], cb[idx])
    assert np.array_equal(auto[idx], want)


def test_wide_mux_level_auto_vs_pinned(keyset, ctx, oracle_keys):
    """A wide MUX level (700 gates = 1,400 blind rotations: a full v4 wave plus
    a remainder, then the split-K key switch over 6 tiles with two extracted
    samples per gate) under the auto selection equals the same level on
    pinned kernels (v4 6085 + unsplit tcgen05 key switch), and decrypts."""
    from paper_2101_03403_b200._native import lib, check
    n = 700
    s, t, f = _bits(n, 50), _bits(n, 51), _bits(n, 52)
    cs, ct, cf = keyset.encrypt(s, 93), keyset.encrypt(t, 94), keyset.encrypt(f, 95)
    base = ctx.alloc(5 * n)
    for k, c in enumerate((cs, ct, cf)):
        ctx.upload(base + k * n, c)
    mux = lambda dst: [("MUX", [(base + i, 1, 0), (base + n + i, 1, 0),  # noqa: E731
                                (base + 2 * n + i, 1, 0)], dst + i) for i in range(n)]
    ob, ok = lib.cvm_get_br_variant(), lib.cvm_get_ks_variant()
    try:
        check(lib.cvm_set_br_variant(0))
        check(lib.cvm_set_ks_variant(0))
        ctx.submit_level(mux(base + 3 * n))
        check(lib.cvm_set_br_variant(6085))
        check(lib.cvm_set_ks_variant(8))
        ctx.submit_level(mux(base + 4 * n))
        ctx.sync()
    finally:
        check(lib.cvm_set_br_variant(ob))
        check(lib.cvm_set_ks_variant(ok))
    auto, pinned = ctx.download(base + 3 * n, n), ctx.download(base + 4 * n, n)
    assert np.array_equal(auto, pinned)
    assert np.array_equal(keyset.decrypt(auto), np.where(s == 1, t, f))
    idx = np.unique(np.concatenate([np.arange(0, n, 29), [n - 1]]))
    want = oracle_keys.gates(np.full(len(idx), O.MUX, np.uint8), cs[idx], ct[idx], cf[idx])
    assert np.array_equal(auto[idx], want)


@pytest.mark.parametrize("op", ["add", "cmp"])
def test_wave_packing_same_results(op, keyset, ctx):
    """The wave-packing levelizer (backend.cpp pack_levels) moves gates
    between their earliest and latest levels: same number of launches, same
    ciphertexts as plain dataflow levels, correct decryptions."""
    from paper_2101_03403_b200._native import lib, check
    rng = np.random.default_rng(12)
    batch = 64  # 12,480 (add) / 13,888 (cmp) gates: packing is active
    av, bv = rng.integers(0, 1 << 16, batch), rng.integers(0, 1 << 16, batch)
    a = keyset.encrypt_words(av, 16, 91)
    b = keyset.encrypt_words(bv, 16, 92)
    old = lib.cvm_get_level_packing()
    res = {}
    try:
        for pack in (1, 0):
            check(lib.cvm_set_level_packing(pack))
            res[pack] = fu_batch(ctx, op, 16, a, b)
    finally:
        check(lib.cvm_set_level_packing(old))
    (o1, s1), (o0, s0) = res[1], res[0]
    assert np.array_equal(o1, o0)
    assert s1["last_flush_levels"] == s0["last_flush_levels"]
    if op == "add":
        vals = keyset.decrypt_words(o1.reshape(-1, 631), 17)
        assert np.array_equal(vals, (av + bv) % (1 << 17))


@pytest.mark.parametrize("ks_variant", [8, 9])
def test_key_switch_variants_bit_identical(ks_variant, keyset, ctx, oracle_keys):
    """Single- and multi-gate key-switch kernels, with plain gates and MUX
    (two extracted samples + 1/8) and a partially filled last CTA."""
    from paper_2101_03403_b200._native import lib, check
    n = 11
    s, t, f = _bits(n, 8), _bits(n, 9), _bits(n, 10)
    cs, ct, cf = keyset.encrypt(s, 61), keyset.encrypt(t, 62), keyset.encrypt(f, 63)
    old = lib.cvm_get_ks_variant()
    check(lib.cvm_set_ks_variant(ks_variant))
    try:
        base = ctx.alloc(5 * n)
        for k, c in enumerate((cs, ct, cf)):
            ctx.upload(base + k * n, c)
        gates = [("MUX", [(base + i, 1, 0), (base + n + i, 1, 0), (base + 2 * n + i, 1, 0)],
                  base + 3 * n + i) for i in range(n)]
        gates += [("ORYN", [(base + i, 1, 0), (base + n + i, 1, 0)], base + 4 * n + i)
                  for i in range(n)]
        ctx.submit_level(gates)
        ctx.sync()
        mux, oryn = ctx.download(base + 3 * n, n), ctx.download(base + 4 * n, n)
    finally:
        check(lib.cvm_set_ks_variant(old))
    assert np.array_equal(mux, oracle_keys.gates(np.full(n, O.MUX, np.uint8), cs, ct, cf))
    assert np.array_equal(oryn, oracle_keys.gates(np.full(n, O.ORYN, np.uint8), cs, ct))


@pytest.mark.parametrize("kind", list(TRUTH))
def test_every_binary_gate_truth_table_and_raw(kind, keyset, ctx, oracle_keys):
    a = np.array([0, 0, 1, 1, 0, 1, 1, 0], np.uint8)
    b = np.array([0, 1, 0, 1, 1, 1, 0, 0], np.uint8)
    ca, cb = keyset.encrypt(a, 21), keyset.encrypt(b, 22)
    bk = P.Backend(ctx, keyset)
    ha, hb = bk.import_lwe(ca), bk.import_lwe(cb)
    hs = [bk.binary_gate(kind, x, y) for x, y in zip(ha, hb)]
    got = bk.export_lwe(hs)
    ref = oracle_keys.gates(np.full(8, O.__dict__[kind], np.uint8), ca, cb)
    assert np.array_equal(got, ref)
    assert np.array_equal(bk.decrypt_bits(hs), TRUTH[kind](a, b))


def test_mux_and_folded_free_ops(keyset, ctx, oracle_keys):
    """MUX (2 bootstraps + 1 key switch) and NOT/COPY/CONSTANT folded into the
    next gate's input combination must equal the oracle evaluating them as
    explicit ciphertext operations."""
    n = 8
    s, t, f = _bits(n, 5), _bits(n, 6), _bits(n, 7)
    cs, ct, cf = keyset.encrypt(s, 31), keyset.encrypt(t, 32), keyset.encrypt(f, 33)
    bk = P.Backend(ctx, keyset)
    hs, ht, hf = bk.import_lwe(cs), bk.import_lwe(ct), bk.import_lwe(cf)
    mux = [bk.mux_gate(x, y, z) for x, y, z in zip(hs, ht, hf)]
    one = bk.constant(True)
    # NOT(s) AND COPY(t), then NOT(that) XOR CONSTANT(1)
    g1 = [bk.binary_gate("AND", bk.unary_gate("NOT", x), bk.unary_gate("COPY", y))
          for x, y in zip(hs, ht)]
    g2 = [bk.binary_gate("XOR", bk.unary_gate("NOT", x), one) for x in g1]
    got_mux, got_g2 = bk.export_lwe(mux), bk.export_lwe(g2)
    ref_mux = oracle_keys.gates(np.full(n, O.MUX, np.uint8), cs, ct, cf)
    neg = lambda c: (np.uint32(0) - c).astype(np.uint32)  # noqa: E731
    r1 = oracle_keys.gates(np.full(n, O.AND, np.uint8), neg(cs), ct)
    r2 = oracle_keys.gates(np.full(n, O.XOR, np.uint8), neg(r1), np.tile(O.trivial(1), (n, 1)))
    assert np.array_equal(got_mux, ref_mux)
    assert np.array_equal(got_g2, r2)
    assert np.array_equal(bk.decrypt_bits(mux), np.where(s == 1, t, f))
    assert np.array_equal(bk.decrypt_bits(g2), ((1 - ((1 - s) & t)) ^ 1))


def test_gate_on_trivial_inputs(keyset, ctx, oracle_keys):
    """Both operands CONSTANT: still bootstrapped (TFHE semantics), still exact."""
    bk = P.Backend(ctx, keyset)
    h = bk.binary_gate("NAND", bk.constant(True), bk.constant(True))
    got = bk.export_lwe([h])
    ref = oracle_keys.gates(np.array([O.NAND], np.uint8), O.trivial(1)[None], O.trivial(1)[None])
    assert np.array_equal(got, ref)
    assert bk.decrypt_bit(h) is False


def test_add16_through_backend_matches_oracle_dag(keyset, ctx, oracle_keys):
    """One ADD16 (195 bootstraps, 9 levels) node-for-node against the oracle
    replaying the reference DAG (tests/golden/dags.npz)."""
    d = np.load("tests/golden/dags.npz")
    nodes = d["add_16_nodes"]
    outs = d["add_16_out"]
    av, bv = 0xBEEF, 0x1234
    ca = keyset.encrypt_words([av], 16, 41)[0]
    cb = keyset.encrypt_words([bv], 16, 42)[0]
    ref = O.eval_dag(oracle_keys, nodes, np.concatenate([ca, cb]))
    bk = P.Backend(ctx, keyset)
    ha, hb = bk.import_lwe(ca), bk.import_lwe(cb)
    out = fu(bk, "add", ha, hb)
    got = bk.export_lwe(out)
    assert np.array_equal(got, ref[outs - 1])
    assert bk.decrypt_word(out[:16]) == (av + bv) & 0xFFFF
    assert bk.decrypt_bit(out[16]) == ((av + bv) >> 16)


def test_fu_batch_add16_decrypts(keyset, ctx):
    rng = np.random.default_rng(11)
    batch = 32
    av = rng.integers(0, 1 << 16, batch)
    bv = rng.integers(0, 1 << 16, batch)
    a = keyset.encrypt_words(av, 16, 51)
    b = keyset.encrypt_words(bv, 16, 52)
    out, st = fu_batch(ctx, "add", 16, a, b)
    vals = keyset.decrypt_words(out.reshape(-1, 631), 17)
    assert np.array_equal(vals, (av + bv) % (1 << 17))
    assert st["last_flush_levels"] == 9
    assert st["bootstrapped"] == 195 * batch


def test_key_switch_tensor_core_multi_tile(keyset, ctx, oracle_keys):
    """The tcgen05 key switch over several 128-gate tiles with a partial last
    tile, MUX and binary gates mixed: unsplit (variant 8) and split along K
    (variant 9: 2 tiles x 5 x 8 CTAs + ks_reduce) equal the oracle."""
    from paper_2101_03403_b200._native import lib, check
    n = 300
    s, t, f = _bits(n, 18), _bits(n, 19), _bits(n, 20)
    cs, ct, cf = keyset.encrypt(s, 71), keyset.encrypt(t, 72), keyset.encrypt(f, 73)
    base = ctx.alloc(5 * n)
    for k, c in enumerate((cs, ct, cf)):
        ctx.upload(base + k * n, c)
    gates = [("MUX", [(base + i, 1, 0), (base + n + i, 1, 0), (base + 2 * n + i, 1, 0)],
              base + 3 * n + i) for i in range(n)]
    gates += [("XNOR", [(base + i, 1, 0), (base + n + i, 1, 0)], base + 4 * n + i)
              for i in range(n)]
    outs = {}
    old = lib.cvm_get_ks_variant()
    try:
        for v in (8, 9):
            check(lib.cvm_set_ks_variant(v))
            ctx.submit_level(gates)
            ctx.sync()
            outs[v] = ctx.download(base + 3 * n, 2 * n)
    finally:
        check(lib.cvm_set_ks_variant(old))
    assert np.array_equal(outs[8], outs[9])
    idx = np.arange(0, n, 7)
    ref_mux = oracle_keys.gates(np.full(len(idx), O.MUX, np.uint8), cs[idx], ct[idx], cf[idx])
    ref_xnor = oracle_keys.gates(np.full(len(idx), O.XNOR, np.uint8), cs[idx], ct[idx])
    assert np.array_equal(outs[9][idx], ref_mux)
    assert np.array_equal(outs[9][n + idx], ref_xnor)
    bits = keyset.decrypt(outs[9])
    assert np.array_equal(bits[:n], np.where(s == 1, t, f))
    assert np.array_equal(bits[n:], 1 - (s ^ t))


def test_per_context_kernel_choice(keyset, ctx):
    """cvm_ctx_set_kernels pins this context's kernels without touching the
    process-wide setting; results are unchanged (every variant is
    bit-identical) and -1 restores 'follow the process'."""
    from paper_2101_03403_b200._native import lib
    n = 40
    a, b = _bits(n, 30), _bits(n, 31)
    ca, cb = keyset.encrypt(a, 32), keyset.encrypt(b, 33)
    base = ctx.alloc(3 * n)
    ctx.upload(base, ca)
    ctx.upload(base + n, cb)
    gates = [("XOR", [(base + i, 1, 0), (base + n + i, 1, 0)], base + 2 * n + i)
             for i in range(n)]
    glob = lib.cvm_get_br_variant(), lib.cvm_get_ks_variant()
    outs = []
    try:
        for br, ks in ((-1, -1), (9, 8), (5247, 9), (6045, 8)):
            ctx.set_kernels(br, ks, -1)
            assert ctx.kernels()["br_variant"] == br
            ctx.submit_level(gates)
            ctx.sync()
            outs.append(ctx.download(base + 2 * n, n))
            assert (lib.cvm_get_br_variant(), lib.cvm_get_ks_variant()) == glob
    finally:
        ctx.set_kernels(-1, -1, -1)
    assert all(np.array_equal(o, outs[0]) for o in outs)
    assert np.array_equal(keyset.decrypt(outs[0]), a ^ b)
    with pytest.raises(P.CvmInputError):
        ctx.set_kernels(4044, -1, -1)  # retired variant


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_random_circuits_bit_exact(seed, keyset, ctx, oracle_keys):
    """Random DAGs over every gate kind (MUX, the ten binary gates, NOT / COPY /
    CONSTANT folded into operands), recorded through the Backend and evaluated
    by dataflow level on the GPU: every node's 631 words equal the oracle
    evaluating the same node table gate by gate."""
    rng = np.random.default_rng(seed)
    bits = rng.integers(0, 2, 8).astype(np.uint8)
    cins = keyset.encrypt(bits, 300 + seed)
    bk = P.Backend(ctx, keyset)
    hs = list(bk.import_lwe(cins))
    kinds = list(TRUTH) + ["MUX", "NOT", "COPY", "CONSTANT"]

    def pick():
        return int(hs[rng.integers(len(hs))])

    for _ in range(40):
        k = kinds[rng.integers(len(kinds))]
        if k == "MUX":
            h = bk.mux_gate(pick(), pick(), pick())
        elif k in ("NOT", "COPY"):
            h = bk.unary_gate(k, pick())
        elif k == "CONSTANT":
            h = bk.constant(bool(rng.integers(2)))
        else:
            h = bk.binary_gate(k, pick(), pick())
        hs.append(h)
    nodes = bk.nodes()
    ref = O.eval_dag(oracle_keys, nodes, cins)
    got = bk.export_lwe(np.arange(1, len(nodes) + 1, dtype=np.uint64))
    assert np.array_equal(got, ref)


def test_random_wide_levels_bit_exact(keyset, ctx, oracle_keys):
    """Two random 320-gate levels (binary gates and MUX mixed, operands with
    folded NOT / COPY): wide enough for the throughput kernel and the tcgen05
    key switch; every node bit-exact against the oracle."""
    rng = np.random.default_rng(99)
    bits = rng.integers(0, 2, 16).astype(np.uint8)
    cins = keyset.encrypt(bits, 400)
    bk = P.Backend(ctx, keyset)
    layer = [int(h) for h in bk.import_lwe(cins)]
    kinds = list(TRUTH) + ["MUX"]
    for _ in range(2):
        src = layer + [int(bk.unary_gate("NOT", h)) for h in layer[:8]]
        nxt = []
        for _ in range(320):
            k = kinds[rng.integers(len(kinds))]
            pick = [src[i] for i in rng.integers(0, len(src), 3)]
            nxt.append(int(bk.mux_gate(*pick) if k == "MUX" else bk.binary_gate(k, *pick[:2])))
        layer = nxt
    nodes = bk.nodes()
    ref = O.eval_dag(oracle_keys, nodes, cins)
    got = bk.export_lwe(np.arange(1, len(nodes) + 1, dtype=np.uint64))
    assert np.array_equal(got, ref)
