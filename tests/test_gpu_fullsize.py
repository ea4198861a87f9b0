"""Full-size raw-ciphertext parity and determinism of the asynchronous kernels.

* Configs 1 and 2 at BASELINE.json's sizes (4,096 NAND; 256 x ADD16 =
  49,920 bootstraps): every node's 631 torus32 words against the CPU oracle
  evaluating the same recorded DAG level by level (double-FFT mode, the TFHE
  library's method), with any mismatching gate re-checked against the exact
  NTT oracle -- the GPU must equal the exact product.
* Determinism: the kernels whose correctness rests on asynchronous protocols
  -- the v4 key ring refilled by each slot's last reader
  (blind_rotate_v4.cu), the pair kernel's st.async partial-product exchange
  (variant 96), the split-K tcgen05 key switch + ks_reduce (variant 9) -- are
  re-run 50 times on the same level and must reproduce the first,
  oracle-checked run bit for bit (compute-sanitizer is not available on this
  pool, so repetition is the race evidence).
"""
import os

import numpy as np
import pytest

import oracle as O
import paper_2101_03403_b200 as P
from conftest import fu_dag

pytestmark = pytest.mark.gpu
THREADS = os.cpu_count() or 1


def _recheck_exact(oracle_keys, kinds, a, b, c, got):
    """Gates whose FFT-oracle output differed: recompute exactly (NTT)."""
    ck = O.CloudKeys(oracle_keys._bk, oracle_keys._ksk, O.MODE_NTT)
    return np.array_equal(ck.gates(kinds, a, b, c, THREADS), got)


@pytest.mark.slow
def test_config1_full_size_every_ciphertext(keyset, ctx, oracle_keys):
    n = 4096
    rng = np.random.default_rng(2024)
    a, b = rng.integers(0, 2, n).astype(np.uint8), rng.integers(0, 2, n).astype(np.uint8)
    ca, cb = keyset.encrypt(a, 61), keyset.encrypt(b, 62)
    base = ctx.alloc(3 * n)
    ctx.upload(base, ca)
    ctx.upload(base + n, cb)
    ctx.submit_level([("NAND", [(base + i, 1, 0), (base + n + i, 1, 0)], base + 2 * n + i)
                      for i in range(n)])
    ctx.sync()
    got = ctx.download(base + 2 * n, n)
    kinds = np.full(n, O.NAND, np.uint8)
    ck = O.CloudKeys(oracle_keys._bk, oracle_keys._ksk, O.MODE_FFT)
    ref = ck.gates(kinds, ca, cb, None, THREADS)
    bad = np.flatnonzero((got != ref).any(axis=1))
    if len(bad):
        assert _recheck_exact(oracle_keys, kinds[bad], ca[bad], cb[bad], None, got[bad])
    assert np.array_equal(keyset.decrypt(got), 1 - (a & b))


def _replicate(rows, k):
    n = len(rows)
    out = np.tile(rows, (k, 1))
    for i in range(1, k):
        blk = out[i * n:(i + 1) * n]
        blk[:, 3:6] = np.where(blk[:, 3:6] > 0, blk[:, 3:6] + i * n, 0)
    return out


@pytest.mark.slow
def test_config2_full_size_every_node(keyset, ctx, oracle_keys):
    """256 x ADD16 (the headline workload), all ~58k nodes' ciphertexts."""
    batch, dag = 256, fu_dag("add", 16)
    rng = np.random.default_rng(4242)
    av, bv = rng.integers(0, 1 << 16, batch), rng.integers(0, 1 << 16, batch)
    lwe = np.concatenate([keyset.encrypt_words(av, 16, 71), keyset.encrypt_words(bv, 16, 72)],
                         axis=1)  # (256, 32, 631)
    bk = P.Backend(ctx, keyset)
    bk.set_flush_policy("all")
    hin = bk.import_lwe(lwe.reshape(-1, 631)).reshape(batch, -1)
    handles = np.concatenate([bk.replay(dag, hin[i]) for i in range(batch)])
    got = bk.export_lwe(handles)
    rows = _replicate(dag.rows(), batch)
    ck = O.CloudKeys(oracle_keys._bk, oracle_keys._ksk, O.MODE_FFT)
    ref = O.eval_dag(ck, rows, lwe.reshape(-1, 631), THREADS)
    bad = np.flatnonzero((got != ref).any(axis=1))
    if len(bad):
        # every mismatch must be the FFT oracle's, not the GPU's: recompute
        # those gates exactly from the (matching) GPU inputs
        assert (rows[bad, 0] >= O.NAND).all() and not rows[bad, 1].any()
        deps = rows[bad, 3:6]
        c_in = got[np.maximum(deps[:, 2], 1) - 1]
        assert _recheck_exact(oracle_keys, rows[bad, 0].astype(np.uint8), got[deps[:, 0] - 1],
                              got[deps[:, 1] - 1], c_in, got[bad])
    outs = np.concatenate([dag.outputs.astype(np.int64) - 1 + i * dag.n_nodes
                           for i in range(batch)])
    sums = keyset.decrypt_words(got[outs], 17)
    assert np.array_equal(sums, av + bv)


def _repeat_level(ctx, gates, out_slot, n, reps):
    first = None
    for r in range(reps):
        ctx.submit_level(gates)
        ctx.sync()
        cur = ctx.download(out_slot, n)
        if first is None:
            first = cur
        elif not np.array_equal(cur, first):
            return first, r
    return first, None


@pytest.mark.parametrize("n,what", [(2368, "two full v4 waves (last-reader key ring)"),
                                    (74, "pair kernel 96 (st.async exchange)"),
                                    (148, "wide kernel 9 (per-group key rows)"),
                                    (300, "v3 round + split-K tcgen05 key switch, MUX")])
def test_async_kernels_are_deterministic(n, what, keyset, ctx, oracle_keys):
    rng = np.random.default_rng(n)
    s, t, f = (rng.integers(0, 2, n).astype(np.uint8) for _ in range(3))
    cs, ct, cf = keyset.encrypt(s, 81), keyset.encrypt(t, 82), keyset.encrypt(f, 83)
    base = ctx.alloc(4 * n)
    for k, c in enumerate((cs, ct, cf)):
        ctx.upload(base + k * n, c)
    mux = n == 300
    gates = [("MUX" if (mux and i % 2) else "XOR",
              [(base + i, 1, 0), (base + n + i, 1, 0), (base + 2 * n + i, 1, 0)],
              base + 3 * n + i) for i in range(n)]
    reps = int(os.environ.get("CVM_DETERMINISM_REPS", 50))  # evidence runs use 1000
    first, bad_rep = _repeat_level(ctx, gates, base + 3 * n, n, reps)
    assert bad_rep is None, f"{what}: run {bad_rep} differs from run 0"
    # the first run against the exact oracle (a sample of the level)
    idx = np.arange(0, n, max(1, n // 48))
    kinds = np.array([O.MUX if (mux and i % 2) else O.XOR for i in idx], np.uint8)
    ref = oracle_keys.gates(kinds, cs[idx], ct[idx], cf[idx], THREADS)
    assert np.array_equal(first[idx], ref), what
    want = np.where(np.arange(n) % 2 & mux, np.where(s == 1, t, f), s ^ t)
    assert np.array_equal(keyset.decrypt(first), want)
