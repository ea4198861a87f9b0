"""Known-answer tests pinning the CPU TFHE oracle (oracle/tfhe_oracle.c).

The reference ships no TFHE code, so ciphertext-level
parity cannot be pinned to reference outputs; these tests pin the oracle to
exact arithmetic instead; tests/test_gpu_parity.py replays the reference's
recorded DAGs on the oracle and decrypts them to the reference SimBackend's
golden results, and test_keygen_byte_identical_to_product below pins the
product keygen to the oracle's.
"""
import numpy as np
import pytest

import oracle as O

SEED = 20260808


@pytest.fixture(scope="module")
def sk():
    return O.SecretKeys(SEED)


@pytest.fixture(scope="module")
def ck_ntt(sk):
    return O.CloudKeys(sk.bk, sk.ksk, O.MODE_NTT)


def _schoolbook_py(d, p):
    """Pure-numpy negacyclic product mod 2^32 (small-case reference)."""
    # |d| <= 64, p < 2^32: every partial sum stays below 2^48, exact in int64
    full = np.convolve(d.astype(np.int64), p.astype(np.int64))
    full = np.concatenate([full, [0]])
    res = (full[:1024] - full[1024:]) % (1 << 32)
    return res.astype(np.uint32)


@pytest.mark.parametrize("trial", range(4))
def test_negacyclic_products_agree(trial):
    rng = np.random.default_rng(trial)
    d = rng.integers(-64, 64, 1024).astype(np.int32)
    p = rng.integers(0, 2**32, 1024, dtype=np.uint64).astype(np.uint32)
    sb = O.negacyclic_mul(d, p, O.MODE_SCHOOLBOOK)
    assert np.array_equal(sb, _schoolbook_py(d, p))
    assert np.array_equal(O.negacyclic_mul(d, p, O.MODE_NTT), sb)
    assert np.array_equal(O.negacyclic_mul(d, p, O.MODE_FFT), sb)


def test_negacyclic_extremes():
    """Largest-magnitude operands (|d| = 64, |p| = 2^31): exact in NTT mode."""
    d = np.full(1024, -64, np.int32)
    p = np.full(1024, 0x80000000, np.uint32)
    sb = O.negacyclic_mul(d, p, O.MODE_SCHOOLBOOK)
    assert np.array_equal(O.negacyclic_mul(d, p, O.MODE_NTT), sb)


def test_modswitch_rounding():
    # round(phase * 2048 / 2^32) mod 2048
    for ph in [0, 1, (1 << 20) - 1, 1 << 20, (1 << 21) - 1, 0xFFFFFFFF, 0x80000000, 0x7FF00000]:
        want = ((ph * 2048 + (1 << 31)) >> 32) % 2048
        assert O.lib().oracle_modswitch(ph) == want


def test_keygen_deterministic_and_shaped(sk):
    again = O.SecretKeys(SEED)
    assert np.array_equal(again.bk, sk.bk) and np.array_equal(again.ksk, sk.ksk)
    assert set(np.unique(sk.lwe_key)) <= {0, 1} and set(np.unique(sk.tlwe_key)) <= {0, 1}
    # KSK rows for digit value 0 are zero (trivial), others are not
    ksk = sk.ksk.reshape(1024, 8, 4, 631)
    assert not ksk[:, :, 0, :].any() and ksk[:, :, 1:, :].any()


def test_encrypt_decrypt_noise(sk):
    bits = np.random.default_rng(3).integers(0, 2, 2000).astype(np.uint8)
    ct = sk.encrypt(bits, 99)
    dec, ph = sk.decrypt(ct, with_phase=True)
    assert np.array_equal(dec, bits)
    # phase = +-2^29 + e, e ~ N(0, (2^-15 * 2^32)^2) = N(0, 2^17 std)
    err = ph.astype(np.int64) - np.where(bits == 1, 1 << 29, -(1 << 29))
    assert abs(err.std() / 2**17 - 1) < 0.1
    assert np.abs(err).max() < 8 * 2**17


def test_bootstrapped_gates_truth_tables(sk, ck_ntt):
    a = np.array([0, 0, 1, 1], np.uint8)
    b = np.array([0, 1, 0, 1], np.uint8)
    ca, cb = sk.encrypt(a, 1), sk.encrypt(b, 2)
    table = {O.NAND: 1 - (a & b), O.OR: a | b, O.XNOR: 1 - (a ^ b), O.ORYN: a | (1 - b)}
    kinds = np.array([k for k in table for _ in range(4)], np.uint8)
    out = ck_ntt.gates(kinds, np.tile(ca, (len(table), 1)), np.tile(cb, (len(table), 1)))
    dec, ph = sk.decrypt(out, with_phase=True)
    assert np.array_equal(dec, np.concatenate(list(table.values())))
    # fresh gate outputs are +-1/8 with bootstrapping + key-switch noise
    assert np.abs(np.abs(ph.astype(np.int64)) - (1 << 29)).max() < (1 << 25)


def test_mux_order(sk, ck_ntt):
    s = np.array([0, 1, 0, 1], np.uint8)
    t = np.array([1, 1, 0, 0], np.uint8)
    f = np.array([0, 1, 1, 0], np.uint8)
    out = ck_ntt.gates(np.full(4, O.MUX, np.uint8), sk.encrypt(s, 1), sk.encrypt(t, 2),
                       sk.encrypt(f, 3))
    assert np.array_equal(sk.decrypt(out), np.where(s == 1, t, f))


def test_fft_mode_matches_ntt_mode(sk, ck_ntt):
    """The CPU speed baseline (double FFT, the TFHE library's method) produces
    the same ciphertexts as the exact oracle."""
    ckf = O.CloudKeys(sk.bk, sk.ksk, O.MODE_FFT)
    a, b = sk.encrypt(np.array([1, 0], np.uint8), 5), sk.encrypt(np.array([1, 1], np.uint8), 6)
    kinds = np.array([O.XOR, O.AND], np.uint8)
    assert np.array_equal(ckf.gates(kinds, a, b), ck_ntt.gates(kinds, a, b))


def test_rejects_non_bootstrapped_kind(sk, ck_ntt):
    a = sk.encrypt(np.array([1], np.uint8), 1)
    with pytest.raises(ValueError):
        ck_ntt.gates(np.array([O.NOT], np.uint8), a, a)


def test_eval_dag_free_ops_after_same_level_gates(sk, ck_ntt):
    """A NOT / COPY shares the dataflow level of the gate it reads: eval_dag
    must run it after that level's bootstrapped batch (regression: it once
    read the gate's output before it was computed)."""
    I, C, NT, CP, AND, XOR = 1, O.CONSTANT, O.NOT, O.COPY, O.AND, O.XOR
    # ids: 1 a, 2 b, 3 AND(a,b), 4 COPY(3), 5 NOT(3), 6 XOR(4,5), 7 NOT(4)
    nodes = np.array([[C, I, 0, 0, 0, 0, 0], [C, I, 0, 0, 0, 0, 0],
                      [AND, 0, 2, 1, 2, 0, 0], [CP, 0, 1, 3, 0, 0, 0],
                      [NT, 0, 1, 3, 0, 0, 0], [XOR, 0, 2, 4, 5, 0, 0],
                      [NT, 0, 1, 4, 0, 0, 0]], np.int64)
    ins = sk.encrypt(np.array([1, 1], np.uint8), 5)
    ct = O.eval_dag(ck_ntt, nodes, ins)
    assert np.array_equal(ct[3], ct[2])
    assert np.array_equal(ct[4], (np.uint32(0) - ct[2]).astype(np.uint32))
    assert np.array_equal(ct[6], ct[4])
    assert list(sk.decrypt(ct[2:])) == [1, 1, 0, 1, 0]


@pytest.mark.parametrize("seed", [SEED, 7])
def test_keygen_byte_identical_to_product(seed):
    """The product keygen (csrc/keys.cpp) and the oracle keygen
    (oracle/tfhe_oracle.c) are independent implementations of one spec
    (DESIGN.md section 3); they must produce the same key bytes and the same
    fresh encryptions, which bench.py's CPU legs rely on."""
    import paper_2101_03403_b200 as P
    prod = P.KeySet(seed)
    mine = prod.export()
    ref = O.SecretKeys(seed)
    for name in ("lwe_key", "tlwe_key", "bk", "ksk"):
        a, b = mine[name], getattr(ref, name)
        assert a.dtype.itemsize == b.dtype.itemsize and a.tobytes() == b.tobytes(), name
    bits = np.random.default_rng(seed).integers(0, 2, 257).astype(np.uint8)
    for enc_seed in (1, 12345):
        assert prod.encrypt(bits, enc_seed).tobytes() == ref.encrypt(bits, enc_seed).tobytes()
