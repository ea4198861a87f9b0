"""ctypes/numpy front end of the CPU TFHE oracle (liboracle.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
CPU-baseline legs of bench.py -- never by the product package.  See
tfhe_oracle.h for what is restated and from where.

Also holds a small DAG evaluator (levelised, NOT/COPY/CONSTANT as linear ops
on the ciphertext, bootstrapped gates through the C library) that replays a
reference gate DAG (tests/golden/*.npz, node layout of GateDag::append,
proj/core/src/dag.cpp:57-73) on real ciphertexts.
"""
import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")

N_LWE, N_POLY, LWE_WORDS, XLWE_WORDS = 630, 1024, 631, 1025
BK_WORDS = 630 * 6 * 2 * 1024
KSK_WORDS = 1024 * 8 * 4 * 631
MU = 1 << 29
MODE_NTT, MODE_FFT, MODE_SCHOOLBOOK = 0, 1, 2
CONSTANT, NOT, COPY, NAND, AND, OR, XOR, XNOR, NOR, ANDNY, ANDYN, ORNY, ORYN, MUX = range(14)

_u32p = ctypes.POINTER(ctypes.c_uint32)
_i32p = ctypes.POINTER(ctypes.c_int32)
_u8p = ctypes.POINTER(ctypes.c_uint8)


def _ptr(a, t):
    return a.ctypes.data_as(t) if a is not None else None


def load():
    if not os.path.exists(LIB_PATH):
        raise RuntimeError("oracle library missing: run `make -C oracle`")
    lib = ctypes.CDLL(LIB_PATH)
    lib.oracle_keygen.argtypes = [ctypes.c_uint64, _i32p, _i32p, _u32p, _u32p]
    lib.oracle_encrypt.argtypes = [ctypes.c_uint64, _i32p, ctypes.c_int, _u8p, _u32p]
    lib.oracle_decrypt.argtypes = [_i32p, ctypes.c_int, _u32p, _u8p, _i32p]
    lib.oracle_decrypt_x.argtypes = [_i32p, ctypes.c_int, _u32p, _u8p, _i32p]
    lib.oracle_keys_load.argtypes = [_u32p, _u32p, ctypes.c_int]
    lib.oracle_keys_load.restype = ctypes.c_void_p
    lib.oracle_keys_free.argtypes = [ctypes.c_void_p]
    lib.oracle_gates.argtypes = [ctypes.c_void_p, ctypes.c_int, _u8p, _u32p, _u32p,
                                 _u32p, _u32p, ctypes.c_int]
    lib.oracle_gates.restype = ctypes.c_int
    lib.oracle_blind_rotate_extract.argtypes = [ctypes.c_void_p, _u32p, ctypes.c_uint32, _u32p]
    lib.oracle_key_switch.argtypes = [ctypes.c_void_p, _u32p, _u32p]
    lib.oracle_negacyclic_mul.argtypes = [ctypes.c_int, _i32p, _u32p, _u32p]
    lib.oracle_modswitch.argtypes = [ctypes.c_uint32]
    lib.oracle_modswitch.restype = ctypes.c_uint32
    return lib


_LIB = None


def lib():
    global _LIB
    if _LIB is None:
        _LIB = load()
    return _LIB


class SecretKeys:
    """Key-owner material from oracle_keygen (same spec as the product keygen)."""

    def __init__(self, seed):
        self.seed = seed
        self.lwe_key = np.zeros(N_LWE, np.int32)
        self.tlwe_key = np.zeros(N_POLY, np.int32)
        self.bk = np.zeros(BK_WORDS, np.uint32)
        self.ksk = np.zeros(KSK_WORDS, np.uint32)
        lib().oracle_keygen(seed, _ptr(self.lwe_key, _i32p), _ptr(self.tlwe_key, _i32p),
                            _ptr(self.bk, _u32p), _ptr(self.ksk, _u32p))

    def encrypt(self, bits, seed):
        bits = np.ascontiguousarray(bits, dtype=np.uint8)
        out = np.zeros((len(bits), LWE_WORDS), np.uint32)
        lib().oracle_encrypt(seed, _ptr(self.lwe_key, _i32p), len(bits), _ptr(bits, _u8p),
                             _ptr(out, _u32p))
        return out

    def decrypt(self, cts, with_phase=False):
        return decrypt(self.lwe_key, cts, with_phase)


def decrypt(lwe_key, cts, with_phase=False):
    cts = np.ascontiguousarray(cts, dtype=np.uint32).reshape(-1, LWE_WORDS)
    bits = np.zeros(len(cts), np.uint8)
    ph = np.zeros(len(cts), np.int32)
    lib().oracle_decrypt(_ptr(np.ascontiguousarray(lwe_key, np.int32), _i32p), len(cts),
                         _ptr(cts, _u32p), _ptr(bits, _u8p), _ptr(ph, _i32p))
    return (bits, ph) if with_phase else bits


class CloudKeys:
    """BK/KSK loaded into the oracle (NTT exact / FFT / schoolbook mode)."""

    def __init__(self, bk, ksk, mode=MODE_NTT):
        self._bk = np.ascontiguousarray(bk, np.uint32)
        self._ksk = np.ascontiguousarray(ksk, np.uint32)
        self.mode = mode
        self.h = lib().oracle_keys_load(_ptr(self._bk, _u32p), _ptr(self._ksk, _u32p), mode)

    def __del__(self):
        if getattr(self, "h", None):
            lib().oracle_keys_free(self.h)
            self.h = None

    def gates(self, kinds, a, b, c=None, threads=None):
        kinds = np.ascontiguousarray(kinds, np.uint8)
        n = len(kinds)
        a = np.ascontiguousarray(a, np.uint32).reshape(n, LWE_WORDS)
        b = np.ascontiguousarray(b, np.uint32).reshape(n, LWE_WORDS)
        if c is not None:
            c = np.ascontiguousarray(c, np.uint32).reshape(n, LWE_WORDS)
        out = np.zeros((n, LWE_WORDS), np.uint32)
        if n == 0:
            return out
        threads = threads or os.cpu_count() or 1
        rc = lib().oracle_gates(self.h, n, _ptr(kinds, _u8p), _ptr(a, _u32p), _ptr(b, _u32p),
                                _ptr(c, _u32p), _ptr(out, _u32p), threads)
        if rc:
            raise ValueError("oracle_gates rejected a gate kind")
        return out

    def blind_rotate_extract(self, lwe, mu=MU):
        lwe = np.ascontiguousarray(lwe, np.uint32)
        out = np.zeros(XLWE_WORDS, np.uint32)
        lib().oracle_blind_rotate_extract(self.h, _ptr(lwe, _u32p), mu, _ptr(out, _u32p))
        return out

    def key_switch(self, xlwe):
        xlwe = np.ascontiguousarray(xlwe, np.uint32)
        out = np.zeros(LWE_WORDS, np.uint32)
        lib().oracle_key_switch(self.h, _ptr(xlwe, _u32p), _ptr(out, _u32p))
        return out


def negacyclic_mul(digits, poly, mode):
    d = np.ascontiguousarray(digits, np.int32)
    p = np.ascontiguousarray(poly, np.uint32)
    out = np.zeros(N_POLY, np.uint32)
    lib().oracle_negacyclic_mul(mode, _ptr(d, _i32p), _ptr(p, _u32p), _ptr(out, _u32p))
    return out


def trivial(bit):
    c = np.zeros(LWE_WORDS, np.uint32)
    c[-1] = np.uint32(MU if bit else (1 << 32) - MU)
    return c


def dag_levels(nodes):
    """Dataflow level per node: inputs / free ops inherit, bootstrapped +1."""
    lv = np.zeros(len(nodes), np.int64)
    for i, (kind, inp, nd, d0, d1, d2) in enumerate(nodes[:, :6]):
        deps = [d for d in (d0, d1, d2)[:nd]]
        base = max((lv[d - 1] for d in deps), default=0)
        lv[i] = base + (1 if (not inp and kind >= NAND) else 0)
    return lv


def eval_dag(ck, nodes, inputs, threads=None):
    """Evaluate a reference GateDag on ciphertexts.

    nodes: (n, 7) int array [kind, input, ndeps, d0, d1, d2, const_value]
           (ids 1-based; const_value is the CONSTANT node's bit).
    inputs: (n_inputs, 631) ciphertexts, consumed in order by input nodes.
    Returns (n, 631) ciphertexts, one per node.
    """
    n = len(nodes)
    ct = np.zeros((n, LWE_WORDS), np.uint32)
    done = np.zeros(n, bool)
    lv = dag_levels(nodes)
    k_in = 0
    order = np.argsort(lv, kind="stable")

    def free_op(i):
        kind, inp, nd, d0, d1, d2, val = nodes[i]
        if kind == CONSTANT:
            ct[i] = trivial(bool(val))
        elif kind == NOT:
            ct[i] = (np.uint32(0) - ct[d0 - 1]).astype(np.uint32)
        else:  # COPY
            ct[i] = ct[d0 - 1]
        done[i] = True

    # By level.  A free op (NOT / COPY) shares the level of the gate it reads,
    # so inside a level: inputs and the free ops whose operand is ready, in id
    # order; then the bootstrapped batch; then the remaining free ops in id
    # order (they read this batch or earlier free ops of the same pass).
    for level in range(int(lv.max()) + 1 if n else 0):
        ids = order[lv[order] == level]
        boot, later = [], []
        for i in ids:
            kind, inp, nd, d0 = nodes[i][:4]
            if inp:
                ct[i] = inputs[k_in]
                k_in += 1
                done[i] = True
            elif kind >= NAND:
                boot.append(i)
            elif kind == CONSTANT or done[d0 - 1]:
                free_op(i)
            else:
                later.append(i)
        if boot:
            boot = np.array(boot)
            kinds = nodes[boot, 0].astype(np.uint8)
            a = ct[nodes[boot, 3] - 1]
            b = ct[nodes[boot, 4] - 1]
            c = ct[np.maximum(nodes[boot, 5], 1) - 1]
            ct[boot] = ck.gates(kinds, a, b, c, threads)
            done[boot] = True
        for i in later:
            free_op(i)
    return ct
