"""Python front end of the B200 backend (thin; the product is libcvm_b200.so).

Names follow the reference interface (cryptovm::Backend, gates.hpp:109-132;
alu.hpp; Machine, emulator.hpp) so tests read like the reference's own.
"""
import ctypes

import numpy as np

from . import _native as N
from ._native import check, lib

GATE_KINDS = ["CONSTANT", "NOT", "COPY", "NAND", "AND", "OR", "XOR", "XNOR", "NOR",
              "ANDNY", "ANDYN", "ORNY", "ORYN", "MUX"]
KIND = {n: i for i, n in enumerate(GATE_KINDS)}

FU_OPS = ["add", "add_cin", "sub", "addsub", "cmp", "and", "orr", "eor", "orn", "lsl",
          "lsr", "asr", "umul", "smul", "udiv", "udiv_exact", "mul_lo"]
FU = {n: i for i, n in enumerate(FU_OPS)}

OPCODES = ["LOAD", "STORE", "MOV", "ADD", "ADDS", "SUB", "SUBS", "MUL", "MULS", "SMUL",
           "SMULS", "UDIV", "LLS", "LRS", "ARS", "AND", "OR", "XOR", "ORN", "NOT", "BFC",
           "BFI", "RBIT", "REV", "CMP", "B", "HALT"]
OPCODE = {n: i for i, n in enumerate(OPCODES)}


def _vp(a):
    return ctypes.c_void_p(a.ctypes.data) if a is not None else None


def _u32(a, shape=None):
    a = np.ascontiguousarray(a, dtype=np.uint32)
    return a if shape is None else a.reshape(shape)


class KeySet:
    """Key owner's material (host only): LWE/TRLWE secret keys, BK and KSK."""

    def __init__(self, seed):
        h = ctypes.c_void_p()
        check(lib.cvm_keyset_generate(seed, ctypes.byref(h)))
        self._h = h
        self.seed = seed

    def close(self):
        if self._h:
            lib.cvm_keyset_destroy(self._h)
            self._h = None

    __del__ = close

    @property
    def handle(self):
        return self._h

    def export(self):
        lwe = np.zeros(N.LWE_N, np.int32)
        tl = np.zeros(N.POLY_N, np.int32)
        bk = np.zeros(N.BK_WORDS, np.uint32)
        ksk = np.zeros(N.KSK_WORDS, np.uint32)
        check(lib.cvm_keyset_export(self._h, _vp(lwe), _vp(tl), _vp(bk), _vp(ksk)))
        return {"lwe_key": lwe, "tlwe_key": tl, "bk": bk, "ksk": ksk}

    def encrypt(self, bits, seed):
        bits = np.ascontiguousarray(bits, dtype=np.uint8).ravel()
        out = np.zeros((len(bits), N.LWE_WORDS), np.uint32)
        check(lib.cvm_encrypt_bits(self._h, seed, len(bits), _vp(bits), _vp(out)))
        return out

    def decrypt(self, lwe, with_phase=False):
        lwe = _u32(lwe).reshape(-1, N.LWE_WORDS)
        bits = np.zeros(len(lwe), np.uint8)
        ph = np.zeros(len(lwe), np.int32)
        check(lib.cvm_decrypt_bits(self._h, len(lwe), _vp(lwe), _vp(bits), _vp(ph)))
        return (bits, ph) if with_phase else bits

    def encrypt_words(self, values, width, seed):
        """LSB-first bit ciphertexts of integers: shape (len(values), width, 631)."""
        values = np.asarray(values, dtype=np.uint64)
        bits = ((values[:, None] >> np.arange(width, dtype=np.uint64)) & 1).astype(np.uint8)
        return self.encrypt(bits.ravel(), seed).reshape(len(values), width, N.LWE_WORDS)

    def decrypt_words(self, lwe, width):
        bits = self.decrypt(lwe).reshape(-1, width).astype(np.uint64)
        return (bits << np.arange(width, dtype=np.uint64)).sum(axis=1)


class Context:
    """Device context on one B200: resident BK (FFT domain) / KSK, LWE slots."""

    def __init__(self, device=0):
        h = ctypes.c_void_p()
        check(lib.cvm_ctx_create(device, ctypes.byref(h)))
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            lib.cvm_ctx_destroy(self._h)
            self._h = None

    __del__ = close

    @property
    def handle(self):
        return self._h

    def upload_keyset(self, ks):
        check(lib.cvm_upload_keyset(self._h, ks.handle))

    def upload_keys(self, bk, ksk):
        bk, ksk = _u32(bk), _u32(ksk)
        check(lib.cvm_upload_keys(self._h, _vp(bk), _vp(ksk)))

    def alloc(self, n):
        """n fresh slot ids (first id returned); capacity reserved."""
        first = ctypes.c_uint64()
        check(lib.cvm_slots_alloc(self._h, n, ctypes.byref(first)))
        return first.value

    def reserve(self, n):
        check(lib.cvm_slots_reserve(self._h, n))

    def upload(self, slot, lwe):
        lwe = _u32(lwe).reshape(-1, N.LWE_WORDS)
        check(lib.cvm_upload_lwe(self._h, slot, len(lwe), _vp(lwe)))

    def download(self, slot, count):
        out = np.zeros((count, N.LWE_WORDS), np.uint32)
        check(lib.cvm_download_lwe(self._h, slot, count, _vp(out)))
        return out

    @staticmethod
    def pack_level(gates):
        """gates: list of (kind, [(slot, sign, const), ...], out_slot) ->
        the C `cvm_gate` array `submit_level` takes (pack once, submit many)."""
        arr = (N.Gate * len(gates))()
        for g, (kind, ins, out) in zip(arr, gates):
            g.kind = KIND[kind] if isinstance(kind, str) else kind
            for i in range(3):
                s, sg, c = ins[i] if i < len(ins) else (-1, 1, 0)
                g.inp[i].slot, g.inp[i].sign, g.inp[i].constant = s, sg, c & 0xFFFFFFFF
            g.out_slot = out
        return arr

    def submit_level(self, gates):
        """gates: a gate list (see `pack_level`) or an already packed array."""
        arr = gates if isinstance(gates, ctypes.Array) else self.pack_level(gates)
        check(lib.cvm_submit_level(self._h, arr, len(arr)))

    def sync(self):
        check(lib.cvm_sync(self._h))

    def set_profiling(self, on=True):
        check(lib.cvm_ctx_set_profiling(self._h, 1 if on else 0))

    def kernel_stats(self):
        s = N.KernelStats()
        check(lib.cvm_ctx_kernel_stats(self._h, ctypes.byref(s)))
        return s.as_dict()

    def reset_stats(self):
        check(lib.cvm_ctx_reset_stats(self._h))

    def flush_l2(self):
        check(lib.cvm_ctx_flush_l2(self._h))

    def fp64_peak_tflops(self, reps=3):
        v = ctypes.c_double()
        check(lib.cvm_ctx_fp64_peak(self._h, reps, ctypes.byref(v)))
        return v.value

    def sm_count(self):
        v = ctypes.c_int()
        check(lib.cvm_ctx_sm_count(self._h, ctypes.byref(v)))
        return v.value

    def event(self, which):
        check(lib.cvm_ctx_event_record(self._h, which))

    def event_elapsed_ms(self):
        v = ctypes.c_double()
        check(lib.cvm_ctx_event_elapsed_ms(self._h, ctypes.byref(v)))
        return v.value


class Backend:
    """cryptovm::Backend over the device (ctx given) or the cleartext recorder
    (ctx=None: SimBackend semantics, node table only -- no ciphertexts)."""

    def __init__(self, ctx=None, owner=None, enc_seed=1):
        h = ctypes.c_void_p()
        check(lib.cvm_backend_create(ctx.handle if ctx else None,
                                     owner.handle if owner else None, enc_seed,
                                     ctypes.byref(h)))
        self._h = h
        self._ctx, self._owner = ctx, owner  # keep alive

    def close(self):
        if getattr(self, "_h", None):
            lib.cvm_backend_destroy(self._h)
            self._h = None

    __del__ = close

    @property
    def handle(self):
        return self._h

    def _out(self, fn, *args):
        o = ctypes.c_uint64()
        check(fn(self._h, *args, ctypes.byref(o)))
        return o.value

    def constant(self, v):
        return self._out(lib.cvm_backend_constant, 1 if v else 0)

    def unary_gate(self, kind, a):
        return self._out(lib.cvm_backend_unary_gate, KIND.get(kind, kind), a)

    def binary_gate(self, kind, a, b):
        return self._out(lib.cvm_backend_binary_gate, KIND.get(kind, kind), a, b)

    def mux_gate(self, sel, t, f):
        return self._out(lib.cvm_backend_mux_gate, sel, t, f)

    def encrypt_bit(self, v):
        return self._out(lib.cvm_backend_encrypt_bit, 1 if v else 0)

    def decrypt_bit(self, h):
        v = ctypes.c_int()
        check(lib.cvm_backend_decrypt_bit(self._h, h, ctypes.byref(v)))
        return bool(v.value)

    def decrypt_bits(self, hs):
        hs = np.ascontiguousarray(hs, dtype=np.uint64).ravel()
        out = np.zeros(len(hs), np.uint8)
        check(lib.cvm_backend_decrypt_bits(self._h, len(hs), _vp(hs), _vp(out)))
        return out

    def import_lwe(self, lwe):
        lwe = _u32(lwe).reshape(-1, N.LWE_WORDS)
        out = np.zeros(len(lwe), np.uint64)
        check(lib.cvm_backend_import_lwe(self._h, len(lwe), _vp(lwe), _vp(out)))
        return out

    def export_lwe(self, hs):
        hs = np.ascontiguousarray(hs, dtype=np.uint64).ravel()
        out = np.zeros((len(hs), N.LWE_WORDS), np.uint32)
        check(lib.cvm_backend_export_lwe(self._h, len(hs), _vp(hs), _vp(out)))
        return out

    def export_bit(self, h):
        blob = (ctypes.c_uint8 * (4 * N.LWE_WORDS))()
        check(lib.cvm_backend_export_bit(self._h, h, blob, len(blob)))
        return bytes(blob)

    def import_bit(self, blob):
        buf = (ctypes.c_uint8 * len(blob)).from_buffer_copy(blob)
        return self._out(lib.cvm_backend_import_bit, buf, len(blob))

    def push_region(self, name):
        check(lib.cvm_backend_push_region(self._h, name.encode()))

    def pop_region(self):
        check(lib.cvm_backend_pop_region(self._h))

    def fence(self):
        check(lib.cvm_backend_fence(self._h))

    def flush(self):
        check(lib.cvm_backend_flush(self._h))

    def set_flush_policy(self, policy):
        """"cone" (default: decrypt/export evaluate only what they need) or "all"."""
        check(lib.cvm_backend_set_flush_policy(self._h, {"cone": 0, "all": 1}[policy]))

    def capture_plan(self):
        h = ctypes.c_void_p()
        check(lib.cvm_backend_capture_plan(self._h, ctypes.byref(h)))
        return Plan(h)

    def handle_slot(self, h):
        s, sg, c = ctypes.c_int64(), ctypes.c_int32(), ctypes.c_uint32()
        check(lib.cvm_backend_handle_slot(self._h, h, ctypes.byref(s), ctypes.byref(sg),
                                          ctypes.byref(c)))
        return s.value, sg.value, c.value

    def stats(self):
        s = N.BackendStats()
        check(lib.cvm_backend_stats_get(self._h, ctypes.byref(s)))
        return s.as_dict()

    def nodes(self):
        n = ctypes.c_uint64()
        check(lib.cvm_backend_node_count(self._h, ctypes.byref(n)))
        rows = np.zeros((n.value, 7), np.int64)
        check(lib.cvm_backend_nodes(self._h, 0, n.value, _vp(rows)))
        return rows

    # -- functional units (alu.hpp) --
    def fu(self, op, a, b, c=0):
        a = np.ascontiguousarray(a, dtype=np.uint64)
        b = np.ascontiguousarray(b, dtype=np.uint64)
        w = len(a)
        opi = FU[op] if isinstance(op, str) else op
        ow = lib.cvm_fu_out_width(opi, w)
        if ow < 0:
            raise N.CvmInputError(f"unknown op {op}")
        out = np.zeros(ow, np.uint64)
        cc = np.array([c], np.uint64)
        check(lib.cvm_fu_apply(self._h, opi, w, _vp(a), _vp(b), _vp(cc), _vp(out)))
        return out

    def encrypt_word(self, value, width):
        return np.array([self.encrypt_bit((value >> i) & 1) for i in range(width)], np.uint64)

    def decrypt_word(self, hs):
        bits = self.decrypt_bits(hs).astype(np.uint64)
        return int((bits << np.arange(len(bits), dtype=np.uint64)).sum())

    def machine_run(self, program, memory, word_size=16, register_count=8):
        """program: list of (op, rd, rn, rm, imm, sets_flags[, imm2]); memory:
        list of handle arrays (width each).  Returns (regs handles, nzcv handles)."""
        arr = (N.Insn * len(program))()
        for x, ins in zip(arr, program):
            op, rd, rn, rm, imm, sf = ins[:6]
            x.op = OPCODE[op] if isinstance(op, str) else op
            x.rd, x.rn, x.rm, x.imm, x.sets_flags = rd, rn, rm, imm, sf
            x.imm2 = ins[6] if len(ins) > 6 else -1
        mem = np.ascontiguousarray(np.array(memory, dtype=np.uint64).reshape(-1)) \
            if len(memory) else np.zeros(1, np.uint64)
        regs = np.zeros(register_count * word_size, np.uint64)
        nzcv = np.zeros(4, np.uint64)
        check(lib.cvm_machine_run(self._h, word_size, register_count, _vp(mem), len(memory),
                                  arr, len(program), _vp(regs), _vp(nzcv)))
        return regs.reshape(register_count, word_size), nzcv


class Plan:
    """A recorded circuit (levels with device-resident job tables)."""

    def __init__(self, h):
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            lib.cvm_plan_destroy(self._h)
            self._h = None

    __del__ = close

    def run(self, ctx, graph=True):
        check(lib.cvm_plan_run(ctx.handle, self._h, 1 if graph else 0))

    def info(self):
        lv, g, b = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
        check(lib.cvm_plan_info(self._h, ctypes.byref(lv), ctypes.byref(g), ctypes.byref(b)))
        return {"levels": lv.value, "gates": g.value, "bootstraps": b.value}


def fu_batch(ctx, op, width, a_lwe, b_lwe, c_lwe=None):
    """Batched functional unit through the public path (host buffers)."""
    opi = FU[op] if isinstance(op, str) else op
    a = _u32(a_lwe)
    b = _u32(b_lwe)
    batch = a.size // (width * N.LWE_WORDS)
    c = _u32(c_lwe) if c_lwe is not None else None
    ow = lib.cvm_fu_out_width(opi, width)
    out = np.empty((batch, ow, N.LWE_WORDS), np.uint32)
    st = N.BackendStats()
    check(lib.cvm_fu_batch(ctx.handle, opi, width, batch, _vp(a), _vp(b), _vp(c), _vp(out),
                           ctypes.byref(st)))
    return out, st.as_dict()
