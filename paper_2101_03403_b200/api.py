"""Python front end of the B200 backend (thin; the product is libcvm_b200.so).

Names follow the reference interface (cryptovm::Backend, gates.hpp:109-132) so
tests read like the reference's own.  Circuits (the reference's functional
units and emulator) are not re-implemented here: they arrive as recorded gate
tables (`Dag`, the reference GateDag's node list) and are replayed on the
device (`Backend.replay`, `dag_batch`).
"""
import ctypes

import numpy as np

from . import _native as N
from ._native import check, lib

GATE_KINDS = ["CONSTANT", "NOT", "COPY", "NAND", "AND", "OR", "XOR", "XNOR", "NOR",
              "ANDNY", "ANDYN", "ORNY", "ORYN", "MUX"]
KIND = {n: i for i, n in enumerate(GATE_KINDS)}

# cvm_dag_node (include/cvm_gpu.h): 32 bytes per node
DAG_DTYPE = np.dtype([("kind", "u1"), ("input", "u1"), ("value", "u1"), ("ndeps", "u1"),
                      ("region", "<u4"), ("dep", "<u8", (3,))])
assert DAG_DTYPE.itemsize == ctypes.sizeof(N.DagNode)


class Dag:
    """A recorded circuit: the reference GateDag's nodes (dag.hpp:33-42, ids
    1-based in creation order) plus each CONSTANT's value, and the ids of its
    output bits (LSB first).  Inputs are the input nodes in id order."""

    def __init__(self, nodes, outputs, name="", regions=None):
        self.nodes = np.ascontiguousarray(nodes, dtype=DAG_DTYPE)
        self.outputs = np.ascontiguousarray(outputs, dtype=np.uint64)
        self.name = name
        # region path of each node.region index (GateDag::regions(); [0] = "")
        self.regions = list(regions) if regions else None

    def _region_array(self):
        if not self.regions:
            return None, 0
        arr = (ctypes.c_char_p * len(self.regions))(*[r.encode() for r in self.regions])
        return arr, len(self.regions)

    @classmethod
    def from_rows(cls, rows, outputs, name=""):
        """rows: (n, 7) ints [kind, input, ndeps, d0, d1, d2, const_value] -- the
        oracle / golden-fixture layout."""
        rows = np.asarray(rows, dtype=np.int64).reshape(-1, 7)
        nodes = np.zeros(len(rows), DAG_DTYPE)
        nodes["kind"], nodes["input"], nodes["ndeps"] = rows[:, 0], rows[:, 1], rows[:, 2]
        nodes["dep"] = rows[:, 3:6]
        nodes["value"] = rows[:, 6]
        return cls(nodes, outputs, name)

    def rows(self):
        r = np.zeros((len(self.nodes), 7), np.int64)
        r[:, 0], r[:, 1], r[:, 2] = self.nodes["kind"], self.nodes["input"], self.nodes["ndeps"]
        r[:, 3:6] = self.nodes["dep"]
        r[:, 6] = self.nodes["value"]
        return r

    @property
    def n_inputs(self):
        return int(self.nodes["input"].sum())

    @property
    def n_nodes(self):
        return len(self.nodes)

    def bootstrapped(self):
        k = self.nodes["kind"][self.nodes["input"] == 0]
        return int((k >= KIND["NAND"]).sum())


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

    def set_kernels(self, br_variant=-1, ks_variant=-1, level_packing=-1):
        """This context's kernel choices (-1 = follow the process-wide setting)."""
        check(lib.cvm_ctx_set_kernels(self._h, br_variant, ks_variant, level_packing))

    def kernels(self):
        b, k, p = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        check(lib.cvm_ctx_get_kernels(self._h, ctypes.byref(b), ctypes.byref(k), ctypes.byref(p)))
        return {"br_variant": b.value, "ks_variant": k.value, "level_packing": p.value}

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

    def regions(self):
        """{region path: (recorded bootstrapped gates, executed)}."""
        n = ctypes.c_uint64()
        check(lib.cvm_backend_region_count(self._h, ctypes.byref(n)))
        out = {}
        buf = ctypes.create_string_buffer(512)
        rec, exe = ctypes.c_uint64(), ctypes.c_uint64()
        for i in range(n.value):
            check(lib.cvm_backend_region_info(self._h, i, buf, len(buf), ctypes.byref(rec),
                                              ctypes.byref(exe)))
            out[buf.value.decode()] = (rec.value, exe.value)
        return out

    def nodes(self):
        n = ctypes.c_uint64()
        check(lib.cvm_backend_node_count(self._h, ctypes.byref(n)))
        rows = np.zeros((n.value, 7), np.int64)
        check(lib.cvm_backend_nodes(self._h, 0, n.value, _vp(rows)))
        return rows

    # -- recorded circuits --
    def replay(self, dag, inputs):
        """Re-issue a recorded circuit on this backend; returns the handle of
        every node (index = node id - 1)."""
        inputs = np.ascontiguousarray(inputs, dtype=np.uint64).ravel()
        out = np.zeros(dag.n_nodes, np.uint64)
        names, n = dag._region_array()
        check(lib.cvm_backend_set_dag_regions(self._h, names, n))
        check(lib.cvm_backend_replay_dag(self._h, dag.nodes.ctypes.data, dag.n_nodes,
                                         _vp(inputs), len(inputs), _vp(out)))
        return out

    def replay_outputs(self, dag, inputs):
        return self.replay(dag, inputs)[dag.outputs.astype(np.int64) - 1]

    def evaluate(self, hs):
        """Evaluate the cone of `hs` now (one flush)."""
        hs = np.ascontiguousarray(hs, dtype=np.uint64).ravel()
        check(lib.cvm_backend_evaluate(self._h, len(hs), _vp(hs)))

    def encrypt_word(self, value, width):
        return np.array([self.encrypt_bit((value >> i) & 1) for i in range(width)], np.uint64)

    def decrypt_word(self, hs):
        bits = self.decrypt_bits(hs).astype(np.uint64)
        return int((bits << np.arange(len(bits), dtype=np.uint64)).sum())


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


def dag_batch(ctx, dag, in_lwe):
    """`batch` independent instances of a recorded circuit through the public
    C-ABI call cvm_dag_batch with host buffers: in_lwe (batch, n_inputs, 631)
    -> (batch, n_outputs, 631) ciphertexts, backend stats."""
    a = _u32(in_lwe)
    per = dag.n_inputs * N.LWE_WORDS
    if per == 0 or a.size % per:
        raise N.CvmInputError(f"in_lwe has {a.size} words, not a multiple of "
                              f"{dag.n_inputs} inputs x {N.LWE_WORDS}")
    batch = a.size // per
    out = np.empty((batch, len(dag.outputs), N.LWE_WORDS), np.uint32)
    st = N.BackendStats()
    names, n = dag._region_array()
    check(lib.cvm_dag_batch_regions(ctx.handle, dag.nodes.ctypes.data, dag.n_nodes, names, n,
                                    _vp(dag.outputs), len(dag.outputs), batch, _vp(a), a.size,
                                    _vp(out), out.size, ctypes.byref(st)))
    return out, st.as_dict()
