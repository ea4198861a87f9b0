"""ctypes binding of libcvm_b200.so (include/cvm_gpu.h).

The library is the product: CUDA kernels for sm_100a plus the C++ host side
(GpuBackend, functional units, machine).  There is no Python or CPU fallback:
if the library is missing this module raises at import time, and creating a
device context without an sm_100a GPU raises CvmDeviceError.
"""
import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# CVM_LIB_PATH: an alternative build of the same library (developer A/B runs)
LIB_PATH = os.environ.get("CVM_LIB_PATH") or os.path.join(_HERE, "_lib", "libcvm_b200.so")

LWE_N, POLY_N, LWE_WORDS = 630, 1024, 631
BK_WORDS = 630 * 6 * 2 * 1024
KSK_WORDS = 1024 * 8 * 4 * 631


class CvmError(RuntimeError):
    pass


class CvmInputError(CvmError, ValueError):
    """cryptovm::InputError (errors.hpp) -- a precondition was violated."""


class CvmDeviceError(CvmError):
    pass


class CvmStateError(CvmError):
    pass


class Operand(ctypes.Structure):
    _fields_ = [("slot", ctypes.c_int64), ("sign", ctypes.c_int32),
                ("constant", ctypes.c_uint32)]


class Gate(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_uint32), ("pad", ctypes.c_uint32),
                ("inp", Operand * 3), ("out_slot", ctypes.c_uint64)]


class KernelStats(ctypes.Structure):
    _fields_ = [("br_launches", ctypes.c_uint64), ("br_jobs", ctypes.c_uint64),
                ("ks_launches", ctypes.c_uint64), ("ks_jobs", ctypes.c_uint64),
                ("other_launches", ctypes.c_uint64),
                ("br_ms", ctypes.c_double), ("ks_ms", ctypes.c_double)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class BackendStats(ctypes.Structure):
    _fields_ = [(n, ctypes.c_uint64) for n in
                ("nodes", "bootstrapped", "bootstraps", "levels_run", "flushes", "decrypts",
                 "last_flush_levels", "last_flush_gates", "max_level_width", "executed",
                 "executed_bootstraps", "pending")]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class DagNode(ctypes.Structure):
    """cvm_dag_node: one node of a recorded circuit (the reference DagNode)."""
    _fields_ = [("kind", ctypes.c_uint8), ("input", ctypes.c_uint8), ("value", ctypes.c_uint8),
                ("ndeps", ctypes.c_uint8), ("region", ctypes.c_uint32),
                ("dep", ctypes.c_uint64 * 3)]



_p = ctypes.c_void_p
_u64 = ctypes.c_uint64
_i = ctypes.c_int
_u32 = ctypes.c_uint32
_u64p = ctypes.POINTER(ctypes.c_uint64)

# name: (restype, argtypes)
_SIGS = {
    "cvm_last_error": (ctypes.c_char_p, []),
    "cvm_version": (ctypes.c_char_p, []),
    "cvm_keyset_generate": (_i, [_u64, ctypes.POINTER(_p)]),
    "cvm_keyset_destroy": (None, [_p]),
    "cvm_keyset_export": (_i, [_p, _p, _p, _p, _p]),
    "cvm_encrypt_bits": (_i, [_p, _u64, ctypes.c_size_t, _p, _p]),
    "cvm_decrypt_bits": (_i, [_p, ctypes.c_size_t, _p, _p, _p]),
    "cvm_ctx_create": (_i, [_i, ctypes.POINTER(_p)]),
    "cvm_ctx_destroy": (None, [_p]),
    "cvm_upload_keys": (_i, [_p, _p, _p]),
    "cvm_upload_keyset": (_i, [_p, _p]),
    "cvm_slots_alloc": (_i, [_p, _u64, _u64p]),
    "cvm_slots_reserve": (_i, [_p, _u64]),
    "cvm_slots_capacity": (_u64, [_p]),
    "cvm_upload_lwe": (_i, [_p, _u64, _u64, _p]),
    "cvm_download_lwe": (_i, [_p, _u64, _u64, _p]),
    "cvm_submit_level": (_i, [_p, _p, _u64]),
    "cvm_sync": (_i, [_p]),
    "cvm_ctx_set_profiling": (_i, [_p, _i]),
    "cvm_ctx_kernel_stats": (_i, [_p, ctypes.POINTER(KernelStats)]),
    "cvm_ctx_reset_stats": (_i, [_p]),
    "cvm_ctx_flush_l2": (_i, [_p]),
    "cvm_ctx_event_record": (_i, [_p, _i]),
    "cvm_ctx_event_elapsed_ms": (_i, [_p, ctypes.POINTER(ctypes.c_double)]),
    "cvm_ctx_fp64_peak": (_i, [_p, _i, ctypes.POINTER(ctypes.c_double)]),
    "cvm_ctx_sm_count": (_i, [_p, ctypes.POINTER(_i)]),
    "cvm_set_br_variant": (_i, [_i]),
    "cvm_get_br_variant": (_i, []),
    "cvm_set_level_packing": (_i, [_i]),
    "cvm_get_level_packing": (_i, []),
    "cvm_set_ks_variant": (_i, [_i]),
    "cvm_get_ks_variant": (_i, []),
    "cvm_ctx_set_kernels": (_i, [_p, _i, _i, _i]),
    "cvm_ctx_get_kernels": (_i, [_p, ctypes.POINTER(_i), ctypes.POINTER(_i), ctypes.POINTER(_i)]),
    "cvm_backend_create":(_i, [_p, _p, _u64, ctypes.POINTER(_p)]),
    "cvm_backend_destroy": (None, [_p]),
    "cvm_backend_constant": (_i, [_p, _i, _u64p]),
    "cvm_backend_unary_gate": (_i, [_p, _u32, _u64, _u64p]),
    "cvm_backend_binary_gate": (_i, [_p, _u32, _u64, _u64, _u64p]),
    "cvm_backend_mux_gate": (_i, [_p, _u64, _u64, _u64, _u64p]),
    "cvm_backend_encrypt_bit": (_i, [_p, _i, _u64p]),
    "cvm_backend_decrypt_bit": (_i, [_p, _u64, ctypes.POINTER(_i)]),
    "cvm_backend_decrypt_bits": (_i, [_p, ctypes.c_size_t, _p, _p]),
    "cvm_backend_import_lwe": (_i, [_p, ctypes.c_size_t, _p, _p]),
    "cvm_backend_export_lwe": (_i, [_p, ctypes.c_size_t, _p, _p]),
    "cvm_backend_export_bit": (_i, [_p, _u64, _p, ctypes.c_size_t]),
    "cvm_backend_import_bit": (_i, [_p, _p, ctypes.c_size_t, _u64p]),
    "cvm_backend_push_region": (_i, [_p, ctypes.c_char_p]),
    "cvm_backend_pop_region": (_i, [_p]),
    "cvm_backend_fence": (_i, [_p]),
    "cvm_backend_flush": (_i, [_p]),
    "cvm_backend_set_flush_policy": (_i, [_p, _i]),
    "cvm_backend_stats_get":(_i, [_p, ctypes.POINTER(BackendStats)]),
    "cvm_backend_region_count": (_i, [_p, _u64p]),
    "cvm_backend_region_info": (_i, [_p, _u64, ctypes.c_char_p, ctypes.c_size_t, _u64p, _u64p]),
    "cvm_backend_node_count": (_i, [_p, _u64p]),
    "cvm_backend_nodes": (_i, [_p, _u64, _u64, _p]),
    "cvm_backend_capture_plan": (_i, [_p, ctypes.POINTER(_p)]),
    "cvm_plan_run": (_i, [_p, _p, _i]),
    "cvm_plan_info": (_i, [_p, _u64p, _u64p, _u64p]),
    "cvm_plan_destroy": (None, [_p]),
    "cvm_backend_handle_slot": (_i, [_p, _u64, ctypes.POINTER(ctypes.c_int64),
                                     ctypes.POINTER(ctypes.c_int32),
                                     ctypes.POINTER(ctypes.c_uint32)]),
    "cvm_backend_replay_dag": (_i, [_p, _p, _u64, _p, _u64, _p]),
    "cvm_backend_evaluate": (_i, [_p, ctypes.c_size_t, _p]),
    "cvm_backend_set_dag_regions": (_i, [_p, _p, _u64]),
    "cvm_dag_batch_regions": (_i, [_p, _p, _u64, _p, _u64, _p, _u64, _u64, _p, _u64, _p, _u64,
                                   ctypes.POINTER(BackendStats)]),
    "cvm_dag_batch": (_i, [_p, _p, _u64, _p, _u64, _u64, _p, _u64, _p, _u64,
                           ctypes.POINTER(BackendStats)]),
}

EXPORTED = tuple(_SIGS)


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2101_03403_b200.build` "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()

_ERRORS = {-1: CvmInputError, -2: CvmDeviceError, -3: CvmStateError, -4: MemoryError}


def check(rc):
    if rc != 0:
        msg = (lib.cvm_last_error() or b"").decode(errors="replace")
        raise _ERRORS.get(rc, CvmError)(msg)
    return rc
