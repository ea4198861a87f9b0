"""The C-ABI library loads, exports every symbol include/cvm_gpu.h declares,
and fails loudly (no CPU fallback) when no sm_100a device is present."""
import ctypes
import os
import re

import pytest

import paper_2101_03403_b200 as P
from paper_2101_03403_b200 import _native as N

HEADER = os.path.join(os.path.dirname(os.path.dirname(__file__)), "include", "cvm_gpu.h")


def _declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"CVM_API\s+[\w\s\*]+?\b(cvm_\w+)\s*\(", src)))


def test_header_declares_entry_points():
    names = _declared()
    assert len(names) > 40
    assert "cvm_submit_level" in names and "cvm_backend_binary_gate" in names


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(N.LIB_PATH)
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_python_binding_covers_header():
    assert sorted(N.EXPORTED) == _declared()


def test_struct_layouts():
    # cvm_gate: kind, pad, 3 x cvm_operand(16 B), out_slot
    assert ctypes.sizeof(N.Operand) == 16
    assert ctypes.sizeof(N.Gate) == 8 + 48 + 8
    # cvm_dag_node: kind, input, value, ndeps, pad, dep[3]
    assert ctypes.sizeof(N.DagNode) == 32 == P.DAG_DTYPE.itemsize


def test_dag_batch_checks_buffer_sizes_before_touching_them():
    """cvm_dag_batch validates the table and the element counts of both host
    buffers against it (no over-read on mismatched shapes).  A
    NULL context is rejected first, so this runs without a GPU."""
    import numpy as np
    st = N.BackendStats()
    nodes = np.zeros(3, P.DAG_DTYPE)
    nodes["input"][:2] = 1
    nodes["kind"][2], nodes["ndeps"][2] = P.KIND["AND"], 2
    nodes["dep"][2, :2] = (1, 2)
    outs = np.array([3], np.uint64)
    with pytest.raises(P.CvmInputError):
        N.check(N.lib.cvm_dag_batch(None, nodes.ctypes.data, 3, outs.ctypes.data, 1, 1,
                                    None, 0, None, 0, ctypes.byref(st)))


def test_version_and_errors():
    assert b"sm_100a" in N.lib.cvm_version()
    with pytest.raises(P.CvmInputError):
        N.check(N.lib.cvm_keyset_generate(1, None))
    assert b"null" in N.lib.cvm_last_error()


def test_process_wide_kernel_knobs():
    """Variant / packing setters validate their argument (host-only, no GPU):
    every documented value is accepted and restored, anything else raises
    InputError and leaves the setting unchanged."""
    lib = N.lib
    br, ks, pack = lib.cvm_get_br_variant(), lib.cvm_get_ks_variant(), lib.cvm_get_level_packing()
    try:
        for v in (0, 9, 96, 5247, 6085, 6015, 6045):
            N.check(lib.cvm_set_br_variant(v))
            assert lib.cvm_get_br_variant() == v
        # retired round-1 variants and malformed numbers are rejected
        for v in (1, 13, 92, 4044, 5044, 6185, 6084, 6095, 6005, 7000):
            with pytest.raises(P.CvmInputError):
                N.check(lib.cvm_set_br_variant(v))
            assert lib.cvm_get_br_variant() == 6045
        for v in (0, 8, 9):
            N.check(lib.cvm_set_ks_variant(v))
            assert lib.cvm_get_ks_variant() == v
        for v in (1, 5, 6, 7):
            with pytest.raises(P.CvmInputError):
                N.check(lib.cvm_set_ks_variant(v))
        for v in (0, 1):
            N.check(lib.cvm_set_level_packing(v))
            assert lib.cvm_get_level_packing() == v
        with pytest.raises(P.CvmInputError):
            N.check(lib.cvm_set_level_packing(2))
    finally:
        N.check(lib.cvm_set_br_variant(br))
        N.check(lib.cvm_set_ks_variant(ks))
        N.check(lib.cvm_set_level_packing(pack))


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(_has_gpu(), reason="checks the no-device failure path")
def test_no_device_fails_loudly():
    with pytest.raises(P.CvmDeviceError):
        P.Context(0)
