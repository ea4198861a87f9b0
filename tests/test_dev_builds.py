"""The developer instrumentation builds (clock64 phase marks behind
-DCVM_PHASE_PROF, read by tools/v4_phases.py and tools/pair_phases.py) still
compile for sm_100a, and export their read-out entry points only there."""
import os
import shutil
import subprocess

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(REPO, "paper_2101_03403_b200", "csrc")
NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"


@pytest.mark.skipif(not os.path.exists(NVCC), reason="needs nvcc")
@pytest.mark.parametrize("src,symbol", [("blind_rotate.cu", "cvm_debug_pair_phases"),
                                        ("blind_rotate_v4.cu", "cvm_debug_v4_phases")])
def test_phase_instrumented_build_compiles(tmp_path, src, symbol):
    objs = {}
    for tag, extra in (("prof", ["-DCVM_PHASE_PROF"]), ("product", [])):
        obj = tmp_path / f"{tag}.o"
        subprocess.run([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++20",
                        "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC", *extra, "-c",
                        os.path.join(CSRC, src), "-o", str(obj)], check=True)
        syms = subprocess.run(["nm", "-g", str(obj)], capture_output=True, text=True).stdout
        objs[tag] = symbol in syms
    assert objs == {"prof": True, "product": False}
