"""Runs the kernel's FFT arithmetic (csrc/fft512.cuh, the same __host__
__device__ functions) on the CPU with 64 emulated threads: exchange
permutations, swizzle conflict-freedom and bit-exact negacyclic products."""
import os
import shutil
import subprocess

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(shutil.which("g++") is None, reason="needs g++")
def test_fft_emulation_bit_exact(tmp_path):
    exe = tmp_path / "fft_emul"
    subprocess.run(["g++", "-O2", "-std=c++17", "-ffp-contract=off",
                    "-I", os.path.join(REPO, "paper_2101_03403_b200", "csrc"),
                    os.path.join(REPO, "tests", "native", "fft_emul.cpp"), "-o", str(exe)],
                   check=True)
    r = subprocess.run([str(exe), "30"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "bit-exact" in r.stdout
