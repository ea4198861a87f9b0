"""Runs the kernel's FFT arithmetic (csrc/fft512.cuh, the same __host__
__device__ functions) on the CPU with 64 emulated threads: exchange
permutations, swizzle conflict-freedom and bit-exact negacyclic products,
with the table twiddles and with the generated twiddles (TwPow8) of the
v3 throughput kernel, and the warp-wide transform of the v4 kernel
(csrc/fft512w.cuh: one transpose plus a lane-pair swap, 32 emulated lanes);
the rounding margin of every mode is asserted."""
import os
import re
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
    r = subprocess.run([str(exe), "60"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "bit-exact" in r.stdout
    tab, rec = (float(x) for x in re.findall(r"twiddles: (?:max distance to integer )?([0-9.e-]+)",
                                             r.stdout))
    warp = float(re.search(r"warp FFT: ([0-9.e-]+)", r.stdout).group(1))
    # a rounding flip needs 0.5; every mode keeps a > 20x margin
    assert tab < 0.025 and rec < 0.025 and warp < 0.025, r.stdout
