"""Developer probe: per-phase cycle breakdown of the v4 blind-rotation kernel.

Needs a library built with CVM_NVCC_EXTRA=-DCVM_PHASE_PROF (tools/gpu/v4_phases.sh).
Prints cycles per CMux step in each phase (PH4(k) marks in blind_rotate_v4.cu),
lane 0 of every warp, mean over warps of one full wave.
"""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2101_03403_b200 as P  # noqa: E402
from paper_2101_03403_b200._native import check, lib  # noqa: E402

NAMES = ["digits (6 rows)", "forward FFT (6)", "key wait (6)", "MAC + release (6)",
         "inverse FFT (2)", "round + ACC (2)"]


def main():
    n = int(os.environ.get("N_NAND", 1184))
    ks = P.KeySet(1)
    ctx = P.Context(0)
    ctx.upload_keyset(ks)
    rng = np.random.default_rng(0)
    a, b = rng.integers(0, 2, n), rng.integers(0, 2, n)
    base = ctx.alloc(3 * n)
    ctx.upload(base, ks.encrypt(a, 1))
    ctx.upload(base + n, ks.encrypt(b, 2))
    gates = [("NAND", [(base + i, 1, 0), (base + n + i, 1, 0)], base + 2 * n + i)
             for i in range(n)]
    check(lib.cvm_set_br_variant(int(os.environ.get("VARIANT", 6085))))
    ctx.set_profiling(True)
    for _ in range(3):
        ctx.reset_stats()
        ctx.submit_level(gates)
        ctx.sync()
    br = ctx.kernel_stats()["br_ms"]
    assert np.array_equal(ks.decrypt(ctx.download(base + 2 * n, n)), 1 - (a & b))
    buf = (ctypes.c_ulonglong * (148 * 8 * 8))()
    fn = lib.cvm_debug_v4_phases
    fn.argtypes = [ctypes.c_void_p]
    assert fn(buf) == 0
    ph = np.frombuffer(buf, dtype=np.uint64).reshape(148, 8, 8).astype(float) / 630
    ph = ph[:, :, :6].reshape(-1, 6)
    print(f"N={n} br_ms {br:.3f}; cycles per CMux step, mean (min..max) over {len(ph)} warps")
    for k, nm in enumerate(NAMES):
        print(f"  {nm:20s} {ph[:, k].mean():8.1f} ({ph[:, k].min():.0f}..{ph[:, k].max():.0f})")
    tot = ph.sum(1)
    print(f"  {'total':20s} {tot.mean():8.1f} -> {tot.mean() * 630 / 1.965e6:.2f} ms at 1.965 GHz")


if __name__ == "__main__":
    main()
