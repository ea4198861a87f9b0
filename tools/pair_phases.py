"""Developer probe: per-phase cycle breakdown of the pair kernel's CMux step.

Needs a library built with CVM_NVCC_EXTRA=-DCVM_PHASE_PROF (tools/gpu/pair_phases.sh).
Prints, for groups 0 and 1 (thread 0) averaged over the CTAs, cycles per step in
each phase of blind_rotate_pair_kernel (blind_rotate.cu, PH(k) marks).
"""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2101_03403_b200 as P  # noqa: E402
from paper_2101_03403_b200._native import check, lib  # noqa: E402

NAMES = ["top barrier", "rotate+digits", "fwd FFT", "key wait",
         "MAC + all-partials barrier", "next-row copy issue", "own sum / send", "peer wait",
         "inv A+ex", "inv B+ex", "inv C", "add_rounded"]


def main():
    n = int(os.environ.get("N_NAND", 74))
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
    check(lib.cvm_set_br_variant(int(os.environ.get("VARIANT", 96))))
    ctx.set_profiling(True)
    for _ in range(3):
        ctx.reset_stats()
        ctx.submit_level(gates)
        ctx.sync()
    print("br_ms", ctx.kernel_stats()["br_ms"])
    assert np.array_equal(ks.decrypt(ctx.download(base + 2 * n, n)), 1 - (a & b))
    buf = (ctypes.c_ulonglong * (296 * 2 * 12))()
    fn = lib.cvm_debug_pair_phases
    fn.argtypes = [ctypes.c_void_p]
    assert fn(buf) == 0
    ph = np.frombuffer(buf, dtype=np.uint64).reshape(296, 2, 12)[: 2 * n].astype(float) / 630
    for r in (0, 1):
        sel = ph[r::2]
        print(f"CTA rank {r}: cycles per step (mean over {len(sel)} CTAs)")
        for k, nm in enumerate(NAMES):
            print(f"  {nm:22s} g0 {sel[:, 0, k].mean():8.1f}   g1 {sel[:, 1, k].mean():8.1f}")
        print(f"  {'total':22s} g0 {sel[:, 0].sum(1).mean():8.1f}   g1 {sel[:, 1].sum(1).mean():8.1f}")


if __name__ == "__main__":
    main()
