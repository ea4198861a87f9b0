"""Tiny workload for compute-sanitizer (racecheck / memcheck / synccheck):
one small level per blind-rotation and key-switch kernel variant, plus a MUX
level, checked for decryption."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2101_03403_b200 as P  # noqa: E402
from paper_2101_03403_b200._native import check, lib  # noqa: E402


def main():
    n = int(os.environ.get("N", 6))
    variants = [int(v) for v in os.environ.get("VARIANTS", "6015,5247,9,96").split(",")]
    ks = P.KeySet(3)
    ctx = P.Context(0)
    ctx.upload_keyset(ks)
    rng = np.random.default_rng(0)
    a, b, c = (rng.integers(0, 2, n) for _ in range(3))
    base = ctx.alloc(4 * n)
    for k, bits in enumerate((a, b, c)):
        ctx.upload(base + k * n, ks.encrypt(bits, 10 + k))
    for v in variants:
        check(lib.cvm_set_br_variant(v))
        for kv in (8, 9):
            check(lib.cvm_set_ks_variant(kv))
            ctx.submit_level([("MUX", [(base + i, 1, 0), (base + n + i, 1, 0),
                                       (base + 2 * n + i, 1, 0)], base + 3 * n + i)
                              for i in range(n)])
            ctx.sync()
            got = ks.decrypt(ctx.download(base + 3 * n, n))
            ok = np.array_equal(got, np.where(a == 1, b, c))
            print(f"br={v} ks={kv} ok={ok}", flush=True)
            assert ok


if __name__ == "__main__":
    main()
