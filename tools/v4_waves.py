"""Developer probe: time of one full wave of each blind-rotation
organisation at its natural width (v4 with w warps per SM = 148*w
bootstraps, v3 5247 at 4 per SM, the wide kernel at 1 per SM) -- the
constants of the auto cost model in blind_rotate.cu."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2101_03403_b200 as P  # noqa: E402
from paper_2101_03403_b200._native import check, lib  # noqa: E402


def main():
    ks = P.KeySet(1)
    ctx = P.Context(0)
    ctx.upload_keyset(ks)
    ctx.set_profiling(True)
    rng = np.random.default_rng(0)
    nmax = 148 * 12
    a, b = rng.integers(0, 2, nmax), rng.integers(0, 2, nmax)
    base = ctx.alloc(3 * nmax)
    ctx.upload(base, ks.encrypt(a, 1))
    ctx.upload(base + nmax, ks.encrypt(b, 2))
    plan = [(6000 + 10 * w + 5, 148 * w) for w in range(1, 9)]
    plan += [(5247, 148 * 4), (5247, 148 * 2), (9, 148), (13, 296)]
    if os.environ.get("PLAN"):  # "variant:count,..."
        plan = [tuple(int(x) for x in it.split(":")) for it in os.environ["PLAN"].split(",")]
    res = {}
    for v, n in plan:
        gates = [("NAND", [(base + i, 1, 0), (base + nmax + i, 1, 0)], base + 2 * nmax + i)
                 for i in range(n)]
        check(lib.cvm_set_br_variant(v))
        best = None
        for _ in range(3):
            ctx.reset_stats()
            ctx.flush_l2()
            ctx.submit_level(gates)
            ctx.sync()
            st = ctx.kernel_stats()
            best = st["br_ms"] if best is None else min(best, st["br_ms"])
        out = ctx.download(base + 2 * nmax, n)
        ok = bool(np.array_equal(ks.decrypt(out), 1 - (a[:n] & b[:n])))
        res[f"{v}@{n}"] = {"br_ms": round(best, 3), "per_bootstrap_us": round(1e3 * best / n, 2),
                           "decrypt_ok": ok}
        print(v, n, res[f"{v}@{n}"], flush=True)
    check(lib.cvm_set_br_variant(0))
    print(json.dumps(res))


if __name__ == "__main__":
    main()
