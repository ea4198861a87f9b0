"""Developer probe: time each blind-rotation kernel variant on a config-1
style NAND level and check they produce identical ciphertexts."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2101_03403_b200 as P  # noqa: E402
from paper_2101_03403_b200._native import check, lib  # noqa: E402


def main():
    n = int(os.environ.get("N_NAND", 4096))
    variants = [int(v) for v in os.environ.get("VARIANTS", "6085,5247,9,96").split(",")]
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
    ctx.set_profiling(True)
    res, ref = {}, None
    for v in variants:
        check(lib.cvm_set_br_variant(v))
        best = None
        for _ in range(3):
            ctx.reset_stats()
            ctx.flush_l2()
            ctx.submit_level(gates)
            ctx.sync()
            st = ctx.kernel_stats()
            best = st["br_ms"] if best is None else min(best, st["br_ms"])
        out = ctx.download(base + 2 * n, n)
        same = bool(ref is None or np.array_equal(out, ref))
        ref = out if ref is None else ref
        ok = bool(np.array_equal(ks.decrypt(out), 1 - (a & b)))
        res[v] = {"br_ms": best, "bootstraps_per_s": n / (best * 1e-3), "identical": same,
                  "decrypt_ok": ok}
        print(v, res[v], flush=True)
    check(lib.cvm_set_br_variant(0))
    for kv in [int(v) for v in os.environ.get("KS_VARIANTS", "8,9").split(",")]:
        check(lib.cvm_set_ks_variant(kv))
        best = None
        for _ in range(3):
            ctx.reset_stats()
            ctx.flush_l2()
            ctx.submit_level(gates)
            ctx.sync()
            st = ctx.kernel_stats()
            best = st["ks_ms"] if best is None else min(best, st["ks_ms"])
        out = ctx.download(base + 2 * n, n)
        res[f"ks{kv}"] = {"ks_ms": best, "identical": bool(np.array_equal(out, ref))}
        print(f"ks{kv}", res[f"ks{kv}"], flush=True)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
