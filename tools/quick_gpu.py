"""Developer probe for one gpurun call: FP64 peak, config-1 NAND level and
config-2 ADD16 batch throughput with kernel-event accounting."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2101_03403_b200 as P  # noqa: E402


def main():
    n_nand = int(os.environ.get("N_NAND", 4096))
    ks = P.KeySet(1)
    ctx = P.Context(0)
    t = time.time()
    ctx.upload_keyset(ks)
    res = {"upload_keys_s": time.time() - t, "sms": ctx.sm_count(),
           "fp64_peak_tflops": ctx.fp64_peak_tflops(3)}
    rng = np.random.default_rng(0)
    a, b = rng.integers(0, 2, n_nand), rng.integers(0, 2, n_nand)
    ca, cb = ks.encrypt(a, 1), ks.encrypt(b, 2)
    base = ctx.alloc(3 * n_nand)
    ctx.upload(base, ca)
    ctx.upload(base + n_nand, cb)
    gates = [("NAND", [(base + i, 1, 0), (base + n_nand + i, 1, 0)], base + 2 * n_nand + i)
             for i in range(n_nand)]
    ctx.set_profiling(True)
    times = []
    for rep in range(4):
        ctx.reset_stats()
        ctx.flush_l2()
        ctx.submit_level(gates)
        ctx.sync()
        st = ctx.kernel_stats()
        times.append((st["br_ms"], st["ks_ms"]))
    out = ctx.download(base + 2 * n_nand, n_nand)
    ok = bool(np.array_equal(ks.decrypt(out), 1 - (a & b)))
    br, ksm = min(times)
    res["c1"] = {"gates": n_nand, "br_ms": br, "ks_ms": ksm, "ok": ok,
                 "gates_per_s": n_nand / ((br + ksm) * 1e-3), "all": times}
    if os.environ.get("ONLY_C1"):
        print(json.dumps(res, indent=1))
        return
    # config 2
    batch = int(os.environ.get("ADD_BATCH", 256))
    av, bv = rng.integers(0, 1 << 16, batch), rng.integers(0, 1 << 16, batch)
    wa, wb = ks.encrypt_words(av, 16, 3), ks.encrypt_words(bv, 16, 4)
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                    "integration"))
    import refshim
    add16 = refshim.record_fu("add", 16)
    for rep in range(2):
        ctx.reset_stats()
        t = time.time()
        out, st = P.dag_batch(ctx, add16, np.concatenate([wa, wb], axis=1))
        wall = time.time() - t
    ks_ = ctx.kernel_stats()
    vals = ks.decrypt_words(out.reshape(-1, 631), 17)
    res["c2"] = {"batch": batch, "wall_s": wall, "ok": bool(np.array_equal(vals, av + bv)),
                 "kernel": ks_, "backend": st,
                 "gates_per_s_wall": st["bootstrapped"] / wall}
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
