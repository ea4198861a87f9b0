"""Where does the e2e (cvm_fu_batch) time go?  Host recording vs device time
for the config-2 batch (256 x ADD16).  Run with CVM_FU_TIMING=1."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2101_03403_b200 as P  # noqa: E402


def main():
    batch = int(os.environ.get("BATCH", 256))
    ks = P.KeySet(1)
    ctx = P.Context(0)
    ctx.upload_keyset(ks)
    rng = np.random.default_rng(0)
    av, bv = rng.integers(0, 1 << 16, batch), rng.integers(0, 1 << 16, batch)
    a, b = ks.encrypt_words(av, 16, 5), ks.encrypt_words(bv, 16, 6)
    for rep in range(4):
        ctx.set_profiling(rep > 0)
        ctx.reset_stats()
        t = time.perf_counter()
        res, st = P.fu_batch(ctx, os.environ.get("OP", "add"), 16, a, b)
        wall = (time.perf_counter() - t) * 1e3
        k = ctx.kernel_stats()
        print(f"rep {rep}: wall {wall:.1f} ms, device br {k['br_ms']:.1f} + ks {k['ks_ms']:.1f} ms,"
              f" levels {st['last_flush_levels']}", flush=True)


if __name__ == "__main__":
    main()
