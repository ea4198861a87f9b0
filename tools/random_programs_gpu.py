"""Evidence run: the reference's random-program cross-check (emulator_test.cc:
486-640's shape -- seeded straight-line programs over the data-path ISA) at a
scale the test suite cannot afford.  Each program is recorded once by the
reference Machine (refshim.record_program) and run by cvm_dag_batch for a
batch of memory images; every final register and NZCV flag is compared with
the reference Machine on SimBackend (refshim.sim_program) for the same image.
Summary: profiles/r02_random_programs_gpu.json.

    python tools/random_programs_gpu.py [OUT.json]
"""
import json
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "integration"))
import paper_2101_03403_b200 as P  # noqa: E402
import refshim  # noqa: E402

PLAN = [(8, 200, 64), (16, 100, 32), (32, 20, 8)]  # (word size, programs, images)
N_MEM, N_REGS = 4, 8


def main():
    out_path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/random_programs.json"
    only = {int(x) for x in sys.argv[2:]}  # optional word sizes to run
    ks = P.KeySet(9)
    ctx = P.Context(0)
    ctx.upload_keyset(ks)
    rng = np.random.default_rng(2026)
    res = {}
    for w, n_prog, n_img in PLAN:
        if only and w not in only:
            continue
        bad_runs, runs, gates, t0 = 0, 0, 0, time.time()
        for k in range(n_prog):
            prog = refshim.random_program(rng, w, n_mem=N_MEM, n_regs=N_REGS)
            dag = refshim.record_program(prog, N_MEM, w, N_REGS)
            mems = rng.integers(0, 1 << w, (n_img, N_MEM), dtype=np.uint64)
            lwe = ks.encrypt_words(mems.ravel(), w, 3000 + 7 * k).reshape(n_img, -1, 631)
            out, st = P.dag_batch(ctx, dag, lwe)
            bits = ks.decrypt(out.reshape(-1, 631)).reshape(n_img, -1).astype(np.uint64)
            for m in range(n_img):
                regs, nzcv = refshim.sim_program(prog, mems[m], w, N_REGS)
                got = [int((bits[m, w * r:w * r + w] << np.arange(w, dtype=np.uint64)).sum())
                       for r in range(N_REGS)]
                ok = got == [int(x) for x in regs] and list(bits[m, w * N_REGS:]) == list(nzcv)
                bad_runs += not ok
                runs += 1
            gates += int(st["executed_bootstraps"])
        dt = time.time() - t0
        res[f"width{w}"] = {"programs": n_prog, "images_per_program": n_img, "runs": runs,
                            "mismatching_runs": bad_runs, "bootstraps": gates,
                            "seconds": round(dt, 1)}
        print(w, res[f"width{w}"], flush=True)
    json.dump({"what": "random straight-line programs (emulator_test.cc cross-check shape): "
                       "cvm_dag_batch on the reference-recorded program vs the reference "
                       "Machine on SimBackend, registers + NZCV", "results": res},
              open(out_path, "w"), indent=1)
    return 0 if all(r["mismatching_runs"] == 0 for r in res.values()) else 1


if __name__ == "__main__":
    sys.exit(main())
