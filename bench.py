#!/usr/bin/env python3
"""Benchmark: batched TFHE gate bootstrapping under CryptoEmu's functional units.

Workload (BASELINE.json configs[1], the config the headline metric is quoted
on): 256 independent 16-bit homomorphic ADDs (Kogge-Stone, 195 bootstrapped
gates each, 9 dataflow levels -> 49,920 bootstraps per step), n=630, N=1024,
l=3, Bg=2^7, t=8, base 4, torus32, seeded synthetic operands (no dataset is
involved; inputs are uniform random 16-bit integers encrypted under seeded keys).
The adder circuit is the reference's own alu::add, recorded once by the
reference code (integration/refshim.py -> libcvm_refshim.so) and replayed by
the B200 library (cvm_backend_replay_dag / cvm_dag_batch).

  value   bootstrapped gates/s with inputs resident in HBM: one step = the
          recorded 256-adder plan replayed on the device.
  e2e     the same metric through the public C-ABI call cvm_dag_batch with host
          buffers: pinned H2D of the 512 operand words (20.7 MB), replay of the
          recorded table, levelised execution, D2H of the 256 x 17 result bits.
          cvm_dag_batch evaluates only the outputs' cone (180 of 195 gates per
          ADD16), so e2e counts the gates it executes; ADD16/s is beside it.
          e2e.reference_api: the reference's own API through the drop-in
          (Word::encrypt, alu::add on cryptovm::GpuBackend, decrypt_word per
          result; host encryption and decryption inside the timed region).
  roofline  the blind-rotation kernels (99% of the device time): algorithmic
          FP64 flops per bootstrap (147,087,360) x
          bootstraps / summed kernel event time, against the FP64 DFMA peak
          measured live (MEASURED_PEAKS.json has no FP64 figure).

Multi-GPU (--gpus N under torchrun): weak scaling, each rank runs its own 256
independent adders (no data-path collective; gates of a level are
independent), barrier + max-over-ranks device time.

--impl reference: the reference's path on the host CPU.  The reference ships
no TFHE code, so this arm times the CPU restatement
of the TFHE library's gate bootstrapping (oracle/, double-precision FFT: the
library's own method) on all host threads, evaluating whole ADD16 circuits
(the same recorded DAG, several adders level by level in lockstep).
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

ALG_FLOP_PER_BOOTSTRAP = 147_087_360  # n[(k+1)(l+1)5(N/2)log(N/2) + (k+1)^2 l (N/2) 8]
WIDTH, BATCH = 16, 256
GATES_PER_ADD = 195
METRIC = "bootstrapped gates/s (batched) on 1 B200; 16-bit FHE ADD ops/s & latency"
KEY_SEED, DATA_SEED = 20260808, 4242
USES_C = {"add_cin", "addsub"}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                     "--format=csv,noheader,nounits"], capture_output=True, text=True,
                    timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 4 + i and r[4 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows),
                "power_w_max": max((float(r[2]) for r in self.rows
                                    if r[2].replace(".", "").isdigit()), default=None)}


def workload_operands(rank):
    rng = np.random.default_rng(DATA_SEED + rank)
    return rng.integers(0, 1 << WIDTH, BATCH), rng.integers(0, 1 << WIDTH, BATCH)


# --------------------------------------------------------- recorded circuits --
def load_dag(op, width):
    """The unit's gate table as the reference records it: live from the
    reference code (integration/_build/libcvm_refshim.so); if that library
    was not built, the same table the reference run stored in
    tests/golden/dags.npz (tests/golden/make_golden.py)."""
    import paper_2101_03403_b200 as P
    sys.path.insert(0, os.path.join(REPO, "integration"))
    import refshim
    if refshim.available():
        d = refshim.record_fu(op, width)
        d.source = "reference alu recorded live (libcvm_refshim.so)"
        return d
    g = np.load(os.path.join(REPO, "tests", "golden", "dags.npz"))
    src = "umul" if op == "mul_lo" else op
    outs = g[f"{src}_{width}_out"][:width] if op == "mul_lo" else g[f"{src}_{width}_out"]
    d = P.Dag.from_rows(g[f"{src}_{width}_nodes"], outs, f"{op}{width}")
    d.source = "reference alu table from tests/golden/dags.npz"
    return d


def operand_lwe(ks, op, width, av, bv, seed, cv=None):
    """(batch, n_inputs, 631): a's bits, b's bits (LSB first)[, c]."""
    parts = [ks.encrypt_words(av, width, seed), ks.encrypt_words(bv, width, seed + 1)]
    if op in USES_C:
        parts.append(ks.encrypt(np.asarray(cv, np.uint8), seed + 2).reshape(-1, 1, 631))
    return np.concatenate(parts, axis=1)


def replicate_rows(rows, k):
    """k independent copies of a gate table ((n, 7) oracle layout) in one."""
    n = len(rows)
    out = np.tile(rows, (k, 1))
    for i in range(1, k):
        blk = out[i * n:(i + 1) * n]
        dep = blk[:, 3:6]
        blk[:, 3:6] = np.where(dep > 0, dep + i * n, 0)
    return out


# ------------------------------------------------------------ CPU baseline --
def cpu_info():
    info = {"cpu_model": "unknown", "nproc": os.cpu_count()}
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    info["cpu_model"] = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        import psutil
        info["physical_cores"] = psutil.cpu_count(logical=False)
        info["logical_cpus"] = psutil.cpu_count(logical=True)
    except Exception:
        pass
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=5).stdout
        for line in out.splitlines():
            if line.startswith("Thread(s) per core"):
                info["threads_per_core"] = int(line.split(":")[1])
    except Exception:
        pass
    return info


def cpu_add16_circuits(adders, threads, rounds=1):
    """The oracle (double-FFT TFHE, the library's method) evaluating `adders`
    whole ADD16 circuits (the reference's recorded DAG) level by level, all
    adders of a level in one multi-threaded lockstep batch.  Returns
    (bootstrapped gates per second, seconds, gates evaluated, decrypted ok)."""
    sys.path.insert(0, os.path.join(REPO, "oracle"))
    import oracle as O
    sk = O.SecretKeys(KEY_SEED)
    ck = O.CloudKeys(sk.bk, sk.ksk, O.MODE_FFT)
    dag = load_dag("add", WIDTH)
    rows = replicate_rows(dag.rows(), adders)
    rng = np.random.default_rng(7)
    av, bv = rng.integers(0, 1 << WIDTH, adders), rng.integers(0, 1 << WIDTH, adders)
    lanes = np.arange(WIDTH)
    bits = np.concatenate([np.concatenate([(av[i] >> lanes) & 1, (bv[i] >> lanes) & 1])
                           for i in range(adders)]).astype(np.uint8)
    cts = sk.encrypt(bits, 8)
    t = time.perf_counter()
    for _ in range(rounds):
        ct = O.eval_dag(ck, rows, cts, threads)
    dt = time.perf_counter() - t
    outs = np.concatenate([dag.outputs.astype(np.int64) - 1 + i * dag.n_nodes
                           for i in range(adders)])
    dec = sk.decrypt(ct[outs]).reshape(adders, WIDTH + 1).astype(np.int64)
    ok = bool(np.array_equal((dec << np.arange(WIDTH + 1)).sum(axis=1), av + bv))
    gates = adders * dag.bootstrapped() * rounds
    return gates / dt, dt, gates, ok


def cpu_baseline():
    """Bounded CPU sample on rank 0 at N=1: whole ADD16 circuits on the
    oracle with every host thread (about 10-20 s)."""
    info = cpu_info()
    threads = os.cpu_count() or 1
    adders = int(os.environ.get("CPU_ADDERS", max(4, threads)))
    rate, dt, gates, ok = cpu_add16_circuits(adders, threads)
    # one bootstrap on one thread, for comparison with the paper's single-core
    # 25.6 ms per gate (a 2014 Xeon core with the TFHE
    # library's AVX FFT)
    sys.path.insert(0, os.path.join(REPO, "oracle"))
    import oracle as O
    sk = O.SecretKeys(KEY_SEED)
    ck = O.CloudKeys(sk.bk, sk.ksk, O.MODE_FFT)
    a1, b1 = sk.encrypt(np.array([1, 0], np.uint8), 3), sk.encrypt(np.array([1, 1], np.uint8), 4)
    t = time.perf_counter()
    ck.gates(np.array([O.AND, O.XOR], np.uint8), a1, b1, None, 1)
    one = (time.perf_counter() - t) / 2
    return {"value": rate, "unit": "bootstrapped gates/s", "cores": threads, "kind": "port",
            "seconds": dt, **info, "single_thread_ms_per_gate": 1e3 * one,
            "sample": f"{adders} whole ADD16 circuits ({gates} bootstrapped gates, all 9 "
                      f"levels, adders in lockstep per level), oracle/ double-FFT TFHE "
                      f"(the TFHE library's method), {threads} threads",
            "add16_ops_per_s": rate / GATES_PER_ADD, "decrypted_correct": ok}


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    adders = int(os.environ.get("REF_ADDERS", max(4, threads)))
    cpu_add16_circuits(max(1, adders // 4), threads)  # warm-up: keys, caches
    times, gates, ok = [], 0, True
    for _ in range(args.warmup):
        cpu_add16_circuits(1, threads)
    for _ in range(args.steps):
        rate, dt, g, good = cpu_add16_circuits(adders, threads)
        times.append(dt)
        gates += g
        ok &= good
    total = sum(times)
    value = gates / total
    info = cpu_info()
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "bootstrapped gates/s",
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u32 torus / f64 FFT", "data": "synthetic",
        "config": {"workload": "config2: ADD16 circuits (n=630,N=1024,l=3,Bg=2^7,t=8,base 4)",
                   "sample_per_step": f"{adders} whole ADD16 circuits "
                                      f"({adders * GATES_PER_ADD} bootstraps, 9 levels)",
                   "parallelism": f"cpu threads={threads}"},
        "add16_ops_per_s": value / GATES_PER_ADD,
        "cpu_baseline": {"value": value, "unit": "bootstrapped gates/s", "cores": threads,
                         "kind": "port", **info, "decrypted_correct": ok,
                         "sample": f"{adders} ADD16 circuits per step, double-FFT TFHE "
                                   f"(oracle/), adders in lockstep per level"},
        "e2e": {"value": value, "unit": "bootstrapped gates/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "note": "reference repo has no TFHE implementation (cleartext SimBackend only); "
                "this arm is the CPU restatement of the TFHE library's bootstrapping "
                "evaluating the reference's recorded ADD16 circuit",
    }
    print(json.dumps(line))
    return 0


# ------------------------------------------------------- other configs ---
# (op, batch, reference for the decrypted check)
EXTRA_OPS = [
    ("sub", 256, lambda a, b, w: (a - b) % (1 << w), WIDTH),
    ("cmp", 256, lambda a, b, w: (a - b) % (1 << w), WIDTH),
    ("and", 256, lambda a, b, w: a & b, WIDTH),
    ("orr", 256, lambda a, b, w: a | b, WIDTH),
    ("eor", 256, lambda a, b, w: a ^ b, WIDTH),
    ("lsl", 256, lambda a, b, w: (a << (b % w)) % (1 << w), WIDTH),
    ("lsr", 256, lambda a, b, w: a >> (b % w), WIDTH),
    ("mul_lo", 64, lambda a, b, w: (a * b) % (1 << w), WIDTH),
    ("umul", 64, lambda a, b, w: a * b, 2 * WIDTH),
    ("udiv", 16, lambda a, b, w: a // b, WIDTH),
]


def extra_configs(P, ctx, ks, fp64_peak):
    """Configs 1, 3, 4 and 5 (BASELINE.json configs[0,2,3,4]) plus the other
    16-bit units, each run once through the public batched API (host buffers
    in and out, cvm_dag_batch) with the device time of its kernels, its
    batch-1 latency, its roofline fraction, and the reference's cleartext
    SimBackend on the same circuit; reported beside the headline line."""
    sys.path.insert(0, os.path.join(REPO, "integration"))
    import refshim
    rng = np.random.default_rng(77)
    out = {}
    # cvm_dag_batch returns its scratch slots, so the slab only holds the
    # largest single call; size it once (config 4: 216k gates + inputs).
    ctx.reserve(ctx.alloc(0) + 300_000)
    ctx.set_profiling(True)

    def frac(boots, ms):
        return boots * ALG_FLOP_PER_BOOTSTRAP / (ms * 1e-3) / 1e12 / fp64_peak

    def run(dag, lwe):
        ctx.reset_stats()
        t = time.perf_counter()
        res, st = P.dag_batch(ctx, dag, lwe)
        wall = time.perf_counter() - t
        k = ctx.kernel_stats()
        return res, st, wall, k["br_ms"] + k["ks_ms"], k["br_ms"]

    # config 1: 4096 independent NAND, one level
    n = 4096
    a_bits, b_bits = rng.integers(0, 2, n), rng.integers(0, 2, n)
    base = ctx.alloc(3 * n)
    ctx.upload(base, ks.encrypt(a_bits, 901))
    ctx.upload(base + n, ks.encrypt(b_bits, 902))
    ctx.reset_stats()
    ctx.submit_level([("NAND", [(base + i, 1, 0), (base + n + i, 1, 0)], base + 2 * n + i)
                      for i in range(n)])
    ctx.sync()
    k = ctx.kernel_stats()
    ok = np.array_equal(ks.decrypt(ctx.download(base + 2 * n, n)), 1 - (a_bits & b_bits))
    dev = k["br_ms"] + k["ks_ms"]
    out["config1_nand4096"] = {"gates_per_s_device": n / (dev * 1e-3), "device_ms": dev,
                               "roofline_frac": frac(n, k["br_ms"]), "correct": bool(ok)}
    for op, batch, want, ow in EXTRA_OPS:
        dag = load_dag(op, WIDTH)
        av = rng.integers(0, 1 << WIDTH, batch)
        bv = rng.integers(1 if op == "udiv" else 0, 1 << WIDTH, batch)
        lwe = operand_lwe(ks, op, WIDTH, av, bv, 910 + 10 * len(out))
        run(dag, lwe[:2])  # first use of this table's kernel shapes: untimed
        res, st, wall, dev, br = run(dag, lwe)
        # the value bits (SUB / CMP also return carry or NZCV after them)
        vals = ks.decrypt_words(np.ascontiguousarray(res[:, :ow]).reshape(-1, 631), ow)
        boots = st["executed_bootstraps"]
        d = {"batch": batch, "recorded_gates": st["bootstrapped"],
             "executed_gates": st["executed"], "executed_bootstraps": boots,
             "levels": st["last_flush_levels"], "wall_s": wall, "device_ms": dev,
             "ops_per_s_e2e": batch / wall, "ops_per_s_device": batch / (dev * 1e-3),
             "gates_per_s_device": st["executed"] / (dev * 1e-3),
             "bootstraps_per_s_device": boots / (dev * 1e-3),
             "roofline_frac": frac(boots, br),
             "correct": bool(np.array_equal(vals, want(av, bv, WIDTH)))}
        # batch-1 latency: one unit alone (the latency kernels)
        _, _, w1, dev1, _ = run(dag, lwe[:1])
        d["latency_batch1_ms_device"], d["latency_batch1_ms_wall"] = dev1, 1e3 * w1
        # the reference's own CPU path on the same circuit (cleartext booleans)
        sim_out, sim_s, nodes = refshim.sim_fu_batch(op, WIDTH, av, bv) \
            if refshim.available() else (None, None, None)
        if sim_s:
            d["reference_simbackend"] = {"gates_per_s": st["bootstrapped"] / sim_s,
                                         "ops_per_s": batch / sim_s, "dag_nodes": nodes,
                                         "note": "cleartext booleans, not FHE work"}
        out[f"{op}16"] = d
    # config 5: the golden seeded 64-instruction program + UDIV on 8 encrypted
    # registers, recorded by the reference Machine (dataflow across fences)
    meta = json.load(open(os.path.join(REPO, "tests", "golden", "programs.json")))[0]
    prog = [tuple(i) for i in meta["insns"]]
    if refshim.available():
        dag = refshim.record_program(prog, len(meta["mem"]))
        mem = ks.encrypt_words(meta["mem"], WIDTH, 940).reshape(1, -1, 631)
        res, st, wall, dev, br = run(dag, mem)
        bits = ks.decrypt(res.reshape(-1, 631))
        words = bits[:8 * WIDTH].reshape(8, WIDTH).astype(np.int64)
        vals = [int((w << np.arange(WIDTH)).sum()) for w in words]
        ok = vals == meta["regs"] and list(bits[8 * WIDTH:]) == meta["nzcv"]
        out["config5_program"] = {"instructions": len(prog), "recorded_gates": st["bootstrapped"],
                                  "executed_gates": st["executed"],
                                  "dataflow_levels": st["last_flush_levels"],
                                  "latency_s": wall, "device_ms": dev,
                                  "instructions_per_s": len(prog) / wall, "correct": bool(ok)}
        # the same program on the reference's own Machine through the drop-in
        # (cryptovm::GpuBackend, demand-driven): record + evaluate + decrypt
        t = time.perf_counter()
        regs, nzcv, st2, _ = refshim.run_program_gpu(ctx, ks, prog, meta["mem"])
        wall2 = time.perf_counter() - t
        out["config5_reference_machine"] = {
            "latency_s": wall2, "executed_gates": st2["executed"],
            "recorded_gates": st2["bootstrapped"],
            "correct": bool([int(r) for r in regs] == meta["regs"]
                            and list(nzcv) == meta["nzcv"])}
    ctx.set_profiling(False)
    return out


# ------------------------------------------------------------------ ours --
def pinned_copy(a):
    try:
        import torch
        p = torch.empty(a.shape, dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
        p[...] = a
        return p
    except Exception:
        return a


def run_ours(args):
    import paper_2101_03403_b200 as P
    ws, rank, local = dist_env()
    dist = None
    if ws > 1:
        import torch
        import torch.distributed as tdist
        torch.cuda.set_device(local)
        tdist.init_process_group("nccl", device_id=torch.device("cuda", local))
        dist = tdist

    def barrier():
        if dist:
            dist.barrier()

    def max_over_ranks(x):
        if not dist:
            return x
        import torch
        t = torch.tensor([x], device=f"cuda:{local}", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    ks = P.KeySet(KEY_SEED)
    ctx = P.Context(local)
    ctx.upload_keyset(ks)
    add16 = load_dag("add", WIDTH)
    assert add16.bootstrapped() == GATES_PER_ADD and add16.n_inputs == 2 * WIDTH
    av, bv = workload_operands(rank)
    lwe = operand_lwe(ks, "add", WIDTH, av, bv, 100 + 2 * rank)  # (256, 32, 631)
    pin = pinned_copy(lwe)  # pinned host buffer for the e2e leg

    # Record the 256 adders once (replay of the reference's table); replay the
    # levelised plan each step.
    bk = P.Backend(ctx)
    hin = bk.import_lwe(lwe.reshape(-1, 631)).reshape(BATCH, -1)
    outs = np.stack([bk.replay_outputs(add16, hin[i]) for i in range(BATCH)])
    plan = bk.capture_plan()
    info = plan.info()
    assert info["gates"] == BATCH * GATES_PER_ADD and info["levels"] == 9, info
    ctx.sync()

    fp64_peak = ctx.fp64_peak_tflops(3)
    ctx.set_profiling(True)
    for _ in range(args.warmup):
        plan.run(ctx)
        ctx.sync()
    # correctness of the replayed plan
    got = ks.decrypt_words(bk.export_lwe(outs.reshape(-1)).reshape(-1, 631), WIDTH + 1)
    assert np.array_equal(got, av + bv), "plan replay produced wrong sums"

    step_ms = []
    ctx.reset_stats()
    barrier()
    ctx.sync()
    with ClockSampler(local) as clocks:
        for _ in range(args.steps):
            ctx.flush_l2()  # cold L2 between steps (outside the timed events)
            ctx.event(0)
            plan.run(ctx)
            ctx.event(1)
            step_ms.append(ctx.event_elapsed_ms())
    ctx.sync()
    barrier()
    kst = ctx.kernel_stats()
    total_ms = max_over_ranks(sum(step_ms))
    gates_step = info["gates"]
    boots_step = info["bootstraps"]
    value = ws * gates_step * args.steps / (total_ms * 1e-3)

    br_ms_per_step = kst["br_ms"] / args.steps
    achieved = boots_step * ALG_FLOP_PER_BOOTSTRAP / (br_ms_per_step * 1e-3) / 1e12
    launches = kst["br_launches"] + kst["ks_launches"]

    # e2e through the public C ABI with host buffers (pinned)
    ctx.set_profiling(False)
    e2e_times = []
    for i in range(args.warmup + args.steps):
        barrier()
        t = time.perf_counter()
        res, st = P.dag_batch(ctx, add16, pin)
        dt = time.perf_counter() - t
        if i >= args.warmup:
            e2e_times.append(dt)
    vals = ks.decrypt_words(res.reshape(-1, 631), WIDTH + 1)
    assert np.array_equal(vals, av + bv), "e2e produced wrong sums"
    e2e_total = max_over_ranks(sum(e2e_times))
    # cvm_dag_batch evaluates only the exported outputs' cone (dead-gate
    # elimination: 180 of an ADD16's 195 gates feed sum + carry), so its rate
    # counts the gates it actually bootstraps; ADD16/s is the application rate.
    e2e_gates = int(st["executed"])
    e2e_value = ws * e2e_gates * args.steps / e2e_total
    e2e_add16 = ws * BATCH * args.steps / e2e_total

    # the reference's own API through the drop-in shim: Word::encrypt, alu::add
    # on cryptovm::GpuBackend, one evaluate, decrypt_word per result
    ref_api = None
    sys.path.insert(0, os.path.join(REPO, "integration"))
    import refshim
    if refshim.available():
        times = []
        for i in range(1 + min(args.steps, 10)):  # host-side work: more runs, less noise
            barrier()
            t = time.perf_counter()
            sums, carries, st_r = refshim.add_batch_gpu(ctx, ks, av, bv, WIDTH)
            if i:
                times.append(time.perf_counter() - t)
        ok = np.array_equal(sums + (carries.astype(np.uint64) << WIDTH), av + bv)
        tot = max_over_ranks(sum(times))
        ref_api = {"value": ws * st_r["executed"] * len(times) / tot,
                   "unit": "bootstrapped gates/s", "add16_ops_per_s": ws * BATCH * len(times) / tot,
                   "ms_per_step": 1e3 * tot / len(times), "correct": bool(ok),
                   "path": "reference Word::encrypt + alu::add on cryptovm::GpuBackend "
                           "(integration/), evaluate, decrypt_word per result; host "
                           "encryption / decryption inside the timed region"}

    # batch-1 latency of one ADD16 (9 levels of <= 32 gates)
    lat = None
    if rank == 0:
        b1 = P.Backend(ctx)
        o1 = b1.replay_outputs(add16, b1.import_lwe(lwe[0]))
        p1 = b1.capture_plan()
        p1.run(ctx)
        ctx.sync()
        ctx.event(0)
        p1.run(ctx)
        ctx.event(1)
        lat = ctx.event_elapsed_ms()
        s1 = ks.decrypt_words(b1.export_lwe(o1), WIDTH + 1)[0]
        assert s1 == av[0] + bv[0], "batch-1 adder produced a wrong sum"

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return 0
    extras = extra_configs(P, ctx, ks, fp64_peak) if (ws == 1 and not args.no_extras) else None
    cpu = cpu_baseline() if (ws == 1 and not args.no_cpu) else None
    # DRAM bytes per blind-rotation launch of this workload, from the committed
    # ncu capture of the same command (profiles/ncu_blind_rotate.json)
    traffic, traffic_src = None, None
    prof = os.path.join(REPO, "profiles", "ncu_blind_rotate.json")
    if os.path.exists(prof):
        try:
            pj = json.load(open(prof))
            traffic = pj[pj.get("dominant", "blind_rotate_v4")]["avg_dram_bytes_per_launch"]
            traffic_src = pj.get("source")
        except (KeyError, ValueError):
            traffic = None
    line = {
        "metric": METRIC, "value": value, "unit": "bootstrapped gates/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "u32 torus / f64 FFT", "data": "synthetic",
        "config": {"workload": "config2: 256 x ADD16 per GPU (Kogge-Stone, 195 bootstraps, "
                               "9 dataflow levels), n=630 N=1024 l=3 Bg=2^7 t=8 base 4",
                   "global_batch": BATCH * ws, "gates_per_step": gates_step * ws,
                   "parallelism": f"dp{ws} (independent adders per GPU)",
                   "circuit": add16.source,
                   "l2": "flushed (256 MB memset) before every timed step"},
        "add16_ops_per_s": value / GATES_PER_ADD,
        "add16_batch_latency_ms": total_ms / args.steps,
        "add16_latency_batch1_ms": lat,
        "e2e": {"value": e2e_value, "unit": "bootstrapped gates/s",
                "h2d_bytes_per_step": int(pin.nbytes),
                "d2h_bytes_per_step": int(BATCH * (WIDTH + 1) * 631 * 4),
                "gates_executed_per_step": e2e_gates * ws,
                "add16_ops_per_s": e2e_add16,
                "call": "cvm_dag_batch (C ABI), pinned host buffers",
                "reference_api": ref_api},
        "roofline": {"bound": "fp64", "kernel": "blind rotation (v4 waves + remainder kernels)",
                     "achieved": achieved, "peak": fp64_peak, "unit": "TFLOP/s",
                     "frac": achieved / fp64_peak, "traffic": traffic,
                     "traffic_unit": "DRAM bytes per blind_rotate launch (ncu)",
                     "traffic_source": traffic_src,
                     "algorithmic_bytes_per_launch": 61_931_520 + (2524 + 4112) * boots_step
                     / max(1.0, kst["br_launches"] / args.steps),
                     "peak_source": "DFMA peak measured live in bench.py (cvm_ctx_fp64_peak); "
                                    "MEASURED_PEAKS.json has no FP64 figure",
                     "algorithmic_flop_per_bootstrap": ALG_FLOP_PER_BOOTSTRAP},
        "kernel_share": {"blind_rotate": kst["br_ms"] / max(1e-9, kst["br_ms"] + kst["ks_ms"]),
                         "key_switch": kst["ks_ms"] / max(1e-9, kst["br_ms"] + kst["ks_ms"])},
        "gpu_launches": int(launches),
        "clocks": clocks.summary(),
        "cpu_baseline": cpu,
        "kernels": {"blind_rotate_variant": P.api.lib.cvm_get_br_variant(),
                    "key_switch_variant": P.api.lib.cvm_get_ks_variant()},
        "other_configs": extras,
    }
    print(json.dumps(line))
    if dist:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the one-shot configs 1/3/4/5 measurements")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
