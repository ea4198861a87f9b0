#!/usr/bin/env python3
"""Benchmark: batched TFHE gate bootstrapping under CryptoEmu's functional units.

Workload (BASELINE.json configs[1], the config the headline metric is quoted
on): 256 independent 16-bit homomorphic ADDs (Kogge-Stone, 195 bootstrapped
gates each, 9 dataflow levels -> 49,920 bootstraps per step), n=630, N=1024,
l=3, Bg=2^7, t=8, base 4, torus32, seeded synthetic operands (no dataset is
involved; inputs are uniform random 16-bit integers encrypted under seeded keys).

  value   bootstrapped gates/s with inputs resident in HBM: one step = the
          recorded 9-level plan replayed on the device (18 launches).
  e2e     the same metric through the public C-ABI call cvm_fu_batch with host
          buffers: pinned H2D of the 512 operand words (20.7 MB), circuit
          recording, levelised execution, D2H of the 256 x 17 result bits.
          cvm_fu_batch evaluates only the outputs' cone (180 of 195 gates per
          ADD16), so e2e counts the gates it executes; ADD16/s is reported
          beside it.
  roofline  blind_rotate_kernel (dominant): algorithmic FP64 flops per
          bootstrap (147,087,360) x bootstraps /
          summed kernel event time, against the FP64 DFMA peak measured live.

Multi-GPU (--gpus N under torchrun): weak scaling, each rank runs its own 256
independent adders (no data-path collective; gates of a level are
independent), barrier + max-over-ranks device time.

--impl reference: the reference's path on the host CPU.  The reference ships
no TFHE code, so this arm times the CPU restatement of
the TFHE library's gate bootstrapping (oracle/, double-precision FFT: the
library's own method) on all host threads, on a bounded sample of the same
workload (the first dataflow level's AND/XOR gates).
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


# ------------------------------------------------------------ CPU baseline --
def cpu_sample_inputs(sk, n_gates, seed=7):
    """First dataflow level of the ADD16 batch: per bit an AND and an XOR of
    the two operand bits (alu.cpp:106-108), as fresh ciphertexts under the
    oracle's keys (same seed, same key bytes as the product keygen)."""
    import oracle as O
    rng = np.random.default_rng(seed)
    bits_a = rng.integers(0, 2, n_gates).astype(np.uint8)
    bits_b = rng.integers(0, 2, n_gates).astype(np.uint8)
    a, b = sk.encrypt(bits_a, 1), sk.encrypt(bits_b, 2)
    kinds = np.where(np.arange(n_gates) % 2 == 0, O.AND, O.XOR).astype(np.uint8)
    return kinds, a, b


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_baseline(target_s=12.0, threads=None):
    """Oracle (double-FFT TFHE, the library's method) on all host threads."""
    sys.path.insert(0, os.path.join(REPO, "oracle"))
    import oracle as O
    threads = threads or os.cpu_count() or 1
    sk = O.SecretKeys(KEY_SEED)
    ck = O.CloudKeys(sk.bk, sk.ksk, O.MODE_FFT)
    kinds, a, b = cpu_sample_inputs(sk, threads)
    t = time.perf_counter()
    ck.gates(kinds, a, b, threads=threads)  # calibration, one gate per thread
    per_round = time.perf_counter() - t
    rounds = max(1, int(target_s / max(per_round, 1e-3)))
    n = threads * rounds
    kinds, a, b = cpu_sample_inputs(sk, n)
    t = time.perf_counter()
    out = ck.gates(kinds, a, b, threads=threads)
    dt = time.perf_counter() - t
    dec = sk.decrypt(out)
    return {"value": n / dt, "unit": "bootstrapped gates/s", "cores": threads,
            "kind": "port", "seconds": dt, "cpu_model": cpu_model(),
            "nproc": os.cpu_count(),
            "sample": f"{n} AND/XOR gates of the ADD16 batch's first dataflow level, "
                      f"oracle/ double-FFT TFHE (the TFHE library's method), {threads} threads",
            "decrypt_sanity": int(dec.size)}


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    sys.path.insert(0, os.path.join(REPO, "oracle"))
    import oracle as O
    threads = os.cpu_count() or 1
    sk = O.SecretKeys(KEY_SEED)
    ck = O.CloudKeys(sk.bk, sk.ksk, O.MODE_FFT)
    # 32 gates per thread per step, evaluated in lockstep (the oracle's batched
    # mode): enough bootstraps that thread start-up and the per-CMux-step
    # barrier do not depress the CPU rate, short enough for a few-minute run
    n = threads * int(os.environ.get("REF_ROUNDS", "32"))
    kinds, a, b = cpu_sample_inputs(sk, n)
    for _ in range(args.warmup):
        ck.gates(kinds[:threads], a[:threads], b[:threads], threads=threads)
    times = []
    for _ in range(args.steps):
        t = time.perf_counter()
        ck.gates(kinds, a, b, threads=threads)
        times.append(time.perf_counter() - t)
    total = sum(times)
    value = n * args.steps / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "bootstrapped gates/s",
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u32 torus / f64 FFT", "data": "synthetic",
        "config": {"workload": "config2: 256 x ADD16 (n=630,N=1024,l=3,Bg=2^7,t=8,base 4)",
                   "sample_per_step": f"{n} gates of the first dataflow level",
                   "parallelism": f"cpu threads={threads}"},
        "cpu_baseline": {"value": value, "unit": "bootstrapped gates/s", "cores": threads,
                         "kind": "port", "cpu_model": cpu_model(), "nproc": os.cpu_count(),
                         "sample": f"{n} AND/XOR gates per step, double-FFT TFHE (oracle/)"},
        "e2e": {"value": value, "unit": "bootstrapped gates/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "note": "reference repo has no TFHE implementation (cleartext SimBackend only); "
                "this arm is the CPU restatement of the TFHE library's bootstrapping",
    }
    print(json.dumps(line))
    return 0


# ------------------------------------------------------- other configs ---
def extra_configs(P, ctx, ks):
    """Configs 1, 3, 4 and 5 (BASELINE.json configs[0,2,3,4]) run once each
    through the public batched API (host buffers in and out), with the device
    time of their kernels; reported beside the headline config-2 line."""
    import json as _json
    rng = np.random.default_rng(77)
    out = {}
    # cvm_fu_batch returns its scratch slots, so the slab only holds the
    # largest single call; size it once for config 4 (216k gates + inputs)
    # instead of growing it by doubling inside a timed call.
    ctx.reserve(ctx.alloc(0) + 300_000)

    def fu(op, batch, seed):
        av = rng.integers(0, 1 << WIDTH, batch)
        bv = rng.integers(0, 1 << WIDTH, batch)
        a = ks.encrypt_words(av, WIDTH, seed)
        b = ks.encrypt_words(bv, WIDTH, seed + 1)
        ctx.reset_stats()
        t = time.perf_counter()
        res, st = P.fu_batch(ctx, op, WIDTH, a, b)
        wall = time.perf_counter() - t
        k = ctx.kernel_stats()
        dev_ms = k["br_ms"] + k["ks_ms"]
        return av, bv, res, {"batch": batch, "recorded_gates": st["bootstrapped"],
                             "executed_gates": st["executed"],
                             "levels": st["last_flush_levels"], "wall_s": wall,
                             "device_ms": dev_ms,
                             "ops_per_s_e2e": batch / wall,
                             "ops_per_s_device": batch / (dev_ms * 1e-3),
                             "gates_per_s_device": st["executed"] / (dev_ms * 1e-3)}

    ctx.set_profiling(True)
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
    out["config1_nand4096"] = {"gates_per_s_device": n / ((k["br_ms"] + k["ks_ms"]) * 1e-3),
                               "device_ms": k["br_ms"] + k["ks_ms"], "correct": bool(ok)}
    # config 3: SUBS/CMP (sub + NZCV) and LSL by an encrypted amount, 256 each
    def latency1(op, seed):
        """Device time of one unit alone (batch 1: the latency kernels)."""
        return fu(op, 1, seed)[3]["device_ms"]

    av, bv, res, d = fu("cmp", 256, 910)
    vals = ks.decrypt_words(res[:, :WIDTH].reshape(-1, 631), WIDTH)
    d["correct"] = bool(np.array_equal(vals, (av - bv) % (1 << WIDTH)))
    d["latency_batch1_ms"] = latency1("cmp", 915)
    out["config3_cmp16"] = d
    av, bv, res, d = fu("lsl", 256, 920)
    vals = ks.decrypt_words(res.reshape(-1, 631), WIDTH)
    d["correct"] = bool(np.array_equal(vals, (av << (bv % WIDTH)) % (1 << WIDTH)))
    d["bootstraps_per_s_device"] = 2 * d["gates_per_s_device"]  # MUX = 2 bootstraps
    d["latency_batch1_ms"] = latency1("lsl", 925)
    out["config3_lsl16"] = d
    # config 4: 64 x MUL16 producing the low 16 bits (the emulator's MUL):
    # the high half's 2,083 gates per multiplier are dead and never run
    av, bv, res, d = fu("mul_lo", 64, 930)
    vals = ks.decrypt_words(res.reshape(-1, 631), WIDTH)
    d["correct"] = bool(np.array_equal(vals, (av * bv) % (1 << WIDTH)))
    d["latency_batch1_ms"] = latency1("mul_lo", 935)
    out["config4_mul16"] = d
    av, bv, res, d = fu("umul", 64, 931)
    vals = ks.decrypt_words(res.reshape(-1, 631), 2 * WIDTH)
    d["correct"] = bool(np.array_equal(vals, av * bv))
    out["config4_mul16_full_product"] = d
    # config 5: a seeded 64-instruction program + UDIV on 8 encrypted registers
    meta = _json.load(open(os.path.join(REPO, "tests", "golden", "programs.json")))[0]
    bk = P.Backend(ctx, ks)
    mem = [bk.import_lwe(w) for w in ks.encrypt_words(meta["mem"], WIDTH, 940)]
    regs, nzcv = bk.machine_run([tuple(i) for i in meta["insns"]], mem)
    ctx.reset_stats()
    t = time.perf_counter()
    # the key owner reads the final register file and flags: one flush that
    # evaluates the live cone only
    bits = bk.decrypt_bits(np.concatenate([regs.ravel(), nzcv]))
    wall = time.perf_counter() - t
    k = ctx.kernel_stats()
    st = bk.stats()
    words = bits[:8 * WIDTH].reshape(8, WIDTH).astype(np.int64)
    vals = [int((w << np.arange(WIDTH)).sum()) for w in words]
    ok = vals == meta["regs"] and list(bits[8 * WIDTH:]) == meta["nzcv"]
    out["config5_program"] = {"instructions": len(meta["insns"]),
                              "recorded_gates": st["bootstrapped"],
                              "executed_gates": st["executed"],
                              "dataflow_levels": st["last_flush_levels"],
                              "latency_s": wall, "device_ms": k["br_ms"] + k["ks_ms"],
                              "instructions_per_s": len(meta["insns"]) / wall,
                              "correct": bool(ok)}
    ctx.set_profiling(False)
    return out


# ------------------------------------------------------------------ ours --
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

    ks = P.KeySet(KEY_SEED)
    ctx = P.Context(local)
    ctx.upload_keyset(ks)
    av, bv = workload_operands(rank)
    a_lwe = ks.encrypt_words(av, WIDTH, 100 + rank)
    b_lwe = ks.encrypt_words(bv, WIDTH, 200 + rank)
    # pinned host copies for the e2e leg
    try:
        import torch
        pa = torch.empty(a_lwe.shape, dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
        pb = torch.empty(b_lwe.shape, dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
        pa[...] = a_lwe
        pb[...] = b_lwe
    except Exception:
        pa, pb = a_lwe, b_lwe

    # Record the 256 adders once; replay the levelised plan each step.
    bk = P.Backend(ctx)
    ha = bk.import_lwe(a_lwe.reshape(-1, 631)).reshape(BATCH, WIDTH)
    hb = bk.import_lwe(b_lwe.reshape(-1, 631)).reshape(BATCH, WIDTH)
    outs = np.stack([bk.fu("add", ha[i], hb[i]) for i in range(BATCH)])
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
    total_ms = sum(step_ms)
    if dist:
        import torch
        t = torch.tensor([total_ms], device=f"cuda:{local}", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
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
        out, st = P.fu_batch(ctx, "add", WIDTH, pa, pb)
        dt = time.perf_counter() - t
        if i >= args.warmup:
            e2e_times.append(dt)
    vals = ks.decrypt_words(out.reshape(-1, 631), WIDTH + 1)
    assert np.array_equal(vals, av + bv), "e2e produced wrong sums"
    e2e_total = sum(e2e_times)
    if dist:
        import torch
        t = torch.tensor([e2e_total], device=f"cuda:{local}", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_total = float(t.item())
    # cvm_fu_batch evaluates only the exported outputs' cone (dead-gate
    # elimination: 180 of an ADD16's 195 gates feed sum + carry), so its rate
    # counts the gates it actually bootstraps; ADD16/s is the application rate.
    e2e_gates = int(st["executed"])
    e2e_value = ws * e2e_gates * args.steps / e2e_total
    e2e_add16 = ws * BATCH * args.steps / e2e_total

    # batch-1 latency of one ADD16 (9 levels of <= 32 gates)
    lat = None
    if rank == 0:
        b1 = P.Backend(ctx)
        o1 = b1.fu("add", b1.import_lwe(a_lwe[0]), b1.import_lwe(b_lwe[0]))
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
        return 0
    extras = extra_configs(P, ctx, ks) if (ws == 1 and not args.no_extras) else None
    cpu = cpu_baseline() if (ws == 1 and not args.no_cpu) else None
    # DRAM bytes per blind-rotation launch of this workload, from the committed
    # ncu capture of the same command (profiles/ncu_blind_rotate.json)
    traffic = None
    prof = os.path.join(REPO, "profiles", "ncu_blind_rotate.json")
    if os.path.exists(prof):
        try:
            pj = json.load(open(prof))
            traffic = pj[pj.get("dominant", "blind_rotate_v3")]["avg_dram_bytes_per_launch"]
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
                   "l2": "flushed (256 MB memset) before every timed step"},
        "add16_ops_per_s": value / GATES_PER_ADD,
        "add16_batch_latency_ms": total_ms / args.steps,
        "add16_latency_batch1_ms": lat,
        "e2e": {"value": e2e_value, "unit": "bootstrapped gates/s",
                "h2d_bytes_per_step": int(pa.nbytes + pb.nbytes),
                "d2h_bytes_per_step": int(BATCH * (WIDTH + 1) * 631 * 4),
                "gates_executed_per_step": e2e_gates * ws,
                "add16_ops_per_s": e2e_add16},
        "roofline": {"bound": "fp64", "kernel": "blind_rotate_kernel_v4 (+ v3/wide remainders)",
                     "achieved": achieved, "peak": fp64_peak, "unit": "TFLOP/s",
                     "frac": achieved / fp64_peak, "traffic": traffic,
                     "traffic_unit": "DRAM bytes per blind_rotate launch (ncu)",
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
