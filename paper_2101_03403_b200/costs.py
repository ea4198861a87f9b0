"""Measured B200 gate costs in the reference's cost-table format.

The reference prices gates with a `CostTable` read by `CostTable::parse`
(`core/src/gates.cpp:99-134`): one `KIND = <milliseconds>` line per gate kind,
`#` comments, blank lines allowed.  `SimBackend(costs)` stamps those costs on
DAG nodes (`cryptovm.cpp:147-151`) and `repriced()` re-stamps a saved trace
(`cryptovm.cpp:71-81`) so `analyze()` (`sched.cpp:188-233`) can report the
critical path and W-worker makespans.  Its defaults are the paper's one-core
CPU latencies (`gates.cpp:36-49`, ~25.6 ms per bootstrap).

A GPU has two honest prices per gate, so two tables are produced:
  * latency    -- device time of a level holding ONE gate of that kind (the
                  latency kernels).  `analyze()`'s unbounded-worker makespan
                  with this table is the critical-path time of a program on
                  the device.
  * throughput -- device time per gate of a full-width level (the batched
                  kernels).  The 1-worker makespan (sum of node costs) with
                  this table is the time of a wide, throughput-bound job.
NOT / COPY / CONSTANT are folded into their consumers' operands and launch
nothing, so they cost 0 on the device.
"""
import numpy as np

from ._native import CvmInputError
from .api import GATE_KINDS

FREE_KINDS = ("CONSTANT", "NOT", "COPY")
BINARY_KINDS = tuple(k for k in GATE_KINDS if k not in FREE_KINDS and k != "MUX")


def _time_level(ctx, kind, width, base, reps):
    """Average device ms of one level of `width` gates of `kind` (L2 flushed
    before every repetition; CUDA events around the level only)."""
    n_in = 3 if kind == "MUX" else 2
    gates = ctx.pack_level([(kind, [(base + k * width + i, 1, 0) for k in range(n_in)],
                             base + 3 * width + i) for i in range(width)])
    ctx.submit_level(gates)  # warm-up (kernel selection, first-touch)
    ctx.sync()
    total = 0.0
    for _ in range(reps):
        ctx.flush_l2()
        ctx.event(0)
        ctx.submit_level(gates)
        ctx.event(1)
        ctx.sync()
        total += ctx.event_elapsed_ms()
    return total / reps


def measure(ctx, keyset, mode="throughput", width=None, reps=3, kinds=GATE_KINDS):
    """Return {KIND: ms} measured on `ctx` (keys already uploaded).

    mode "latency": one gate per level.  mode "throughput": `width` gates per
    level (default 8192 bootstraps = 8192 binary gates or 4096 MUX), cost =
    level time / gates."""
    if mode not in ("latency", "throughput"):
        raise ValueError("mode must be 'latency' or 'throughput'")
    full = 8192 if width is None else int(width)
    max_w = 1 if mode == "latency" else full
    base = ctx.alloc(4 * max_w)
    rng = np.random.default_rng(7)
    for k in range(3):
        ctx.upload(base + k * max_w, keyset.encrypt(rng.integers(0, 2, max_w), 100 + k))
    out = {}
    for kind in kinds:
        if kind in FREE_KINDS:
            out[kind] = 0.0
            continue
        w = 1 if mode == "latency" else (max_w // 2 if kind == "MUX" else max_w)
        out[kind] = _time_level(ctx, kind, w, base, reps) / w
    return out


def format_table(costs, header=()):
    """Render {KIND: ms} in the `CostTable::parse` grammar (gates.cpp:99-134)."""
    lines = ["# " + h for h in header]
    for kind in GATE_KINDS:
        if kind in costs:
            lines.append(f"{kind} = {costs[kind]:.9g}")
    return "\n".join(lines) + "\n"


def parse_table(text):
    """Restatement of `CostTable::parse` (gates.cpp:99-134) for tests: same
    grammar, same rejections (missing `=`, trailing junk, unknown kind,
    negative latency).  Kinds absent from the text keep the reference
    defaults, which are not needed here, so they are simply absent."""
    table = {}
    for no, line in enumerate(text.splitlines(), 1):
        line = line.split("#", 1)[0]
        f = line.split()
        if not f:
            continue
        if len(f) < 3 or f[1] != "=":
            raise CvmInputError(f"cost table line {no}: expected `KIND = <milliseconds>`")
        if len(f) > 3:
            raise CvmInputError(f"cost table line {no}: trailing junk `{f[3]}`")
        if f[0] not in GATE_KINDS:
            raise CvmInputError(f"cost table line {no}: unknown gate kind `{f[0]}`")
        ms = float(f[2])
        if ms < 0:
            raise CvmInputError(f"cost table line {no}: negative latency")
        table[f[0]] = ms
    return table
