"""Summarise a `ncu --set full` report (.ncu-rep) into a small JSON per kernel
launch: duration, launch shape, pipe utilisation, issue, stalls and DRAM
traffic (bytes and GB/s against the HBM peak in MEASURED_PEAKS.json).

    python tools/ncu_summary.py gpurun_out/x.ncu-rep profiles/r02_ncu_x.json ["note"]
"""
import csv
import io
import json
import os
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum", "launch__grid_size", "launch__block_size",
    "launch__registers_per_thread", "launch__cluster_dim_x",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_subpipe_imma_cycles_active_realtime.avg",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_tmem.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct", "smsp__inst_executed.sum", "sm__cycles_active.avg",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_membar_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_sleeping_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_selected_per_issue_active.ratio",
]


def _num(s):
    try:
        return float(s.replace(",", ""))
    except ValueError:
        return s


def summarise(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units, data = rows[0], rows[1], rows[2:]
    peaks = {}
    mp = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                      "MEASURED_PEAKS.json")
    if os.path.exists(mp):
        peaks = json.load(open(mp))
    hbm = None
    for k, v in peaks.items():
        if "hbm" in k.lower() and isinstance(v, (int, float)):
            hbm = float(v)
    res = []
    for r in data:
        d = {"kernel": r[head.index("Kernel Name")][:120], "id": r[head.index("ID")]}
        for m in METRICS:
            if m in head:
                i = head.index(m)
                d[m] = _num(r[i])
                if units[i]:
                    d[m + " [unit]"] = units[i]
        t = d.get("gpu__time_duration.sum")
        rd, wr = d.get("dram__bytes_read.sum"), d.get("dram__bytes_write.sum")
        if isinstance(t, float) and isinstance(rd, float) and isinstance(wr, float):
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
            su = scale.get(d.get("dram__bytes_read.sum [unit]", "byte"), 1)
            wu = scale.get(d.get("dram__bytes_write.sum [unit]", "byte"), 1)
            tu = {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "ns": 1e-9, "us": 1e-6,
                  "ms": 1e-3}.get(
                d.get("gpu__time_duration.sum [unit]", "nsecond"), 1e-9)
            d["dram_bytes_total"] = rd * su + wr * wu
            d["dram_GBps"] = d["dram_bytes_total"] / (t * tu) / 1e9
            if hbm:
                d["dram_frac_of_hbm_peak"] = d["dram_GBps"] / hbm
                d["hbm_peak_GBps"] = hbm
        res.append(d)
    return res


def main():
    rep, dst = sys.argv[1], sys.argv[2]
    note = sys.argv[3] if len(sys.argv) > 3 else ""
    res = summarise(rep)
    json.dump({"source": os.path.basename(rep), "note": note, "launches": res},
              open(dst, "w"), indent=1)
    for d in res:
        print(d["kernel"][:60], d.get("gpu__time_duration.sum"), d.get("dram_GBps"))


if __name__ == "__main__":
    main()
