"""Summarise an ncu --metrics CSV of the bench command into
profiles/ncu_blind_rotate.json (per-launch DRAM traffic of the blind-rotation
and key-switch kernels; bench.py reads the average of the dominant kernel as
roofline.traffic) and, given a third path, the launch list (per-kernel launch
count, time and share of the device time).

    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
        --clock-control none --csv --log-file gpurun_out/traffic.csv \
        python bench.py --steps 1 --warmup 1 --no-cpu --no-extras
    python tools/ncu_traffic.py gpurun_out/traffic.csv profiles/ncu_blind_rotate.json \
        profiles/r01_ncu_launches_summary.txt
"""
import collections
import csv
import json
import sys


def main():
    src, dst = sys.argv[1], sys.argv[2]
    rows = list(csv.reader(open(src)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ik, ig, im, iv = (h.index(x) for x in ("Kernel Name", "Grid Size", "Metric Name",
                                            "Metric Value"))
    iid = h.index("ID")
    launches = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= iv:
            continue
        key = r[iid]
        d = launches.setdefault(key, {"kernel": r[ik], "grid": r[ig]})
        d[r[im]] = float(r[iv].replace(",", ""))
    out = {"source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,"
                     "gpu__time_duration.sum --clock-control none, python bench.py --steps 1 "
                     "--warmup 1 --no-cpu --no-extras (tools/ncu_traffic.py); per launch"}
    groups = {"blind_rotate_v4": "blind_rotate_kernel_v4", "blind_rotate_v3": "blind_rotate_kernel_v3", "blind_rotate_wide": "wide_kernel",
              "blind_rotate_pair": "pair_kernel", "key_switch_mma": "key_switch_mma",
              "key_switch_tc": "key_switch_tc", "key_switch_wide": "key_switch_wide"}
    for name, pat in groups.items():
        ls = [d for d in launches.values() if pat in d["kernel"]]
        if not ls:
            continue
        per = [{"grid": d["grid"],
                "dram_bytes": d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0),
                "ncu_ms": d.get("gpu__time_duration.sum", 0) / 1e6} for d in ls]
        out[name] = {"kernel": ls[0]["kernel"], "launches": len(per),
                     "avg_dram_bytes_per_launch": sum(p["dram_bytes"] for p in per) / len(per),
                     "per_launch": per}
    # the dominant blind-rotation kernel (most device time)
    br = [k for k in out if k.startswith("blind_rotate") and isinstance(out[k], dict)]
    if br:
        out["dominant"] = max(br, key=lambda k: sum(p["ncu_ms"] for p in out[k]["per_launch"]))
    json.dump(out, open(dst, "w"), indent=1)
    if len(sys.argv) > 3:
        per_kernel = collections.OrderedDict()
        for d in launches.values():
            k = per_kernel.setdefault(d["kernel"], [0, 0.0])
            k[0] += 1
            k[1] += d.get("gpu__time_duration.sum", 0) / 1e6
        total = sum(v[1] for v in per_kernel.values()) or 1.0
        with open(sys.argv[3], "w") as f:
            f.write("ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                    "--clock-control none (per-launch, cold-cache, serialised: compare shares, not "
                    "absolutes); command: python bench.py --steps 1 --warmup 1 --no-cpu --no-extras\n")
            for name, (n, ms) in sorted(per_kernel.items(), key=lambda kv: -kv[1][1]):
                f.write(f"{name}: launches={n} total_ms={ms:.2f} avg_ms={ms / n:.3f} "
                        f"share={100 * ms / total:.1f}%\n")
    for k, v in out.items():
        if isinstance(v, dict):
            print(k, v["launches"], v["avg_dram_bytes_per_launch"], v["kernel"][:60])


if __name__ == "__main__":
    main()
