"""Summarise ncu captures into profiles/<round>/ (run here, no GPU needed).

    python scripts/summarize_ncu.py --launches gpurun_out/launches_bench.csv \
        --report gpurun_out/prof_round_v3.ncu-rep --out profiles/r01

Writes launches.md (every kernel's share of the captured device time),
kernels.md (the --set full metrics per captured launch) and traffic.json
(DRAM bytes per launch of the rounding kernel, by launch index), which
bench.py reads for roofline.traffic.
"""
import argparse
import csv
import io
import json
import os
import subprocess
from collections import defaultdict


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        scale = {"ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(r[ui], 1e-3)
        name = r[ki].split("(")[0]
        tot[name] += v * scale
        cnt[name] += 1
    grand = sum(tot.values())
    out = ["| kernel | launches | device time (us) | share |", "|---|---|---|---|"]
    for k in sorted(tot, key=lambda x: -tot[x]):
        out.append(f"| `{k}` | {cnt[k]} | {tot[k]:.1f} | {100 * tot[k] / grand:.1f}% |")
    return "\n".join(out), tot, cnt


def ncu_csv(report, page, extra=()):
    res = subprocess.run(["ncu", "-i", report, "--page", page, "--csv", *extra],
                         capture_output=True, text=True, check=True)
    return list(csv.reader(io.StringIO(res.stdout)))


def kernels(report):
    rows = ncu_csv(report, "details")
    h = rows[0]
    ii, mn, mv, mu = (h.index(x) for x in ("ID", "Metric Name", "Metric Value", "Metric Unit"))
    kn = h.index("Kernel Name")
    want = ["Duration", "DRAM Throughput", "Compute (SM) Throughput", "Registers Per Thread",
            "Dynamic Shared Memory Per Block", "Theoretical Occupancy", "Achieved Occupancy",
            "Issue Slots Busy", "Executed Ipc Active", "Grid Size", "Executed Instructions"]
    d = defaultdict(dict)
    names = {}
    for r in rows[1:]:
        if r[mn] in want:
            d[r[ii]][r[mn]] = f"{r[mv]} {r[mu]}".strip()
            names[r[ii]] = r[kn].split("(")[0]
    raw = ncu_csv(report, "raw")
    rh = raw[0]
    extra = ["dram__bytes_read.sum", "dram__bytes_write.sum",
             "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
             "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"]
    units = raw[1]
    traffic = {}
    for li, r in enumerate(raw[2:]):
        rid = str(li)
        for e in extra:
            if e in rh:
                d[rid][e] = f"{r[rh.index(e)]} {units[rh.index(e)]}".strip()
        try:
            rb = float(r[rh.index("dram__bytes_read.sum")].replace(",", ""))
            wb = float(r[rh.index("dram__bytes_write.sum")].replace(",", ""))
            ub = units[rh.index("dram__bytes_read.sum")]
            mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(ub, 1)
            traffic[rid] = (rb + wb) * mult
        except (ValueError, KeyError, IndexError):
            pass
    cols = want + extra
    out = ["| id | kernel | " + " | ".join(cols) + " |", "|" + "---|" * (len(cols) + 2)]
    for k in sorted(d, key=int):
        out.append(f"| {k} | `{names.get(k, '?')}` | " + " | ".join(d[k].get(c, "") for c in cols) + " |")
    return "\n".join(out), traffic


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--report")
    ap.add_argument("--out", required=True)
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    os.makedirs(a.out, exist_ok=True)
    if a.launches:
        md, _, _ = launches(a.launches)
        open(os.path.join(a.out, "launches.md"), "w").write(
            "# Launch list (ncu --metrics gpu__time_duration.sum --clock-control none)\n\n"
            f"{a.note}\n\nSource: `{os.path.basename(a.launches)}`. Per-launch times are "
            "cold-cache and serialised; compare shares, not absolutes.\n\n" + md + "\n")
    if a.report:
        md, traffic = kernels(a.report)
        open(os.path.join(a.out, "kernels.md"), "w").write(
            "# ncu --set full, captured launches\n\n"
            f"{a.note}\n\nSource: `{os.path.basename(a.report)}`.\n\n" + md + "\n")
        json.dump({"per_launch_dram_bytes": traffic}, open(os.path.join(a.out, "traffic_raw.json"), "w"),
                  indent=1)


if __name__ == "__main__":
    main()
