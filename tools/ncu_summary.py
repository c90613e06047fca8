"""Summarise ncu captures into profiles/: per-kernel launch list (shares, DRAM bytes) and the
full-capture counters bench.py quotes as roofline.traffic.

  python tools/ncu_summary.py <launches.csv> <full_*.ncu-rep ...> --tag r1b
"""
from __future__ import annotations

import collections
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def launch_list(path):
    rows = list(csv.reader(open(path)))
    i = [n for n, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[i]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
    for r in rows[i + 1:]:
        k = r[ki].split("(")[0].replace("void ", "")
        v = float(r[vi].replace(",", ""))
        if r[mi] == "gpu__time_duration.sum":
            agg[k][0] += 1
            agg[k][1] += v
        elif r[mi] == "dram__bytes_read.sum":
            agg[k][2] += v
        elif r[mi] == "dram__bytes_write.sum":
            agg[k][3] += v
    return agg


METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
           "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
           "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
           "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_sectors_srcunit_tex_op_write.sum",
           "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_elapsed",
           "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
           "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
           "smsp__inst_executed.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]


def full_capture(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h, u, v = r[0], r[1], r[2]
    name = v[h.index("Kernel Name")].split("(")[0].replace("void ", "")
    d = {"kernel": name}
    for m in METRICS:
        if m in h:
            j = h.index(m)
            d[m] = {"value": v[j], "unit": u[j]}
    return d


def to_bytes(e):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[e["unit"]]
    return float(e["value"].replace(",", "")) * scale


def main():
    args = sys.argv[1:]
    tag = args[args.index("--tag") + 1]
    args = [a for a in args if a not in ("--tag", tag)]
    md = [f"# {tag} ncu summary\n"]
    js = {"tag": tag, "kernels": {}}
    for a in args:
        if a.endswith(".csv"):
            agg = launch_list(a)
            tot = sum(v[1] for v in agg.values())
            md.append("Launch list (`--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                      "--clock-control none`, one bench step). Cold-cache, serialised: compare shares.\n")
            md.append("| kernel | launches | time (ms) | share | DRAM read (GB) | DRAM write (GB) |")
            md.append("|---|---|---|---|---|---|")
            for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
                md.append(f"| `{k}` | {v[0]} | {v[1] / 1e6:.3f} | {100 * v[1] / tot:.1f}% | {v[2] / 1e9:.3f} | "
                          f"{v[3] / 1e9:.3f} |")
            md.append(f"| total | {sum(v[0] for v in agg.values())} | {tot / 1e6:.3f} | 100% | | |\n")
            js["launch_list"] = {k: {"launches": v[0], "ns": v[1], "dram_read": v[2], "dram_write": v[3]}
                                 for k, v in agg.items()}
        else:
            d = full_capture(a)
            name = d.pop("kernel")
            if "dram__bytes_read.sum" in d:
                d["traffic_bytes"] = to_bytes(d["dram__bytes_read.sum"]) + to_bytes(d["dram__bytes_write.sum"])
            js["kernels"][name] = d
            md.append(f"## `{name}` (ncu --set full, {os.path.basename(a)})\n")
            md.append("| metric | value |")
            md.append("|---|---|")
            for m, e in d.items():
                if isinstance(e, dict):
                    md.append(f"| {m} | {e['value']} {e['unit']} |")
                else:
                    md.append(f"| {m} | {e:.0f} |")
            md.append("")
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    open(os.path.join(ROOT, "profiles", f"{tag}_ncu.md"), "w").write("\n".join(md) + "\n")
    json.dump(js, open(os.path.join(ROOT, "profiles", f"{tag}_ncu.json"), "w"), indent=1)
    print("\n".join(md))


if __name__ == "__main__":
    main()
