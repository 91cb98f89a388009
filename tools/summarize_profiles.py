"""Turns gpurun_out/ ncu artifacts into the committed profiles/ summaries.

    python tools/summarize_profiles.py r01

Reads gpurun_out/launches.csv (ncu --metrics gpu__time_duration.sum,
dram__bytes_read.sum,dram__bytes_write.sum launch list of
`bench.py --steps 2 --warmup 1`) and gpurun_out/prof_<kernel>.ncu-rep (one
--set full capture per hot kernel), writes profiles/<tag>_launches.csv,
profiles/<tag>_summary.md and profiles/k1_traffic.json (read by bench.py for
roofline.traffic).
"""
from __future__ import annotations

import csv
import json
import os
import re
import shutil
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")
FRAMES = 300
FRAME_BYTES = 3840 * 2160 * 3


def launches():
    rows = list(csv.reader(open(os.path.join(OUT, "launches.csv"))))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, mi, vi, ii = (h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"),
                      h.index("ID"))
    d = defaultdict(dict)
    for r in rows[hdr + 1:]:
        name = r[ki].split("(")[0].replace("void ", "")
        d[(int(r[ii]), name)][r[mi]] = float(r[vi].replace(",", ""))
    return d


def details(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[0]
    mi, vi, ui = h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    return {r[mi]: f"{r[vi]} {r[ui]}".strip() for r in rows[1:]}


def stalls(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, v = rows[0], rows[2]
    res = []
    for i, name in enumerate(h):
        m = re.match(r"smsp__average_warps_issue_stalled_(.*)_per_issue_active\.ratio", name)
        if m:
            try:
                res.append((float(v[i].replace(",", "")), m.group(1)))
            except ValueError:
                pass
    return sorted(res, reverse=True)[:5]


def main(tag):
    os.makedirs(PROF, exist_ok=True)
    shutil.copy(os.path.join(OUT, "launches.csv"), os.path.join(PROF, f"{tag}_launches.csv"))
    d = launches()
    # steady-state launches: skip the synthesis kernels and the first (warm-up) step
    per = defaultdict(list)
    for (i, name), m in sorted(d.items()):
        per[name].append(m)
    lines = [f"# ncu summary {tag}", "",
             "Source: `bash tools/profile.sh` under gpurun (ncu --clock-control none; launch list of "
             "`bench.py --steps 2 --warmup 1`, 300 4K frames per launch). ncu times are serialized "
             "cold-cache replays: compare shares, not absolutes.", "",
             "| kernel | launches | mean ms | DRAM read GB | DRAM write GB | DRAM GB/s |",
             "|---|---|---|---|---|---|"]
    k1 = None
    for name, ms in per.items():
        if name.startswith("synth"):
            continue
        t = sum(m["gpu__time_duration.sum"] for m in ms) / len(ms) / 1e6
        rd = sum(m["dram__bytes_read.sum"] for m in ms) / len(ms)
        wr = sum(m["dram__bytes_write.sum"] for m in ms) / len(ms)
        lines.append(f"| {name} | {len(ms)} | {t:.4f} | {rd/1e9:.3f} | {wr/1e9:.3f} | "
                     f"{(rd+wr)/t/1e6:.0f} |")
        if name.startswith("mask_fg_kernel"):
            k1 = dict(ms=t, read=rd, write=wr)
    total = sum(sum(m["gpu__time_duration.sum"] for m in ms) / len(ms)
                for n, ms in per.items() if not n.startswith("synth"))
    lines += ["", f"Step total (sum of mean kernel times): {total/1e6:.4f} ms", ""]
    for kern in ("mask_fg", "plan_kernel", "gather_kernel"):
        rep = os.path.join(OUT, f"prof_{kern}.ncu-rep")
        if not os.path.exists(rep):
            continue
        det = details(rep)
        lines.append(f"## {kern} (ncu --set full)")
        for key in ("Duration", "DRAM Throughput", "Memory Throughput", "L2 Hit Rate",
                    "Compute (SM) Throughput", "Issue Slots Busy", "Achieved Occupancy",
                    "Registers Per Thread", "Dynamic Shared Memory Per Block"):
            if key in det:
                lines.append(f"- {key}: {det[key]}")
        lines.append("- top stall reasons (warps per issue): " +
                     ", ".join(f"{n} {v:.2f}" for v, n in stalls(rep)))
        lines.append("")
    with open(os.path.join(PROF, f"{tag}_summary.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    if k1:
        traffic = k1["read"] + k1["write"]
        raw = 2160 * 120 * 4
        cells = 135 * (240 + 8) * 4
        json.dump({"kernel": "mask_fg_kernel (K1, K1b fused)", "frames_per_launch": FRAMES,
                   "dram_bytes_per_launch": traffic, "dram_bytes_per_frame": traffic / FRAMES,
                   "algorithmic_bytes_per_launch":
                       (FRAMES + 1) * FRAME_BYTES + FRAMES * (2 * raw + cells),
                   "source": f"profiles/{tag}_launches.csv"},
                  open(os.path.join(PROF, "k1_traffic.json"), "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r01")
