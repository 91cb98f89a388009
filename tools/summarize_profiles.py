"""Turns gpurun_out/ ncu artifacts into the committed profiles/ summaries.

    python tools/summarize_profiles.py <tag> <frame reads per step> <traffic json> [title]

Reads gpurun_out/<tag>_launches.csv (ncu --metrics gpu__time_duration.sum,
dram__bytes_read.sum,dram__bytes_write.sum launch list of a short bench run,
tools/gpu/r02_profile.sh) and gpurun_out/<tag>_prof_<kernel>.ncu-rep (one
--set full capture per hot kernel); writes profiles/<tag>_launches.csv,
profiles/<tag>_summary.md and the traffic record bench.py reads for
roofline.traffic (DRAM bytes of one mask_fg launch per frame read) and
path.dram (every kernel's DRAM bytes per step).
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
FRAME_BYTES = 3840 * 2160 * 3
KERNELS = ("mask_fg", "dilate_cells", "plan_kernel", "gather_kernel")


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, mi, vi, ii = (h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"),
                      h.index("ID"))
    d = defaultdict(dict)
    for r in rows[hdr + 1:]:
        name = r[ki].split("(")[0].replace("void ", "")
        d[(int(r[ii]), name)][r[mi]] = float(r[vi].replace(",", ""))
    return d


def page(rep, name):
    """One report page as CSV text: from the .ncu-rep, or from the
    <rep>.<page>.csv the box exported (reports too large to copy back)."""
    if os.path.exists(rep):
        return subprocess.run(["ncu", "-i", rep, "--page", name, "--csv"], capture_output=True,
                              text=True).stdout
    return open(f"{rep[:-len('.ncu-rep')]}.{name}.csv").read()


def details(rep):
    out = page(rep, "details")
    rows = list(csv.reader(out.splitlines()))
    h = rows[0]
    mi, vi, ui = h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    return {r[mi]: f"{r[vi]} {r[ui]}".strip() for r in rows[1:]}


def raw(rep):
    out = page(rep, "raw")
    rows = list(csv.reader(out.splitlines()))
    return dict(zip(rows[0], rows[2]))


def stalls(r):
    res = []
    for name, v in r.items():
        m = re.match(r"smsp__average_warps_issue_stalled_(.*)_per_issue_active\.ratio", name)
        if m:
            try:
                res.append((float(v.replace(",", "")), m.group(1)))
            except ValueError:
                pass
    return sorted(res, reverse=True)[:5]


def main(tag, reads, traffic_json, title):
    os.makedirs(PROF, exist_ok=True)
    src = os.path.join(OUT, f"{tag}_launches.csv")
    shutil.copy(src, os.path.join(PROF, f"{tag}_launches.csv"))
    per = defaultdict(list)
    for (_, name), m in sorted(launches(src).items()):
        per[name].append(m)
    lines = [f"# ncu summary {tag}", "", title, "",
             "Launch list: `tools/gpu/r02_profile.sh` under gpurun (`ncu --metrics "
             "gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control "
             "none`). ncu times are serialized cold-cache replays: compare shares, not absolutes.",
             "", "| kernel | launches | mean ms | DRAM read GB | DRAM write GB | DRAM GB/s |",
             "|---|---|---|---|---|---|"]
    k1 = None
    total = 0.0
    step_bytes = 0.0  # every kernel's mean DRAM bytes per launch (one launch per step each)
    for name, ms in per.items():
        if name.startswith("synth"):
            continue
        t = sum(m["gpu__time_duration.sum"] for m in ms) / len(ms) / 1e6
        rd = sum(m["dram__bytes_read.sum"] for m in ms) / len(ms)
        wr = sum(m["dram__bytes_write.sum"] for m in ms) / len(ms)
        total += t
        step_bytes += rd + wr
        lines.append(f"| {name} | {len(ms)} | {t:.4f} | {rd/1e9:.3f} | {wr/1e9:.3f} | "
                     f"{(rd+wr)/t/1e6:.0f} |")
        if name.startswith("mask_fg_kernel"):
            k1 = dict(ms=t, read=rd, write=wr)
    lines += ["", f"Sum of mean kernel times per step: {total:.4f} ms", ""]
    if k1:
        alg = reads * FRAME_BYTES
        lines += [f"K1 (mask_fg_kernel): {alg/1e9:.2f} GB of frames per launch ({reads} frame "
                  f"reads); DRAM traffic {(k1['read']+k1['write'])/1e9:.2f} GB = "
                  f"{(k1['read']+k1['write'])/alg:.3f}x the algorithmic bytes.", ""]
    for kern in KERNELS:
        rep = os.path.join(OUT, f"{tag}_prof_{kern}.ncu-rep")
        if not (os.path.exists(rep) or os.path.exists(rep[:-len(".ncu-rep")] + ".raw.csv")):
            continue
        det, r = details(rep), raw(rep)
        lines.append(f"## {kern} (ncu --set full)")
        for key in ("Duration", "DRAM Throughput", "Memory Throughput", "L2 Hit Rate",
                    "Compute (SM) Throughput", "Issue Slots Busy", "Achieved Occupancy",
                    "Registers Per Thread", "Dynamic Shared Memory Per Block"):
            if key in det:
                lines.append(f"- {key}: {det[key]}")
        for key in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            if key in r:
                lines.append(f"- {key}: {r[key]}")
        lines.append("- top stall reasons (warps per issue): " +
                     ", ".join(f"{n} {v:.2f}" for v, n in stalls(r)))
        lines.append("")
    with open(os.path.join(PROF, f"{tag}_summary.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    if k1 and traffic_json:
        traffic = k1["read"] + k1["write"]
        json.dump({"kernel": "mask_fg_kernel", "frame_reads_per_launch": reads,
                   "dram_bytes_per_launch": traffic, "dram_bytes_per_frame": traffic / reads,
                   "algorithmic_bytes_per_launch": reads * FRAME_BYTES,
                   "dram_bytes_per_step": step_bytes,
                   "dram_bytes_per_step_def": "sum over the step's kernels (one launch each) of "
                                              "the mean dram__bytes_read + dram__bytes_write",
                   "source": f"profiles/{tag}_launches.csv"},
                  open(os.path.join(ROOT, traffic_json), "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]), sys.argv[3] if len(sys.argv) > 3 else "",
         sys.argv[4] if len(sys.argv) > 4 else "")
