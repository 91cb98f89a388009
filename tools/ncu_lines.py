"""Per-CUDA-source-line totals (instructions executed, stall samples) from an ncu report."""
import csv, subprocess, sys
from collections import defaultdict
rep, n = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
inst, samp, src = defaultdict(int), defaultdict(int), {}
fname = None
hdr = None
cur_line = None
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No":
        hdr = r; continue
    if hdr is None or len(r) != len(hdr):
        continue
    if r[0]:
        cur_line = (fname, int(r[0])); src[cur_line] = r[1].strip()
    try:
        inst[cur_line] += int(r[hdr.index("Instructions Executed")] or 0)
        samp[cur_line] += int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
    except (ValueError, IndexError):
        pass
ti, ts = sum(inst.values()) or 1, sum(samp.values()) or 1
print("total warp-instructions", ti)
for k in sorted(inst, key=lambda k: -inst[k])[:n]:
    print(f"{100*inst[k]/ti:5.1f}% inst {100*samp[k]/ts:5.1f}% stall  {k[0]}:{k[1]}  {src.get(k,'')[:70]}")
