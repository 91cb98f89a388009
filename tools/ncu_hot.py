"""Top stall-sampled SASS instructions of an ncu report (reads the CSV source page)."""
import csv, subprocess, sys
rep, n = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
si, ai, ii = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source"), hdr.index("Instructions Executed")
data = [(int(r[si] or 0), i, r[ai].strip(), int(r[ii] or 0)) for i, r in enumerate(rows[2:]) if len(r) == len(hdr)]
tot = sum(d[0] for d in data) or 1
print("total samples", tot, "instructions", len(data))
for s, i, src, ex in sorted(data, reverse=True)[:n]:
    print(f"{100*s/tot:5.1f}% #{i:5d} exec={ex:9d} {src[:80]}")
