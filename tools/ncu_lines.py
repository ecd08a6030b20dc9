"""Summarise an ncu report per CUDA source line: stall samples and instructions."""
import csv, subprocess, sys
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
files, cur = [], None
agg = {}
hdr = None
for r in rows:
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8 or not r[0]:
        continue
    iS = hdr.index("Warp Stall Sampling (All Samples)")
    iI = hdr.index("Instructions Executed")
    key = (cur, int(r[0]))
    a = agg.setdefault(key, [0, 0, r[1].strip()[:100]])
    a[0] += int(r[iS]) if r[iS].isdigit() else 0
    a[1] += int(r[iI]) if r[iI].isdigit() else 0
ts = sum(v[0] for v in agg.values()) or 1
ti = sum(v[1] for v in agg.values()) or 1
print(f"total stall samples {ts}, instructions {ti}")
for (f, l), (s, i, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:n]:
    print(f"{s/ts*100:5.1f}% stall {i/ti*100:5.1f}% inst {f}:{l}: {src}")
