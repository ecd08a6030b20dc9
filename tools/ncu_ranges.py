"""Stall samples / instructions / stall reasons of an ncu report summed over
source-line ranges of one file (role or phase breakdown of a kernel).

    python tools/ncu_ranges.py report.ncu-rep pipe.cuh name:a-b name:a-b ...
"""
import csv
import subprocess
import sys

rep, fname, specs = sys.argv[1], sys.argv[2], sys.argv[3:]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
ranges = []
for s in specs:
    name, ab = s.split(":")
    a, b = ab.split("-")
    ranges.append((name, int(a), int(b)))
hdr, cur = None, None
agg = {n: {} for n, _, _ in ranges}
agg["other"] = {}
tot = {}
for r in rows:
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r or not r[0].isdigit():
        continue
    line = int(r[0])
    key = "other"
    if cur == fname:
        for n, a, b in ranges:
            if a <= line <= b:
                key = n
                break
    d = agg[key]
    for i, h in enumerate(hdr):
        if h in ("Warp Stall Sampling (All Samples)", "Instructions Executed") or (h.startswith("stall_") and "Not Issued" not in h):
            try:
                v = float(r[i])
            except ValueError:
                continue
            d[h] = d.get(h, 0) + v
            tot[h] = tot.get(h, 0) + v
S, I = "Warp Stall Sampling (All Samples)", "Instructions Executed"
print(f"total samples {tot.get(S, 0):.0f}, instructions {tot.get(I, 0):.0f}")
for n, d in agg.items():
    if not d:
        continue
    reasons = sorted(((k[6:], v) for k, v in d.items() if k.startswith("stall_")), key=lambda kv: -kv[1])[:6]
    print(f"{n:>10}: {d.get(S, 0) / tot[S] * 100:5.1f}% samples {d.get(I, 0) / tot[I] * 100:5.1f}% inst  "
          + " ".join(f"{k}={v / max(d.get(S, 1), 1) * 100:.0f}%" for k, v in reasons))
