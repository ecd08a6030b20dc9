"""Per CUDA source line of an ncu report (--set full --import-source on):
share of shared-memory wavefronts, excessive wavefronts (bank conflicts),
instructions and stall samples; plus the kernel's stall-reason mix.

    python tools/ncu_smem_lines.py gpurun_out/full_sylv64.ncu-rep [top]
"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 24
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur = hdr = None
agg = {}
stalls = {}


def num(x):
    try:
        return int(x)
    except ValueError:
        return 0


for r in rows:
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr) or not r[0].isdigit():
        continue
    iw, ie = hdr.index("L1 Wavefronts Shared"), hdr.index("L1 Wavefronts Shared Excessive")
    ii, ist = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
    a = agg.setdefault((cur, int(r[0])), [0, 0, 0, 0, r[1].strip()[:84]])
    a[0] += num(r[iw]); a[1] += num(r[ie]); a[2] += num(r[ii]); a[3] += num(r[ist])
    for k, name in enumerate(hdr):
        if name.startswith("stall_") and "Not Issued" not in name:
            stalls[name] = stalls.get(name, 0) + num(r[k])
tw = sum(a[0] for a in agg.values()) or 1
te = sum(a[1] for a in agg.values()) or 1
ti = sum(a[2] for a in agg.values()) or 1
ts = sum(a[3] for a in agg.values()) or 1
print(f"shared wavefronts {tw}, excessive {te} ({100 * te / tw:.1f} %), instructions {ti}, stall samples {ts}")
print("stall mix: " + ", ".join(f"{k[6:]} {100 * v / ts:.1f}%" for k, v in sorted(stalls.items(), key=lambda kv: -kv[1])[:8]))
print("by wavefronts:")
for (f, l), a in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{a[0]/tw*100:5.1f}% wf {a[1]/te*100:5.1f}% exc {a[2]/ti*100:5.1f}% inst {a[3]/ts*100:5.1f}% stall  {f}:{l}: {a[4]}")
print("by stall samples:")
for (f, l), a in sorted(agg.items(), key=lambda kv: -kv[1][3])[:top]:
    print(f"{a[3]/ts*100:5.1f}% stall {a[2]/ti*100:5.1f}% inst {a[0]/tw*100:5.1f}% wf  {f}:{l}: {a[4]}")
