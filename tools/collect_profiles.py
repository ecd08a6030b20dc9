"""Copy one evidence run (tools/evidence.sh -> gpurun_out/) into profiles/:
the bench line, the per-sweep ncu launch lists (time + DRAM bytes of the last
sweep step's launches) and the ncu --set full metrics of the top kernels.

    python tools/collect_profiles.py --round 1
"""
import argparse
import csv
import io
import json
import shutil
import subprocess
from pathlib import Path

REPO = Path(__file__).resolve().parents[1]
OUT = REPO / "gpurun_out"
PROF = REPO / "profiles"
FULL_ALL = [("chol128_rows_v1b8", "full_chol128"), ("chol92_rowsmix_v1", "full_chol92"),
        ("sylv128_pipe_v13", "full_sylv128"), ("lyap64_pipe_v5", "full_lyap64"),
        ("sylv64_pipe_v13", "full_sylv64"), ("lyap128_pipe_v5", "full_lyap128")]
METRICS = ["dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "gpu__time_duration.sum",
           "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "launch__block_size", "launch__grid_size",
           "launch__registers_per_thread", "sm__inst_executed.sum.per_cycle_active",
           "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
           "smsp__inst_executed.sum"]


def _csv_rows(path):
    text = path.read_text().splitlines()
    start = next(i for i, l in enumerate(text) if l.startswith('"ID"'))
    return list(csv.reader(text[start:]))


def launches(name, nlaunch):
    rows = _csv_rows(OUT / f"launches_{name}.csv")
    hdr = rows[0]
    iK, iM, iU, iV = (hdr.index(h) for h in ("Kernel Name", "Metric Name", "Metric Unit", "Metric Value"))
    iID, iG, iB = hdr.index("ID"), hdr.index("Grid Size"), hdr.index("Block Size")
    per = {}
    for r in rows[1:]:
        if len(r) <= iV:
            continue
        k = per.setdefault(int(r[iID]), {"kernel": r[iK], "grid": r[iG], "block": r[iB]})
        v = float(r[iV].replace(",", ""))
        unit = r[iU]
        if r[iM] == "gpu__time_duration.sum":
            k["us"] = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(unit, 1.0) * v
        else:
            k["mb"] = k.get("mb", 0.0) + v * {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "B": 1e-6, "KB": 1e-3, "MB": 1.0, "GB": 1e3}.get(unit, 1.0)
    solver = [per[i] for i in sorted(per) if "gen_" not in per[i]["kernel"]]
    return solver[-nlaunch:]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--round", type=int, default=1)
    a = ap.parse_args()
    tag = f"r{a.round:02d}"
    line = (OUT / "bench_final.log").read_text().strip().splitlines()[-1]
    bench = json.loads(line)
    (PROF / f"{tag}_bench.json").write_text(json.dumps(bench) + "\n")
    if (OUT / "bench_detail.json").exists():
        shutil.copy(OUT / "bench_detail.json", PROF / f"{tag}_bench_detail.json")
    for extra, dst in (("bench_reference.log", f"{tag}_bench_reference_arm.json"), ("pytest_gpu.log", f"{tag}_pytest_gpu.log")):
        if (OUT / extra).exists():
            shutil.copy(OUT / extra, PROF / dst)
    md = []
    for name in ("chol-sweep", "lyap-sweep", "sylv-sweep"):
        ls = launches(name, 32)
        tot = sum(k["us"] for k in ls)
        md.append(f"## {name}: last {len(ls)} solver launches (= one sweep step), ncu --metrics "
                  "gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none "
                  "(cold, serialised)")
        md.append(f"sum of launch times {tot / 1000:.3f} ms")
        md.append("| # | kernel | grid x block | us | share | DRAM MB |")
        md.append("|---|---|---|---|---|---|")
        for i, k in enumerate(ls):
            md.append(f"| {i} | `{k['kernel'][:90]}` | {k['grid']} x {k['block']} | {k['us']:.1f} | "
                      f"{100 * k['us'] / tot:.1f}% | {k.get('mb', 0):.0f} |")
        md.append("")
    (PROF / f"{tag}_ncu_launches_sweeps.md").write_text("\n".join(md))
    shutil.copy(OUT / "launches_chol-sweep.csv", PROF / f"{tag}_ncu_launches_chol_sweep.csv")
    FULL = [(l, r) for l, r in FULL_ALL if (OUT / f"{r}.ncu-rep").exists()]
    cols = {}
    for label, rep in FULL:
        out = subprocess.run(["ncu", "-i", str(OUT / f"{rep}.ncu-rep"), "--page", "raw", "--csv", "--metrics",
                              ",".join(METRICS)], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(out)))
        hdr, units, vals = rows[0], rows[1], rows[2]
        cols[label] = {m: f"{vals[hdr.index(m)]} {units[hdr.index(m)]}".strip() for m in METRICS if m in hdr}
    lines = ["# ncu --set full --clock-control none, one launch each (tools/evidence.sh): " +
             "; ".join(l for l, _ in FULL), "metric," + ",".join(l for l, _ in FULL)]
    for m in METRICS:
        lines.append(m + "," + ",".join(cols[l].get(m, "") for l, _ in FULL))
    (PROF / f"{tag}_ncu_full_top_kernels.csv").write_text("\n".join(lines) + "\n")
    print(f"wrote {tag}_bench.json, {tag}_ncu_launches_sweeps.md, {tag}_ncu_launches_chol_sweep.csv, "
          f"{tag}_ncu_full_top_kernels.csv")


if __name__ == "__main__":
    main()
