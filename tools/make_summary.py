"""Write profiles/r<NN>_summary.md from the committed measurement files.

    python tools/make_summary.py --round 1
"""
import argparse
import json
from pathlib import Path

PROF = Path(__file__).resolve().parents[1] / "profiles"


def table(per_n):
    rows = ["| n | engine / variant / b | ms | GFLOP/s | GB/s | bound | frac (measured roof) |",
            "|---|---|---|---|---|---|---|"]
    for r in per_n:
        rows.append(f"| {r['n']} | {r.get('engine', '?')} v{r['variant']} b{r['b']} | {r['ms']:.4f} | "
                    f"{r['gflops']} | {r['gbs']} | {r['bound']} | {r['roofline_frac_measured']} |")
    return "\n".join(rows)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--round", type=int, default=1)
    a = ap.parse_args()
    tag = f"r{a.round:02d}"
    b = json.loads((PROF / f"{tag}_bench.json").read_text())
    rf = b["roofline"]
    cpu = b.get("cpu_baseline", {})
    e2e = b.get("e2e", {})
    out = [f"# Round {a.round} — measurement summary (B200, 1 GPU)", "",
           "Files in this directory: `" + tag + "_bench.json` (the bench.py JSON line), "
           "`" + tag + "_autotune_report.json` (every engine x variant x b timed per (eq, n)), "
           "`" + tag + "_ncu_launches_chol_sweep.csv` (ncu launch list, `--metrics gpu__time_duration.sum "
           "--clock-control none`), `" + tag + "_ncu_full_*.csv` (`ncu --set full` of top kernels), "
           "`fp64_peaks.json` / `fp64_latency.json` (tools/fp64_peaks.cu, tools/fp64_latency.cu), "
           "`" + tag + "_rows_modes.txt` (rows-engine work-split sweep), `" + tag + "_phase_profile.txt`, "
           "`" + tag + "_ncu_launches_sweeps.md` (per-launch time and DRAM bytes of one step of each sweep), "
           "`" + tag + "_ncu_full_top_kernels.csv` (ncu --set full metrics of the top kernels), "
           "`" + tag + "_traffic.json`, `" + tag + "_wave_traffic.txt`, `" + tag + "_rows_db.txt`, "
           "`" + tag + "_e2e_bands.txt`; A/B records of this round's tuning: `" + tag + "_chol_lookahead.md`, "
           "`" + tag + "_wave_geometry.md`, `" + tag + "_rows_tune.txt`, `" + tag + "_rowspad_tune.txt`, "
           "`" + tag + "_rowloop_ab.txt`, `" + tag + "_col_wide_ab.txt`, `" + tag + "_spread_ab.txt`; other BASELINE configs: "
           "`" + tag + "_bench_c1.json` (configs[0]), `" + tag + "_bench_c5.jsonl` (config 5 on one GPU), "
           "`" + tag + "_bench_reference_arm.json` (`bench.py --impl reference`); GPU parity run of the same tree: `" + tag + "_pytest_gpu_rerun.log` (`tools/gpu_round_end.sh`).", "",
           "## Peaks used", "",
           f"- HBM: {b['peaks']['hbm_gbs']} GB/s ({b['peaks']['source']['hbm_gbs']}).",
           f"- FP64: {b['peaks']['fp64_tflops']} TFLOP/s ({b['peaks']['source']['fp64_tflops']}).", ""]
    lat = PROF / "fp64_latency.json"
    if lat.exists():
        out += [f"- Measured dependent-chain latencies (cycles): {lat.read_text().strip()}", ""]
    out += ["## Headline (BASELINE configs[1], Cholesky sweep n = 4..128)", "",
            f"- value: **{b['value']} {b['unit']}** (nominal n^3/3 flops), {b['ms_per_step']} ms per sweep step "
            f"({b.get('gpu_launches', '?')} kernel launches in the timed region, one CUDA graph per step).",
            f"- roofline ({rf['bound']}-bound): achieved {rf['achieved']} {rf['unit']} of compulsory bytes = "
            f"{rf['frac']} of the measured peak; {rf.get('frac_of_nominal_roofline')} of the BASELINE.md nominal roofline.",
            f"- CPU reference ({cpu.get('kind')}, {cpu.get('cores')} cores): {cpu.get('value')} {cpu.get('unit')} — "
            f"{cpu.get('sample', '')}",
            f"- e2e (host buffers through executor.solve_host, H2D + D2H inside the timed region): "
            f"{e2e.get('value')} {e2e.get('unit')}",
            f"- clocks during the timed region: {b.get('clocks')}", "",
            table(b["per_n"]), ""]
    for eq, r in b.get("extra", {}).items():
        rr = r["roofline"]
        c = r.get("cpu_baseline", {})
        out += [f"## {eq.capitalize()} sweep (BASELINE configs: {r.get('description', '')})", "",
                f"- value: **{r['value']} {r['unit']}**, {r['ms_per_step']} ms per sweep; roofline "
                f"{rr['bound']}: {rr['achieved']} {rr['unit']} = {rr['frac']} of the measured peak.",
                f"- CPU reference: {c.get('value')} {c.get('unit')} ({c.get('cores')} cores).", "",
                table(r["per_n"]), ""]
    (PROF / f"{tag}_summary.md").write_text("\n".join(out))
    print(PROF / f"{tag}_summary.md")


if __name__ == "__main__":
    main()
