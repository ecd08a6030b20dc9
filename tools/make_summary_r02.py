"""Regenerate profiles/r02_summary.md and profiles/r02_bench_c1_c5.jsonl from
one evidence run (tools/gpu_r02_final.sh -> gpurun_out/, then
tools/collect_profiles.py --round 2).

    python tools/make_summary_r02.py
"""
import json
import shutil
from pathlib import Path

REPO = Path(__file__).resolve().parents[1]
OUT = REPO / "gpurun_out"
PROF = REPO / "profiles"


def last_json_line(path):
    for line in reversed(path.read_text().splitlines()):
        line = line.strip()
        if line.startswith("{") and line.endswith("}"):
            return json.loads(line)
    raise RuntimeError(f"no JSON line in {path}")


def table(rows):
    out = ["| n | engine / variant / b | ms | GFLOP/s | GB/s | bound | frac (measured roof) |", "|---|---|---|---|---|---|---|"]
    for r in rows:
        out.append(f"| {r['n']} | {r['engine']} v{r['variant']} b{r['b']} | {r['ms']:.4f} | {r['gflops']} | {r['gbs']} | "
                   f"{r['bound']} | {r['roofline_frac_measured']} |")
    return out


def main():
    b = json.loads((PROF / "r02_bench.json").read_text())
    d = json.loads((PROF / "r02_bench_detail.json").read_text())
    ref = json.loads((PROF / "r02_bench_reference_arm.json").read_text())
    lines = []
    for w in ("c1", "c5-chol", "c5-lyap", "c5-sylv"):
        p = OUT / f"bench_{w}.log"
        if p.exists():
            lines.append((w, last_json_line(p)))
    if lines:
        (PROF / "r02_bench_c1_c5.jsonl").write_text("".join(json.dumps(j, separators=(",", ":")) + "\n" for _, j in lines))
    else:
        lines = list(zip(("c1", "c5-chol", "c5-lyap", "c5-sylv"),
                         (json.loads(l) for l in (PROF / "r02_bench_c1_c5.jsonl").read_text().splitlines())))
    for src, dst in (("e2e_hybrid.txt", "r02_e2e_hybrid.txt"), ("e2e_nosplit.txt", "r02_e2e_nosplit.txt"),
                     ("pytest_gpu.log", "r02_pytest_gpu.log")):
        if (OUT / src).exists():
            shutil.copyfile(OUT / src, PROF / dst)
    rf, cpu, e2e = b["roofline"], b["cpu_baseline"], b["e2e"]
    out = ["# Round 2 — measurement summary (B200, 1 GPU)", "",
           "Files: `r02_bench.json` (the bench.py line), `r02_bench_detail.json` (`--json-out`, per-n tables), "
           "`r02_bench_reference_arm.json` (`bench.py --impl reference`), `r02_bench_c1_c5.jsonl` (BASELINE configs 1 and 5 "
           "on one GPU), `r02_pytest_gpu.log` (GPU parity run of the same tree), `r02_ncu_launches_sweeps.md` / "
           "`r02_ncu_launches_chol_sweep.csv` (ncu launch lists: time and DRAM bytes per launch of one step of each sweep), "
           "`r02_ncu_full_top_kernels.csv` (`ncu --set full` of the top kernels), `r02_traffic.json` (DRAM bytes vs "
           "algorithmic bytes), A/B and tuning records: `r02_pipe_solver_ab.txt` (tile-solve formulations, columns per "
           "updater warp, predication, single-warp issue rates), `r02_ncu_pipe_solver_stalls.txt` (stall reasons inside the tile solve), "
           "`r02_rows_trim.txt` (rows / column engine instruction trimming), `r02_rowsmix_ab.txt`, `r02_rowsmix_tune.txt`, "
           "`r02_pipe_minb_sweep.txt`, `r02_pipe_minb_resweep.txt`, `r02_pipe_lsu_fix.txt`, `r02_pipe_solo.txt`, "
           "`r02_rowsweep_sweep.txt`, `r02_rowsweep_symk.txt`, `r02_e2e_hybrid.txt`, `r02_e2e_nosplit.txt`, "
           "`r02_ncu_rows128_smem_lines.txt`, `r02_ncu_pipe_sylv64_smem_lines_before.txt`, `r02_chol_gang_experiment.md` "
           "(+ `_v5_ioonly`, `_v6`). Produced by `tools/gpu_r02_final.sh` / `tools/evidence.sh` / "
           "`tools/collect_profiles.py --round 2` / `tools/make_summary_r02.py`.", "",
           "## Headline (BASELINE configs[1], Cholesky sweep n = 4..128)", "",
           f"- value: **{b['value']} GFLOP/s** (nominal n^3/3 flops), {b['ms_per_step']} ms per sweep step "
           f"({b['gpu_launches']} launches in the timed region, one CUDA graph per step); round 1: 4108.",
           f"- roofline ({rf['bound']}-bound): {rf['achieved']} GB/s of compulsory bytes = **{rf['frac']}** of the measured "
           f"peak ({rf['peak']}); minimum over n >= 32: {rf['frac_min_n_ge_32']} (n = {rf['dominant']['n']}, "
           f"{rf['dominant']['engine']}).",
           f"- DRAM traffic of the n = 128 launch: {rf['traffic']} B = {rf['traffic_ratio']} x its algorithmic bytes.",
           f"- CPU reference in the same run ({cpu['kind']}, {cpu['cores']} cores): {cpu['value']} GFLOP/s; "
           f"`--impl reference` arm on the same box: {ref['value']} GFLOP/s.",
           f"- e2e (host buffers through executor.solve_host, H2D + D2H inside the timed region): {e2e['value']} GFLOP/s "
           f"({e2e['h2d_bytes_per_step']} B in, {e2e['d2h_bytes_per_step']} B out per step).",
           f"- clocks: {b['clocks']}", ""]
    out += table(d["per_n"]) + [""]
    for eq, name in (("lyapunov", "Lyapunov"), ("sylvester", "Sylvester")):
        x, xd = b["extra"][eq], d["extra_detail"][eq]
        out += [f"## {name} sweep", "",
                f"- value: **{x['value']} GFLOP/s**, {x['ms_per_step']} ms per sweep; roofline {x['roofline_bound']}: "
                f"{x['roofline_frac']} of the measured peak (bytes), {x['frac_roofline_time']} by roofline time, minimum over "
                f"n >= 32: {x['frac_min_n_ge_32']}; e2e {x['e2e']} GFLOP/s; CPU reference {x['cpu_baseline']} GFLOP/s.", ""]
        out += table(xd["per_n"]) + [""]
    out += ["## BASELINE configs 1 and 5 (one GPU)", "", "| workload | GFLOP/s | ms per step | roofline frac | e2e GFLOP/s |",
            "|---|---|---|---|---|"]
    for w, j in lines:
        out.append(f"| {w} | {j['value']} | {j['ms_per_step']} | {j['roofline']['frac']} | {j.get('e2e', {}).get('value')} |")
    (PROF / "r02_summary.md").write_text("\n".join(out) + "\n")
    print("wrote r02_summary.md")


if __name__ == "__main__":
    main()
