"""Large-n golden vectors from the REFERENCE implementation (n = 48 ... 128).

Run in the build container, where the reference package is importable:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_large.py

For every equation, n in SIZES, every synthesised variant and every default
block size b (cli.default_blocks, /root/reference/pkg/src/lagen/cli.py:89-93)
it runs the reference executor (`interpret_algorithm`,
/root/reference/pkg/src/lagen/verify.py:221-303) on the first NPROB problems of
the BASELINE-distribution stream (the oracle's CPU generator, seed = n) and
stores, per output X, two right projections X V and two left projections
W^T X (V, W: fixed seeded Gaussian n x 2) and ||X||_F — 4n + 1 numbers
instead of n^2, so the fixture stays small at n = 128.  A relative error
||X - X_ref||_F <= tol * ||X_ref||_F bounds both projection errors by
tol * ||X_ref||_F * ||V||_F, which is what tests check.  The inputs are not
stored: the tests regenerate them with the same CPU generator and check the
stored input checksums first.

Output: tests/golden/large_<equation>.npz + large_meta.json.
"""

import json
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parents[1]
sys.path.insert(0, str(REPO))

SIZES = (48, 64, 96, 128)
NPROB = 2
CASES = {"cholesky": "cholesky.la", "lyapunov": "lyapunov.la", "sylvester": "sylvester.la"}


def projectors(n):
    rng = np.random.default_rng(1000 + n)
    return rng.standard_normal((n, 2)), rng.standard_normal((n, 2))


def input_checksum(arrs):
    return [float(np.sum(a)) for a in arrs] + [float(np.sum(a * a)) for a in arrs]


def main():
    from lagen.lang import parse_equation
    from lagen.verify import Instance, interpret_algorithm
    from lagen.worksheet import enumerate_algorithms

    from oracle import oracle
    from paper_1906_08613_b200.variants import EQ_INPUTS, default_blocks

    ref_root = Path(__import__("lagen").__file__).resolve().parents[2]
    meta = {"sizes": list(SIZES), "nprob": NPROB, "generator": "oracle.generate(eq, n, seed=n, first=0)",
            "reference": "lagen interpret_algorithm", "script": "tests/golden/make_golden_large.py"}
    for eq_name, fname in CASES.items():
        text = (ref_root / "cases" / fname).read_text()
        eq = parse_equation(text, name=eq_name)
        algs = enumerate_algorithms(eq)
        data, entries = {}, []
        t0 = time.time()
        for n in SIZES:
            gen = oracle.generate(eq_name, n, seed=n, first=0, batch=NPROB)
            data[f"checksum_{n}"] = np.array(input_checksum(gen))
            V, W = projectors(n)
            for p in range(NPROB):
                inst = Instance(eq, n, n, {nm: g[p] for nm, g in zip(EQ_INPUTS[eq_name], gen)})
                for alg in algs:
                    for b in default_blocks(n):
                        out, flops = interpret_algorithm(alg, inst, b)
                        X = out["X"]
                        key = f"{n}_p{p}_v{alg.index}_b{b}"
                        data["xv_" + key] = X @ V
                        data["wx_" + key] = W.T @ X
                        data["nrm_" + key] = np.array([np.linalg.norm(X)])
                        entries.append({"key": key, "n": n, "p": p, "variant": alg.index, "b": b, "flops": flops})
        np.savez_compressed(HERE / f"large_{eq_name}.npz", **data)
        meta[eq_name] = entries
        print(eq_name, len(entries), "outputs", f"{time.time() - t0:.1f} s")
    (HERE / "large_meta.json").write_text(json.dumps(meta, indent=1) + "\n")


if __name__ == "__main__":
    main()
