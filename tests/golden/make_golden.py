"""Generate golden vectors from the REFERENCE implementation.

Run in the build container, where the reference package is importable:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

For every equation, n in SIZES, every synthesised variant and every default
block size b (cli.default_blocks, /root/reference/pkg/src/lagen/cli.py:89-93)
plus b = n (one block: the leaf kernel on the whole matrix, admissible for
interpret_algorithm, verify.py:232-233)
it records the reference executor's output
(`interpret_algorithm`, /root/reference/pkg/src/lagen/verify.py:221-303) and
dynamic flop count on two instances:

  * "ref":  the reference's own `random_instance(eq, n, seed=11)`
            (verify.py:64-102, splitmix64 uniform fills), and
  * "base": the BASELINE.json distributions from the oracle's generator
            (seed = n, problem 0), stored verbatim so the fixture does not
            depend on generator stability.

plus the independent oracle (`oracle_solve`, verify.py:163-183) for n <= 16.
Output: tests/golden/<equation>.npz (+ golden_meta.json).  These fixtures pin
both the CPU oracle (tests/test_oracle_golden.py) and the CUDA path
(tests/test_gpu_parity.py) to the reference's numbers.
"""

import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parents[1]
sys.path.insert(0, str(REPO))

SIZES = (4, 8, 12, 16, 24, 32)
CASES = {"cholesky": "cholesky.la", "lyapunov": "lyapunov.la", "sylvester": "sylvester.la"}


def main():
    from lagen.lang import parse_equation
    from lagen.verify import Instance, interpret_algorithm, oracle_solve, random_instance
    from lagen.worksheet import enumerate_algorithms

    from oracle import oracle
    from paper_1906_08613_b200.variants import EQ_INPUTS, default_blocks

    ref_root = Path(__import__("lagen").__file__).resolve().parents[2]
    meta = {}
    for eq_name, fname in CASES.items():
        text = (ref_root / "cases" / fname).read_text()
        eq = parse_equation(text, name=eq_name)
        algs = enumerate_algorithms(eq)
        data = {}
        entries = []
        for n in SIZES:
            insts = {"ref": random_instance(eq, n, seed=11)}
            gen = oracle.generate(eq_name, n, seed=n, first=0, batch=1)
            insts["base"] = Instance(eq, n, n, {nm: g[0] for nm, g in zip(EQ_INPUTS[eq_name], gen)})
            for case, inst in insts.items():
                for nm in EQ_INPUTS[eq_name]:
                    data[f"in_{case}_{n}_{nm}"] = inst.bindings[nm]
                if n <= 16:
                    data[f"oracle_{case}_{n}"] = oracle_solve(inst)["X"]
                for alg in algs:
                    for b in sorted(set(default_blocks(n)) | {n}):
                        out, flops = interpret_algorithm(alg, inst, b)
                        key = f"x_{case}_{n}_v{alg.index}_b{b}"
                        data[key] = out["X"]
                        entries.append({"key": key, "case": case, "n": n,
                                        "variant": alg.index, "b": b, "flops": flops})
        np.savez_compressed(HERE / f"{eq_name}.npz", **data)
        meta[eq_name] = {"sizes": list(SIZES), "entries": entries,
                         "generator": "tests/golden/make_golden.py",
                         "reference": "lagen 0.1.0 interpret_algorithm"}
        print(eq_name, len(entries), "outputs")
    (HERE / "golden_meta.json").write_text(json.dumps(meta, indent=1) + "\n")


if __name__ == "__main__":
    main()
