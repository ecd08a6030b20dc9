"""Serialise the reference's live `Algorithm` objects (worksheet.py:70-87) and
what its own interpreter computes from them, so the drop-in path
`executor.interpret_algorithm(alg, inst, b)` (the replacement of
/root/reference/pkg/src/lagen/verify.py:221) is tested on the GPU box, where
the reference package does not exist.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_algorithm_fixtures.py

Writes tests/golden/algorithms.json (every field encode_algorithm reads, for
every algorithm enumerate_algorithms synthesises: equation name and operands,
traversal, rhs_source, output, index, and the statements with their views) and
tests/golden/algorithms_n16.npz (random_instance(eq, 16, seed=42) bindings and
the reference interpret_algorithm's X and flop count for b in {4, 8}).  The
test rebuilds objects with the same attribute names from the JSON and feeds
them to the executor unchanged.
"""

import json
from pathlib import Path

import numpy as np

from lagen.lang import parse_equation
from lagen.verify import interpret_algorithm, random_instance
from lagen.worksheet import enumerate_algorithms

HERE = Path(__file__).resolve().parent
N, SEED, BLOCKS = 16, 42, (4, 8)
CASES = {
    "cholesky": "Equation: X^T * X = A\nA: Matrix(n,n), spd, input\nX: Matrix(n,n), upper_triangular, output\n",
    "lyapunov": "Equation: L * X + X * L^T = S\nL: Matrix(n,n), lower_triangular, input\n"
                "S: Matrix(n,n), symmetric, input\nX: Matrix(n,n), symmetric, output\n",
    "sylvester": "Equation: L * X + X * U = C\nL: Matrix(n,n), lower_triangular, input\n"
                 "U: Matrix(n,n), upper_triangular, input\nC: Matrix(n,n), general, input\n"
                 "X: Matrix(n,n), general, output\n",
}


def view(v):
    return {"op": v.op, "r": v.r, "c": v.c, "trans": bool(v.trans)}


def main():
    meta, arrays = {}, {}
    for name, text in CASES.items():
        eq = parse_equation(text, name=name)
        inst = random_instance(eq, N, seed=SEED)
        for nm, a in inst.bindings.items():
            arrays[f"{name}_in_{nm}"] = np.asarray(a, dtype=np.float64)
        algs = []
        for alg in enumerate_algorithms(eq):
            algs.append({
                "index": alg.index, "traversal": alg.traversal, "rhs_source": alg.rhs_source, "output": alg.output,
                "statements": [{"kind": s.kind, "sign": s.sign, "out": view(s.out), "ins": [view(v) for v in s.ins]}
                               for s in alg.statements],
            })
            for b in BLOCKS:
                got, flops = interpret_algorithm(alg, inst, b)
                arrays[f"{name}_v{alg.index}_b{b}_X"] = got[alg.output]
                algs[-1][f"flops_b{b}"] = int(flops)
        meta[name] = {
            "operands": [{"name": op.name, "is_output": bool(op.is_output)} for op in eq.operands],
            "inputs": list(inst.bindings.keys()),
            "algorithms": algs,
        }
    (HERE / "algorithms.json").write_text(json.dumps({"n": N, "seed": SEED, "blocks": BLOCKS, "equations": meta}, separators=(",", ":")))
    np.savez_compressed(HERE / "algorithms_n16.npz", **arrays)
    print({k: len(v["algorithms"]) for k, v in meta.items()})


if __name__ == "__main__":
    main()
