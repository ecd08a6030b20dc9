"""Writes tests/golden/nu_defect.json: the observed error of the reference's
nu-mode Lyapunov kernel (b = 8 > nu = 4) against its own interpreter, next to
its scalar twin.  Run where /root/reference and gcc exist:

    python tests/golden/make_nu_defect.py
"""
import json
import sys
import tempfile
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))
sys.path.insert(0, str(HERE.parent))
import test_ref_nu_defects as t  # noqa: E402

t._lagen()
from lagen.verify import interpret_algorithm, random_instance  # noqa: E402

n, out = 16, {}
with tempfile.TemporaryDirectory() as d:
    for b, mode in ((8, "nu"), (8, "scalar"), (4, "nu")):
        eq, alg, fn, header = t._emit("lyapunov", 5, n, b, mode)
        inst = random_instance(eq, n, seed=31)
        want, _ = interpret_algorithm(alg, inst, b)
        got = t._compile_and_run(fn, header, Path(d) / f"{fn.name}_{mode}.so", inst, n)
        out[f"b{b}_{mode}_rel_err"] = t._rel(got, want["X"])
out.update({"equation": "lyapunov", "variant": 5, "n": n, "b": 8, "mode": "nu", "seed": 31,
            "b8_nu_rel_err_min": out["b8_nu_rel_err"] / 10,
            "reference": "lowering.py:628-636 (_nu_gemm symmetric gather), test_acceptance.py:257-267 (.so path)"})
(HERE / "nu_defect.json").write_text(json.dumps(out, indent=1) + "\n")
print(out)
