"""Rebuild the reference's `Algorithm` / `Statement` / `View` / `Instance`
objects (worksheet.py:29-87, verify.py Instance) from
tests/golden/algorithms.json + algorithms_n16.npz — written from the live
objects by tests/golden/make_algorithm_fixtures.py — with the same attribute
names, so code written against the reference's objects runs on them where the
reference package itself is absent (the GPU box)."""

import json
from dataclasses import dataclass
from pathlib import Path
from types import SimpleNamespace

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"


@dataclass(frozen=True)
class View:
    op: str
    r: int
    c: int
    trans: bool = False


@dataclass(frozen=True)
class Statement:
    kind: str
    out: View
    ins: tuple = ()
    sign: int = 1


@dataclass(frozen=True)
class Algorithm:
    equation: object
    traversal: str
    statements: tuple
    rhs_source: str
    output: str
    index: int = 0


def load():
    """{eq: (algorithms, instance, {(index, b): (X, flops)})}"""
    meta = json.loads((GOLDEN / "algorithms.json").read_text())
    data = np.load(GOLDEN / "algorithms_n16.npz")
    out = {}
    for name, m in meta["equations"].items():
        eq = SimpleNamespace(name=name, operands=tuple(SimpleNamespace(**o) for o in m["operands"]))
        algs, want = [], {}
        for a in m["algorithms"]:
            stmts = tuple(Statement(s["kind"], View(**s["out"]), tuple(View(**v) for v in s["ins"]), s["sign"])
                          for s in a["statements"])
            algs.append(Algorithm(eq, a["traversal"], stmts, a["rhs_source"], a["output"], a["index"]))
            for b in meta["blocks"]:
                want[(a["index"], b)] = (data[f"{name}_v{a['index']}_b{b}_X"], a[f"flops_b{b}"])
        inst = SimpleNamespace(n=meta["n"], bindings={nm: data[f"{name}_in_{nm}"] for nm in m["inputs"]})
        out[name] = (algs, inst, want)
    return out, meta["blocks"]
