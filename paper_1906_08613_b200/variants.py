"""Blocked-variant descriptors: the statement lists the backend executes.

A variant is the per-iteration statement list of one blocked algorithm on the
2x2 -> 3x3 repartition (reference: `Algorithm`/`Statement`/`View`,
/root/reference/pkg/src/lagen/worksheet.py:29-87).  The backend consumes it
in an integer encoding shared by the Python host, the C-ABI
(`lagen_stmt`, include/lagen_b200.h) and the CUDA kernels:

  kind:  GEMM_update=0, CHOL=1, TRSM_left_transposed=2, SYLV=3, LYAP=4
  op:    0 = the unknown's storage X, 1.. = coefficient operands (the inputs
         other than the rhs source) in declaration order: L=1, U=2
  view:  (op, r, c, trans) with r, c in {0, 1, 2}

Two sources of statement lists:
  * `builtin_variants(eq)`: the frozen output of the reference's
    `enumerate_algorithms` for the three shipped cases (variants_table.json,
    produced by tools/extract_variants.py);
  * `encode_algorithm(alg)`: any live `lagen.worksheet.Algorithm`.
"""

import json
from dataclasses import dataclass
from functools import lru_cache
from pathlib import Path

from .errors import VariantError

KIND_CODES = {
    "GEMM_update": 0,
    "CHOL": 1,
    "TRSM_left_transposed": 2,
    "SYLV": 3,
    "LYAP": 4,
}
KIND_NAMES = {v: k for k, v in KIND_CODES.items()}

EQUATIONS = ("cholesky", "lyapunov", "sylvester")
EQ_CODES = {name: i for i, name in enumerate(EQUATIONS)}
# _signature order (codegen.py:143-152): inputs in declaration order, then X
EQ_INPUTS = {
    "cholesky": ("A",),
    "lyapunov": ("L", "S"),
    "sylvester": ("L", "U", "C"),
}
EQ_RHS = {"cholesky": "A", "lyapunov": "S", "sylvester": "C"}
EQ_COEFFS = {"cholesky": (), "lyapunov": ("L",), "sylvester": ("L", "U")}
# structure of each operand as the reference declares it (cases/*.la)
EQ_STRUCT = {
    "cholesky": {"A": "spd", "X": "upper_triangular"},
    "lyapunov": {"L": "lower_triangular", "S": "symmetric", "X": "symmetric"},
    "sylvester": {"L": "lower_triangular", "U": "upper_triangular",
                  "C": "general", "X": "general"},
}

_TABLE_PATH = Path(__file__).with_name("variants_table.json")


def _op_code(name, output, coeffs):
    if name == output:
        return 0
    if name in coeffs:
        return 1 + coeffs.index(name)
    raise VariantError(f"statement reads operand {name!r}, which is neither "
                       "the unknown nor a coefficient")


def classify_equation(eq):
    """Map a reference Equation onto one of the three supported classes.

    Uses the reference's own classifier when available (verify.py:134-160)."""
    name = getattr(eq, "name", None)
    try:
        from lagen.verify import classify
        kind = classify(eq)
    except Exception:  # pragma: no cover - reference not importable
        kind = None
    mapping = {"chol": "cholesky", "lyap": "lyapunov", "sylv": "sylvester"}
    if kind in mapping:
        return mapping[kind]
    if name in EQUATIONS:
        return name
    raise VariantError(f"equation {name!r} is not one of {EQUATIONS}")


def encode_algorithm(alg):
    """Encode a reference `Algorithm` (worksheet.py:70-87) as statement dicts."""
    if getattr(alg, "traversal", "TL_to_BR") != "TL_to_BR":
        raise VariantError("only TL_to_BR traversals are synthesised")
    eq = alg.equation
    output = alg.output
    rhs = alg.rhs_source
    coeffs = tuple(op.name for op in eq.operands
                   if not op.is_output and op.name != rhs)
    out = []
    for stmt in alg.statements:
        if stmt.kind not in KIND_CODES:
            raise VariantError(f"statement kind {stmt.kind} has no B200 kernel")
        if stmt.out.op != output:
            raise VariantError("statement writes outside the output")
        if stmt.out.trans:
            raise VariantError("transposed output views are not synthesised")
        ins = [[_op_code(v.op, output, coeffs), v.r, v.c, int(bool(v.trans))]
               for v in stmt.ins]
        while len(ins) < 2:
            ins.append([-1, 0, 0, 0])
        out.append({
            "kind": KIND_CODES[stmt.kind],
            "sign": int(stmt.sign),
            "out": [0, stmt.out.r, stmt.out.c],
            "ins": ins,
        })
    return out


def validate(eq_name, stmts):
    """Structural checks mirroring what the executor needs (and the C-ABI
    re-checks): arity per kind, block indices, triangular coefficients."""
    if not stmts:
        raise VariantError("empty statement list")
    if len(stmts) > 16:
        raise VariantError("more than LAGEN_MAX_STMTS statements")
    ncoef = len(EQ_COEFFS[eq_name])
    arity = {0: 2, 1: 0, 2: 1, 3: 2, 4: 1}
    for s in stmts:
        k = s["kind"]
        if k not in arity:
            raise VariantError(f"unknown statement kind {k}")
        if s["out"][0] != 0:
            raise VariantError("statement writes outside the output")
        for idx in (1, 2):
            if s["out"][idx] not in (0, 1, 2):
                raise VariantError("block index out of range")
        for j in range(2):
            v = s["ins"][j]
            if j < arity[k]:
                if not (0 <= v[0] <= ncoef) or v[1] not in (0, 1, 2) or v[2] not in (0, 1, 2):
                    raise VariantError(f"bad input view {v}")
            elif v[0] != -1:
                raise VariantError(f"unexpected input view {v} for kind {k}")
        if k == 0 and s["sign"] not in (1, -1):
            raise VariantError("GEMM sign must be +-1")
    return stmts


@dataclass(frozen=True)
class Variant:
    """One built-in blocked variant of one equation."""

    equation: str
    index: int
    invariant: str
    statements: tuple          # encoded statement dicts
    display: tuple             # reference worksheet lines (Statement.display)
    mirror_output: bool

    @property
    def name(self):
        return f"{self.equation}_v{self.index}"


@lru_cache(maxsize=None)
def _table():
    return json.loads(_TABLE_PATH.read_text())


def builtin_variants(eq_name):
    entry = _table()[eq_name]
    return [Variant(eq_name, v["index"], v["invariant"],
                    tuple(_freeze(s) for s in v["statements"]),
                    tuple(v["display"]), v["mirror_output"])
            for v in entry["variants"]]


def _freeze(s):
    return {"kind": s["kind"], "sign": s["sign"], "out": tuple(s["out"]),
            "ins": tuple(tuple(v) for v in s["ins"])}


def stmts_key(stmts):
    return tuple((s["kind"], s["sign"], tuple(s["out"]),
                  tuple(tuple(v) for v in s["ins"])) for s in stmts)


def match_builtin(eq_name, stmts):
    """Index of the built-in variant with this exact statement list, or None."""
    key = stmts_key(stmts)
    for v in builtin_variants(eq_name):
        if stmts_key(v.statements) == key:
            return v.index
    return None


def default_blocks(n):
    """Admissible block sizes, restating cli.default_blocks (cli.py:89-93)."""
    blocks = [b for b in (4, 8, 16) if n % b == 0 and b < n]
    if not blocks and n in (4, 8, 16):
        blocks = [n]
    return blocks


def statement_flops(eq_name, s, ext):
    """Exact count of one statement, restating worksheet.statement_flops
    (/root/reference/pkg/src/lagen/worksheet.py:313-351)."""
    def shape(v):
        r, c = ext[v[1]], ext[v[2]]
        return (c, r) if len(v) > 3 and v[3] else (r, c)

    m, q = shape(s["out"])
    if m == 0 or q == 0:
        return 0
    k = s["kind"]
    if k == 0:
        p = shape(s["ins"][0])[1]
        if p == 0:
            return 0
        if eq_name != "sylvester" and s["out"][1] == s["out"][2]:
            return q * (q + 1) * p
        return 2 * m * p * q
    if k == 1:
        return m * (m + 1) * (2 * m + 1) // 6
    if k == 2:
        p = shape(s["ins"][0])[0]
        return q * p * p
    if k == 3:
        return m * q * (m + q)
    if k == 4:
        return m * m * (m + 1)
    raise VariantError(f"no cost model for kind {k}")


def flop_count(eq_name, stmts, n, b):
    """Dynamic scalar-op count of a variant (worksheet.flop_count, :354-367)."""
    if n % b:
        raise VariantError(f"block size {b} does not divide {n}")
    total = 0
    for k in range(n // b):
        ext = {0: k * b, 1: b, 2: n - (k + 1) * b}
        for s in stmts:
            total += statement_flops(eq_name, s, ext)
    return total


def flops_alg(eq_name, n):
    """Exact structure-exploiting count (worksheet.py:313-367 closed forms)."""
    if eq_name == "cholesky":
        return n * (n + 1) * (2 * n + 1) // 6
    if eq_name == "lyapunov":
        return n * n * (n + 1)
    return 2 * n ** 3


def flops_nominal(eq_name, n):
    """Metric convention of BASELINE.json / PAPER.md:84-86."""
    if eq_name == "cholesky":
        return n ** 3 / 3.0
    return 2.0 * n ** 3


def bytes_compulsory(eq_name, n):
    """needed input triangles read once, full X written once."""
    tri = n * (n + 1) // 2
    if eq_name == "cholesky":
        return 8 * (tri + n * n)
    if eq_name == "lyapunov":
        return 8 * (tri + tri + n * n)
    return 8 * (tri + tri + n * n + n * n)
