"""Variant x block-size dispatch per (equation, n): the GPU analogue of the
reference's empirical selection `_select` (/root/reference/pkg/src/lagen/cli.py:175-181,
fastest median, ties broken by flops then id).

The table (dispatch_table.json) is written by tools/autotune.py from timings
of every (variant, b) on a B200; entries missing from it fall back to a
static choice.
"""

import json
from functools import lru_cache
from pathlib import Path

from .variants import default_blocks

TABLE = Path(__file__).with_name("dispatch_table.json")

# static fallback (right-looking / trailing-update variants, largest block)
_FALLBACK_VARIANT = {"cholesky": 2, "lyapunov": 5, "sylvester": 13}


@lru_cache(maxsize=None)
def _table():
    if TABLE.exists():
        return json.loads(TABLE.read_text())
    return {}


def reload():
    _table.cache_clear()


def select(eq_name, n):
    entry = _table().get(eq_name, {}).get(str(n))
    if entry is not None:
        return {"variant": int(entry["variant"]), "b": int(entry["b"]), "source": "autotune",
                "engine": entry.get("engine", "auto")}
    # sizes without an admissible reference block (n not a multiple of 4) run
    # as the identity-padded problem (lagen_b200.h); b = its largest divisor
    # of n from (8, 4, 2, 1) keeps the reference's b | n condition
    blocks = default_blocks(n) or [max(d for d in (8, 4, 2, 1) if n % d == 0)]
    return {"variant": _FALLBACK_VARIANT[eq_name], "b": max(blocks), "source": "fallback"}
