"""Build oracle/_ref: the REFERENCE's own CPU path, compiled.

The reference's CPU kernels are not shipped as source: `lagen` emits them
at run time (`emit_function(build_program(cfg, n))`,
/root/reference/pkg/src/lagen/codegen.py:155-201 and cli.py:123-128, plus the
nu micro-kernel header codegen.py:208-310).  This script runs that emitter
(in the build container, where /root/reference is importable) and writes

  oracle/_ref/src/ref_<eq>_n<n>.c   the emitted kernels, one TU per (eq, n)
  oracle/_ref/src/nu_kernels_4.h    the emitted nu = 4 micro-kernel header
  oracle/_ref/src/ref_driver.c      a batch driver (ours): OpenMP over problems
  oracle/_ref/manifest.json         kernels, parameters, verification status

Every emitted kernel is compiled here once and checked against the
reference interpreter (verify.interpret_algorithm) on one random instance;
kernels that disagree (the nu-Lyapunov gather defect) are
marked unverified and never used.  `compile_lib()` builds the shared
library with the reference's test flags `gcc -O3 -march=native -std=c99`
(pkg/tests/test_acceptance.py:261-263) on whatever host runs it:
the build directory is keyed by the host's CPU model + ISA flags + gcc version
(host_tag), so a GPU box whose CPU differs from the build container's
recompiles for its own CPU on first use (~15 s on 8 cores).  Nothing here is copied from the
reference sources: the .c files are the reference program's output.

TEST / BASELINE INFRASTRUCTURE ONLY (bench.py cpu_baseline and
--impl reference; tests).  The product never loads it.
"""

import ctypes
import hashlib
import json
import os
import platform
import subprocess
import sys
import tempfile
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF = HERE / "_ref"
SRC = REF / "src"
MANIFEST = REF / "manifest.json"

SIZES = list(range(4, 129, 4))
# candidate (variant, b, mode) per equation: the variants `lagen tune` picked
# on CPU during the survey plus neighbours; b = 16 only where it
# is a default block (16 | n, 16 < n)
# ("the fastest by batch timing among scalar variants and those nu
# variants that match interpret_algorithm on a sample" — both modes are
# emitted; bench.py times every verified candidate of a size and keeps the
# fastest)
CANDIDATES = {
    "cholesky": [(1, 4, "nu"), (2, 4, "nu"), (2, 16, "nu"), (1, 16, "nu"),
                 (1, 4, "scalar"), (2, 4, "scalar"), (1, 8, "scalar")],
    "lyapunov": [(1, 4, "nu"), (2, 4, "nu"), (4, 4, "nu"), (5, 4, "nu"),
                 (5, 4, "scalar"), (1, 8, "scalar")],
    "sylvester": [(0, 4, "nu"), (3, 4, "nu"), (11, 4, "nu"), (12, 16, "nu"),
                  (13, 4, "scalar"), (0, 8, "scalar")],
}
CASE_FILES = {"cholesky": "cholesky.la", "lyapunov": "lyapunov.la", "sylvester": "sylvester.la"}
EQ_CODES = {"cholesky": 0, "lyapunov": 1, "sylvester": 2}
NIN = {"cholesky": 1, "lyapunov": 2, "sylvester": 3}


def _gomp_flags():
    for d in sorted(Path("/usr/lib/gcc/x86_64-linux-gnu").glob("*/libgomp.spec")):
        return ["-fopenmp", f"-B{d.parent}"]
    return []


DRIVER = r"""
/* Batch driver for the reference's emitted kernels (ours, not emitted).
 * The emitted contract: X zero-initialised by the caller, row-major, ld = n
 * (codegen.py:4-7).  Problems are independent: OpenMP static schedule. */
#include <string.h>
#include <stddef.h>
#ifdef _OPENMP
#include <omp.h>
#endif
typedef void (*k1)(const double*, double*);
typedef void (*k2)(const double*, const double*, double*);
typedef void (*k3)(const double*, const double*, const double*, double*);
struct ref_kernel { int eq, n, variant, b; const char* name; void* fn; };
extern const struct ref_kernel ref_kernels[];
extern const int ref_num_kernels;

int ref_count(void) { return ref_num_kernels; }
int ref_info(int idx, int* eq, int* n, int* variant, int* b) {
  if (idx < 0 || idx >= ref_num_kernels) return -1;
  *eq = ref_kernels[idx].eq; *n = ref_kernels[idx].n;
  *variant = ref_kernels[idx].variant; *b = ref_kernels[idx].b;
  return 0;
}
const char* ref_name(int idx) { return (idx >= 0 && idx < ref_num_kernels) ? ref_kernels[idx].name : ""; }

int ref_run(int idx, long long batch, const double* const* in, double* X, int nthreads) {
  if (idx < 0 || idx >= ref_num_kernels) return -1;
  const struct ref_kernel* k = &ref_kernels[idx];
  const long long nn = (long long)k->n * k->n;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#else
  (void)nthreads;
#endif
#pragma omp parallel for schedule(static)
  for (long long p = 0; p < batch; ++p) {
    double* x = X + p * nn;
    if (k->eq == 0) {
      memset(x, 0, sizeof(double) * (size_t)nn);
      ((k1)k->fn)(in[0] + p * nn, x);
    } else if (k->eq == 1) {
      ((k2)k->fn)(in[0] + p * nn, in[1] + p * nn, x);
    } else {
      ((k3)k->fn)(in[0] + p * nn, in[1] + p * nn, in[2] + p * nn, x);
    }
  }
  return 0;
}
"""


def generate(reference=None):
    """Emit all candidate kernels with the reference generator; verify them."""
    reference = Path(reference or os.environ.get("LAGEN_REFERENCE", "/root/reference"))
    sys.path.insert(0, str(reference / "pkg" / "src"))
    from lagen.cli import VariantConfig, build_program
    from lagen.codegen import emit_function, emit_nu_kernel_header
    from lagen.lang import parse_equation
    from lagen.verify import interpret_algorithm, random_instance
    from lagen.worksheet import enumerate_algorithms

    SRC.mkdir(parents=True, exist_ok=True)
    (SRC / "nu_kernels_4.h").write_text(emit_nu_kernel_header(4).text)
    (SRC / "ref_driver.c").write_text(DRIVER)
    kernels = []
    for eq_name, fname in CASE_FILES.items():
        eq = parse_equation((reference / "pkg" / "cases" / fname).read_text(), name=eq_name)
        algs = enumerate_algorithms(eq)
        for n in SIZES:
            parts = ["#include <math.h>", '#include "nu_kernels_4.h"', ""]
            for v, b, mode in CANDIDATES[eq_name]:
                if n % b or (b >= n and n != b) or (b == 16 and not (16 < n)):
                    continue
                cfg = VariantConfig(algs[v], v, b, b, mode, 4 if mode == "nu" else None)
                fn = emit_function(build_program(cfg, n))
                cname = f"ref_{fn.name}_{mode}"
                body = fn.text.replace(f"void {fn.name}(", f"void {cname}(")
                body = "\n".join(l for l in body.splitlines() if not l.startswith("#include"))
                parts.append(body)
                kernels.append({"eq": eq_name, "n": n, "variant": v, "b": b, "mode": mode,
                                "name": cname, "file": f"ref_{eq_name}_n{n}.c"})
            (SRC / f"ref_{eq_name}_n{n}.c").write_text("\n".join(parts) + "\n")
    _write_table(kernels)
    # verify every kernel against the reference interpreter
    lib_path = compile_lib(opt=["-O1"], tag="verify")
    lib = ctypes.CDLL(str(lib_path))
    _bind(lib)
    cache = {}
    for idx, k in enumerate(kernels):
        eq_name = k["eq"]
        if eq_name not in cache:
            eq = parse_equation((reference / "pkg" / "cases" / CASE_FILES[eq_name]).read_text(), name=eq_name)
            cache[eq_name] = (eq, enumerate_algorithms(eq))
        eq, algs = cache[eq_name]
        inst = random_instance(eq, k["n"], seed=19)
        want, _ = interpret_algorithm(algs[k["variant"]], inst, k["b"])
        names = [op.name for op in eq.operands if not op.is_output]
        ins = [np.ascontiguousarray(inst.bindings[nm])[None] for nm in names]
        X = _run(lib, idx, ins, k["n"], 1)
        err = float(np.max(np.abs(X[0] - want["X"])) / max(1.0, np.max(np.abs(want["X"]))))
        k["max_rel_err_vs_interpreter"] = err
        k["verified"] = bool(err <= 1e-12)
    MANIFEST.write_text(json.dumps({"kernels": kernels, "flags": "gcc -O3 -march=native -std=c99",
                                    "emitter": "lagen 0.1.0 emit_function(build_program(cfg, n))"},
                                   indent=1) + "\n")
    bad = [k["name"] for k in kernels if not k["verified"]]
    print(f"emitted {len(kernels)} kernels; unverified: {bad}")
    return kernels


def _write_table(kernels):
    lines = ["#include <stddef.h>",
             "struct ref_kernel { int eq, n, variant, b; const char* name; void* fn; };"]
    for k in kernels:
        nin = NIN[k["eq"]]
        args = ", ".join(["const double*"] * nin + ["double*"])
        lines.append(f"void {k['name']}({args});")
    lines.append("const struct ref_kernel ref_kernels[] = {")
    for k in kernels:
        lines.append(f"  {{{EQ_CODES[k['eq']]}, {k['n']}, {k['variant']}, {k['b']}, \"{k['name']}\", "
                     f"(void*){k['name']}}},")
    lines.append("};")
    lines.append(f"const int ref_num_kernels = {len(kernels)};")
    (SRC / "ref_table.c").write_text("\n".join(lines) + "\n")


def host_tag():
    """Key of the -march=native build: the CPU's model AND its ISA flags (two
    hosts can report the same model string with different feature sets, e.g.
    "Intel(R) Xeon(R) Processor" in VMs), plus the compiler version."""
    cpu = [platform.processor() or ""]
    try:
        seen = set()
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            key = line.split(":", 1)[0].strip()
            if key in ("model name", "flags") and key not in seen:
                seen.add(key)
                cpu.append(" ".join(sorted(line.split(":", 1)[1].split())) if key == "flags"
                           else line.split(":", 1)[1].strip())
    except OSError:
        pass
    try:
        cpu.append(subprocess.run(["gcc", "-dumpfullversion"], capture_output=True, text=True).stdout.strip())
    except OSError:
        pass
    return hashlib.sha1("|".join(cpu).encode()).hexdigest()[:10]


def lib_path(tag=None):
    return REF / f"build-{tag or host_tag()}" / "libref.so"


def compile_lib(opt=("-O3", "-march=native"), tag=None, jobs=None):
    """Compile oracle/_ref/src into a shared library for THIS host."""
    out = lib_path(tag)
    srcs = sorted(SRC.glob("*.c"))
    if not srcs:
        raise FileNotFoundError("oracle/_ref/src is empty: run oracle/build_ref.py where the reference exists")
    if out.exists() and out.stat().st_mtime >= max(s.stat().st_mtime for s in srcs):
        return out
    out.parent.mkdir(parents=True, exist_ok=True)
    objdir = out.parent / "obj"
    objdir.mkdir(exist_ok=True)
    omp = _gomp_flags()

    def cc(src):
        obj = objdir / (src.stem + ".o")
        cmd = ["gcc", *opt, "-std=c99", "-fPIC", *omp, f"-I{SRC}", "-c", str(src), "-o", str(obj)]
        subprocess.run(cmd, check=True, capture_output=True)
        return obj

    with ThreadPoolExecutor(jobs or os.cpu_count() or 4) as ex:
        objs = list(ex.map(cc, srcs))
    tmp = out.with_suffix(".tmp")
    subprocess.run(["gcc", "-shared", *omp, "-o", str(tmp), *map(str, objs), "-lm"], check=True)
    os.replace(tmp, out)
    return out


def _bind(lib):
    lib.ref_run.argtypes = [ctypes.c_int, ctypes.c_longlong, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
    lib.ref_info.argtypes = [ctypes.c_int] + [ctypes.POINTER(ctypes.c_int)] * 4
    lib.ref_name.restype = ctypes.c_char_p


def _run(lib, idx, ins, n, nthreads):
    batch = ins[0].shape[0]
    X = np.empty((batch, n, n))
    ptrs = (ctypes.c_void_p * 3)(*([a.ctypes.data for a in ins] + [0] * (3 - len(ins))))
    rc = lib.ref_run(idx, batch, ctypes.addressof(ptrs), X.ctypes.data, nthreads)
    if rc:
        raise RuntimeError("ref_run failed")
    return X


class RefLib:
    """The compiled reference CPU path (emitted kernels + OpenMP batch driver)."""

    def __init__(self, path=None):
        self.path = Path(path) if path else compile_lib()
        self.lib = ctypes.CDLL(str(self.path))
        _bind(self.lib)
        self.manifest = json.loads(MANIFEST.read_text())["kernels"]

    def kernels(self, eq, n):
        return [(i, k) for i, k in enumerate(self.manifest)
                if k["eq"] == eq and k["n"] == n and k.get("verified")]

    def run(self, idx, ins, nthreads=None):
        n = self.manifest[idx]["n"]
        return _run(self.lib, idx, [np.ascontiguousarray(a) for a in ins], n,
                    nthreads or len(os.sched_getaffinity(0)))


def available():
    return MANIFEST.exists() and (SRC / "ref_driver.c").exists()


if __name__ == "__main__":
    generate(sys.argv[1] if len(sys.argv) > 1 else None)
    print(compile_lib())
