"""Build the sm_100a kernel library in-tree (no JIT cache, so it travels with
the repo snapshot to the GPU box).

    python -m paper_1906_08613_b200.build        # incremental
    python -m paper_1906_08613_b200.build --force

Produces paper_1906_08613_b200/lib/liblagen_b200.so: every .cu under csrc/
compiled with `nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3`
and linked against the static CUDA runtime.  The C ABI is include/lagen_b200.h.
"""

import argparse
import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
REPO = PKG.parent
CSRC = PKG / "csrc"
INCLUDE = REPO / "include"
OBJ = PKG / "lib" / "obj"
LIB = PKG / "lib" / "liblagen_b200.so"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++20", "-Xcompiler", "-fPIC,-O2",
              "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills"]


def nvcc():
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found: cannot build the sm_100a kernel library")


def _headers():
    return list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h")) + list(INCLUDE.glob("*.h"))


def _stale(target, deps):
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def _deps(src, obj, headers):
    """Headers src includes, from the nvcc -MD file of its last compile (all
    headers when unknown)."""
    dfile = obj.with_suffix(".d")
    if not dfile.exists():
        return headers
    text = dfile.read_text().replace("\\\n", " ")
    names = text.split(":", 1)[1].split() if ":" in text else []
    deps = [Path(n) for n in names if n.endswith((".cuh", ".h")) and str(REPO) in str(Path(n).resolve())]
    return [d for d in deps if d.exists()] + [h for h in headers if h.name == "lagen_b200.h"]


def build(force=False, verbose=False, jobs=None):
    sources = sorted(CSRC.glob("*.cu"))
    if not sources:
        raise RuntimeError(f"no CUDA sources under {CSRC}")
    OBJ.mkdir(parents=True, exist_ok=True)
    headers = _headers()
    todo = []
    objs = []
    for src in sources:
        obj = OBJ / (src.stem + ".o")
        objs.append(obj)
        if force or _stale(obj, [src] + _deps(src, obj, headers)):
            todo.append((src, obj))
    cc = nvcc()

    def compile_one(item):
        src, obj = item
        cmd = [cc, *ARCH, *NVCC_FLAGS, *os.environ.get("LAGEN_NVCC_EXTRA", "").split(), f"-I{INCLUDE}", f"-I{CSRC}", "-MD", "-MF", str(obj.with_suffix(".d")),
               "-c", str(src), "-o", str(obj)]
        proc = subprocess.run(cmd, capture_output=True, text=True)
        if proc.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src.name}:\n{proc.stderr}")
        if verbose and proc.stderr.strip():
            print(proc.stderr, file=sys.stderr)
        return src.name

    if todo:
        jobs = jobs or max(1, min(len(todo), os.cpu_count() or 4))
        with ThreadPoolExecutor(jobs) as ex:
            for name in ex.map(compile_one, todo):
                if verbose:
                    print("compiled", name)
    if force or todo or _stale(LIB, objs):
        tmp = LIB.with_suffix(".so.tmp")
        cmd = [cc, *ARCH, "-shared", "-cudart", "static", "-o", str(tmp), *map(str, objs)]
        proc = subprocess.run(cmd, capture_output=True, text=True)
        if proc.returncode != 0:
            raise RuntimeError(f"link failed:\n{proc.stderr}")
        os.replace(tmp, LIB)
    return LIB


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", "--verbose", action="store_true")
    args = ap.parse_args()
    print(build(force=args.force, verbose=args.verbose))


if __name__ == "__main__":
    main()
