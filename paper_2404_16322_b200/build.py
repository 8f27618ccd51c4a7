"""Build libdade.so in-tree with nvcc for sm_100a (no GPU needed: nvcc cross-compiles).

Each translation unit is compiled to an object in parallel (build/obj/), then linked; a unit is
recompiled only when it or a header is newer than its object."""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libdade.so")
OBJ = os.path.join(HERE, "build", "obj")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
INC = os.path.join(HERE, "..", "include")
FLAGS = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-I", INC]


def sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cu", ".cpp")))


def headers():
    h = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    h.append(os.path.join(INC, "dade.h"))
    return h


def _obj(src: str, extra=()) -> str:
    d = OBJ if not extra else OBJ + "_" + "_".join(e.strip("-").replace("=", "") for e in extra)
    return os.path.join(d, os.path.basename(src) + ".o")


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(d) > t for d in sources() + headers())


def _compile(src: str, verbose: bool, extra: list) -> tuple:
    o = _obj(src, extra)
    cmd = [NVCC, *FLAGS, *extra, *(["-Xptxas", "-v"] if verbose else []), "-c", src, "-o", o + ".tmp"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode == 0:
        os.replace(o + ".tmp", o)
    return src, r


def build(force: bool = False, verbose: bool = False, extra: list | None = None, out: str | None = None) -> str:
    """Compile every csrc/ unit for sm_100a and link libdade.so (or `out` with `extra` nvcc flags,
    e.g. an experiment build)."""
    extra = list(extra or [])
    lib = out or LIB
    if not force and not extra and out is None and not stale():
        return LIB
    os.makedirs(os.path.dirname(_obj("x", extra)), exist_ok=True)
    hdr_t = max(os.path.getmtime(h) for h in headers())
    todo = [s for s in sources()
            if force or not os.path.exists(_obj(s, extra))
            or os.path.getmtime(_obj(s, extra)) < max(os.path.getmtime(s), hdr_t)]
    with ThreadPoolExecutor(max_workers=min(len(todo), os.cpu_count() or 4) or 1) as ex:
        res = list(ex.map(lambda s: _compile(s, verbose, extra), todo))
    failed = [(s, r) for s, r in res if r.returncode != 0]
    for s, r in res:
        if verbose or r.returncode != 0:
            sys.stderr.write(f"== {os.path.basename(s)}\n{r.stdout}{r.stderr}")
    if failed:
        raise RuntimeError("nvcc failed: " + ", ".join(os.path.basename(s) for s, _ in failed))
    cmd = [NVCC, *ARCH, "-shared", "-o", lib + ".tmp", *[_obj(s, extra) for s in sources()], "-lcudart", "-ldl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc link failed")
    os.replace(lib + ".tmp", lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
