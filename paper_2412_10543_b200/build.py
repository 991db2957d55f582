"""Build the CUDA library in-tree: ``paper_2412_10543_b200/libragsched_b200.so``.

One nvcc invocation per translation unit (parallel), linked with a static
cudart.  sm_100a only: ``-gencode arch=compute_100a,code=sm_100a`` (tcgen05,
TMEM and TMA are arch-specific features).  Run ``python -m
paper_2412_10543_b200.build`` or ``__graft_entry__.build()``.
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(ROOT, "include")
OBJ = os.path.join(HERE, "_obj")
LIB = os.path.join(HERE, "libragsched_b200.so")
SOURCES = ["abi.cu", "select.cu", "gate.cu", "plan.cu", "retrieval.cu", "score_topk_sm100.cu", "score_topk_sm100_pair.cu",
           "parse.cpp", "costs.cu", "peer.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _flags():
    return [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
            "--expt-relaxed-constexpr", f"-I{INCLUDE}", f"-I{CSRC}",
            "-ccbin", "/usr/bin/g++"]


def _deps(src):
    hdrs = [os.path.join(CSRC, h) for h in os.listdir(CSRC) if h.endswith((".cuh", ".h"))]
    hdrs.append(os.path.join(INCLUDE, "ragsched_b200.h"))
    return [os.path.join(CSRC, src), *hdrs]


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src, verbose, objdir=None, defines=()):
    objdir = objdir or OBJ
    obj = os.path.join(objdir, os.path.splitext(src)[0] + ".o")
    if not _stale(obj, _deps(src)):
        return obj, ""
    cmd = [nvcc(), *_flags(), *[f"-D{d}" for d in defines], "-c", os.path.join(CSRC, src), "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    return obj, r.stderr


def build(verbose: bool = False, force: bool = False, *, defines=(), out: str | None = None) -> str:
    """Build the library.  ``defines``/``out`` build a tuning variant (e.g.
    ``RS_PAIR_EPI_COLS=64``) into its own object dir and .so, selected at
    run time with ``RAGSCHED_B200_LIB=<path>``."""
    lib = out or LIB
    objdir = OBJ if not defines else os.path.join(OBJ, "_".join(d.replace("=", "") for d in defines))
    os.makedirs(objdir, exist_ok=True)
    if force:
        for f in os.listdir(objdir):
            p = os.path.join(objdir, f)
            if os.path.isfile(p):
                os.remove(p)
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        results = list(ex.map(lambda s: _compile(s, verbose, objdir, defines), SOURCES))
    objs = [o for o, _ in results]
    if verbose:
        for _, log in results:
            if log:
                sys.stderr.write(log)
    if force or _stale(lib, objs):
        cmd = [nvcc(), *ARCH, "-shared", "-cudart", "static", "-ccbin", "/usr/bin/g++", *objs, "-o", lib]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return lib


if __name__ == "__main__":
    defs = [a[2:] for a in sys.argv[1:] if a.startswith("-D")]
    outs = [a[6:] for a in sys.argv[1:] if a.startswith("--out=")]
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv, defines=defs, out=outs[0] if outs else None))
