"""Builds the product library paper_2603_06101_b200/libsbg.so (sm_100a only) with nvcc.

    python -m paper_2603_06101_b200.build [--verbose-ptxas]

Objects go to build/ (git-ignored); the .so lands in-tree next to this file so it travels to the
GPU box with the repo snapshot. tables.cu is compiled with --fmad=false (bit-exact diagonal).
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
# developer knobs for A/B builds: SBG_NVCC_FLAGS (extra nvcc flags), SBG_LIB_OUT (library path)
EXTRA = os.environ.get("SBG_NVCC_FLAGS", "").split()
LIB = os.environ.get("SBG_LIB_OUT", os.path.join(PKG, "libsbg.so"))
OBJ = os.path.join(ROOT, "build", "sbg" if not EXTRA else "sbg_" + str(abs(hash(" ".join(EXTRA)))))
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
         "--expt-relaxed-constexpr", "-I" + os.path.join(ROOT, "include")]
SOURCES = ["tables.cu", "sigma_ab.cu", "sigma_ss.cu", "vec.cu", "selftest.cu", "context.cu", "solver.cu", "sbci2.cu",
           "davidson.cu", "spin.cu", "step_scalars.cu", "api.cu"]
# bit-exact with the reference / the host: no FMA contraction in the diagonal and the step scalars
PER_FILE = {"tables.cu": ["--fmad=false"], "step_scalars.cu": ["--fmad=false"]}


def nvcc():
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def nccl_link():
    """Link the NCCL that PyTorch ships (nvidia-nccl wheel, 2.28) when present, else the system one.
    Both arrive as soname libnccl.so.2 in one process: whichever loads first serves both, so libsbg
    must bind the newer one or a later `import torch` fails on symbols 2.27 lacks."""
    try:
        import nvidia.nccl
        d = os.path.join(list(nvidia.nccl.__path__)[0], "lib")
        if os.path.exists(os.path.join(d, "libnccl.so.2")):
            return ["-L" + d, "-l:libnccl.so.2", "-Xlinker", "-rpath," + d]
    except ImportError:
        pass
    return ["-lnccl", "-Xlinker", "-rpath,/usr/lib/x86_64-linux-gnu"]


def _headers_mtime():
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".hpp", ".h"))]
    hs.append(os.path.join(ROOT, "include", "sbg.h"))
    return max(os.path.getmtime(h) for h in hs)


def _compile(src, ptxas_verbose, force=True):
    out = os.path.join(OBJ, src.replace(".cu", ".o"))
    # incremental: an object newer than its source and every header is kept
    if (not force and not ptxas_verbose and os.path.exists(out)
            and os.path.getmtime(out) > max(os.path.getmtime(os.path.join(CSRC, src)), _headers_mtime())):
        return out, ""
    cmd = [nvcc(), *ARCH, *FLAGS, *EXTRA, *PER_FILE.get(src, []), "-c", os.path.join(CSRC, src), "-o", out]
    if ptxas_verbose:
        cmd += ["-Xptxas", "-v"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
    return out, r.stderr


def build(ptxas_verbose=False, force=False):
    os.makedirs(OBJ, exist_ok=True)
    newest_src = max(os.path.getmtime(os.path.join(CSRC, f)) for f in os.listdir(CSRC))
    newest_src = max(newest_src, os.path.getmtime(os.path.join(ROOT, "include", "sbg.h")))
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) > newest_src and not ptxas_verbose:
        return LIB
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        results = list(ex.map(lambda s: _compile(s, ptxas_verbose, force), SOURCES))
    if ptxas_verbose:
        for _, err in results:
            sys.stderr.write(err)
    objs = [o for o, _ in results]
    cmd = [nvcc(), *ARCH, "-shared", "-o", LIB + ".tmp", *objs, *nccl_link()]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("link failed:\n" + r.stderr)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(ptxas_verbose="--verbose-ptxas" in sys.argv, force="--force" in sys.argv))
