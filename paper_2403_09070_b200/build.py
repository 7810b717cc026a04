"""Build libp3d.so in-tree with nvcc for sm_100a (no JIT, no torch extension).

Translation units whose arithmetic must round exactly like numpy (density
overlaps, the optimiser) are compiled with ``-fmad=false``; the others keep FMA
contraction.  Object files are rebuilt only when a source or header changed,
or when the nvcc flags differ from the ones the object dir was built with
(a flags stamp in the object dir).
"""

from __future__ import annotations

import concurrent.futures as cf
import hashlib
import os
import shutil
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")
OBJDIR = os.path.join(HERE, "build")
LIB = os.path.join(HERE, "libp3d.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
          "--expt-relaxed-constexpr", "-I", CSRC, "-I", INCLUDE]
NO_FMA = {"p3d_density.cu", "p3d_loop.cu", "p3d_gp2d.cu", "p3d_score.cu", "p3d_post.cu", "p3d_ops.cu"}
SOURCES = ["p3d_api.cu", "p3d_wl.cu", "p3d_wl_fused.cu", "p3d_density.cu", "p3d_spectral.cu", "p3d_spectral_fast.cu", "p3d_loop.cu", "p3d_gp2d.cu", "p3d_score.cu", "p3d_post.cu", "p3d_ops.cu", "p3d_parse.cu"]


def _nvcc():
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.isabs(c) and os.path.exists(c) or not os.path.isabs(c)):
            return c
    return "nvcc"


def _headers():
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    hs.append(os.path.join(INCLUDE, "p3d.h"))
    return max(os.path.getmtime(h) for h in hs)


def _compile(src, extra, objdir=OBJDIR):
    obj = os.path.join(objdir, src.replace(".cu", ".o"))
    path = os.path.join(CSRC, src)
    if os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(path), _headers()):
        return obj, None
    cmd = [_nvcc(), *ARCH, *COMMON, *extra, "-c", path, "-o", obj]
    if src in NO_FMA:
        cmd.insert(1, "-fmad=false")
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}\n{r.stdout}")
    return obj, r.stderr


def build(verbose=False, extra=(), variant=""):
    """Build libp3d.so; with `variant`, an A/B copy libp3d_<variant>.so built
    with the `extra` nvcc flags (e.g. -D switches) in its own object dir."""
    objdir = OBJDIR + (f"_{variant}" if variant else "")
    lib_path = LIB if not variant else os.path.join(HERE, f"libp3d_{variant}.so")
    stamp = hashlib.sha256(" ".join([_nvcc(), *ARCH, *COMMON, *extra, "|", *sorted(NO_FMA)])
                           .encode()).hexdigest()
    stamp_path = os.path.join(objdir, "FLAGS")
    if os.path.isdir(objdir) and (not os.path.exists(stamp_path) or
                                  open(stamp_path).read().strip() != stamp):
        shutil.rmtree(objdir)  # built with other flags (e.g. -D switches): rebuild all
    os.makedirs(objdir, exist_ok=True)
    with open(stamp_path, "w") as fh:
        fh.write(stamp + "\n")
    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        results = list(ex.map(lambda s: _compile(s, list(extra), objdir), SOURCES))
    objs = [o for o, _ in results]
    if verbose:
        for o, log in results:
            if log:
                print(o, log)
    if not os.path.exists(lib_path) or os.path.getmtime(lib_path) < max(os.path.getmtime(o) for o in objs):
        cmd = [_nvcc(), *ARCH, "-shared", "-o", lib_path, *objs]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc link failed:\n{r.stderr}")
    return lib_path


if __name__ == "__main__":
    import sys
    print(build(verbose=True, extra=sys.argv[1:]))
