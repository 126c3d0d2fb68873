"""Build libchessfad.so in-tree with nvcc for sm_100a (no JIT cache, no torch extension).

Each translation unit in csrc/ is compiled in parallel (-gencode arch=compute_100a,
code=sm_100a -O3 -lineinfo), ptxas register/spill reports go to build/ptxas_<unit>.log,
and the objects are linked with -shared into paper_2410_22575_b200/libchessfad.so.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(ROOT, "build")
LIB = os.path.join(HERE, "libchessfad.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
              "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include")]


def _nvcc():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    return "nvcc"


def source_hash() -> str:
    """sha256 over the CUDA sources, the header and the compile flags: identifies the SASS
    that the ncu-measured executed-FLOP table (profiles/executed_flops.json) describes."""
    import hashlib
    h = hashlib.sha256()
    for f in sorted(glob.glob(os.path.join(CSRC, "*.cu*"))) + _public_headers():
        h.update(os.path.basename(f).encode())
        h.update(open(f, "rb").read())
    h.update(" ".join(ARCH + NVCC_FLAGS[:-2]).encode())
    return h.hexdigest()[:16]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _public_headers():
    inc = os.path.join(ROOT, "include")
    return [os.path.join(inc, "chessfad.h")] + sorted(glob.glob(os.path.join(inc, "chessfad", "*.cuh")))


def _deps():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu*"))) + _public_headers() + [__file__]


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(d) <= t for d in _deps())


def _compile(src: str, defines=(), tag: str = "") -> str:
    name = os.path.splitext(os.path.basename(src))[0] + tag
    obj = os.path.join(BUILD, name + ".o")
    cmd = [_nvcc(), *ARCH, *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    with open(os.path.join(BUILD, f"ptxas_{name}.log"), "w") as f:
        f.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr[-6000:]}")
    return obj


def build(force: bool = False, jobs: int | None = None, defines=(), out: str | None = None) -> str:
    """Build the library; `defines`/`out` build an experimental variant elsewhere (tuning).
    Serialised across processes by an fcntl lock on build/.lock (concurrent ranks would
    otherwise write the same object files); a process that waited re-checks staleness."""
    if not force and not defines and out is None and up_to_date():
        return LIB
    import fcntl
    os.makedirs(BUILD, exist_ok=True)
    with open(os.path.join(BUILD, ".lock"), "w") as lk:
        fcntl.flock(lk, fcntl.LOCK_EX)
        if not force and not defines and out is None and up_to_date():
            return LIB
        return _build_locked(jobs, defines, out)


def _build_locked(jobs, defines, out) -> str:
    srcs = sources()
    tag = "_" + "_".join(d.replace("=", "") for d in defines) if defines else ""
    with cf.ThreadPoolExecutor(max_workers=jobs or min(len(srcs), os.cpu_count() or 4)) as ex:
        objs = list(ex.map(lambda f: _compile(f, defines, tag), srcs))
    target = out or LIB
    tmp = target + f".tmp{os.getpid()}"
    cmd = [_nvcc(), *ARCH, "-shared", "-o", tmp, *objs, "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr[-4000:]}")
    os.replace(tmp, target)
    try:  # per-kernel SASS fingerprints, cached next to the library (sass.py)
        from . import sass as _sass
    except ImportError:
        import sass as _sass  # run as a script
    _sass.kernel_sass_hashes.cache_clear()
    _sass.kernel_sass_hashes(target)
    return target


if __name__ == "__main__":
    defs = [a[2:] for a in sys.argv[1:] if a.startswith("-D")]
    outp = next((a.split("=", 1)[1] for a in sys.argv[1:] if a.startswith("--out=")), None)
    print(build(force="--force" in sys.argv, defines=defs, out=outp))
