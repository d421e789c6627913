"""Build libturbo.so (the C-ABI library, include/turbo.h) in-tree for sm_100a with nvcc."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
CHECKED = bool(os.environ.get("TURBO_CHECKS"))        # bounds-checked build (device TCHECK reports)
LIB = os.path.join(PKG, "checked", "libturbo.so") if CHECKED else os.path.join(PKG, "libturbo.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-O2",
    "-Xptxas", "-v",
    "--expt-relaxed-constexpr",
]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _flags() -> str:
    return " ".join(NVCC_FLAGS) + (" -DTURBO_TRACE" if os.environ.get("TURBO_TRACE") else "") + \
        (" -DTURBO_CHECKS" if CHECKED else "")


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    stamp = os.path.join(PKG, "build_checked" if CHECKED else "build", ".flags")
    if not os.path.exists(stamp) or open(stamp).read() != _flags():
        return True                       # built with other flags (e.g. the trace marks)
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(INCLUDE, "*.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src: str, obj: str):
    extra = ["-DTURBO_TRACE"] if os.environ.get("TURBO_TRACE") else []   # profiling build (trace marks)
    if CHECKED:
        extra.append("-DTURBO_CHECKS")
    cmd = [NVCC, *NVCC_FLAGS, *extra, "-I", INCLUDE, "-I", CSRC, "-c", "-o", obj, src]
    return subprocess.run(cmd, capture_output=True, text=True)


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile every csrc/*.cu to an object in parallel (one nvcc per file), link libturbo.so."""
    if not force and not _stale():
        return LIB
    from concurrent.futures import ThreadPoolExecutor
    objdir = os.path.join(PKG, "build_checked" if CHECKED else "build")
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    os.makedirs(objdir, exist_ok=True)
    srcs = sources()
    objs = [os.path.join(objdir, os.path.basename(s)[:-3] + ".o") for s in srcs]
    # incremental: an object is rebuilt when its source, any header, or the build flags changed
    headers = glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(INCLUDE, "*.h")) + [__file__]
    t_hdr = max(os.path.getmtime(h) for h in headers)
    stamp = os.path.join(objdir, ".flags")
    flags = _flags()
    same_flags = os.path.exists(stamp) and open(stamp).read() == flags
    todo = [i for i, (s, o) in enumerate(zip(srcs, objs))
            if force or not same_flags or not os.path.exists(o)
            or os.path.getmtime(o) < max(os.path.getmtime(s), t_hdr)]
    with ThreadPoolExecutor(max_workers=max(1, min(len(todo) or 1, os.cpu_count() or 1))) as ex:
        done = list(ex.map(_compile, [srcs[i] for i in todo], [objs[i] for i in todo]))
    with open(stamp, "w") as f:
        f.write(flags)
    results = {i: r for i, r in zip(todo, done)}
    log = []
    for i, s in enumerate(srcs):
        if i not in results:
            continue
        r = results[i]
        log.append(f"==== {os.path.basename(s)}\n{r.stdout}{r.stderr}")
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed on {s}")
    link = subprocess.run([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", LIB + ".tmp",
                           *objs], capture_output=True, text=True)
    if link.returncode != 0:
        sys.stderr.write(link.stdout + link.stderr)
        raise RuntimeError("nvcc link of libturbo.so failed")
    with open(os.path.join(objdir if CHECKED else PKG, "ptxas.log"), "a" if len(todo) < len(srcs) else "w") as f:
        f.write("\n".join(log))
    if verbose:
        sys.stderr.write("\n".join(log))
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
