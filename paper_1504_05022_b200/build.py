"""Build libspgemm.so in-tree with nvcc for sm_100a (no JIT, no torch extension).

    python -m paper_1504_05022_b200.build            # incremental
    python -m paper_1504_05022_b200.build --force    # rebuild everything

Each csrc/*.cu is compiled to an object in build/ (in parallel), then linked into
paper_1504_05022_b200/libspgemm.so against the NCCL that torch itself loads
(site-packages/nvidia/nccl), so one libnccl.so.2 lives in the process.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(ROOT, "build")
LIB = os.path.join(PKG, "libspgemm.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_dirs():
    try:
        import nvidia.nccl  # noqa: F401
        base = list(nvidia.nccl.__path__)[0]
        inc, lib = os.path.join(base, "include"), os.path.join(base, "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc, lib
    except Exception:
        pass
    return "/usr/include", "/usr/lib/x86_64-linux-gnu"


def _deps():
    hdrs = glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(ROOT, "include", "*.h"))
    return max((os.path.getmtime(h) for h in hdrs), default=0.0)


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    inc, libdir = _nccl_dirs()
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    hdr_t = _deps()
    flags = ["-O3", "-std=c++17", *ARCH, "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-O3",
             "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include"), "-I", inc]
    if os.environ.get("SPGEMM_PTXAS_V"):
        flags += ["-Xptxas", "-v"]
    if os.environ.get("SPGEMM_DEFS"):  # development A/B builds: extra -D definitions
        flags += ["-D" + d for d in os.environ["SPGEMM_DEFS"].split()]

    def one(src):
        obj = os.path.join(BUILD, os.path.basename(src)[:-3] + ".o")
        if not force and os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(src), hdr_t):
            return obj, False, ""
        cmd = [NVCC, *flags, "-c", src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("nvcc failed for %s:\n%s\n%s" % (src, r.stdout, r.stderr))
        return obj, True, r.stderr

    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        res = list(ex.map(one, srcs))
    objs = [o for o, _, _ in res]
    if verbose:
        for _, _, err in res:
            if err:
                sys.stderr.write(err)
    rebuilt = any(b for _, b, _ in res)
    if force or rebuilt or not os.path.exists(LIB):
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB + ".tmp", *objs, "-L", libdir, "-l:libnccl.so.2",
               "-Xlinker", "-rpath=" + libdir]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("link failed:\n%s\n%s" % (r.stdout, r.stderr))
        os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
