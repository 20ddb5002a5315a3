"""In-tree build of the sm_100a C-ABI library `libhs_b200.so`.

    python paper_2404_11912_b200/build.py          # or __graft_entry__.build()

Compiles every `csrc/*.cu` with nvcc for `-gencode arch=compute_100a,code=sm_100a`
into one shared library next to this file (git-ignored, travels to the GPU box
with the gpurun snapshot).  Rebuilds only when a source or header is newer.
"""

from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(HERE, "libhs_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_root() -> str:
    """NCCL 2.28 shipped with torch (nvidia-nccl wheel); /usr/include has 2.27."""
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    for base in (spec.submodule_search_locations if spec else []):
        root = os.path.join(base, "nccl")
        if os.path.exists(os.path.join(root, "include", "nccl.h")):
            return root
    raise RuntimeError("nccl.h not found (expected the nvidia-nccl wheel next to torch)")


NCCL = _nccl_root()


FLAGS = ["-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC",
         "-Xptxas", "-O3"]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(INCLUDE, "*.h"))
    return any(os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    objdir = os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    objs = []
    extra = ["-Xptxas", "-v"] if verbose else []
    if os.environ.get("HS_TRACE_BUILD") == "1":   # per-CTA timeline (tools/cta_timeline.py); slower
        extra.append("-DHS_CTA_TRACE")
    extra += os.environ.get("HS_NVCC_DEFINES", "").split()   # experiment builds, e.g. "-DHS_TC_STAGES=4"
    cmds = []
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src).replace(".cu", ".o"))
        cmds.append([NVCC, *ARCH, *FLAGS, *extra, "-I", INCLUDE, "-I", CSRC, "-I", os.path.join(NCCL, "include"),
                     "-c", src, "-o", obj])
        objs.append(obj)
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=min(len(cmds), os.cpu_count() or 1)) as pool:
        for r in pool.map(lambda c: subprocess.run(c, check=True), cmds):
            pass
    tmp = LIB + ".tmp"
    nccl_lib = os.path.join(NCCL, "lib")
    subprocess.run([NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-lcudart", "-L", nccl_lib, "-l:libnccl.so.2",
                    "-Xlinker", "-rpath," + nccl_lib], check=True)
    # every hs:: symbol must resolve inside the library (a declaration that
    # drifted from its definition links as an undefined symbol and only fails
    # at dlopen on the GPU box)
    und = subprocess.run(["nm", "-u", "-C", tmp], capture_output=True, text=True).stdout.splitlines()
    bad = [u.strip() for u in und if "hs::" in u]
    if bad:
        os.remove(tmp)
        raise RuntimeError("unresolved library-internal symbols: " + "; ".join(bad))
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
