"""Build libpearl_b200.so (sm_100a) in-tree with nvcc.

    python -m paper_2408_11850_b200.build        # or __graft_entry__.build()

Every translation unit under csrc/ is compiled with
``-gencode arch=compute_100a,code=sm_100a -lineinfo -O3`` and linked into
``paper_2408_11850_b200/libpearl_b200.so``, which the package loads with
ctypes.  Objects are rebuilt only when a source or header is newer.
"""

from __future__ import annotations

import glob
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(REPO, "build", "obj")
LIB = os.path.join(PKG, "libpearl_b200.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O3",
                  "--expt-relaxed-constexpr", "-I", os.path.join(REPO, "include")]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: cannot build the sm_100a extension")


def _newest_header() -> float:
    hs = glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h"))
    hs += glob.glob(os.path.join(REPO, "include", "*.h"))
    return max((os.path.getmtime(h) for h in hs), default=0.0)


def build(verbose: bool = False, force: bool = False, defines=(), variant: str = "") -> str:
    """Build the library; ``defines`` / ``variant`` make a diagnostic build
    (e.g. ``-DPEARL_TIMELINE``) under build/var_<variant>/ that the package
    loads only through PEARL_LIB_PATH."""
    nvcc = _nvcc()
    obj_dir = os.path.join(REPO, "build", f"var_{variant}") if variant else OBJ
    lib = os.path.join(obj_dir, f"libpearl_{variant}.so") if variant else LIB
    os.makedirs(obj_dir, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))
    hdr_t = _newest_header()
    objs = []
    for src in srcs:
        obj = os.path.join(obj_dir, os.path.basename(src) + ".o")
        objs.append(obj)
        if (not force and os.path.exists(obj)
                and os.path.getmtime(obj) >= max(os.path.getmtime(src), hdr_t)):
            continue
        cmd = [nvcc, *NVFLAGS, *defines, "-c", src, "-o", obj]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    if force or not os.path.exists(lib) or os.path.getmtime(lib) < max(os.path.getmtime(o) for o in objs):
        cmd = [nvcc, *ARCH, "-shared", "-o", lib, *objs, "-lcuda"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    return lib


if __name__ == "__main__":
    if "--timeline" in sys.argv:  # diagnostic build for tools/timeline.py
        print(build(verbose="-v" in sys.argv, force="-f" in sys.argv, defines=("-DPEARL_TIMELINE",),
                    variant="tl"))
    elif "--variant" in sys.argv:  # --variant NAME -DX=Y ...: A/B builds loaded via PEARL_LIB_PATH
        i = sys.argv.index("--variant")
        print(build(verbose="-v" in sys.argv, force="-f" in sys.argv,
                    defines=tuple(a for a in sys.argv[i + 2:] if a.startswith("-D")), variant=sys.argv[i + 1]))
    else:
        print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
