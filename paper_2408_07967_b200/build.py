"""In-tree build of libflashgs_b200.so with nvcc for sm_100a.

    python -m paper_2408_07967_b200.build [--force]

The shared library is the C-ABI product (include/flashgs_b200.h).  It is
built next to the sources so it travels with the repo snapshot to the GPU box;
it is git-ignored.  No fallback exists: without this library the package
raises at first use.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT_DIR = os.path.join(HERE, "_lib")
LIB = os.path.join(OUT_DIR, "libflashgs_b200.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC"]
# (file, extra flags).  The preprocess unit must keep every float32 operation
# individually rounded (bit-exact pair lists), hence -fmad=false on top of the
# explicit _rn intrinsics it uses.
UNITS = [
    ("fgs_preprocess.cu", ["-fmad=false", "-prec-div=true", "-prec-sqrt=true"]),
    ("fgs_sort.cu", []),
    ("fgs_blend.cu", ["-prec-div=true", "-prec-sqrt=true"]),
    ("fgs_capi.cu", []),
]


def _nvcc() -> str:
    cand = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(cand):
        raise RuntimeError("nvcc not found; the CUDA library cannot be built")
    return cand


def sources():
    deps = [os.path.join(CSRC, "fgs_common.cuh"),
            os.path.join(os.path.dirname(HERE), "include", "flashgs_b200.h")]
    return [os.path.join(CSRC, u) for u, _ in UNITS] + deps


def is_stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(s) > t for s in sources())


def build(force: bool = False, verbose: bool = False, variant: str = "", defines=()) -> str:
    """Build the library.  ``variant`` / ``defines`` are for tuning experiments only:
    a variant is built with extra -D flags into _lib/variants/<variant>/ and is
    picked up when FGS_LIB points at it (see _capi.LIB_PATH)."""
    out_dir = os.path.join(OUT_DIR, "variants", variant) if variant else OUT_DIR
    lib = os.path.join(out_dir, "libflashgs_b200.so")
    if not variant and not force and not is_stale():
        return LIB
    nvcc = _nvcc()
    os.makedirs(out_dir, exist_ok=True)
    objs = []
    procs = []
    for unit, extra in UNITS:
        obj = os.path.join(out_dir, unit.replace(".cu", ".o"))
        cmd = [nvcc, *ARCH, *COMMON, *extra, *[f"-D{d}" for d in defines],
               "-c", os.path.join(CSRC, unit), "-o", obj]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
            print(" ".join(cmd))
        procs.append((unit, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
        objs.append(obj)
    for unit, p in procs:
        out, _ = p.communicate()
        if verbose and out:
            print(out.decode())
        if p.returncode != 0:
            raise RuntimeError(f"nvcc failed on {unit}:\n{out.decode()}")
    cmd = [nvcc, *ARCH, "-shared", "-o", lib, *objs, "-cudart", "static"]
    r = subprocess.run(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)
    if r.returncode != 0:
        raise RuntimeError("link failed:\n" + r.stdout.decode())
    return lib


if __name__ == "__main__":
    # python -m paper_2408_07967_b200.build [--force] [-v] [--variant NAME -DX=1 -DY=2]
    var = sys.argv[sys.argv.index("--variant") + 1] if "--variant" in sys.argv else ""
    defs = [a[2:] for a in sys.argv if a.startswith("-D")]
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, variant=var, defines=defs))
