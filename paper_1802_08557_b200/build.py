"""Build libblp.so in-tree with nvcc for sm_100a (no GPU needed to compile).

    python -m paper_1802_08557_b200.build

-fmad=false keeps every multiply and add separately rounded (numpy parity),
on top of the explicit __dmul_rn/__dsub_rn in the kernels; -lineinfo maps
ncu source pages back to the .cuh files.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
OUT = PKG / "libblp.so"
SOURCES = [CSRC / "blp_capi.cu", CSRC / "blp_cluster.cu", CSRC / "blp_condensed.cu"]
OBJDIR = PKG / "build"
DEPS = SOURCES + sorted(CSRC.glob("*.cuh")) + sorted(CSRC.glob("*.h")) + [PKG.parent / "include" / "blp.h"]

NVCC_FLAGS = [
    "-O3", "-std=c++17",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo", "-fmad=false",
    "-Xcompiler", "-fPIC",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def up_to_date() -> bool:
    if not OUT.exists():
        return False
    t = OUT.stat().st_mtime
    return all(p.stat().st_mtime <= t for p in DEPS if p.exists())


PYOBJ_SRC = CSRC / "blp_pyobj.c"


def pyobj_path() -> Path:
    import sysconfig
    return PKG / ("_pyobj" + sysconfig.get_config_var("EXT_SUFFIX"))


def build_pyobj(force: bool = False) -> Path:
    """gcc the CPython marshalling extension (_pyobj: StandardFormLP list -> per-LP pointers)."""
    import sysconfig

    import numpy
    out = pyobj_path()
    if not force and out.exists() and out.stat().st_mtime >= PYOBJ_SRC.stat().st_mtime:
        return out
    cmd = [os.environ.get("CC", "gcc"), "-O2", "-shared", "-fPIC", "-Wall",
           "-I" + sysconfig.get_paths()["include"], "-I" + numpy.get_include(),
           "-o", str(out), str(PYOBJ_SRC)]
    subprocess.run(cmd, check=True)
    return out


def build(force: bool = False, verbose: bool = False) -> Path:
    build_pyobj(force)
    if not force and up_to_date():
        return OUT
    # one object per translation unit, compiled in parallel, then one shared link
    OBJDIR.mkdir(exist_ok=True)
    objs, procs = [], []
    for src in SOURCES:
        obj = OBJDIR / (src.stem + ".o")
        extra = os.environ.get("BLP_EXTRA_NVCC", "").split()      # experiment knobs (-D...), A/B builds only
        cmd = [nvcc(), *NVCC_FLAGS, *extra, *(["-Xptxas", "-v"] if verbose else []), "-c", "-o", str(obj), str(src)]
        procs.append((cmd, subprocess.Popen(cmd)))
        objs.append(obj)
    for cmd, p in procs:
        if p.wait() != 0:
            raise subprocess.CalledProcessError(p.returncode, cmd)
    link = [nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "static",
            "-o", str(OUT), *map(str, objs)]
    subprocess.run(link, check=True)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
