"""In-tree build of the sm_100a library libemie_cu.so (C ABI: include/emie_cu.h).

Compiled with nvcc for `-gencode arch=compute_100a,code=sm_100a -lineinfo`
only; nvcc cross-compiles without a GPU, so this runs in the CPU container.
The .so lands next to this file (git-ignored, travels to the GPU box).
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libemie_cu.so"
CPPLIB = PKG / "libemie_b200.so"  # C++ drop-in of the reference emie:: API over the C ABI
SOURCES = ["capi.cu", "operator.cu", "lateral.cu", "solver.cu", "greens.cu", "shard.cu", "peer.cu", "dense.cu", "layered.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.sep not in c or Path(c).exists()):
            return c
    raise RuntimeError("nvcc not found")


def stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = (list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cuh")) + [ROOT / "include" / "emie_cu.h"]
            + list((PKG / "cpp").glob("*.cpp")) + list((ROOT / "include" / "emie").glob("*.hpp")))
    if not CPPLIB.exists():
        return True
    return any(p.stat().st_mtime > t for p in deps)


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not stale():
        return LIB
    objs = []
    tmp = PKG / "build_obj"
    tmp.mkdir(exist_ok=True)
    flags = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2",
                    "-I", str(ROOT / "include"), "--expt-relaxed-constexpr"]
    if verbose:
        flags += ["-Xptxas", "-v"]
    procs = []
    for s in SOURCES:
        o = tmp / (s + ".o")
        objs.append(o)
        cmd = [nvcc()] + flags + ["-c", str(CSRC / s), "-o", str(o)]
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
    for cmd, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0 or verbose:
            sys.stderr.write(out.decode())
        if p.returncode != 0:
            raise RuntimeError("nvcc failed: " + " ".join(cmd))
    link = [nvcc()] + ARCH + ["-shared", "-o", str(LIB)] + [str(o) for o in objs] + ["-cudart", "static"]
    r = subprocess.run(link, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("link failed:\n" + r.stdout + r.stderr)
    build_cpp()
    return LIB


def build_cpp() -> Path:
    """libemie_b200.so: include/emie/*.hpp implemented over libemie_cu.so."""
    cmd = ["g++", "-std=c++20", "-O2", "-fPIC", "-shared", "-I", str(ROOT / "include"),
           str(PKG / "cpp" / "emie_dropin.cpp"), str(PKG / "cpp" / "emie_quad.cpp"), "-L", str(PKG), "-lemie_cu",
           "-Wl,-rpath,$ORIGIN", "-o", str(CPPLIB)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("drop-in build failed:\n" + r.stdout + r.stderr)
    return CPPLIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
