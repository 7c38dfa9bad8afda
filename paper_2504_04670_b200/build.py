"""In-tree build of the native libraries (no JIT cache: the .so files travel
with the repo snapshot to the GPU box).

  lib/libhgs.so         CUDA kernels (sm_100a) + the C ABI of include/hgs.h
  lib/libhitgnn_gpu.so  C++ drop-in of the reference sampler API
                        (include/hitgnn/*.hpp) layered on libhgs.so

Usage: python -m paper_2504_04670_b200.build [--force]
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "lib")
INCLUDE = os.path.join(ROOT, "include")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
              "-Xptxas", "-v"]

HGS_SO = os.path.join(LIB, "libhgs.so")
DROPIN_SO = os.path.join(LIB, "libhitgnn_gpu.so")


def _newer(target: str, sources: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def _run(cmd: list[str], log: str | None = None) -> None:
    res = subprocess.run(cmd, capture_output=True, text=True)
    if log:
        with open(log, "w") as f:
            f.write(" ".join(cmd) + "\n" + res.stdout + res.stderr)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"build failed: {' '.join(cmd[:3])} ...")


def build_hgs(force: bool = False) -> str:
    cu = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    deps = cu + glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(INCLUDE, "hgs.h")]
    if not force and not _newer(HGS_SO, deps):
        return HGS_SO
    os.makedirs(LIB, exist_ok=True)
    objs = []
    for src in cu:
        obj = os.path.join(LIB, os.path.basename(src) + ".o")
        _run([NVCC, *ARCH, *NVCC_FLAGS, "-I", INCLUDE, "-I", CSRC, "-c", src, "-o", obj],
             log=obj + ".log")
        objs.append(obj)
    _run([NVCC, *ARCH, "-shared", "-o", HGS_SO, *objs])
    for o in objs:
        os.remove(o)
    return HGS_SO


def build_variant(name: str, defines: list[str]) -> str:
    """Experiment builds (tuning sweeps): lib/variants/libhgs_<name>.so with
    extra -D flags; select one at run time with HGS_LIB=<path>."""
    out = os.path.join(LIB, "variants", f"libhgs_{name}.so")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    objs = []
    for src in sorted(glob.glob(os.path.join(CSRC, "*.cu"))):
        obj = out + "." + os.path.basename(src) + ".o"
        _run([NVCC, *ARCH, *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-I", INCLUDE, "-I", CSRC, "-c", src,
              "-o", obj])
        objs.append(obj)
    _run([NVCC, *ARCH, "-shared", "-o", out, *objs])
    for o in objs:
        os.remove(o)
    return out


def build_dropin(force: bool = False) -> str | None:
    srcs = sorted(glob.glob(os.path.join(CSRC, "dropin", "*.cpp")))
    if not srcs:
        return None
    deps = srcs + glob.glob(os.path.join(INCLUDE, "hitgnn", "*.hpp")) + [HGS_SO]
    if not force and not _newer(DROPIN_SO, deps):
        return DROPIN_SO
    _run(["g++", "-std=c++20", "-O2", "-fPIC", "-shared", "-Wall", "-Wextra", "-I", INCLUDE,
          *srcs, "-o", DROPIN_SO, f"-L{LIB}", "-lhgs", "-Wl,-rpath,$ORIGIN", "-lpthread"])
    return DROPIN_SO


def build(force: bool = False) -> None:
    build_hgs(force)
    build_dropin(force)


if __name__ == "__main__":
    build(force="--force" in sys.argv)
    print("built", HGS_SO)
