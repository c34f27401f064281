"""Builds lib/libngpulm.so in-tree for sm_100a (nvcc cross-compiles without a GPU)."""
from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "lib")
LIB = os.path.join(LIBDIR, "libngpulm.so")
KERNELS = ["advance.cu", "fused.cu", "decode.cu"]
SOURCES = KERNELS + ["capi.cpp", "build.cpp", "nglm.cpp"]
HEADERS = ["kcommon.cuh", "ngpulm_internal.h", os.path.join("..", "..", "include", "ngpulm.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "--fmad=false", "-Xcompiler", "-fPIC,-ffp-contract=off",
         "-shared"]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in SOURCES + HEADERS]
    return any(os.path.getmtime(d) > t for d in deps)


def build_variant(name: str, defines: list[str], only: list[str] | None = None) -> str:
    """Tuning variants (tools/): same sources, other compile-time constants. `only`: the
    sources the defines affect; the other objects are the main build's (build() first)."""
    out = os.path.join(LIBDIR, f"libngpulm_{name}.so")
    _compile_link(out, [f"-D{d}" for d in defines], os.path.join(HERE, "build", name), only=only)
    return out


def build_phase_timing() -> str:
    """Debug variant with per-CTA phase stamps (tools/phase_timing.py); not the product.
    All kernels in one translation unit (unity_timing.cu): one phase-stamp buffer."""
    out = os.path.join(LIBDIR, "libngpulm_timing.so")
    srcs = ["unity_timing.cu"] + [x for x in SOURCES if x not in KERNELS]
    cmd = [NVCC, *ARCH, *FLAGS, "-DNGPULM_PHASE_TIMING", "-o", out, *[os.path.join(CSRC, s) for s in srcs]]
    subprocess.run(cmd, check=True)
    return out


def _compile_link(out: str, extra: list[str], objdir: str, verbose: bool = False,
                  only: list[str] | None = None) -> None:
    """Each source compiles to an object in parallel, then one nvcc link."""
    from concurrent.futures import ThreadPoolExecutor
    os.makedirs(objdir, exist_ok=True)
    cflags = [f for f in FLAGS if f != "-shared"] + extra

    def compile_one(src):
        obj = os.path.join(objdir, os.path.splitext(src)[0] + ".o")
        if only is not None and src not in only:
            return os.path.join(HERE, "build", "main", os.path.splitext(src)[0] + ".o")
        cmd = [NVCC, *ARCH, *cflags, "-c", "-o", obj, os.path.join(CSRC, src)]
        if verbose and src.endswith(".cu"):
            cmd.insert(1, "-Xptxas=-v")
        subprocess.run(cmd, check=True)
        return obj

    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    subprocess.run([NVCC, *ARCH, "-shared", "-o", out + ".tmp", *objs], check=True)
    os.replace(out + ".tmp", out)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    os.makedirs(LIBDIR, exist_ok=True)
    _compile_link(LIB, [], os.path.join(HERE, "build", "main"), verbose)
    return LIB


if __name__ == "__main__":
    print(build(force=True, verbose=True))
