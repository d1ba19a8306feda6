"""Build libskc.so in-tree with nvcc for sm_100a (no JIT cache: the .so travels with the repo).

    python -m paper_1608_01409_b200.build [--force]
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(ROOT, "build", "skc")
LIB = os.path.join(PKG, "libskc.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-O2", "-I", os.path.join(ROOT, "include"),
          "-I", CSRC, "-I", BUILD]
SOURCES = ["plan.cpp", "jit.cpp", "pad.cu", "sconv_direct.cu", "sconv_regtile.cu", "microbench.cu", "topo.cu", "spmdm.cu"]
# the JIT kernel compiles and links its generated code in-process (no ptxas on PATH needed)
CUDA_LIB = os.path.join(os.path.dirname(os.path.dirname(NVCC)), "lib64")
# the PTX compiler is static (it only exists as an archive); nvJitLink is dlopen'ed at run time
# from the toolkit (jit.cpp: jitlink()), so its 130 MB archive is not linked in
JIT_LIBS = [os.path.join(CUDA_LIB, "libnvptxcompiler_static.a"), "-lpthread", "-ldl", "-lrt"]
HEADERS = ["skc_internal.h", "ptx.cuh"]
GENERATED = os.path.join(BUILD, "regtile_gen.inc")  # gen_regtile.py output (not committed)


def _newer(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src: str, force: bool) -> str:
    path = os.path.join(CSRC, src)
    obj = os.path.join(BUILD, src + ".o")
    deps = [path, os.path.join(ROOT, "include", "skc.h"), GENERATED] + [os.path.join(CSRC, h) for h in HEADERS]
    if force or _newer(obj, deps):
        cmd = [NVCC] + ARCH + COMMON + ["-c", path, "-o", obj]
        if src.endswith(".cu"):
            cmd += ["-Xptxas", "-v"] if os.environ.get("SKC_PTXAS_V") else []
        else:
            cmd += ["-x", "cu"] if False else []
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
        if r.stderr.strip() and os.environ.get("SKC_PTXAS_V"):
            sys.stderr.write(r.stderr)
    return obj


def build(force: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    from paper_1608_01409_b200 import gen_regtile
    gen_regtile.generate(GENERATED)
    with cf.ThreadPoolExecutor(max_workers=min(8, len(SOURCES))) as ex:
        objs = list(ex.map(lambda s: _compile(s, force), SOURCES))
    if force or _newer(LIB, objs):
        cmd = [NVCC] + ARCH + ["-shared", "-cudart", "static", "-o", LIB] + objs + JIT_LIBS
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv))
