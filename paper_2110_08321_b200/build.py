"""In-tree build of libhegpu.so (sm_100a) -- `python -m paper_2110_08321_b200.build`.

Every CUDA/C++ source under csrc/ is compiled with nvcc for
`-gencode arch=compute_100a,code=sm_100a -lineinfo` and linked into one
shared library next to this file, so the built .so travels with the repo
snapshot to the GPU box (it is git-ignored, not gpurun-ignored).
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "_obj")
LIB = os.path.join(HERE, "libhegpu.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-I", os.path.join(ROOT, "include"), "-I", CSRC,
          "-Xcompiler", "-fPIC,-fopenmp,-ffp-contract=off,-fno-fast-math", "-Xptxas", "-O3"]


# translation units that #include another .cu (rebuild when it changes)
INCLUDED_SOURCES = {"ntt_r8.cu": ["ntt.cu"], "ntt_fp16.cu": ["ntt.cu"], "ntt_fp8.cu": ["ntt.cu"],
                    "ntt_fp16n.cu": ["ntt.cu"]}


def sources():
    return sorted(f for f in os.listdir(CSRC) if f.endswith((".cu", ".cpp")))


def headers_mtime():
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".hpp", ".cuh", ".h"))]
    hs.append(os.path.join(ROOT, "include", "hegpu.h"))
    return max(os.path.getmtime(h) for h in hs)


def _compile(src, force):
    obj = os.path.join(OBJ, src + ".o")
    path = os.path.join(CSRC, src)
    deps = [path] + [os.path.join(CSRC, d) for d in INCLUDED_SOURCES.get(src, [])]
    if (not force and os.path.exists(obj)
            and os.path.getmtime(obj) >= max(max(os.path.getmtime(d) for d in deps), headers_mtime())):
        return obj
    cmd = [NVCC, *ARCH, *COMMON, "-c", path, "-o", obj]
    if src.endswith(".cpp"):
        cmd = [NVCC, *COMMON, "-x", "c++", "-c", path, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed on {src}:\n{r.stdout}\n{r.stderr}")
    return obj


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    srcs = sources()
    with ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(lambda s: _compile(s, force), srcs))
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-Xcompiler", "-fopenmp", "-lgomp", "-lcudart"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    build_cli(force)
    if verbose:
        print(LIB)
    return LIB


CLI_SRC = os.path.join(ROOT, "tools", "hegpu_cli.cpp")
CLI = os.path.join(HERE, "hegpu_cli")


def build_cli(force: bool = False) -> str:
    """the hesim-style command-line front end (tools/hegpu_cli.cpp) over libhegpu.so"""
    if (not force and os.path.exists(CLI)
            and os.path.getmtime(CLI) >= max(os.path.getmtime(CLI_SRC), os.path.getmtime(LIB))):
        return CLI
    cmd = ["g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"), CLI_SRC, "-o", CLI, "-L", HERE,
           "-lhegpu", "-Wl,-rpath,$ORIGIN"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"hegpu_cli build failed:\n{r.stdout}\n{r.stderr}")
    return CLI


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
