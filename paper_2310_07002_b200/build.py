"""Builds paper_2310_07002_b200/lib/libpcvg.so in-tree with nvcc for sm_100a.

python -m paper_2310_07002_b200.build [--force]
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
OUT = os.path.join(PKG, "lib")
OBJ = os.path.join(PKG, "lib", "obj")
LIB = os.path.join(OUT, "libpcvg.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-O3",
         "--expt-relaxed-constexpr"]
SOURCES = ["gauss_kernel.cu", "suff_kernel.cu", "lean_kernel.cu", "glm_kernel.cu", "glm32_kernel.cu", "chain_kernels.cu", "api.cpp", "multi_device.cpp", "stats.cpp",
           "host_folds.cpp", "suffstats.cpp"]
HEADERS = ["device_cache.hpp", "device_common.cuh", "types.cuh", "host_common.hpp", "tc_common.cuh", "score_extra.cuh", "suffstats.hpp", "gauss_impl.cuh"]


def _newer(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src, force):
    path = os.path.join(CSRC, src)
    obj = os.path.join(OBJ, src + ".o")
    deps = [path] + [os.path.join(CSRC, h) for h in HEADERS] + [
        os.path.join(PKG, "..", "include", "pcvg.h")]
    if not force and not _newer(obj, deps):
        return obj, None
    lang = [] if src.endswith(".cu") else ["-x", "cu"]
    extra = os.environ.get("PCVG_NVCC_DEFS", "").split()  # tooling only (e.g. -DPCVG_GLM32_TRACE)
    cmd = [NVCC] + ARCH + FLAGS + extra + lang + ["-c", path, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
    return obj, r.stderr


def build(force=False, verbose=False):
    os.makedirs(OBJ, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        results = list(ex.map(lambda s: _compile(s, force), SOURCES))
    objs = [o for o, _ in results]
    if verbose:
        for o, log in results:
            if log:
                print(log)
    if force or _newer(LIB, objs):
        cmd = [NVCC] + ARCH + ["-shared", "-o", LIB] + objs + ["-lcudart"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
    build_cli(force)
    return LIB


# The command-line front end (cli/pcvg_main.cpp) over libpcvg.so; JSON via nlohmann/json, the
# reference's own dependency, from the image (3.11.3 under cudnn_frontend).
CLI_SRC = os.path.join(PKG, "cli", "pcvg_main.cpp")
CLI = os.path.join(OUT, "pcvg")
JSON_DIRS = ["/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty"]


def build_cli(force=False):
    deps = [CLI_SRC, LIB, os.path.join(CSRC, "host_common.hpp"), os.path.join(PKG, "..", "include", "pcvg.h")]
    if not force and not _newer(CLI, deps):
        return CLI
    inc = [d for d in JSON_DIRS if os.path.exists(os.path.join(d, "nlohmann", "json.hpp"))]
    if not inc:
        return None  # no JSON header in this image: the CLI is optional
    cmd = [NVCC, "-O2", "-std=c++17", "-x", "cu", "-I" + inc[0], CLI_SRC, "-o", CLI, "-L" + OUT, "-lpcvg",
           "-Xlinker", "-rpath=$ORIGIN"] + ARCH
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"CLI build failed:\n{r.stderr}")
    return CLI


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
