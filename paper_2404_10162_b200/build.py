"""In-tree build of the engine's shared libraries (no JIT cache, no pip):

  paper_2404_10162_b200/libks_b200.so   CUDA kernels (sm_100a) + the C-ABI

nvcc cross-compiles for sm_100a without a GPU, so this runs in the CPU build
container and the .so travels with the repo snapshot to the GPU box.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(PKG, "build")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CU_SOURCES = ["ks_kernels.cu", "ks_engine.cu", "ks_gemm_tc.cu", "ks_gemm16.cu", "ks_train.cu"]
CPP_SOURCES = ["ks_checkpoint.cpp", "ks_synth.cpp", "ks_group.cpp"]


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"build failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return r.stdout + r.stderr


def _newer(src_list, target):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in src_list)


def build_engine(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    out = os.path.join(PKG, "libks_b200.so")
    headers = [os.path.join(CSRC, h) for h in os.listdir(CSRC) if h.endswith((".cuh", ".h"))]
    headers.append(os.path.join(ROOT, "include", "ks_b200.h"))
    jobs = []
    for s in CU_SOURCES:
        src = os.path.join(CSRC, s)
        obj = os.path.join(BUILD, s + ".o")
        if force or _newer([src] + headers, obj):
            jobs.append([NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                         "--expt-relaxed-constexpr", "-Xptxas", "-v", f"-I{ROOT}/include",
                         "-c", src, "-o", obj])
    for s in CPP_SOURCES:
        src = os.path.join(CSRC, s)
        obj = os.path.join(BUILD, s + ".o")
        if force or _newer([src] + headers, obj):
            jobs.append(["g++", "-std=c++17", "-O2", "-fPIC", "-pthread", f"-I{ROOT}/include",
                         "-I/usr/local/cuda/include", "-c", src, "-o", obj])
    with cf.ThreadPoolExecutor(max_workers=max(1, len(jobs))) as ex:
        logs = list(ex.map(_run, jobs))
    if verbose:
        for log in logs:
            print(log)
    objs = [os.path.join(BUILD, s + ".o") for s in CU_SOURCES + CPP_SOURCES]
    if force or jobs or not os.path.exists(out):
        _run([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", out, *objs, "-L/usr/local/cuda/lib64",
              "-Xlinker", "-rpath,/usr/local/cuda/lib64"])
    return out


def build_host(verbose: bool = False, force: bool = False) -> str:
    """libkernelseer_b200.so (reference-compatible C++ API) and the Python
    module _kernelseer_b200 (reference binding names), both over libks_b200.so."""
    import sysconfig

    import pybind11

    host = os.path.join(CSRC, "host")
    api_src = os.path.join(host, "kernelseer_api.cpp")
    mod_src = os.path.join(host, "pymodule.cpp")
    hdrs = [os.path.join(ROOT, "include", "kernelseer_b200.hpp"), os.path.join(ROOT, "include", "ks_b200.h")]
    engine = os.path.join(PKG, "libks_b200.so")
    api = os.path.join(PKG, "libkernelseer_b200.so")
    mod = os.path.join(PKG, "_kernelseer_b200" + sysconfig.get_config_var("EXT_SUFFIX"))
    common = ["g++", "-std=c++20", "-O2", "-fPIC", "-ffp-contract=off", f"-I{ROOT}/include"]
    rpath = "-Wl,-rpath,$ORIGIN"
    if force or _newer([api_src, engine] + hdrs, api):
        _run(common + ["-shared", "-o", api, api_src, f"-L{PKG}", "-l:libks_b200.so", rpath])
    if force or _newer([mod_src, api] + hdrs, mod):
        _run(common + ["-shared", f"-I{sysconfig.get_paths()['include']}", f"-I{pybind11.get_include()}",
                       "-o", mod, mod_src, f"-L{PKG}", "-l:libkernelseer_b200.so", "-l:libks_b200.so", rpath])
    return mod


if __name__ == "__main__":
    import sys
    print(build_engine(verbose=True, force="--force" in sys.argv))
    print(build_host(verbose=True, force="--force" in sys.argv))
