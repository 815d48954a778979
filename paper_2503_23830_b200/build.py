"""Builds the sm_100a library and the host C++ adapter, in-tree.

    python -m paper_2503_23830_b200.build        (also called by __graft_entry__.build())

Outputs (git-ignored, travel to GPU boxes with the snapshot):
    paper_2503_23830_b200/lib/liborchsim_b200.so       C-ABI + CUDA kernels (include/orchsim_capi.h)
    paper_2503_23830_b200/lib/liborchsim_b200_host.so  the reference's C++ API over the C-ABI
    paper_2503_23830_b200/lib/orchsim_b200_ref_tests   the reference's own unit tests compiled
                                                       unmodified against the host adapter
                                                       (only when /root/reference is present)
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "lib")
INCLUDE = os.path.join(ROOT, "include")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
CXX = os.environ.get("CXX", "g++")
REF_TESTS = "/root/reference/proj/tests"


def _nccl_dirs():
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    cands = []
    if spec and spec.submodule_search_locations:
        for loc in spec.submodule_search_locations:
            cands.append(os.path.join(loc, "nccl"))
    for c in cands:
        if os.path.exists(os.path.join(c, "include", "nccl.h")):
            return os.path.join(c, "include"), os.path.join(c, "lib")
    return "/usr/include", "/usr/lib/x86_64-linux-gnu"


CU_SOURCES = ["context.cu", "balance.cu", "dispatch.cu", "exhaustive.cu", "hosting.cu", "compose.cu",
              "exchange.cu", "nccl_window.cu"]
HOST_SOURCES = ["host/core.cpp", "host/balancers.cpp", "host/topology.cpp", "host/exchange.cpp",
                "host/runtime.cpp"]

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _run(cmd):
    print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build_cuda(force=False, lib_dir=LIB):
    """lib_dir: a diagnostics variant (e.g. ORCH_NVCC_EXTRA=-DORCH_SMALL_PROFILE) can be
    built beside the product library and selected with ORCH_LIB_PATH."""
    os.makedirs(lib_dir, exist_ok=True)
    nccl_inc, nccl_lib = _nccl_dirs()
    out = os.path.join(lib_dir, "liborchsim_b200.so")
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cu", ".cuh"))]
    deps.append(os.path.join(INCLUDE, "orchsim_capi.h"))
    if not force and not _stale(out, deps):
        return out
    objs = []
    for src in CU_SOURCES:
        obj = os.path.join(lib_dir, src.replace(".cu", ".o"))
        _run([NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "--fmad=false",
              "-Xcompiler", "-fPIC", "-Xptxas", "-v" if os.environ.get("ORCH_PTXAS_V") else "-O3",
              *os.environ.get("ORCH_NVCC_EXTRA", "").split(),
              "-I", INCLUDE, "-I", CSRC, "-I", nccl_inc, "-c", os.path.join(CSRC, src), "-o", obj])
        objs.append(obj)
    _run([NVCC, *ARCH, "-shared", "-o", out, *objs, "-L", nccl_lib, "-l:libnccl.so.2",
          "-Xlinker", f"-rpath={nccl_lib}", "-lcudart"])
    for o in objs:
        os.remove(o)
    return out


def build_host(force=False):
    """The reference's C++ API (include/orchsim/*.hpp) over the C-ABI."""
    out = os.path.join(LIB, "liborchsim_b200_host.so")
    srcs = [os.path.join(CSRC, s) for s in HOST_SOURCES]
    hdrs = [os.path.join(INCLUDE, "orchsim", f) for f in os.listdir(os.path.join(INCLUDE, "orchsim"))]
    if not force and not _stale(out, srcs + hdrs + [os.path.join(INCLUDE, "orchsim_capi.h")]):
        return out
    _run([CXX, "-std=c++20", "-O2", "-fPIC", "-shared", "-ffp-contract=off", "-Wall", "-Wextra",
          "-I", INCLUDE, "-I/usr/local/cuda/include", "-o", out, *srcs, "-L", LIB,
          "-l:liborchsim_b200.so",
          "-Wl,-rpath,$ORIGIN", "-L/usr/local/cuda/lib64", "-lcudart",
          "-Wl,-rpath,/usr/local/cuda/lib64"])
    return out


def build_ref_tests(force=False):
    """Compile the reference's unit tests UNCHANGED against the B200 host API."""
    out = os.path.join(LIB, "orchsim_b200_ref_tests")
    if not os.path.isdir(REF_TESTS):
        return None
    srcs = [os.path.join(REF_TESTS, f) for f in ("test_main.cpp", "test_core.cpp",
                                                 "test_balancers.cpp")]
    host = os.path.join(LIB, "liborchsim_b200_host.so")
    if not force and not _stale(out, srcs + [host]):
        return out
    shim = os.path.join(ROOT, "oracle", "shim")
    _run([CXX, "-std=c++20", "-O2", "-w", "-I", INCLUDE, "-I", shim, "-I", REF_TESTS, "-o", out,
          *srcs, "-L", LIB, "-l:liborchsim_b200_host.so", "-Wl,-rpath,$ORIGIN"])
    return out


def build_cpp_api_bench(force=False):
    """scripts/cpp_api_{bench,exchange}.cpp against the B200 C++ API (timing and
    parity tools; the same sources are built against the reference by oracle/Makefile)."""
    host = os.path.join(LIB, "liborchsim_b200_host.so")
    outs = []
    for name in ("cpp_api_bench", "cpp_api_exchange"):
        out = os.path.join(LIB, f"{name}_b200")
        src = os.path.join(ROOT, "scripts", f"{name}.cpp")
        if force or _stale(out, [src, host]):
            _run([CXX, "-std=c++20", "-O2", "-Wall", "-I", INCLUDE, "-o", out, src, "-L", LIB,
                  "-l:liborchsim_b200_host.so", "-Wl,-rpath,$ORIGIN"])
        outs.append(out)
    return outs


def build_p2pbench(force=False):
    """scripts/p2pbench.cu: the NVLink push / pull / copy-engine ceilings (measurement tool)."""
    out = os.path.join(LIB, "p2pbench")
    src = os.path.join(ROOT, "scripts", "p2pbench.cu")
    if force or _stale(out, [src]):
        nccl_inc, nccl_lib = _nccl_dirs()
        _run([NVCC, *ARCH, "-O3", "-std=c++17", "-lineinfo", "-I", nccl_inc, "-o", out, src,
              "-L", nccl_lib, "-l:libnccl.so.2", "-Xlinker", f"-rpath={nccl_lib}"])
    return out


def build_all(force=False):
    build_cuda(force)
    build_host(force)
    build_ref_tests(force)
    build_cpp_api_bench(force)
    build_p2pbench(force)


if __name__ == "__main__":
    build_all(force="--force" in sys.argv)
