"""Build recipe for libstabkit_b200.so (sm_100a only, in-tree).

`python -m paper_2507_03092_b200._build` or `__graft_entry__.build()`.
nvcc cross-compiles without a GPU; the .so travels to the GPU box with the repo snapshot.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libstabkit_b200.so")

NVCC_FLAGS = [
    "-std=c++17", "-O3", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall", "-shared",
]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: the CUDA extension cannot be built (no CPU fallback exists)")


def _sources() -> list[str]:
    out = []
    for name in sorted(os.listdir(CSRC)):
        if name.endswith((".cu", ".cpp")) and not name.startswith("host_"):
            out.append(os.path.join(CSRC, name))
    return out


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    srcs = _sources()
    deps = srcs + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".hpp"))]
    deps += [os.path.join(ROOT, "include", "stabkit_b200.h")]
    if force or _stale(LIB, deps):
        extra = ["-DSK_PANEL_TRACE"] if os.environ.get("SK_BUILD_PANEL_TRACE") else []      # per-panel debug timeline (tools/panel_trace.sh)
        cmd = [_nvcc(), *NVCC_FLAGS, *extra, "-I", os.path.join(ROOT, "include"), "-I", CSRC, "-o", LIB, *srcs]
        if verbose:
            cmd.insert(1, "-Xptxas"); cmd.insert(2, "-v")
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("nvcc failed building libstabkit_b200.so")
        if verbose:
            sys.stderr.write(r.stderr)
    return LIB


def build_host(force: bool = False) -> str | None:
    """Self-test binary of the header-only C++ `stabkit::` host API (g++ -std=c++20, links libstabkit_b200.so)."""
    tsrc = os.path.join(ROOT, "tests", "cpp", "test_host_api.cpp")
    tbin = os.path.join(ROOT, "tests", "cpp", "test_host_api")
    if not os.path.exists(tsrc):
        return None
    inc = os.path.join(ROOT, "include", "stabkit")
    deps = [tsrc, LIB, os.path.join(ROOT, "include", "stabkit_b200.h")] + [os.path.join(inc, f) for f in os.listdir(inc)]
    if force or _stale(tbin, deps):
        cmd = ["g++", "-std=c++20", "-O1", "-Wall", "-I", os.path.join(ROOT, "include"), "-o", tbin, tsrc,
               "-L", PKG, "-lstabkit_b200", f"-Wl,-rpath,{PKG}", "-Wl,-rpath,$ORIGIN/../../paper_2507_03092_b200"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("g++ failed building tests/cpp/test_host_api")
    return tbin


def build_nccl_test(force: bool = False) -> str | None:
    """tests/cpp/test_nccl_exchange: the row-sharded tableau over stabkit::NcclExchange (links the system NCCL + cudart).
    Returns None when nccl.h is not installed."""
    tsrc = os.path.join(ROOT, "tests", "cpp", "test_nccl_exchange.cpp")
    tbin = os.path.join(ROOT, "tests", "cpp", "test_nccl_exchange")
    cuda_inc = "/usr/local/cuda/include"
    if not os.path.exists(tsrc) or not any(os.path.exists(os.path.join(p, "nccl.h")) for p in ("/usr/include", cuda_inc)):
        return None
    inc = os.path.join(ROOT, "include", "stabkit")
    deps = [tsrc, LIB, os.path.join(ROOT, "include", "stabkit_b200.h")] + [os.path.join(inc, f) for f in os.listdir(inc)]
    if force or _stale(tbin, deps):
        cmd = ["g++", "-std=c++20", "-O1", "-Wall", "-I", os.path.join(ROOT, "include"), "-I", cuda_inc, "-o", tbin, tsrc,
               "-L", PKG, "-lstabkit_b200", "-L", "/usr/local/cuda/lib64", "-lcudart", "-lnccl",
               f"-Wl,-rpath,{PKG}", "-Wl,-rpath,$ORIGIN/../../paper_2507_03092_b200", "-Wl,-rpath,/usr/local/cuda/lib64"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("g++ failed building tests/cpp/test_nccl_exchange")
    return tbin


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
    print(build_host(force="--force" in sys.argv))
    print(build_nccl_test(force="--force" in sys.argv))
