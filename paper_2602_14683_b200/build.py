"""In-tree build of the native libraries (sm_100a only).

  libntfg.so      C ABI + CUDA kernels (include/ntfg.h)
  libntf_b200.so  drop-in C++ API, namespace ntf (include/ntf/ntf.hpp),
                  a thin layer over libntfg.so
  ntf-cli         the reference's command-line front end over libntf_b200

Both land in paper_2602_14683_b200/lib/ (git-ignored, shipped to the GPU box
with the repo snapshot).  Objects are rebuilt only when a source or header is
newer than the object.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "lib")
OBJ = os.path.join(PKG, "lib", "obj")
INCLUDE = os.path.join(ROOT, "include")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                  "-Xcompiler", "-fvisibility=hidden", "-I" + INCLUDE, "-I" + CSRC]
if os.environ.get("NTFG_TC_TRACE_BUILD") == "1":  # role wait counters of tc_contract_kernel (tools/tc_wstats.py)
    NVFLAGS = NVFLAGS + ["-DNTFG_TC_TRACE_BUILD"]
CU_SOURCES = ["cp_api.cu", "tucker_api.cu", "io_api.cu", "unfold_api.cu", "capi.cu", "tc_contract.cu", "recon_tc.cu"]
CXX_API_SOURCES = ["ntf_api.cpp"]


def _headers():
    hs = []
    for d in (CSRC, INCLUDE, os.path.join(INCLUDE, "ntf")):
        if os.path.isdir(d):
            hs += [os.path.join(d, f) for f in os.listdir(d) if f.endswith((".cuh", ".h", ".hpp"))]
    return hs


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def _run(cmd):
    import time
    t0 = time.time()
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("build failed:\n" + " ".join(cmd) + "\n" + r.stdout + r.stderr)
    # stamp the output with the time the compile STARTED: a header edited while
    # nvcc was running (minutes per file) must leave the object stale
    if "-o" in cmd:
        out = cmd[cmd.index("-o") + 1]
        if os.path.exists(out):
            os.utime(out, (t0, t0))
    return r


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    hdrs = _headers()
    jobs = []
    objs = []
    for src in CU_SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(OBJ, src.replace(".cu", ".o"))
        objs.append(o)
        if force or _stale(o, [s] + hdrs):
            jobs.append([NVCC] + NVFLAGS + ["-c", s, "-o", o])
    with cf.ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 4))) as ex:
        for r in ex.map(_run, jobs):
            if verbose and (r.stdout or r.stderr):
                print(r.stdout + r.stderr, file=sys.stderr)
    lib = os.path.join(LIB, "libntfg.so")
    if force or jobs or _stale(lib, objs):
        _run([NVCC] + ARCH + ["-shared", "-o", lib] + objs + ["-lcuda", "-lcublas"])
    # drop-in C++ API over the C ABI
    api_srcs = [os.path.join(CSRC, s) for s in CXX_API_SOURCES if os.path.exists(os.path.join(CSRC, s))]
    if api_srcs:
        lib2 = os.path.join(LIB, "libntf_b200.so")
        if force or _stale(lib2, api_srcs + hdrs + [lib]):
            _run(["g++", "-std=c++20", "-O2", "-fPIC", "-shared", "-I" + INCLUDE, "-o", lib2] + api_srcs
                 + ["-L" + LIB, "-lntfg", "-Wl,-rpath,$ORIGIN"])
        # reference CLI front end (tools/ntf_main.cpp) over the drop-in library
        cli_src = os.path.join(CSRC, "ntf_cli.cpp")
        cli = os.path.join(LIB, "ntf-cli")
        if os.path.exists(cli_src) and (force or _stale(cli, [cli_src, lib2] + hdrs)):
            _run(["g++", "-std=c++20", "-O2", "-I" + INCLUDE, "-o", cli, cli_src, "-L" + LIB, "-lntf_b200", "-lntfg",
                  "-Wl,-rpath,$ORIGIN"])
    return lib


if __name__ == "__main__":
    print(build(verbose=True, force="--force" in sys.argv))
