"""Build libowqs.so in-tree: nvcc for the sm_100a kernels, g++ for the host scheduler / C-ABI.

python -m paper_1604_05659_b200._build  [--force]
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
BUILD = os.path.join(PKG, "build")
LIB = os.path.join(PKG, "libowqs.so")
CUDA_HOME = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA_HOME, "bin", "nvcc")
NVRTC_LIB = os.path.join(CUDA_HOME, "lib64", "libnvrtc.so.12")  # loaded by path at run time (jit.cpp)
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]

CU_SOURCES = ["kernels.cu"]
CPP_SOURCES = ["scheduler.cpp", "gflow.cpp", "standardize.cpp", "jit.cpp", "capi.cpp", "host_api.cpp"]
HEADERS = ["owqs_internal.h", "scheduler.h", "device_common.cuh", "jit.h"]
PRELUDE = [("kPreludeInternal", "owqs_internal.h"), ("kPreludeCommon", "device_common.cuh")]


def _run(cmd):
    r = subprocess.run(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
    if r.returncode != 0:
        sys.stderr.write(" ".join(cmd) + "\n" + r.stdout)
        raise RuntimeError(f"build step failed: {cmd[0]} {cmd[-1]}")
    return r.stdout


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _write_prelude():
    """build/jit_prelude.inc: the device headers the generated pass kernels start with (raw strings)."""
    out = []
    for var, name in PRELUDE:
        with open(os.path.join(CSRC, name)) as f:
            text = "".join(l for l in f if not l.startswith("#pragma once"))
        if ')OWQSPRE"' in text:
            raise RuntimeError("raw-string delimiter inside " + name)
        out.append(f'const char* {var} = R"OWQSPRE(\n{text})OWQSPRE";\n')
    path = os.path.join(BUILD, "jit_prelude.inc")
    data = "".join(out)
    if not os.path.exists(path) or open(path).read() != data:
        with open(path, "w") as f:
            f.write(data)
    return path


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    prelude = _write_prelude()
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(INCLUDE, "owqs.h"), os.path.join(INCLUDE, "owqs_host.h")]
    objs = []
    for src in CU_SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src + ".o")
        objs.append(o)
        if force or _stale(o, [s] + hdrs):
            # -rdc: decide_kernel updates graph kernel nodes through the device runtime (cudadevrt)
            out = _run([NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-rdc=true", "-Xcompiler", "-fPIC",
                        "-Xptxas", "-v", "-I", INCLUDE, "-I", CSRC, "-c", s, "-o", o])
            if verbose:
                print(out)
            with open(os.path.join(BUILD, src + ".ptxas.txt"), "w") as f:
                f.write(out)
    for src in CPP_SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src + ".o")
        objs.append(o)
        if force or _stale(o, [s, prelude] + hdrs):
            _run(["g++", "-O2", "-g", "-std=c++17", "-fPIC", "-Wall", "-Wno-unused-function",
                  "-I", INCLUDE, "-I", CSRC, "-I", BUILD, "-I", os.path.join(CUDA_HOME, "include"),
                  f'-DOWQS_NVRTC_PATH="{NVRTC_LIB}"', "-c", s, "-o", o])
    if force or _stale(LIB, objs):
        tmp = LIB + ".tmp"
        _run([NVCC, *ARCH, "-shared", "-rdc=true", "-o", tmp, *objs, "-Xlinker", "--no-undefined",
              "-L/usr/lib/x86_64-linux-gnu", "-lnccl", "-lcudadevrt",
              "-lpthread", "-ldl", "-lrt"])
        shutil.move(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
