"""Build recipe for the in-tree sm_100a library ``paper_2406_04984_b200/libmeft_cuda.so``.

Every ``csrc/*.cu`` is compiled with ``nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3`` into
``build/`` (in parallel) and linked into one shared library with a plain C ABI (include/meft_cuda.h).
The drop-in C++ shim (include/meft/*.hpp over the C ABI) is built by ``build_dropin()``.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(ROOT, "build", "meft_cuda")
LIB = os.path.join(PKG, "libmeft_cuda.so")
DROPIN_LIB = os.path.join(PKG, "libmeft_dropin.so")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
HOST_CXX = "/usr/bin/g++"  # the $CXX wrapper in this image lacks libgomp; nvcc -ccbin must be a real g++
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-ccbin", HOST_CXX, "-Xcompiler", "-fPIC,-O3",
                  "-I" + os.path.join(ROOT, "include")]


def _needs(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _headers():
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh", ".hpp"))]
    hs.append(os.path.join(ROOT, "include", "meft_cuda.h"))
    return hs


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    srcs = sorted(f for f in os.listdir(CSRC) if f.endswith(".cu"))
    hdrs = _headers()
    jobs = []
    for f in srcs:
        src = os.path.join(CSRC, f)
        obj = os.path.join(BUILD, f[:-3] + ".o")
        if force or _needs(obj, [src] + hdrs):
            jobs.append([NVCC] + NVFLAGS + ["-c", src, "-o", obj])

    def run(cmd):
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed:\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        return r

    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        list(ex.map(run, jobs))
    objs = [os.path.join(BUILD, f[:-3] + ".o") for f in srcs]
    if force or jobs or _needs(LIB, objs):
        run([NVCC] + ARCH + ["-shared", "-cudart", "static", "-ccbin", HOST_CXX, "-o", LIB] + objs)
    return LIB


DROPIN_SRC = os.path.join(PKG, "dropin")


def build_dropin(verbose: bool = False, force: bool = False) -> str:
    """libmeft_dropin.so: the reference's C++ API (include/meft/*.hpp) implemented over the C ABI."""
    build()
    srcs = sorted(os.path.join(DROPIN_SRC, f) for f in os.listdir(DROPIN_SRC) if f.endswith(".cpp"))
    hdrs = [os.path.join(DROPIN_SRC, f) for f in os.listdir(DROPIN_SRC) if f.endswith(".hpp")]
    hdrs += [os.path.join(ROOT, "include", "meft", f) for f in os.listdir(os.path.join(ROOT, "include", "meft"))]
    hdrs.append(os.path.join(ROOT, "include", "meft_cuda.h"))
    if force or _needs(DROPIN_LIB, srcs + hdrs + [LIB]):
        cmd = [HOST_CXX, "-O2", "-std=c++17", "-fPIC", "-shared", "-Wall", "-Wno-unused-function",
               "-I" + os.path.join(ROOT, "include"), "-o", DROPIN_LIB] + srcs + \
              ["-L" + PKG, "-lmeft_cuda", "-Wl,-rpath,$ORIGIN"]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"g++ failed:\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return DROPIN_LIB


REF_TESTS = ("test_numerics", "test_adapter", "test_experts", "test_memtier")
# The reference's model / trainer suites exercise its trainer (train(), eval_em, resume, gradient accumulation,
# full-model finite differences) end to end over the drop-in, whose model.hpp runs the toy trunk on the GPU too;
# the out-of-scope parts they call (trainer.cpp, dataset.cpp, report.cpp) are compiled from the reference's own
# sources on top of the shim, exactly as INTEGRATION.md tells a maintainer to build them.
TRAINER_TESTS = ("test_model", "test_trainer")
TRAINER_SRCS = ("trainer.cpp", "dataset.cpp", "report.cpp")  # model.hpp: the drop-in's GPU trunk (dropin/model.cpp)
JSON_INC = "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann"
DROPIN_TEST_BIN = os.path.join(ROOT, "build", "dropin_tests")


def build_reference_tests(ref_proj: str = "/root/reference/proj", verbose: bool = False) -> list:
    """Compile the reference's own unit tests, UNMODIFIED, against the drop-in shim (test infrastructure).
    Needs the reference sources (this container); the binaries travel with the snapshot to the GPU box."""
    if not os.path.isdir(os.path.join(ref_proj, "tests")):
        return []
    lib = build_dropin(verbose)
    os.makedirs(DROPIN_TEST_BIN, exist_ok=True)
    out = []
    for t in REF_TESTS + TRAINER_TESTS + ("trajectory", "layer_bench"):
        src = (os.path.join(ROOT, "tests", "dropin", t + ".cpp") if t in ("trajectory", "layer_bench")
               else os.path.join(ref_proj, "tests", t + ".cpp"))
        exe = os.path.join(DROPIN_TEST_BIN, t)
        extra = ([os.path.join(ref_proj, "src", f) for f in TRAINER_SRCS]
                 if t not in REF_TESTS and t != "layer_bench" else [])
        if _needs(exe, [src, lib] + extra):
            # our include/ first: the hot-path headers resolve to the drop-in's, the rest to the reference's
            cmd = [HOST_CXX, "-O1", "-std=c++20", "-w", "-fopenmp", "-I" + os.path.join(ROOT, "tests", "dropin"),
                   "-I" + os.path.join(ROOT, "include"), "-I" + os.path.join(ref_proj, "include"), "-I" + JSON_INC,
                   "-o", exe, src] + extra + ["-L" + PKG, "-lmeft_dropin", "-lmeft_cuda",
                   "-Wl,-rpath," + PKG + ",-rpath,$ORIGIN/../../paper_2406_04984_b200"]
            if verbose:
                print(" ".join(cmd), file=sys.stderr)
            r = subprocess.run(cmd, capture_output=True, text=True)
            if r.returncode != 0:
                raise RuntimeError(f"g++ failed:\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        out.append(exe)
    return out


CAPI_CHECKS = ("sharded_capi_check", "graph_capi_check")
CAPI_CHECK_BIN = os.path.join(ROOT, "build", "capi_tests")


def build_capi_checks(verbose: bool = False) -> list:
    """C++ programs that use only the C ABI (tests/dropin/*.cpp listed in CAPI_CHECKS), linked against the in-tree
    library; run on the GPU box by the -m gpu tests."""
    lib = build(verbose)
    os.makedirs(CAPI_CHECK_BIN, exist_ok=True)
    out = []
    for t in CAPI_CHECKS:
        src = os.path.join(ROOT, "tests", "dropin", t + ".cpp")
        exe = os.path.join(CAPI_CHECK_BIN, t)
        if _needs(exe, [src, lib, os.path.join(ROOT, "include", "meft_cuda.h")]):
            cmd = [HOST_CXX, "-O1", "-std=c++17", "-Wall", "-I" + os.path.join(ROOT, "include"), "-o", exe, src,
                   "-L" + PKG, "-lmeft_cuda", "-Wl,-rpath," + PKG + ",-rpath,$ORIGIN/../../paper_2406_04984_b200"]
            if verbose:
                print(" ".join(cmd), file=sys.stderr)
            r = subprocess.run(cmd, capture_output=True, text=True)
            if r.returncode != 0:
                raise RuntimeError(f"g++ failed:\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        out.append(exe)
    return out


if __name__ == "__main__":
    print(build(verbose=True, force="--force" in sys.argv))
    print(build_dropin(verbose=True, force="--force" in sys.argv))
    print(build_reference_tests(verbose=True))
