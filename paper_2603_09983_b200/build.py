"""In-tree build of libmoespac.so (CUDA kernels for sm_100a + C++ host engine + C ABI).

Explicit nvcc invocations — no JIT, no torch extension cache — so the built
library sits in ``paper_2603_09983_b200/_lib/`` and travels with the repo
snapshot to the GPU box. cudart is linked statically; libnccl is dlopen'ed at
run time by the expert-parallel path only.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OUT_DIR = os.path.join(PKG, "_lib")
OBJ_DIR = os.path.join(OUT_DIR, "obj")
LIB = os.path.join(OUT_DIR, "libmoespac.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-std=c++20", "-O3", "-Xcompiler", "-fPIC,-ffp-contract=off,-Wall", "-I", os.path.join(ROOT, "include")]
CU_FLAGS = ARCH + ["-lineinfo", "--expt-relaxed-constexpr", "-Xptxas", "-v"] + os.environ.get("MOESPAC_NVCC_EXTRA", "").split()

SOURCES = [
    "kernels/router_hist.cu",
    "kernels/expert_ffn.cu",
    "kernels/expert_ffn_tc.cu",
    "kernels/expert_ffn_grouped.cu",
    "kernels/draft.cu",
    "host/scheduler.cpp",
    "host/step_scheduler.cpp",
    "host/engine.cpp",
    "host/trace_synth.cpp",
    "host/cold_executor.cpp",
    "host/trace_io.cpp",
    "host/estimator.cpp",
    "host/trace_model.cpp",
    "host/metrics.cpp",
    "abi.cpp",
]
HEADERS = [
    "kernels/common.cuh", "kernels/k3_stream.cuh", "kernels/tcgen05.cuh", "kernels/launch.hpp", "host/scheduler.hpp", "host/step_scheduler.hpp",
    "host/engine.hpp", "host/trace_synth.hpp", "host/cold_executor.hpp", "host/trace_io.hpp", "host/metrics.hpp",
    "host/estimator.hpp", "host/trace_model.hpp",
]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _newest(paths):
    return max(os.path.getmtime(p) for p in paths)


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(OBJ_DIR, exist_ok=True)
    nvcc = _nvcc()
    hdr_paths = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "moespac", "moespac.h")]
    hdr_time = _newest(hdr_paths)
    jobs = []
    objs = []
    for src in SOURCES:
        sp = os.path.join(CSRC, src)
        obj = os.path.join(OBJ_DIR, src.replace("/", "_") + ".o")
        objs.append(obj)
        if force or not os.path.exists(obj) or os.path.getmtime(obj) < max(os.path.getmtime(sp), hdr_time):
            flags = COMMON + (CU_FLAGS if src.endswith(".cu") else ["-x", "c++", "-Wno-deprecated-gpu-targets"])
            if src.endswith("cold_executor.cpp"):  # host fp32 SwiGLU loops: let them vectorise
                flags = flags + ["-Xcompiler", "-mavx2,-mfma,-fno-math-errno,-fassociative-math,-fno-signed-zeros,-fno-trapping-math"]
            jobs.append(([nvcc] + flags + ["-c", sp, "-o", obj], src))

    def run(job):
        cmd, src = job
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"compile failed: {src}\n{r.stdout}\n{r.stderr}")
        return src, r.stderr

    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        for src, log in ex.map(run, jobs):
            if verbose:
                print(f"[build] {src}")
                if log.strip():
                    print(log)
    if force or jobs or not os.path.exists(LIB):
        cmd = [nvcc] + ARCH + ["-shared", "-cudart", "static", "-o", LIB] + objs + ["-ldl", "-lpthread"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed\n{r.stdout}\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
