"""In-tree build of libmsfft_b200.so (sm_100a) -- `python -m paper_2011_05698_b200.build`.

Every .cu is compiled with ``-gencode arch=compute_100a,code=sm_100a -lineinfo
--fmad=false`` (no FMA contraction: the reference host build has none, and the
encode is bit-identical to it), host C++ with g++ ``-O2`` (no -march, same
reason).  The CUDA runtime is linked statically and its symbols hidden, so
the library can live in a process that also loaded torch's own cudart.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libmsfft_b200.so")
CUDA_HOME = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA_HOME, "bin", "nvcc")
CU_SOURCES = ["fft.cu", "window.cu", "sigma.cu", "encode.cu", "decode.cu", "fused.cu", "engine.cu",
              "signal_ops.cu", "phase_mc.cu", "wide_decode.cu", "components.cu", "locate_ops.cu"]
CXX_SOURCES = ["host_plan.cpp", "ingest.cpp", "signal_io.cpp", "capi.cpp"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "--fmad=false", "-std=c++17", "-Xcompiler", "-fPIC",
                     "-Xcompiler", "-ffp-contract=off", "--expt-relaxed-constexpr"]
CXX_FLAGS = ["-O2", "-std=c++17", "-fPIC", "-ffp-contract=off", f"-I{CUDA_HOME}/include"]
# the host gather / finiteness scan (integer and copy loops only) wants the
# vectorizer
CXX_FILE_FLAGS = {"ingest.cpp": ["-O3"]}


def _headers():
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".hpp", ".cuh", ".h"))]
    hs.append(os.path.join(REPO, "include", "msfft_b200.h"))
    return hs


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd, verbose):
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"build step failed: {' '.join(cmd[:3])} ...")
    if verbose and (r.stdout.strip() or r.stderr.strip()):
        print((r.stdout + r.stderr).strip(), flush=True)
    return r


def build(verbose: bool = False, ptxas_verbose: bool = False) -> str:
    if not os.path.exists(NVCC):
        raise RuntimeError(f"nvcc not found at {NVCC}")
    os.makedirs(OBJ, exist_ok=True)
    hdrs = _headers()
    objs = []
    for src in CU_SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(OBJ, src + ".o")
        objs.append(o)
        if _stale(o, [s] + hdrs) or ptxas_verbose:
            extra = ["-Xptxas", "-v"] if ptxas_verbose else []
            _run([NVCC] + NVCC_FLAGS + extra + ["-c", s, "-o", o], verbose or ptxas_verbose)
    cxx = shutil.which(os.environ.get("CXX", "g++")) or "g++"
    for src in CXX_SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(OBJ, src + ".o")
        objs.append(o)
        if _stale(o, [s] + hdrs):
            _run([cxx] + CXX_FLAGS + CXX_FILE_FLAGS.get(src, []) + ["-c", s, "-o", o], verbose)
    exports = os.path.join(CSRC, "exports.map")
    if _stale(LIB, objs + [exports]):
        tmp = LIB + ".tmp"
        _run([NVCC] + ARCH + ["-shared", "-cudart", "static", "-o", tmp] + objs +
             ["-Xlinker", "--exclude-libs,ALL", "-Xlinker", f"--version-script={exports}",
              "-lpthread"], verbose)
        os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(verbose=True, ptxas_verbose="-v" in sys.argv))
