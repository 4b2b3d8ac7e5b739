"""Builds a diagnostic variant of libmsfft_b200.so with extra nvcc flags into
tools/variants/lib_<name>.so (git-ignored), e.g.

    python tools/build_variant.py decprof -DMSFFT_DECODE_PROFILE
    MSFFT_B200_LIB=tools/variants/lib_decprof.so python tools/run_c5.py

The product library (paper_2011_05698_b200/libmsfft_b200.so) is untouched."""
import os
import shutil
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2011_05698_b200 import build as B  # noqa: E402

name, extra = sys.argv[1], sys.argv[2:]
CSRC = os.environ.get("VARIANT_CSRC", B.CSRC)  # e.g. the sources of an older commit
here = os.path.dirname(os.path.abspath(__file__))
obj = os.path.join(here, "variants", "_obj_" + name)
os.makedirs(obj, exist_ok=True)
objs = []
for src in B.CU_SOURCES:
    o = os.path.join(obj, src + ".o")
    B._run([B.NVCC] + B.NVCC_FLAGS + extra + ["-c", os.path.join(CSRC, src), "-o", o], True)
    objs.append(o)
cxx = shutil.which(os.environ.get("CXX", "g++")) or "g++"
for src in [f for f in B.CXX_SOURCES if os.path.exists(os.path.join(CSRC, f))]:
    o = os.path.join(obj, src + ".o")
    B._run([cxx] + B.CXX_FLAGS + B.CXX_FILE_FLAGS.get(src, []) + ["-c", os.path.join(CSRC, src),
                                                                 "-o", o], True)
    objs.append(o)
lib = os.path.join(here, "variants", f"lib_{name}.so")
B._run([B.NVCC] + B.ARCH + ["-shared", "-cudart", "static", "-o", lib] + objs +
       ["-Xlinker", "--exclude-libs,ALL", "-lpthread"], True)
print(lib)
