"""The C++ drop-in header (include/msfft_b200.hpp) compiled into a
reference-style caller (tests/cpp/test_dropin.cpp)."""
import os
import shutil
import subprocess

import pytest

from conftest import REPO

SRC = os.path.join(REPO, "tests", "cpp", "test_dropin.cpp")
LIBDIR = os.path.join(REPO, "paper_2011_05698_b200")
REFDIR = os.path.join(REPO, "oracle", "_ref")


def build(tmp_path):
    if not shutil.which("g++"):
        pytest.skip("g++ not available")
    if not os.path.exists(os.path.join(REFDIR, "libmsfft_ref.so")):
        pytest.skip("reference oracle library not built")
    if not os.path.exists(os.path.join(LIBDIR, "libmsfft_b200.so")):
        from paper_2011_05698_b200.build import build as b
        b()
    exe = str(tmp_path / "test_dropin")
    subprocess.run(["g++", "-std=c++17", "-O2", "-I", os.path.join(REPO, "include"), SRC,
                    "-L", LIBDIR, "-lmsfft_b200", "-L", REFDIR, "-lmsfft_ref", "-o", exe],
                   check=True)
    env = dict(os.environ, LD_LIBRARY_PATH=f"{LIBDIR}:{REFDIR}")
    return exe, env


def test_header_compiles(tmp_path):
    build(tmp_path)


@pytest.mark.gpu
def test_dropin_matches_reference(tmp_path):
    exe, env = build(tmp_path)
    r = subprocess.run([exe], env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "dropin ok" in r.stdout
