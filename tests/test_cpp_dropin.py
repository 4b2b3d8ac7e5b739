"""The C++ drop-in header (include/msfft_b200.hpp) compiled into a
reference-style caller (tests/cpp/test_dropin.cpp)."""
import os
import shutil
import subprocess

import pytest

from conftest import REPO

SRC = os.path.join(REPO, "tests", "cpp", "test_dropin.cpp")
SUITE = os.path.join(REPO, "tests", "cpp", "test_reference_suite.cpp")
LIBDIR = os.path.join(REPO, "paper_2011_05698_b200")
REFDIR = os.path.join(REPO, "oracle", "_ref")


def build(tmp_path, src=SRC, std="c++17"):
    if not shutil.which("g++"):
        pytest.skip("g++ not available")
    if not os.path.exists(os.path.join(REFDIR, "libmsfft_ref.so")):
        pytest.skip("reference oracle library not built")
    if not os.path.exists(os.path.join(LIBDIR, "libmsfft_b200.so")):
        from paper_2011_05698_b200.build import build as b
        b()
    exe = str(tmp_path / os.path.splitext(os.path.basename(src))[0])
    subprocess.run(["g++", f"-std={std}", "-O2", "-I", os.path.join(REPO, "include"), src,
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


def test_reference_suite_compiles(tmp_path):
    build(tmp_path, SUITE, "c++20")


@pytest.mark.gpu
def test_reference_suite_on_dropin(tmp_path):
    """proj/tests/test_bucketizer.cpp:73-292 and test_flat_window.cpp:46-112
    (plus the SPEC known answers, the locate helpers and run_iteration)
    re-expressed against the drop-in header."""
    exe, env = build(tmp_path, SUITE, "c++20")
    r = subprocess.run([exe], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "reference suite ok" in r.stdout
