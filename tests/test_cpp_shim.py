"""The C++ host layer (include/dfamin_b200.hpp): compiles against the mirror
types and — where the reference sources are present — against the reference's
own types (drop-in compile check); runs the reference-style test on the GPU."""
import os
import subprocess

import pytest

import paper_2410_22764_b200 as dfm

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "shim_test.cpp")
OUT = os.path.join(ROOT, "build", "shim_test")


def _compile(extra, out):
    os.makedirs(os.path.dirname(out), exist_ok=True)
    libdir = os.path.dirname(dfm.lib_path())
    cmd = ["g++", "-std=c++20", "-O1", "-pthread", "-I" + os.path.join(ROOT, "include"), *extra, SRC, "-o",
           out, "-L" + libdir, "-l:libdfm.so", "-Wl,-rpath," + libdir]
    subprocess.run(cmd, check=True, capture_output=True, text=True)


def test_shim_compiles_with_mirror_types():
    _compile([], OUT)
    assert os.path.exists(OUT)


@pytest.mark.skipif(not os.path.isdir("/root/reference/proj/include"),
                    reason="reference headers only present in the build container")
def test_shim_compiles_against_reference_types():
    _compile(["-DDFAMIN_B200_USE_REFERENCE_TYPES", "-I/root/reference/proj/include", "-pthread"],
             OUT + "_ref")


@pytest.mark.gpu
def test_shim_runs_reference_style_checks():
    _compile([], OUT)
    r = subprocess.run([OUT], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
