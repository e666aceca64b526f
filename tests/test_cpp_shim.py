"""Builds the C++ shim tests (tests/cpp/test_shim.cpp, written like the
reference's optimize_test.cpp) against libsnn_b200.so and runs them on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def build_shim_test(tmp_path):
    from paper_2402_18994_b200.build import build
    lib = build()
    exe = str(tmp_path / "test_shim")
    subprocess.run(["g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "test_shim.cpp"), "-o", exe,
                    lib, "-Wl,-rpath," + os.path.dirname(lib)], check=True)
    return exe


def test_shim_compiles(tmp_path):
    assert os.path.exists(build_shim_test(tmp_path))


@pytest.mark.gpu
def test_shim_runs_on_gpu(tmp_path):
    exe = build_shim_test(tmp_path)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "PASSED" in out.stdout
