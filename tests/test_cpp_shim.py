"""The header-only C++ drop-in (include/rsvd_b200.hpp) compiles against the
C ABI and links librsvd_b200.so (CPU); on a GPU the demo runs the reference's
checks through it."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_1710_01463_b200")


def build(tmp_path):
    exe = str(tmp_path / "shim_demo")
    subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "shim_demo.cpp"), "-L", PKG,
                    "-lrsvd_b200", f"-Wl,-rpath,{PKG}", "-o", exe], check=True)
    return exe


def test_shim_compiles_and_links(tmp_path):
    assert os.path.exists(build(tmp_path))


@pytest.mark.gpu
def test_shim_runs_on_gpu(tmp_path, cuda):
    out = subprocess.run([build(tmp_path)], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "shim ok" in out.stdout
