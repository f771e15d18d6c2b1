"""The C++ drop-in (include/rsvd/*.hpp over the C ABI): reference unit tests
compiled against the headers.  Compiling + linking is checked on CPU; running
needs the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp")
LIBDIR = os.path.join(ROOT, "paper_2402_17794_b200", "lib")


def _build(tmp_path):
    exe = str(tmp_path / "test_dropin")
    cmd = ["g++", "-std=c++20", "-O1", "-Wall", "-Wextra", "-Werror", f"-I{ROOT}/include", SRC,
           f"-L{LIBDIR}", "-lrsvd_b200", f"-Wl,-rpath,{LIBDIR}", "-o", exe]
    subprocess.run(cmd, check=True, capture_output=True)
    return exe


def test_dropin_headers_compile_and_link(tmp_path):
    assert os.path.exists(_build(tmp_path))


@pytest.mark.gpu
def test_dropin_reference_unit_tests_pass_on_gpu(tmp_path):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    exe = _build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "all passed" in r.stdout
