"""The C ABI from plain C (examples/fks_demo.c): it compiles and links against libfks.so with gcc
(CPU), and on a GPU runs ten fused steps with mass and energy conserved to 1e-12 (exit 0)."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_1608_08009_b200")
CUDA = "/usr/local/cuda"


def _build(out):
    if not shutil.which("gcc"):
        pytest.skip("no gcc")
    if not os.path.exists(os.path.join(LIBDIR, "libfks.so")):
        pytest.skip("libfks.so not built")
    cmd = ["gcc", "-std=c11", "-O2", "-Wall", "-Wextra", "-Werror", os.path.join(ROOT, "examples", "fks_demo.c"),
           "-I" + os.path.join(ROOT, "include"), "-I" + os.path.join(CUDA, "include"), "-L" + LIBDIR, "-lfks",
           "-L" + os.path.join(CUDA, "lib64"), "-lcudart", "-Wl,-rpath," + LIBDIR, "-lm", "-o", out]
    subprocess.run(cmd, check=True, capture_output=True, text=True)


def test_c_example_builds(tmp_path):
    _build(str(tmp_path / "fks_demo"))


@pytest.mark.gpu
def test_c_example_runs(tmp_path):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    exe = str(tmp_path / "fks_demo")
    _build(exe)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "10 steps" in r.stdout
