"""The C-ABI used from plain C (examples/c_abi_demo.c): it must compile as C99
against include/mp.h alone (CPU test) and, on a GPU, plan / gather / remap+NMS
a hand-derived tiny case through libmp_b200.so (gpu test)."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2103_14695_b200")
CUDA = "/usr/local/cuda"


def _build(tmp_path):
    gcc = shutil.which("gcc")
    if gcc is None or not os.path.exists(os.path.join(CUDA, "include", "cuda_runtime.h")):
        pytest.skip("gcc or CUDA headers missing")
    import __graft_entry__ as g
    g.build_cuda()
    exe = str(tmp_path / "c_abi_demo")
    cmd = [gcc, "-std=c99", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"), "-I",
           os.path.join(CUDA, "include"), os.path.join(ROOT, "examples", "c_abi_demo.c"), "-L", LIBDIR,
           "-l:libmp_b200.so", "-L", os.path.join(CUDA, "lib64"), "-lcudart", f"-Wl,-rpath,{LIBDIR}", "-o", exe]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe


def test_c_demo_compiles(tmp_path):
    assert os.path.exists(_build(tmp_path))


@pytest.mark.gpu
def test_c_demo_runs(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    exe = _build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "C-ABI demo OK" in r.stdout
