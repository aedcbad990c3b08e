"""CPU-side checks of the C-ABI library (no GPU compute): it loads, exports every
symbol include/*.h declares, and rejects invalid host parameters before any
launch.  Also checks the product package refuses to run without its library
and never imports the oracle."""
import ctypes
import glob
import os
import re
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    sys.path.insert(0, ROOT)
    import __graft_entry__ as g
    g.build_cuda()
    import paper_2103_14695_b200._binding as B
    return B


def _declared_symbols():
    syms = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        txt = open(h).read()
        syms |= set(re.findall(r"\b(mp_[a-z_0-9]+)\s*\(", txt))
    return syms


def test_library_exports_every_declared_symbol(lib):
    syms = _declared_symbols()
    assert {"mp_plan_windows", "mp_gather_resize", "mp_remap_nms"} <= syms
    so = ctypes.CDLL(lib.LIB_PATH)
    for s in sorted(syms):
        assert hasattr(so, s), f"{s} declared in include/ but not exported"
    out = subprocess.run(["nm", "-D", "--defined-only", lib.LIB_PATH], capture_output=True, text=True).stdout
    for s in syms:
        assert re.search(rf"\bT {s}\b", out), s


def test_library_is_sm100a(lib):
    out = subprocess.run(["cuobjdump", "--list-elf", lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_status_strings(lib):
    for code in range(5):
        assert lib.status_string(code).startswith("MP_")
    assert lib.launches_per_call(0) == 4 and lib.launches_per_call(1) == 2 and lib.launches_per_call(2) == 5


def test_workspace_queries(lib):
    p = lib.PlanParams(1920, 1080, [(256, 256), (512, 512), (1920, 1080)], [80, 272, 2056])
    n = lib.mp_plan_workspace_size(p, 1800)
    assert n >= 1800 * 34 * 30 * 16
    assert lib.mp_plan_workspace_size(lib.PlanParams(256, 192, [(64, 64)], [20]), 4) == 0      # no full frame
    assert lib.mp_plan_workspace_size(lib.PlanParams(256, 192, [(64, 64), (256, 192)], [70, 64]), 4) == 0
    assert lib.mp_gather_workspace_size([(192, 192), (384, 384), (1440, 810)], [10, 20, 5]) >= 35 * 16
    assert lib.mp_remap_nms_workspace_size(100, 1000) >= 1000 * 28


def test_gather_sm_reserve_setting(lib):
    """mp_gather_set_sm_reserve validates its range on the host (no launch)."""
    for bad in (-1, 1025):
        with pytest.raises(lib.MPError) as e:
            lib.mp_gather_set_sm_reserve(bad)
        assert e.value.code == lib.MP_ERR_INVALID
    lib.mp_gather_set_sm_reserve(16)
    lib.mp_gather_set_sm_reserve(0)


def test_invalid_host_params_rejected_before_launch(lib):
    """MP_ERR_INVALID is returned synchronously, before any CUDA call (so it
    works without a GPU)."""
    L = lib.lib()
    bad = lib.PlanParams(256, 192, [(64, 64)], [20])                   # (W,H) missing from S (R14)
    st = L.mp_plan_windows(ctypes.byref(bad.c), None, 1, None, None, 0, None, None, None, None, 0, None)
    assert st == lib.MP_ERR_INVALID
    big = lib.PlanParams(20000, 100, [(20000, 100)], [5])
    st = L.mp_plan_windows(ctypes.byref(big.c), None, 1, None, None, 0, None, None, None, None, 0, None)
    assert st == lib.MP_ERR_INVALID
    # remap_nms: k out of range
    st = L.mp_remap_nms(None, None, None, None, 0, 1, 0, None, 10, 10, ctypes.c_float(0.2), ctypes.c_float(0.5),
                        None, None, 0, None, None, 0, None, 0, None)
    assert st == lib.MP_ERR_INVALID
    # gather: pitch not a multiple of 16
    sz = (lib.mp_size * 1)(lib.mp_size(10, 10))
    cap = (ctypes.c_int32 * 1)(1)
    ptr = (ctypes.c_void_p * 1)(None)
    st = L.mp_gather_resize(None, 31, 10, 10, 1, None, None, 0, 1, sz, sz, ptr, cap, 0, None, None, 0, None)
    assert st == lib.MP_ERR_INVALID
    # negative window capacity
    st = L.mp_remap_nms(None, None, None, None, -1, 1, 1, sz, 10, 10, ctypes.c_float(0.2), ctypes.c_float(0.5),
                        None, None, 0, None, None, 0, None, 0, None)
    assert st == lib.MP_ERR_INVALID


def test_product_never_imports_oracle():
    for f in glob.glob(os.path.join(ROOT, "paper_2103_14695_b200", "**", "*"), recursive=True):
        if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
            txt = open(f).read()
            assert "oracle" not in re.sub(r"(#|//).*", "", txt).lower() or f.endswith("__init__.py") and \
                "import oracle" not in txt, f


def test_missing_library_fails_loudly(tmp_path):
    """A copy of the package without libmp_b200.so must raise on import."""
    import shutil
    dst = tmp_path / "paper_2103_14695_b200"
    shutil.copytree(os.path.join(ROOT, "paper_2103_14695_b200"), dst,
                    ignore=shutil.ignore_patterns("*.so", "__pycache__"))
    r = subprocess.run([sys.executable, "-c", "import paper_2103_14695_b200"], cwd=tmp_path, capture_output=True,
                       text=True)
    assert r.returncode != 0 and "not built" in r.stderr
