"""CPU-side checks of the C-ABI library: it loads, exports every symbol
include/kafmm.h declares, and its host-only entry points behave.  No compute
call is made without a GPU."""
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "kafmm.h")


def _declared():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(kafmm_[a-z0-9_]+)\s*\(", txt)))


@pytest.fixture(scope="module")
def lib():
    from paper_2010_15155_b200 import build as B
    B.build()
    from paper_2010_15155_b200.kafmm import load_library
    return load_library()


def test_header_declares_the_north_star_entry_points():
    d = _declared()
    for name in ("kafmm_setup", "kafmm_eval", "kafmm_eval_host", "kafmm_destroy", "kafmm_kernel_dims"):
        assert name in d


def test_every_declared_symbol_is_exported(lib):
    from paper_2010_15155_b200.kafmm import EXPORTED
    for name in _declared():
        assert hasattr(lib, name), name
    assert sorted(EXPORTED) == _declared()


def test_kernel_dims_and_status_strings(lib):
    from paper_2010_15155_b200.kafmm import KafmmError, kernel_dims
    assert kernel_dims("laplace_pgrad") == (1, 4)   # Table XI LapPGrad
    assert kernel_dims("stokeslet") == (3, 3)
    assert kernel_dims("rpy") == (4, 6)
    assert kernel_dims("stokes_reg_vel") == (4, 3)
    assert kernel_dims("stokes_reg_vel_omega") == (7, 6)    # Table XI StokesRegVelOmega
    assert kernel_dims("laplace_pgradgrad") == (4, 10)      # LapPGradGrad, SL + DL at every point
    assert kernel_dims("laplace_qpgradgrad") == (9, 10)     # LapQPGradGrad
    with pytest.raises(KafmmError):
        kernel_dims(8)
    with pytest.raises(KafmmError):
        kernel_dims(0)
    assert lib.kafmm_status_string(2) == b"point outside [0,1)^3"
    assert lib.kafmm_stage_name(4) == b"m2l"


def test_invalid_arguments_rejected_before_any_device_work(lib):
    import ctypes as C
    h = C.c_void_p()
    assert lib.kafmm_setup(None, 10, 2, 8, 50, C.byref(h)) == 1          # null points
    assert lib.kafmm_setup(C.c_void_p(8), 0, 2, 8, 50, C.byref(h)) == 1  # n < 1
    assert lib.kafmm_setup(C.c_void_p(8), 10, 9, 8, 50, C.byref(h)) == 1  # unknown kernel
    assert lib.kafmm_setup(C.c_void_p(8), 10, 2, 1, 50, C.byref(h)) == 1  # p < 2
    assert lib.kafmm_setup(C.c_void_p(8), 10, 2, 8, 0, C.byref(h)) == 1   # cap < 1
    assert lib.kafmm_eval(None, None, None) == 1
    assert h.value is None


def test_product_package_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2010_15155_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle", src, flags=re.M), f
                assert "oracle/" not in src, f


def test_dist_entry_points_host_side(lib):
    """kafmm_get_unique_id (NCCL opened at run time), the in-process test
    communicators, and argument checks of kafmm_setup_dist -- host-only paths."""
    import ctypes as C
    buf = (C.c_ubyte * 128)()
    st = lib.kafmm_get_unique_id(buf)
    assert st in (0, 6), st  # 6 = ENCCL: no libnccl.so.2 in this environment
    if st == 0:
        assert any(bytes(buf))
    h = C.c_void_p()
    assert lib.kafmm_setup_dist(C.c_void_p(8), 10, 2, 8, 50, 2, 2, buf, C.byref(h)) == 1   # rank >= world
    assert lib.kafmm_setup_dist(C.c_void_p(8), 10, 2, 8, 50, 0, 0, buf, C.byref(h)) == 1   # world < 1
    assert lib.kafmm_setup_dist(C.c_void_p(8), 10, 2, 8, 50, 0, 1, None, C.byref(h)) == 1  # no id
    assert h.value is None
    arr = (C.c_void_p * 3)()
    assert lib.kafmm_comm_local_create(3, arr) == 0
    assert all(arr[i] for i in range(3))
    assert lib.kafmm_setup_dist_comm(C.c_void_p(8), 10, 9, 8, 50, arr[0], C.byref(h)) == 1  # unknown kernel
    for i in range(3):
        lib.kafmm_comm_destroy(arr[i])
    assert lib.kafmm_comm_local_create(0, arr) == 1
    out = (C.c_int64 * 16)()
    assert lib.kafmm_dist_query(None, 0, out) == 1
