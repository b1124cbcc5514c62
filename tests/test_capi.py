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
