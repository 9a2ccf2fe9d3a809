"""CPU-side checks of the C-ABI library (no GPU needed): it builds, loads, exports every
symbol include/kx.h declares, its host-side coefficient tables equal the oracle's (written
independently from the same tables), and device entry points fail cleanly without a GPU."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def kx():
    from paper_2310_07551_b200 import build
    build.build()
    from paper_2310_07551_b200 import kx as mod
    return mod


def header_symbols():
    src = open(os.path.join(ROOT, "include", "kx.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(kx_[a-z_0-9]+)\s*\(", src)))


def test_header_symbols_exported(kx):
    syms = header_symbols()
    assert len(syms) >= 20
    lib = ctypes.CDLL(kx.LIB_PATH)
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(kx.EXPORTED)


def test_version(kx):
    assert b"sm_100a" in kx.kx_version()


@pytest.mark.parametrize("scheme,ell,d", [("etd3rkds", 1, 2), ("etd3rkds", 2, 2),
                                          ("etd3rkds", 1, 3), ("etd3rkds", 2, 3),
                                          ("etd3rkds", 1, 4), ("etd3rkds", 2, 5),
                                          ("etd2rkds", 1, 2), ("etd2rkds", 2, 3)])
def test_coefficients_match_oracle(kx, scheme, ell, d):
    from oracle import coeffs
    eta, inner, alpha = kx.scheme_coefficients(scheme, ell, d)
    ref = coeffs.etd3_scheme(ell, d) if scheme == "etd3rkds" else coeffs.second_order(ell, d)
    assert eta == ref.etas          # bitwise: both are correctly rounded (reading R18)
    assert inner == ref.inner
    assert alpha == ref.alphas


def test_unsupported_scheme(kx):
    with pytest.raises(kx.KxError):
        kx.scheme_coefficients("etd3rkds", 1, 1)


def test_create_without_gpu_fails_cleanly(kx):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    h = ctypes.c_void_p()
    st = kx.kx_create(ctypes.byref(h), 0, None)
    assert st == kx.KX_ERR_CUDA
    assert kx.kx_create_error()
    assert kx.kx_set_grid(None, 2, None, 2) == kx.KX_ERR_INVALID


@pytest.mark.parametrize("ell", [1, 2])
@pytest.mark.parametrize("d", [2, 3, 4])
def test_complex_coefficients_match_oracle(kx, ell, d):
    from oracle import coeffs
    eta, inner, alpha = kx.scheme_coefficients_cplx(ell, d)
    ref = coeffs.table2(ell, d)
    assert eta == ref.etas and inner == ref.inner and alpha == ref.alphas
