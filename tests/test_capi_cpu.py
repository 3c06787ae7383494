"""C-ABI library on a box without a GPU: it must load, export every symbol the header
declares, do its host-side arithmetic right, and refuse to compute (no CPU fallback)."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

from oracle import oracle as o
from paper_1808_01995_b200 import capi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "sfb200.h")).read()
    return sorted(set(re.findall(r"SFB_API\s+[\w\s\*]+?\b(sfb_\w+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    declared = header_symbols()
    assert len(declared) >= 30
    out = subprocess.check_output(["nm", "-D", "--defined-only", capi.LIB_PATH], text=True)
    exported = set(re.findall(r"\bT (sfb_\w+)", out))
    assert set(declared) <= exported, sorted(set(declared) - exported)
    assert sorted(capi.SYMBOLS) == declared  # the Python binding lists exactly the header
    for s in declared:
        getattr(capi.lib, s)
    assert capi.lib.sfb_abi_version() == 1


def test_library_has_no_driver_link_dependency():
    out = subprocess.check_output(["ldd", capi.LIB_PATH], text=True)
    assert "libcuda.so" not in out and "libcudart" not in out


def test_sm100_kernel_images_present():
    out = subprocess.check_output(["cuobjdump", "-lelf", capi.LIB_PATH], text=True)
    assert "sm_100a" in out


@pytest.mark.parametrize("order", [2, 4, 6, 8, 10, 12, 14, 16])
def test_fd_weights_match_exact_rationals(order):
    # proj/tests/test_symbolic.cpp:52-97 via the oracle's exact solve
    w2 = capi.fd_weights(2, order)
    assert np.array_equal(w2, o.second_derivative_weights(order))
    w1 = capi.fd_weights(1, order)
    assert w1[0] == 0.0 and np.array_equal(w1[1:], o.first_derivative_weights(order))


def test_fd_weights_reject_bad_orders():
    for bad in (0, 3, 18):
        with pytest.raises(capi.SfbError) as e:
            capi.fd_weights(2, bad)
        assert e.value.code == capi.ERR_ORDER


def test_critical_dt_matches_reference_rule():
    assert capi.critical_dt([10.0, 10.0], 2.0, 2) == pytest.approx(2.5, rel=1e-14)
    m = o.Model([4, 4, 4], [12.5, 10.0, 11.0], [0.0] * 3, np.full(64, 3.7), 0, 12)
    assert capi.critical_dt([12.5, 10.0, 11.0], 3.7, 12) == m.critical_dt(12)


def test_locate_matches_oracle():
    rng = np.random.default_rng(0)
    model = o.Model([9, 11, 13], [10.0, 5.0, 2.5], [1.0, 2.0, 3.0], np.full(9 * 11 * 13, 2.0), 3, 4)
    lo = np.array(model.origin)
    hi = lo + (np.array(model.N) - 1) * np.array(model.spacing)
    pts = rng.uniform(lo, hi, size=(50, 3))
    pts[0], pts[1] = lo, hi  # faces
    base, w = o.locate(model, pts)
    d = capi.PlanDesc()
    d.ndim = 3
    for a in range(3):
        d.shape[a], d.spacing[a] = model.N[a], model.spacing[a]
    b2 = np.zeros((50, 3), dtype=np.int64)
    w2 = np.zeros((50, 8))
    org = np.array(model.origin)
    rc = capi.lib.sfb_locate(C.byref(d), org.ctypes.data, 50, pts.ctypes.data, b2.ctypes.data,
                             w2.ctypes.data)
    assert rc == 0 and np.array_equal(b2, base) and np.array_equal(w2, w)
    pts[3, 1] = hi[1] + 1.0
    rc = capi.lib.sfb_locate(C.byref(d), org.ctypes.data, 50, pts.ctypes.data, b2.ctypes.data,
                             w2.ctypes.data)
    assert rc == capi.ERR_LOCATION


def test_plan_create_validates_before_touching_a_device():
    with pytest.raises(capi.SfbError) as e:
        capi.Plan([32, 32, 32], [10.0] * 3, 7, 1.0, 10)
    assert e.value.code == capi.ERR_ORDER
    with pytest.raises(capi.SfbError) as e:
        capi.Plan([1, 32, 32], [10.0] * 3, 8, 1.0, 10)
    assert e.value.code == capi.ERR_PARAMETER
    with pytest.raises(capi.SfbError) as e:
        capi.Plan([32, 32, 32], [10.0] * 3, 8, -1.0, 10)
    assert e.value.code == capi.ERR_PARAMETER
