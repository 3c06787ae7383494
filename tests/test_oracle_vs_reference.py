"""The oracle restatement against the REFERENCE ITSELF (oracle/_ref/libsf_ref.so: the
reference's unmodified sources compiled in place, see oracle/Makefile).  Skipped when the
library has not been built (it needs /root/reference at build time only)."""
import numpy as np
import pytest

from oracle import oracle as o
from oracle import ref

pytestmark = pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")


def two_layer(n, ndim):
    idx = np.arange(n ** ndim) % n
    return np.where(idx < n // 2, 1.5, 2.5)


def adjoint_case(ndim, n, order, tn, h=10.0, nbl=10, f0=0.01):
    """the configuration of proj/src/verify.cpp:201-253"""
    vel = two_layer(n, ndim)
    L = (n - 1) * h
    if ndim == 2:
        src = [0.5 * L + 0.37 * h, 2.13 * h]
        rec = [[i * h, 4.5 * h] for i in range(n)]
    else:
        src = [0.5 * L + 0.37 * h, 0.5 * L, 2.13 * h]
        rec = [[i * h, 0.5 * L, 4.5 * h] for i in range(n)]
    om = o.Model([n] * ndim, [h] * ndim, [0.0] * ndim, vel, nbl, order)
    dt = 0.8 * om.critical_dt(order)
    og = o.Geometry(om, src, np.array(rec).ravel(), 0.0, tn, dt, f0)
    rp = ref.Problem([n] * ndim, [h] * ndim, [0.0] * ndim, vel, nbl, order, order, src, rec,
                     0.0, tn, dt, f0)
    return om, og, rp


@pytest.mark.parametrize("ndim,n,order", [(1, 17, 2), (2, 19, 4), (3, 11, 6), (3, 9, 16)])
def test_model_and_geometry_bitwise(ndim, n, order):
    rng = np.random.default_rng(ndim)
    vel = rng.uniform(1.5, 3.5, size=[n] * ndim)
    h = [10.0, 7.5, 12.5][:ndim]
    L = [(n - 1) * x for x in h]
    src = [2.0 + 0.37 * x for x in L]
    rec = [[2.0 + f * x for x in L] for f in (0.0, 0.3, 1.0)]
    om = o.Model([n] * ndim, h, [2.0] * ndim, vel, 4, order)
    dt = 0.6 * om.critical_dt(order)
    rp = ref.Problem([n] * ndim, h, [2.0] * ndim, vel, 4, order, order, src, rec, 0.0, 30.0, dt, 0.02)
    m, damp, crit = rp.model()
    assert np.array_equal(m, om.m) and np.array_equal(damp, om.damp) and crit == om.critical_dt(order)
    og = o.Geometry(om, src, np.array(rec).ravel(), 0.0, 30.0, dt, 0.02)
    g = rp.geometry()
    assert g["nt"] == og.nt
    assert np.array_equal(g["src_base"], og.src_base) and np.array_equal(g["rec_base"], og.rec_base)
    assert np.array_equal(g["src_w"], og.src_w) and np.array_equal(g["rec_w"], og.rec_w)
    assert np.array_equal(g["src"], og.src)


@pytest.mark.parametrize("backend", [ref.INTERPRETER, ref.EMITTED])
def test_forward_and_adjoint_2d(backend):
    if backend == ref.EMITTED and not ref.emit_available():
        pytest.skip("no host C compiler")
    om, og, rp = adjoint_case(2, 48, 4, 200.0)
    r = rp.forward(backend=backend)
    mine = o.forward(om, og, 4, want_final=True)
    scale = np.abs(r["rec"]).max()
    assert scale > 0
    assert np.abs(mine["smp"] - r["rec"]).max() <= 1e-12 * scale
    assert np.abs(mine["final"] - r["final"]).max() <= 1e-12 * np.abs(r["final"]).max()
    assert np.abs(mine["prev"] - r["prev"]).max() <= 1e-12 * np.abs(r["prev"]).max()
    a = rp.adjoint(r["rec"], backend=backend)
    mine_a = o.adjoint(om, og, 4, rec=r["rec"], want_final=True)
    assert np.abs(mine_a["smp"] - a["srca"]).max() <= 1e-12 * np.abs(a["srca"]).max()
    assert np.abs(mine_a["final"] - a["level0"]).max() <= 1e-12 * np.abs(a["level0"]).max()


def test_forward_and_adjoint_3d_order6():
    om, og, rp = adjoint_case(3, 24, 6, 150.0)
    r = rp.forward()
    mine = o.forward(om, og, 6, want_final=True)
    assert np.abs(mine["smp"] - r["rec"]).max() <= 1e-12 * np.abs(r["rec"]).max()
    assert np.abs(mine["final"] - r["final"]).max() <= 1e-12 * np.abs(r["final"]).max()
    a = rp.adjoint(r["rec"])
    mine_a = o.adjoint(om, og, 6, rec=r["rec"])
    assert np.abs(mine_a["smp"] - a["srca"]).max() <= 1e-12 * np.abs(a["srca"]).max()
    # the reference's own dot test on its own outputs (test_verify.cpp:68-77)
    fdot, adot = float((r["rec"] ** 2).sum()), float((og.src * a["srca"]).sum())
    assert abs(fdot - adot) / fdot <= 1e-12


def test_forward_3d_order16_damped_corners():
    # order 16 with receivers inside the absorbing layer corners
    n, h, nbl = 14, 12.5, 9
    vel = np.random.default_rng(2).uniform(1.5, 4.5, size=[n] * 3)
    L = (n - 1) * h
    src = [0.41 * L, 0.52 * L, 0.33 * L]
    rec = [[-nbl * h + 1.0, -nbl * h + 2.0, 0.0], [L + nbl * h - 1.0, L, L + 3.0], [0.3 * L] * 3]
    om = o.Model([n] * 3, [h] * 3, [0.0] * 3, vel, nbl, 16)
    dt = om.critical_dt(16)
    og = o.Geometry(om, src, np.array(rec).ravel(), 0.0, 60.5 * dt, dt, 0.02)
    rp = ref.Problem([n] * 3, [h] * 3, [0.0] * 3, vel, nbl, 16, 16, src, rec, 0.0, 60.5 * dt, dt, 0.02)
    r = rp.forward()
    mine = o.forward(om, og, 16, want_final=True)
    assert np.abs(mine["smp"] - r["rec"]).max() <= 1e-11 * np.abs(r["rec"]).max()
    assert np.abs(mine["final"] - r["final"]).max() <= 1e-11 * np.abs(r["final"]).max()


def test_fwi_gradient_tiny_model():
    # the configuration of proj/tests/test_seismic.cpp:199-245
    n, nbl, h = 5, 4, 10.0
    vel_true = np.full(n * n, 1.5)
    vel_true[np.arange(n * n) % n >= n // 2] = 1.8
    om = o.Model([n, n], [h, h], [0.0, 0.0], vel_true, nbl, 2)
    dt = 0.8 * om.critical_dt(2)
    src, rec = [20.0, 10.0], [[10.0, 30.0], [30.0, 30.0]]
    rp_true = ref.Problem([n, n], [h, h], [0.0, 0.0], vel_true, nbl, 2, 2, src, rec, 0.0, 9.0 * dt, dt, 0.05)
    observed = rp_true.forward()["rec"]
    vel0 = np.full(n * n, 1.6)
    rp0 = ref.Problem([n, n], [h, h], [0.0, 0.0], vel0, nbl, 2, 2, src, rec, 0.0, 9.0 * dt, dt, 0.05)
    phi, grad, resid = rp0.fwi_gradient(observed)
    om0 = o.Model([n, n], [h, h], [0.0, 0.0], vel0, nbl, 2)
    og0 = o.Geometry(om0, src, np.array(rec).ravel(), 0.0, 9.0 * dt, dt, 0.05)
    phi2, grad2, resid2 = o.fwi_gradient(om0, og0, observed, 2)
    assert phi > 0 and phi2 == pytest.approx(phi, rel=1e-13)
    assert np.abs(grad2 - grad).max() <= 1e-12 * np.abs(grad).max()
    assert np.abs(resid2 - resid).max() <= 1e-13 * np.abs(resid).max()


def test_fwi_gradient_3d():
    n, nbl, h, order = 10, 5, 10.0, 4
    rng = np.random.default_rng(4)
    vel = rng.uniform(1.5, 2.5, size=[n] * 3)
    L = (n - 1) * h
    src = [0.5 * L + 1.0, 0.5 * L, 15.0]
    rec = [[x, 0.5 * L + 2.0, 25.0] for x in np.linspace(0, L, 7)]
    om = o.Model([n] * 3, [h] * 3, [0.0] * 3, vel, nbl, order)
    dt = 0.9 * om.critical_dt(order)
    tn = 40.5 * dt
    rp = ref.Problem([n] * 3, [h] * 3, [0.0] * 3, vel, nbl, order, order, src, rec, 0.0, tn, dt, 0.03)
    obs = rp.forward()["rec"] * 0.7
    phi, grad, _ = rp.fwi_gradient(obs)
    og = o.Geometry(om, src, np.array(rec).ravel(), 0.0, tn, dt, 0.03)
    phi2, grad2, _ = o.fwi_gradient(om, og, obs, order)
    assert phi2 == pytest.approx(phi, rel=1e-12)
    assert np.abs(grad2 - grad).max() <= 1e-11 * np.abs(grad).max()


def test_unstable_dt_rejected_by_both():
    om, og, rp = adjoint_case(2, 21, 2, 50.0)
    bad = ref.Problem([21, 21], [10.0, 10.0], [0.0, 0.0], two_layer(21, 2), 10, 2, 16,
                      [100.0, 20.0], [[50.0, 50.0]], 0.0, 50.0, og.dt, 0.01)
    with pytest.raises(ref.RefError) as e:
        bad.forward()
    assert e.value.code == 2  # StabilityError
    with pytest.raises(ArithmeticError):
        o.forward(om, og, 16)
