"""Pins the CPU oracle (oracle/) to every known answer the reference's own tests hold
for the wave-propagator path.  Each test cites the reference
test it restates (paths relative to /root/reference/proj)."""
from fractions import Fraction as F

import numpy as np
import pytest

from oracle import oracle as o


# ---- FD tables: tests/test_symbolic.cpp:52-97 ---------------------------------------

def test_second_derivative_weight_tables():
    def check(order, expect):
        assert o.fd_weights_exact(2, o.centered_offsets(order)) == expect
    check(2, [1, -2, 1])
    check(4, [F(-1, 12), F(4, 3), F(-5, 2), F(4, 3), F(-1, 12)])
    check(6, [F(1, 90), F(-3, 20), F(3, 2), F(-49, 18), F(3, 2), F(-3, 20), F(1, 90)])
    check(8, [F(-1, 560), F(8, 315), F(-1, 5), F(8, 5), F(-205, 72), F(8, 5), F(-1, 5),
              F(8, 315), F(-1, 560)])


def test_first_derivative_weight_tables():
    assert o.fd_weights_exact(1, o.centered_offsets(2)) == [F(-1, 2), 0, F(1, 2)]
    assert o.fd_weights_exact(1, [-1, 0]) == [-1, 1]
    assert o.fd_weights_exact(1, [0, 1]) == [-1, 1]


def test_moment_conditions_high_order():
    from math import factorial
    for d in (1, 2):
        for order in (2, 6, 12, 16):
            off = o.centered_offsets(order)
            ws = o.fd_weights_exact(d, off)
            for p in range(len(off)):
                s = sum(w * F(x) ** p for w, x in zip(ws, off))
                assert s == (factorial(d) if p == d else 0)


def test_survey_appendix_tables():
    w16 = o.fd_weights_exact(2, o.centered_offsets(16))
    assert w16[8] == F(-1077749, 352800) and w16[16] == F(-1, 411840)
    w12 = o.fd_weights_exact(1, o.centered_offsets(12))
    assert w12[7:] == [F(6, 7), F(-15, 56), F(5, 63), F(-1, 56), F(1, 385), F(-1, 5544)]
    with pytest.raises(ValueError):
        o.centered_offsets(3)


# ---- locate: tests/test_symbolic.cpp:278-315 ----------------------------------------

def _grid_model(n, h=1.0, ndim=2):
    return o.Model([n] * ndim, [h] * ndim, [0.0] * ndim, np.full(n ** ndim, 1.5), 0, 2)


def test_locate_multilinear_weights():
    base, w = o.locate(_grid_model(11), [0.3, 0.7])
    assert np.allclose(w[0], [0.21, 0.09, 0.49, 0.21], rtol=1e-12)
    assert base.tolist() == [[0, 0]]


def test_locate_far_face_and_outside():
    m = _grid_model(11)
    base, w = o.locate(m, [10.0, 10.0])
    assert base.tolist() == [[9, 9]]
    assert w[0, 0] == pytest.approx(0.0) and w[0, 3] == pytest.approx(1.0)
    with pytest.raises(ValueError):
        o.locate(m, [11.0, 5.0])
    with pytest.raises(ValueError):
        o.locate(m, [-0.5, 5.0])


def test_locate_on_node_single_corner():
    base, w = o.locate(_grid_model(11), [4.0, 6.0])
    assert base.tolist() == [[4, 6]]
    assert w[0].tolist() == [1.0, 0.0, 0.0, 0.0]


# ---- model: tests/test_seismic.cpp:29-83 --------------------------------------------

def _constant_model(n, h, c, nbl, order=8):
    return o.Model([n, n], [h, h], [0.0, 0.0], np.full(n * n, c), nbl, order)


def test_damping_shape():
    m = _constant_model(21, 10.0, 1.5, 6)
    n = 21 + 12
    assert (m.damp[6:n - 6, 6:n - 6] == 0.0).all()
    mid = n // 2
    prev = 0.0
    for i in range(5, -1, -1):
        assert m.damp[i, mid] > prev
        prev = m.damp[i, mid]
    edge = m.damp[0, mid]
    assert (m.damp <= 2.0 * edge + 1e-18).all()
    assert m.damp[0, 0] == pytest.approx(2.0 * edge, rel=1e-12)


def test_nbl_zero():
    m = _constant_model(15, 10.0, 2.0, 0)
    assert (m.damp == 0.0).all() and m.N == [15, 15]


def test_critical_dt_second_order_2d():
    m = _constant_model(15, 10.0, 2.0, 0)
    assert m.critical_dt(2) == pytest.approx(10.0 / (2.0 * 2.0), rel=1e-14)
    assert m.critical_dt(8) < m.critical_dt(2)


def test_survey_critical_dt_table():
    # SURVEY.md section 8 config table
    m = o.Model([4, 4, 4], [12.5] * 3, [0.0] * 3, np.full(64, 4.5), 0, 8)
    assert m.critical_dt(8) == pytest.approx(0.889492, abs=1e-6)
    assert m.critical_dt(16) == pytest.approx(0.832238, abs=1e-6)
    m = o.Model([4, 4, 4], [10.0] * 3, [0.0] * 3, np.full(64, 2.5), 0, 4)
    assert m.critical_dt(4) == pytest.approx(1.414214, abs=1e-6)


def test_velocity_edge_extension():
    n, nbl = 9, 5
    vel = np.array([[1.0 + 0.1 * i + 0.01 * j for j in range(n)] for i in range(n)])
    m = o.Model([n, n], [10.0, 10.0], [0.0, 0.0], vel, nbl, 4)
    slow = lambda v: 1.0 / (v * v)
    assert m.m[0, 0] == pytest.approx(slow(vel[0, 0]), rel=1e-14)
    assert m.m[nbl, nbl] == pytest.approx(slow(vel[0, 0]), rel=1e-14)
    assert m.m[nbl + n - 1 + nbl, nbl] == pytest.approx(slow(vel[n - 1, 0]), rel=1e-14)
    assert m.m[nbl + 3, 0] == pytest.approx(slow(vel[3, 0]), rel=1e-14)


def test_physical_m_roundtrip():
    m = _constant_model(11, 10.0, 1.5, 4)
    vals = m.physical_m().ravel()
    vals = vals + 0.001 * (np.arange(vals.size) % 7)
    m.set_physical_m(vals)
    assert (m.physical_m().ravel() == vals).all()


# ---- geometry / wavelet: tests/test_seismic.cpp:85-114, tests/test_verify.cpp:30-42 --

def test_geometry_time_axis_and_ricker():
    m = _constant_model(21, 10.0, 1.5, 4)
    g = o.Geometry(m, [100.0, 100.0], [50.0, 50.0, 150.0, 50.0], 0.0, 101.0, 2.0, 0.01)
    assert g.nt == int(np.floor(101.0 / 2.0)) + 1 and g.n_src == 1 and g.n_rec == 2
    tr = g.src[:, 0]
    assert tr.max() == pytest.approx(1.0, rel=1e-9)
    assert abs(int(tr.argmax()) * 2.0 - 100.0) <= 2.0
    assert (g.rec == 0.0).all()


def test_geometry_rejects_unstable_dt():
    m = _constant_model(21, 10.0, 1.5, 4)
    with pytest.raises(ArithmeticError):
        o.Geometry(m, [100.0, 100.0], [50.0, 50.0], 0.0, 100.0, m.critical_dt() * 1.5, 0.01)


def test_ricker_peak():
    w = o.ricker(0.01, 0.0, 0.5, 401)
    assert w[200] == pytest.approx(1.0, rel=1e-14)
    assert np.abs(w).max() == pytest.approx(1.0, rel=1e-14)
    assert abs(w[0]) < 1e-3


# ---- operators ------------------------------------------------------------------------

def _adjoint_test(ndim, n, order, tn, h=10.0, nbl=10, f0=0.01):
    """src/verify.cpp:201-253 restated against the oracle."""
    idx = np.arange(n ** ndim) % n
    vel = np.where(idx < n // 2, 1.5, 2.5)
    model = o.Model([n] * ndim, [h] * ndim, [0.0] * ndim, vel, nbl, order)
    L = (n - 1) * h
    if ndim == 2:
        src = [0.5 * L + 0.37 * h, 2.13 * h]
        rec = [[i * h, 4.5 * h] for i in range(n)]
    else:
        src = [0.5 * L + 0.37 * h, 0.5 * L, 2.13 * h]
        rec = [[i * h, 0.5 * L, 4.5 * h] for i in range(n)]
    dt = 0.8 * model.critical_dt(order)
    geom = o.Geometry(model, src, np.array(rec).ravel(), 0.0, tn, dt, f0)
    o.forward(model, geom, order)
    fdot = float((geom.rec ** 2).sum())
    adj = o.adjoint(model, geom, order)
    adot = float((geom.src * adj["smp"]).sum())
    return fdot, adot, abs(fdot - adot) / max(abs(fdot), np.finfo(float).tiny)


def test_dot_test_2d_order4():  # tests/test_seismic.cpp:154-163
    fdot, _, rel = _adjoint_test(2, 48, 4, 200.0)
    assert fdot > 0.0 and rel <= 1e-12


def test_dot_test_3d_order6():  # tests/test_verify.cpp:68-77
    fdot, _, rel = _adjoint_test(3, 24, 6, 150.0)
    assert fdot > 0.0 and rel <= 1e-12


def test_zero_source_zero_receivers():  # tests/test_seismic.cpp:165-174
    m = _constant_model(31, 10.0, 1.5, 8)
    g = o.Geometry(m, [150.0, 150.0], [50.0, 100.0, 250.0, 100.0], 0.0, 150.0,
                   0.9 * m.critical_dt(), 0.01)
    g.src[:] = 0.0
    o.forward(m, g, 8)
    assert (g.rec == 0.0).all()


def test_structural_zero_rows():  # include/sf/seismic_ops.hpp:13-16
    m = _constant_model(31, 10.0, 1.5, 8)
    g = o.Geometry(m, [150.0, 150.0], [50.0, 100.0, 250.0, 100.0], 0.0, 150.0,
                   0.9 * m.critical_dt(), 0.01)
    o.forward(m, g, 8)
    assert (g.rec[[0, 1, g.nt - 1]] == 0.0).all() and np.abs(g.rec).max() > 0


def test_absorbing_layer_dissipates():  # tests/test_seismic.cpp:176-197
    m = _constant_model(41, 10.0, 1.5, 20)
    dt = 0.9 * m.critical_dt()
    g = o.Geometry(m, [200.0, 200.0], [200.0, 300.0], 0.0, 900.0, dt, 0.01)
    r = o.forward(m, g, 8, save_every=1)
    energy = (r["snaps"] ** 2).sum(axis=(1, 2))
    assert energy.max() > 0 and energy[g.nt - 1] < 0.05 * energy.max()


def test_gradient_vs_finite_differences():  # tests/test_seismic.cpp:199-245
    n, nbl, h = 5, 4, 10.0
    vel_true = np.full(n * n, 1.5)
    vel_true[np.arange(n * n) % n >= n // 2] = 1.8
    model = o.Model([n, n], [h, h], [0.0, 0.0], vel_true, nbl, 2)
    dt = 0.8 * model.critical_dt(2)
    geom = o.Geometry(model, [20.0, 10.0], [10.0, 30.0, 30.0, 30.0], 0.0, 9.0 * dt, dt, 0.05)
    assert geom.nt <= 10
    o.forward(model, geom, 2)
    observed = geom.rec.copy()
    model.set_velocity(np.full(n * n, 1.6))
    m0 = model.physical_m().ravel().copy()
    phi, grad, _ = o.fwi_gradient(model, geom, observed, 2)
    grad = grad.ravel()
    assert phi > 0 and np.abs(grad).max() > 0
    gmax = np.abs(grad).max()

    def phi_at(mv):
        model.set_physical_m(mv)
        o.forward(model, geom, 2)
        return o.objective(geom.rec, observed)

    delta = 1e-5
    for i in range(m0.size):
        mp, mm = m0.copy(), m0.copy()
        mp[i] += delta
        mm[i] -= delta
        fd = (phi_at(mp) - phi_at(mm)) / (2 * delta)
        if max(abs(fd), abs(grad[i])) < 1e-9 * gmax:
            continue
        assert abs(fd - grad[i]) <= 1e-5 * max(abs(fd), abs(grad[i]))


def test_zero_residual_zero_gradient():  # tests/test_seismic.cpp:247-260
    m = _constant_model(21, 10.0, 1.5, 6)
    g = o.Geometry(m, [100.0, 20.0], [40.0, 40.0, 160.0, 40.0], 0.0, 120.0,
                   0.8 * m.critical_dt(), 0.01)
    o.forward(m, g, 8)
    phi, grad, _ = o.fwi_gradient(m, g, g.rec.copy(), 8)
    assert phi == 0.0 and (grad == 0.0).all()


def test_injection_known_answer():  # tests/test_compiler.cpp:391-407 (weights only)
    m = o.Model([6, 5], [1.0, 1.0], [0.0, 0.0], np.full(30, 1.0), 0, 2)
    base, w = o.locate(m, [2.25, 1.75])
    assert base.tolist() == [[2, 1]]
    assert np.allclose(10.0 * w[0], [10 * .75 * .25, 10 * .25 * .25, 10 * .75 * .75,
                                     10 * .25 * .75], rtol=1e-15)


def test_unstable_dt_rejected():  # tests/test_seismic.cpp:108-114, seismic_ops.cpp:15-22
    m = _constant_model(21, 10.0, 1.5, 4, order=2)
    g = o.Geometry(m, [100.0, 100.0], [50.0, 50.0], 0.0, 50.0, 0.99 * m.critical_dt(2), 0.01)
    with pytest.raises(ArithmeticError):
        o.forward(m, g, 16)
