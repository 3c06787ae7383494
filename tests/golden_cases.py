"""Deterministic inputs of the golden cases whose outputs, produced by the reference itself,
are stored in tests/golden/reference_outputs.npz (generator: oracle/make_golden.py)."""
import numpy as np

from oracle import oracle as o

SUB = {1: (slice(None, None, 1),), 2: (slice(None, None, 2),) * 2, 3: (slice(None, None, 2),) * 3}


def _adjoint_recipe(ndim, n, order, tn, h=10.0, nbl=10, f0=0.01):
    """proj/src/verify.cpp:201-253"""
    idx = np.arange(n ** ndim) % n
    vel = np.where(idx < n // 2, 1.5, 2.5).astype(np.float64)
    L = (n - 1) * h
    if ndim == 2:
        src = [[0.5 * L + 0.37 * h, 2.13 * h]]
        rec = [[i * h, 4.5 * h] for i in range(n)]
    else:
        src = [[0.5 * L + 0.37 * h, 0.5 * L, 2.13 * h]]
        rec = [[i * h, 0.5 * L, 4.5 * h] for i in range(n)]
    m = o.Model([n] * ndim, [h] * ndim, [0.0] * ndim, vel, nbl, order)
    return dict(shape=[n] * ndim, spacing=[h] * ndim, origin=[0.0] * ndim, velocity=vel, nbl=nbl,
                order=order, src=np.array(src), rec=np.array(rec), tn=tn,
                dt=0.8 * m.critical_dt(order), f0=f0)


def dot2d():  # proj/tests/test_seismic.cpp:154-163
    return _adjoint_recipe(2, 48, 4, 200.0)


def dot3d():  # proj/tests/test_verify.cpp:68-77
    return _adjoint_recipe(3, 24, 6, 150.0)


def cfg1_small():
    """BASELINE.json config 1 shrunk: two layers split on the depth axis, order 4, source at
    the centre at depth 20 m, a receiver line at depth 20 m, dt = the critical dt."""
    n, h, nbl, order = 33, 10.0, 12, 4
    vel = np.empty((n, n, n))
    vel[..., : n // 2] = 1.5
    vel[..., n // 2:] = 2.5
    m = o.Model([n] * 3, [h] * 3, [0.0] * 3, vel, nbl, order)
    L = (n - 1) * h
    dt = m.critical_dt(order)
    return dict(shape=[n] * 3, spacing=[h] * 3, origin=[0.0] * 3, velocity=vel, nbl=nbl,
                order=order, src=np.array([[0.5 * L, 0.5 * L, 20.0]]),
                rec=np.array([[h * i, 0.5 * L, 20.0] for i in range(n)]), tn=250.0, dt=dt, f0=0.01)


def grad3d():
    """a small 3-D FWI gradient: random medium, off-node source, 9 receivers; the gradient is
    taken at a smoothed copy of the medium against 0.6 x the true data"""
    n, h, nbl, order = 12, 10.0, 6, 8
    rng = np.random.default_rng(18080199)
    vel = rng.uniform(1.5, 2.5, size=(n, n, n))
    m = o.Model([n] * 3, [h] * 3, [0.0] * 3, vel, nbl, order)
    L = (n - 1) * h
    c = _base = dict(shape=[n] * 3, spacing=[h] * 3, origin=[0.0] * 3, velocity=vel, nbl=nbl,
                     order=order, src=np.array([[0.5 * L + 1.3, 0.5 * L - 2.1, 17.0]]),
                     rec=np.array([[x, y, 23.0] for x in (10.0, 55.0, 100.0) for y in (15.0, 50.0, 95.0)]),
                     tn=60.5 * 0.9 * m.critical_dt(order), dt=0.9 * m.critical_dt(order), f0=0.03)
    c["gradient"] = True
    c["velocity0"] = np.full((n, n, n), 2.0) + 0.25 * (vel - 2.0)
    return c


CASES = {"dot2d": dot2d, "dot3d": dot3d, "cfg1_small": cfg1_small, "grad3d": grad3d}
