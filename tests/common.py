"""Shared problem builders for the parity tests (oracle inputs -> GPU plan)."""
import numpy as np

from oracle import oracle as o

SEED = 18080199


def smooth_field(shape, seed, sigma, lo, hi):
    """Seeded Gaussian-smoothed noise mapped linearly to [lo, hi] (config 2 recipe)."""
    from scipy.ndimage import gaussian_filter
    g = gaussian_filter(np.random.default_rng(seed).standard_normal(shape), sigma, mode="wrap")
    return lo + (hi - lo) * (g - g.min()) / (g.max() - g.min())


def rel_l2(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    den = np.sqrt((b ** 2).sum())
    return float(np.sqrt(((a - b) ** 2).sum()) / (den if den > 0 else 1.0))


def make_problem(shape, h, nbl, order, nsteps, vel=None, f0=0.015, n_rec_line=None,
                 src=None, rec=None, dt_frac=1.0, seed=SEED):
    ndim = len(shape)
    if vel is None:
        vel = smooth_field(shape, seed, 3.0, 1.5, 4.5)
    model = o.Model(shape, [h] * ndim, [0.0] * ndim, vel, nbl, order)
    dt = dt_frac * model.critical_dt(order)
    tn = (nsteps + 1.5) * dt  # nt = nsteps + 2  (SURVEY.md 8(d), config 2 device)
    L = [(s - 1) * h for s in shape]
    if src is None:
        src = [0.5 * L[a] + 0.37 * h for a in range(ndim - 1)] + [2.13 * h]
    if rec is None:
        n = n_rec_line or shape[0]
        xs = [L[0] * i / max(n - 1, 1) for i in range(n)]
        if ndim == 3:
            rec = [[x, 0.5 * L[1], 4.5 * h] for x in xs]
        elif ndim == 2:
            rec = [[x, 4.5 * h] for x in xs]
        else:
            rec = [[x] for x in xs]
    geom = o.Geometry(model, np.asarray(src, dtype=float).ravel(),
                      np.asarray(rec, dtype=float).ravel(), 0.0, tn, dt, f0)
    assert geom.nt == nsteps + 2, (geom.nt, nsteps)
    return model, geom


def make_plan(model, geom, order, device=0, slab=None):
    from paper_1808_01995_b200 import capi
    plan = capi.Plan(model.N, model.spacing, order, geom.dt, geom.nt, device, slab)
    plan.set_model(model.m, model.damp, model.v_max)
    plan.set_points(capi.CLOUD_SRC, geom.src_base, geom.src_w)
    plan.set_points(capi.CLOUD_REC, geom.rec_base, geom.rec_w)
    return plan
