"""Parity against the f64 oracle on a grid that spans many tiles and several d0 chunks with
ragged edges in every direction (216 x 200 x 232 computed nodes), where the small-grid
parity tests run a single block column: the 64 x 14 tiles of orders 14 and 16, and order 8.
Tolerances are BASELINE.json's: 1e-5 relative L2 after 100 steps, 1e-3 for the gradient.
(tools/parity_sweep.py runs the same for every even order 2..16.)"""
import numpy as np
import pytest

from oracle import oracle as o
from tests.common import make_plan, make_problem, rel_l2

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("order", [8, 14, 16])
def test_midsize_parity(order):
    model, geom = make_problem([200, 184, 216], 10.0, 8, order, 100, dt_frac=0.9, n_rec_line=150)
    ref = o.forward(model, geom, order, want_final=True, save_every=2)
    plan = make_plan(model, geom, order)
    tile = plan.get_tile()
    assert tile["ty"] == (14 if order >= 14 else 16)
    rec, rep = plan.forward(geom.src, save_every=2)
    assert rep.steps == 100 and np.abs(ref["smp"]).max() > 0
    assert rel_l2(rec, ref["smp"]) <= 1e-5
    assert rel_l2(plan.wavefield(geom.nt - 1), ref["final"]) <= 1e-5
    srca, _ = plan.adjoint(geom.rec)
    assert rel_l2(srca, o.adjoint(model, geom, order)["smp"]) <= 1e-5
    resid = geom.rec * 0.5
    plan.forward(geom.src, save_every=2)
    g, _ = plan.gradient(resid)
    assert rel_l2(g, o.gradient_sweep(model, geom, order, resid, ref["snaps"], 2)) <= 1e-3
    plan.close()


@pytest.mark.parametrize("order", [12, 16])
def test_midsize_tti_parity(order):
    """The TTI pair on 120 x 116 x 126 computed nodes (ragged against the 64 x 14 tiles, two
    d0 chunks) against the builder's f64 oracle; tools/parity_sweep_tti.py covers orders 4..16."""
    from tests.common import smooth_field
    model, g0 = make_problem([104, 100, 110], 10.0, 8, order, 100, dt_frac=0.5, n_rec_line=80)
    dt = o.tti_critical_dt(model, order, 0.3)
    geom = o.Geometry(model, g0.src_coords.ravel(), g0.rec_coords.ravel(), 0.0, 101.5 * dt, dt, 0.015)
    eps = smooth_field(model.N, 2, 3.0, 0.0, 0.3)
    delta = np.minimum(smooth_field(model.N, 3, 3.0, 0.0, 0.2), eps)
    theta = smooth_field(model.N, 4, 3.0, 0.0, np.pi / 4)
    phi = smooth_field(model.N, 5, 3.0, 0.0, np.pi / 4)
    ref = o.tti_forward(model, geom, order, eps, delta, theta, phi, want_final=True)
    plan = make_plan(model, geom, order)
    plan.set_model_tti(eps, delta, theta, phi)
    rec, _ = plan.tti_forward(geom.src)
    assert np.abs(ref["smp"]).max() > 0
    assert rel_l2(rec, ref["smp"]) <= 1e-5
    assert rel_l2(plan.wavefield(geom.nt - 1, field=0), ref["p"]) <= 1e-5
    assert rel_l2(plan.wavefield(geom.nt - 1, field=1), ref["r"]) <= 1e-5
    plan.close()
