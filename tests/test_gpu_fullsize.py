"""BASELINE.json's full sizes (592^3 computed nodes, 262 144 receivers) checked through
size-independent properties, since the f64 oracle cannot finish these in seconds:
linearity, zero-in/zero-out, adjointness (dot test), slab-cut invariance, and -- for the
gradient -- agreement of the fused imaging with an imaging recomputed from downloaded
levels on a sub-volume.  A short oracle run on the full grid anchors the absolute values."""
import numpy as np
import pytest

from tests.common import rel_l2

pytestmark = pytest.mark.gpu

N_PHYS, H, NBL, ORDER = 512, 12.5, 40, 8


@pytest.fixture(scope="module")
def full():
    """config 3's medium at config 2/3's size: two layers split on the depth axis."""
    from paper_1808_01995_b200 import _sfb_host as Hst
    from paper_1808_01995_b200 import synthetic as syn
    cfg = syn.config(3, N_PHYS)
    model = Hst.SeismicModel(cfg["shape"], [H] * 3, [0.0] * 3, cfg["velocity"](), NBL, ORDER)
    nsteps = 48
    dt, tn = syn.time_axis(model.critical_dt(ORDER), nsteps)
    geom = Hst.AcquisitionGeometry(model, np.asarray(cfg["src"]).ravel(), cfg["rec"].ravel(),
                                   0.0, tn, dt, 0.03)
    assert geom.nt == nsteps + 2 and geom.n_rec == 512 * 512
    return model, geom


def plan_for(model, geom, slab=None):
    from paper_1808_01995_b200 import capi
    plan = capi.Plan(model.grid.shape, model.grid.spacing, ORDER, geom.dt, geom.nt, 0, slab)
    plan.set_model(model.m.array(), model.damp.array(), model.v_max)
    plan.set_points(capi.CLOUD_SRC, np.array(geom.src.base_table).reshape(-1, 3),
                    np.array(geom.src.weight_table).reshape(-1, 8))
    plan.set_points(capi.CLOUD_REC, np.array(geom.rec.base_table).reshape(-1, 3),
                    np.array(geom.rec.weight_table).reshape(-1, 8))
    return plan


def test_forward_properties_and_dot_test_at_full_size(full):
    model, geom = full
    plan = plan_for(model, geom)
    src = np.ascontiguousarray(geom.src.traces)
    rec, rep = plan.forward(src)
    assert rep.steps == 48 and np.abs(rec).max() > 0 and np.isfinite(rec).all()
    assert (rec[[0, 1, geom.nt - 1]] == 0.0).all()
    # linearity: scaling by a power of two is exact in fp32 except where the wavefront tail
    # underflows into denormals, so F(2x) equals 2 F(x) to far below fp32 round-off
    rec2, _ = plan.forward(2.0 * src)
    assert rel_l2(rec2, 2.0 * rec) <= 1e-7
    zero, _ = plan.forward(np.zeros_like(src))
    assert (zero == 0.0).all()
    # adjointness on random band-limited data: <F x, y> == <x, F^T y> to fp32 accuracy
    rng = np.random.default_rng(18080199 + 11)
    y = rng.standard_normal(rec.shape) * np.hanning(geom.nt)[:, None]
    y[[0, geom.nt - 1]] = 0.0
    xt, _ = plan.adjoint(y)
    lhs, rhs = float((rec * y).sum()), float((src * xt).sum())
    assert abs(lhs - rhs) <= 1e-4 * max(abs(lhs), abs(rhs))
    plan.close()


def test_two_slabs_equal_one_domain_at_full_size(full):
    from paper_1808_01995_b200 import capi
    model, geom = full
    src = np.ascontiguousarray(geom.src.traces)
    plan = plan_for(model, geom)
    rec1, _ = plan.forward(src)
    plan.close()
    n0 = model.grid.shape[0]
    cuts = [0, n0 // 2, n0]
    plans = [plan_for(model, geom, (cuts[i], cuts[i + 1])) for i in range(2)]
    F = capi.OP_FORWARD
    for p in plans:
        p.upload_traces(capi.CLOUD_SRC, src)
        p.step_begin(F)
    for t in range(1, geom.nt - 1):
        for p in plans:
            p.step_compute(F, t, capi.PART_LOW)
            p.step_compute(F, t, capi.PART_HIGH)
            p.step_points(F, t, capi.PART_LOW)
            p.step_compute(F, t, capi.PART_INTERIOR)
            p.step_points(F, t, capi.PART_INTERIOR)
        for p in plans:
            p.sync()
        a, b = plans[0].halo_blocks(F, t), plans[1].halo_blocks(F, t)
        plans[1].copy_halo(b["recv_lo"], a["send_hi"], a["count"])
        plans[0].copy_halo(a["recv_hi"], b["send_lo"], a["count"])
        for p in plans:
            p.sync()
    rec = np.zeros_like(rec1)
    for p in plans:
        p.step_end(F)
        rec += p.download_traces(capi.CLOUD_REC)
        p.close()
    assert np.array_equal(rec, rec1)


def test_gradient_imaging_at_full_size(full):
    """config 3: forward saving every 4th level in HBM, adjoint sweep driven by random
    residuals, fused imaging.  Properties here (zero in / zero out, linearity) and a VALUE
    check of a sub-volume around the source: the imaging condition
    grad -= u_saved[t] (v[t-1] - 2 v[t] + v[t+1]) / dt^2 (proj/src/seismic_ops.cpp:132)
    re-evaluated on the host in f64 from wavefield levels downloaded step by step through
    the stepping entry points.  (The whole gradient is compared with the oracle's sweep in
    tests/test_gpu_parity_fullsize.py.)"""
    from paper_1808_01995_b200 import capi
    model, geom = full
    plan = plan_for(model, geom)
    src = np.ascontiguousarray(geom.src.traces)
    rec, _ = plan.forward(src, save_every=4)
    rng = np.random.default_rng(18080199 + 10)
    resid = rng.standard_normal(rec.shape) * np.abs(rec).max() * np.hanning(geom.nt)[:, None]
    resid[[0, geom.nt - 1]] = 0.0
    g, rep = plan.gradient(resid)
    assert np.isfinite(g).all() and np.abs(g).max() > 0 and rep.steps == 48
    # zero residual -> exactly zero gradient (proj/tests/test_seismic.cpp:247-260)
    g0, _ = plan.gradient(np.zeros_like(resid))
    assert (g0 == 0.0).all()
    # linear in the residual
    g2, _ = plan.gradient(2.0 * resid)
    assert rel_l2(g2, 2.0 * g) <= 1e-7
    # value check on a sub-volume: saved forward levels and adjoint levels, one step at a time
    nt = geom.nt
    b = [int(x) for x in np.array(geom.src.base_table).reshape(-1, 3)[0]]
    box = tuple(slice(max(c - 12, 0), c + 12) for c in b)
    buf = np.zeros(plan.shape)
    saved = {t: plan.wavefield(t, out=buf)[box].copy() for t in range(4, nt - 1, 4)}
    G = capi.OP_ADJOINT   # the gradient sweep's wavefield is the adjoint run of the residual
    plan.upload_traces(capi.CLOUD_REC, resid)
    plan.step_begin(G)
    levels = {nt - 1: np.zeros_like(saved[4]), nt - 2: np.zeros_like(saved[4])}
    want = np.zeros_like(saved[4])
    inv_dt2 = 1.0 / geom.dt ** 2
    for t in range(nt - 2, 0, -1):
        plan.run_steps(G, t, t + 1)                    # writes level t-1
        levels[t - 1] = plan.wavefield(t - 1, out=buf)[box].copy()
        if t % 4 == 0:
            want -= saved[t] * (levels[t - 1] - 2.0 * levels[t] + levels[t + 1]) * inv_dt2
        levels.pop(t + 1)
    assert np.abs(want).max() > 0
    assert rel_l2(g[box], want) <= 1e-4
    plan.close()


def test_short_oracle_anchor_on_the_full_grid(full):
    """12 steps of the f64 oracle on the full 592^3 grid (a few seconds on the host)."""
    from oracle import oracle as o
    from paper_1808_01995_b200 import synthetic as syn
    model, geom = full
    cfg = syn.config(3, N_PHYS)
    om = o.Model(cfg["shape"], [H] * 3, [0.0] * 3, cfg["velocity"](), NBL, ORDER)
    nsteps = 12
    dt = geom.dt
    og = o.Geometry(om, np.asarray(cfg["src"]).ravel(), cfg["rec"].ravel(), 0.0, (nsteps + 1.5) * dt,
                    dt, 0.03)
    src = np.ascontiguousarray(geom.src.traces[: og.nt]) * 1e3  # early Ricker samples are tiny
    ref = o.forward(om, og, ORDER, src=src, want_final=True)
    from paper_1808_01995_b200 import capi
    plan = capi.Plan(om.N, om.spacing, ORDER, dt, og.nt)
    plan.set_model(om.m, om.damp, om.v_max)
    plan.set_points(capi.CLOUD_SRC, og.src_base, og.src_w)
    plan.set_points(capi.CLOUD_REC, og.rec_base, og.rec_w)
    rec, _ = plan.forward(src)
    assert np.abs(ref["smp"]).max() > 0
    assert rel_l2(rec, ref["smp"]) <= 1e-5
    assert rel_l2(plan.wavefield(og.nt - 1), ref["final"]) <= 1e-5
    plan.close()


def test_tti_properties_at_full_size(full):
    """Config 4's grid (592^3, order 12): the f64 oracle cannot run it in seconds, so the TTI
    pair is checked through size-independent properties -- linearity in the source, zero in /
    zero out, and the isotropic limit p == r."""
    from paper_1808_01995_b200 import capi
    model, geom0 = full
    N = list(model.grid.shape)
    steps = 24
    lin = [np.linspace(0.0, 1.0, n) for n in N]
    ones = np.ones(N)
    eps = 0.3 * lin[0][:, None, None] * ones
    delta = 0.2 * lin[1][None, :, None] * lin[0][:, None, None] * ones      # <= eps
    theta = (np.pi / 4) * lin[2][None, None, :] * ones
    phi = (np.pi / 4) * lin[1][None, :, None] * ones
    dt = 0.9 * capi.critical_dt(list(model.grid.spacing), model.v_max, 12) / np.sqrt(1.6)
    plan = capi.Plan(N, model.grid.spacing, 12, dt, steps + 2)
    plan.set_model(model.m.array(), model.damp.array(), model.v_max)
    plan.set_points(capi.CLOUD_SRC, np.array(geom0.src.base_table).reshape(-1, 3),
                    np.array(geom0.src.weight_table).reshape(-1, 8))
    plan.set_points(capi.CLOUD_REC, np.array(geom0.rec.base_table).reshape(-1, 3),
                    np.array(geom0.rec.weight_table).reshape(-1, 8))
    plan.set_model_tti(eps, delta, theta, phi)
    src = np.sin(np.arange(steps + 2) * 0.3).reshape(-1, 1)
    rec, rep = plan.tti_forward(src)
    assert rep.steps == steps and np.isfinite(rec).all() and np.abs(rec).max() > 0
    rec2, _ = plan.tti_forward(2.0 * src)
    assert rel_l2(rec2, 2.0 * rec) <= 1e-7
    zero, _ = plan.tti_forward(np.zeros_like(src))
    assert (zero == 0.0).all()
    # isotropic limit: the two fields of the pair coincide bit for bit
    z = np.zeros(N)
    plan.set_model_tti(z, z, z, z)
    plan.tti_forward(src)
    p = plan.wavefield(steps + 1, field=0)
    r = plan.wavefield(steps + 1, field=1)
    assert np.abs(p).max() > 0 and np.array_equal(p, r)
    plan.close()
