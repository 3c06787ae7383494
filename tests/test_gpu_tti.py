"""TTI forward operator on the GPU against the builder's own f64 oracle restatement.
The reference has no TTI operator: parity here is UNPINNED by the
reference; the pins are the self-checks the survey lists -- the isotropic limit reproduces
the acoustic operator, the wavefield does not grow over 500 steps, the layer dissipates."""
import numpy as np
import pytest

from oracle import oracle as o
from tests.common import make_plan, make_problem, rel_l2, smooth_field

pytestmark = pytest.mark.gpu


def tti_fields(N, seed=1):
    eps = smooth_field(N, seed + 1, 3.0, 0.0, 0.3)
    delta = np.minimum(smooth_field(N, seed + 2, 3.0, 0.0, 0.2), eps)  # eps >= delta
    theta = smooth_field(N, seed + 3, 3.0, 0.0, np.pi / 4)
    phi = smooth_field(N, seed + 4, 3.0, 0.0, np.pi / 4)
    return eps, delta, theta, phi


def tti_problem(shape, order, nsteps, nbl=8, h=10.0):
    model, geom0 = make_problem(shape, h, nbl, order, nsteps, dt_frac=0.5)
    dt = o.tti_critical_dt(model, order, 0.3)
    geom = o.Geometry(model, geom0.src_coords.ravel(), geom0.rec_coords.ravel(), 0.0,
                      (nsteps + 1.5) * dt, dt, 0.015)
    assert geom.nt == nsteps + 2
    return model, geom


@pytest.mark.parametrize("order", [4, 8, 12])
def test_tti_parity_with_oracle(order):
    model, geom = tti_problem([30, 26, 34], order, 100)
    eps, delta, theta, phi = tti_fields(model.N)
    ref = o.tti_forward(model, geom, order, eps, delta, theta, phi, want_final=True)
    plan = make_plan(model, geom, order)
    plan.set_model_tti(eps, delta, theta, phi)
    rec, rep = plan.tti_forward(geom.src)
    assert rep.steps == 100 and np.abs(ref["smp"]).max() > 0
    assert rel_l2(rec, ref["smp"]) <= 1e-5
    assert rel_l2(plan.wavefield(geom.nt - 1, field=0), ref["p"]) <= 1e-5
    assert rel_l2(plan.wavefield(geom.nt - 1, field=1), ref["r"]) <= 1e-5
    plan.close()


def test_tti_isotropic_limit_is_the_acoustic_operator():
    model, geom = make_problem([28, 24, 30], 10.0, 8, 8, 80, dt_frac=0.8)
    z = np.zeros(model.N)
    plan = make_plan(model, geom, 8)
    plan.set_model_tti(z, z, z, z)
    rec_t, _ = plan.tti_forward(geom.src)
    p = plan.wavefield(geom.nt - 1, field=0)
    r = plan.wavefield(geom.nt - 1, field=1)
    rec_a, _ = plan.forward(geom.src)
    u = plan.wavefield(geom.nt - 1)
    assert rel_l2(rec_t, rec_a) <= 2e-6 and rel_l2(p, u) <= 2e-6 and np.array_equal(p, r)
    plan.close()


def test_tti_no_growth_over_500_steps():
    model, geom = tti_problem([24, 22, 26], 8, 500, nbl=6)
    eps, delta, theta, phi = tti_fields(model.N, seed=7)
    plan = make_plan(model, geom, 8)
    plan.set_model_tti(eps, delta, theta, phi)
    rec, _ = plan.tti_forward(geom.src)
    ref = o.tti_forward(model, geom, 8, eps, delta, theta, phi, want_final=True)
    assert np.isfinite(rec).all()
    # late-time amplitude stays below the peak: no exponential growth
    assert np.abs(rec[400:]).max() <= np.abs(rec).max()
    assert rel_l2(rec, ref["smp"]) <= 1e-4                    # full run tolerance
    assert rel_l2(plan.wavefield(geom.nt - 1, field=0), ref["p"]) <= 1e-4
    plan.close()


def test_tti_rejects_ill_posed_medium_and_large_dt():
    from paper_1808_01995_b200 import capi
    model, geom = tti_problem([20, 20, 20], 8, 10, nbl=6)
    eps, delta, theta, phi = tti_fields(model.N)
    plan = make_plan(model, geom, 8)
    with pytest.raises(capi.SfbError) as e:
        plan.set_model_tti(delta * 0.5, delta + 0.01, theta, phi)   # eps < delta
    assert e.value.code == capi.ERR_STABILITY
    with pytest.raises(capi.SfbError) as e:
        plan.tti_forward(geom.src)                                   # fields never bound
    assert e.value.code == capi.ERR_BINDING
    plan.close()
    model2, geom2 = make_problem([20, 20, 20], 10.0, 6, 8, 10)       # acoustic critical dt
    plan = make_plan(model2, geom2, 8)
    with pytest.raises(capi.SfbError) as e:
        plan.set_model_tti(eps, delta, theta, phi)
    assert e.value.code == capi.ERR_STABILITY
    plan.close()


def test_tti_through_the_host_layer():
    from paper_1808_01995_b200 import _sfb_host as H
    n, h, nbl, order = 22, 10.0, 6, 8
    rng = np.random.default_rng(3)
    vel = rng.uniform(1.5, 3.0, size=(n, n, n))
    eps = rng.uniform(0.0, 0.3, size=(n, n, n))
    delta = np.minimum(rng.uniform(0.0, 0.2, size=(n, n, n)), eps)
    theta = rng.uniform(0.0, np.pi / 4, size=(n, n, n))
    phi = rng.uniform(0.0, np.pi / 4, size=(n, n, n))
    model = H.SeismicModel([n] * 3, [h] * 3, [0.0] * 3, vel, nbl, order)
    tti = H.TtiModel(model, eps, delta, theta, phi)
    dt = H.tti_critical_dt(model, tti, order)
    L = (n - 1) * h
    geom = H.AcquisitionGeometry(model, [0.5 * L + 1.0, 0.5 * L, 22.0],
                                 np.array([[x, 0.5 * L, 33.0] for x in np.linspace(0, L, 9)]).ravel(),
                                 0.0, 60.5 * dt, dt, 0.02)
    w = H.tti_forward_operator(model, tti, geom, order)
    rep = H.run_wave(w)
    assert rep.steps == geom.nt - 2
    om = o.Model([n] * 3, [h] * 3, [0.0] * 3, vel, nbl, order)
    og = o.Geometry(om, [0.5 * L + 1.0, 0.5 * L, 22.0],
                    np.array([[x, 0.5 * L, 33.0] for x in np.linspace(0, L, 9)]).ravel(), 0.0, 60.5 * dt, dt, 0.02)
    assert dt == pytest.approx(o.tti_critical_dt(om, order, tti.epsilon_max()), rel=1e-14)
    ref = o.tti_forward(om, og, order, tti.epsilon.array(), tti.delta.array(), tti.theta.array(),
                        tti.phi.array(), want_final=True)
    assert rel_l2(geom.rec.traces, ref["smp"]) <= 1e-5
    assert rel_l2(w.wavefield.array()[(geom.nt - 1) % 3], ref["p"]) <= 1e-5
    assert rel_l2(w.wavefield_r.array()[(geom.nt - 1) % 3], ref["r"]) <= 1e-5
    # the same operator on two slabs driven by this process: bit-identical
    rec1 = geom.rec.traces.copy()
    p1, r1 = w.wavefield.array().copy(), w.wavefield_r.array().copy()
    w2 = H.tti_forward_operator(model, tti, geom, order)
    geom.rec.traces[:] = 0.0
    rep2 = H.run_wave_slabs_tti(w2, model, tti, geom, [0, 0])
    assert rep2.steps == geom.nt - 2
    assert np.array_equal(geom.rec.traces, rec1)
    assert np.array_equal(w2.wavefield.array(), p1) and np.array_equal(w2.wavefield_r.array(), r1)
    geom2 = H.AcquisitionGeometry(model, [0.5 * L, 0.5 * L, 22.0], [10.0, 10.0, 10.0], 0.0, 60.5 * dt,
                                  1.2 * dt, 0.02)
    with pytest.raises(H.StabilityError):
        H.tti_forward_operator(model, tti, geom2, order)


def _run_tti_slabs(model, geom, order, fields, cuts, overlap_parts=True, pushed=False, stall=None):
    """N TTI plans on one device stepping in lockstep with device-to-device ghost copies:
    the single-GPU emulation of the two-exchange slab protocol (include/sfb200.h).  pushed:
    the plans are linked instead and every pass stores its boundary planes straight into the
    neighbours' ghost planes (no copies, no host synchronisation inside the loop)."""
    from paper_1808_01995_b200 import capi
    plans = [make_plan(model, geom, order, slab=(cuts[i], cuts[i + 1])) for i in range(len(cuts) - 1)]
    for p in plans:
        p.set_model_tti(*fields)
        p.upload_traces(capi.CLOUD_SRC, geom.src)
        p.step_begin(capi.OP_TTI_FORWARD)
    if pushed:
        nb = lambda i: [plans[j] for j in (i - 1, i + 1) if 0 <= j < len(plans)]   # noqa: E731
        for i, p in enumerate(plans):
            p.link_peers(plans[i - 1] if i > 0 else None, plans[i + 1] if i + 1 < len(plans) else None)
        for p in plans:
            p.sync()
        for t in range(1, geom.nt - 1):
            for i, p in enumerate(plans):
                if stall and i == stall[0]:
                    p.debug_stall(0, stall[1])
                p.tti_step_rot_fused(t)
            for i, p in enumerate(plans):
                for q in nb(i):
                    p.tti_peer_wait_g(q)
            for p in plans:
                p.tti_step_update_fused(t)
            for i, p in enumerate(plans):
                for q in nb(i):
                    p.peer_wait(q)
        return _collect_tti(plans, model, geom)

    def exchange(which, t):
        for p in plans:
            p.sync()
        for i in range(len(plans) - 1):
            a, b = plans[i].tti_halo_blocks(which, t), plans[i + 1].tti_halo_blocks(which, t)
            plans[i + 1].copy_halo(b["recv_lo"], a["send_hi"], a["count"])
            plans[i].copy_halo(a["recv_hi"], b["send_lo"], a["count"])
        for p in plans:
            p.sync()

    parts = ([capi.PART_LOW, capi.PART_HIGH, capi.PART_INTERIOR] if overlap_parts
             else [capi.PART_ALL])
    for t in range(1, geom.nt - 1):
        for p in plans:
            for part in parts:
                p.tti_step_rot(t, part)
        exchange(capi.TTI_HALO_G_P, t)
        exchange(capi.TTI_HALO_G_R, t)
        for p in plans:
            for part in parts:
                p.tti_step_update(t, part)
        exchange(capi.TTI_HALO_P, t)
        exchange(capi.TTI_HALO_R, t)
    return _collect_tti(plans, model, geom)


def _collect_tti(plans, model, geom):
    from paper_1808_01995_b200 import capi
    rec = np.zeros((geom.nt, geom.n_rec))
    pf, rf = np.zeros(model.N), np.zeros(model.N)
    for p in plans:
        p.step_end(capi.OP_TTI_FORWARD)
        rec += p.download_traces(capi.CLOUD_REC)
        p.wavefield(geom.nt - 1, out=pf, field=0)
        p.wavefield(geom.nt - 1, out=rf, field=1)
        p.close()
    return rec, pf, rf


@pytest.mark.parametrize("order,parts", [(8, True), (8, False), (12, True)])
def test_tti_slab_decomposition_matches_single_domain_bitwise(order, parts):
    """SURVEY.md 8e for the TTI pair: slabs along d0 with K ghost planes of p and r plus one
    exchange of the intermediate a g per step reproduce the single-domain run bit for bit
    (receivers straddling the cuts, the source next to one)."""
    model, geom = tti_problem([48, 26, 30], order, 40)
    fields = tti_fields(model.N, seed=3)
    plan = make_plan(model, geom, order)
    plan.set_model_tti(*fields)
    rec1, _ = plan.tti_forward(geom.src)
    p1 = plan.wavefield(geom.nt - 1, field=0)
    r1 = plan.wavefield(geom.nt - 1, field=1)
    plan.close()
    assert np.abs(rec1).max() > 0
    n0 = model.N[0]
    K = order // 2
    src_plane = int(geom.src_base[0][0])
    cuts = [0, 2 * K + 3, src_plane + 1, n0]      # the source cell straddles the second cut
    rec3, p3, r3 = _run_tti_slabs(model, geom, order, fields, cuts, overlap_parts=parts)
    assert np.array_equal(rec3, rec1)
    assert np.array_equal(p3, p1) and np.array_equal(r3, r1)


@pytest.mark.parametrize("order,stall", [(8, None), (12, None), (8, (1, 300)), (8, (0, 300))])
def test_tti_fused_halo_push_matches_single_domain_bitwise(order, stall):
    """Linked TTI slabs: each pass is one launch per slab whose edge chunks sweep towards the
    interior and push their boundary planes (g in the first pass, the new p and r in the
    second) into the neighbours' ghost planes; events order the slabs.  Bit for bit the
    single-domain run, also with one slab's stream held back 300 us every step."""
    model, geom = tti_problem([48, 26, 30], order, 40)
    fields = tti_fields(model.N, seed=3)
    plan = make_plan(model, geom, order)
    plan.set_model_tti(*fields)
    rec1, _ = plan.tti_forward(geom.src)
    p1 = plan.wavefield(geom.nt - 1, field=0)
    r1 = plan.wavefield(geom.nt - 1, field=1)
    plan.close()
    K = order // 2
    src_plane = int(geom.src_base[0][0])
    cuts = [0, 2 * K + 3, src_plane + 1, model.N[0]]
    rec3, p3, r3 = _run_tti_slabs(model, geom, order, fields, cuts, pushed=True, stall=stall)
    assert np.abs(rec1).max() > 0 and np.array_equal(rec3, rec1)
    assert np.array_equal(p3, p1) and np.array_equal(r3, r1)


def test_tti_step_loop_engine_single_rank():
    """slabs.tti_step_loop over slabs.TtiPlanEngine (two torch streams, the stream joins of
    the protocol) at world size 1 equals sfb_tti_forward bit for bit."""
    import torch
    from paper_1808_01995_b200 import capi, slabs
    model, geom = tti_problem([40, 26, 30], 8, 30)
    fields = tti_fields(model.N, seed=5)
    plan = make_plan(model, geom, 8)
    plan.set_model_tti(*fields)
    rec1, _ = plan.tti_forward(geom.src)
    p1 = plan.wavefield(geom.nt - 1, field=0)
    plan.close()
    plan = make_plan(model, geom, 8)
    plan.set_model_tti(*fields)
    plan.upload_traces(capi.CLOUD_SRC, geom.src)
    eng = slabs.TtiPlanEngine(plan, 0)
    with eng.interior():
        plan.step_begin(capi.OP_TTI_FORWARD)
    slabs.tti_step_loop(eng, slabs.HaloExchanger(0, 1), 1, geom.nt - 1)
    torch.cuda.synchronize()
    plan.step_end(capi.OP_TTI_FORWARD)
    assert np.array_equal(plan.download_traces(capi.CLOUD_REC), rec1)
    assert np.array_equal(plan.wavefield(geom.nt - 1, field=0), p1)
    plan.close()
