"""GPU parity: CUDA path (through the C-ABI) vs the f64 CPU oracle on the same seeded inputs.

Tolerances are BASELINE.json's: wavefields and traces rel-L2 <= 1e-5 after 100 steps and
<= 1e-4 after a full run; gradients <= 1e-3; dot test <= 1e-4 (fp32 arithmetic against an
f64 oracle)."""
import numpy as np
import pytest

from oracle import oracle as o
from tests.common import make_plan, make_problem, rel_l2

pytestmark = pytest.mark.gpu


def _forward_both(shape, h, nbl, order, nsteps, **kw):
    model, geom = make_problem(shape, h, nbl, order, nsteps, **kw)
    ref = o.forward(model, geom, order, want_final=True)
    plan = make_plan(model, geom, order)
    rec, rep = plan.forward(geom.src)
    u = plan.wavefield(geom.nt - 1)
    up = plan.wavefield(geom.nt - 2)
    return model, geom, ref, plan, rec, u, up, rep


@pytest.mark.parametrize("order", [2, 4, 6, 8, 10, 12, 14, 16])
def test_forward_parity_3d_orders(order):
    _, geom, ref, plan, rec, u, up, rep = _forward_both([40, 36, 44], 10.0, 8, order, 100)
    assert rep.steps == 100 and rep.kernel_launches == 200
    assert np.abs(ref["smp"]).max() > 0
    assert rel_l2(rec, ref["smp"]) <= 1e-5
    assert rel_l2(u, ref["final"]) <= 1e-5
    assert rel_l2(up, ref["prev"]) <= 1e-5
    assert (rec[[0, 1, geom.nt - 1]] == 0.0).all()  # structural zeros, seismic_ops.hpp:13-16
    plan.close()


def test_forward_parity_ragged_sizes():
    # extents that are not multiples of any tile or of 4
    _, _, ref, plan, rec, u, _, _ = _forward_both([37, 45, 53], 12.5, 9, 8, 80)
    assert rel_l2(rec, ref["smp"]) <= 1e-5 and rel_l2(u, ref["final"]) <= 1e-5
    plan.close()


def test_forward_parity_2d():
    _, _, ref, plan, rec, u, _, _ = _forward_both([70, 90], 10.0, 10, 4, 120)
    assert rel_l2(rec, ref["smp"]) <= 1e-5 and rel_l2(u, ref["final"]) <= 1e-5
    plan.close()


def test_forward_long_run_two_layer():
    # config-1 style medium (two layers split on the depth axis), 400 steps
    shape = [41, 41, 41]
    vel = np.empty(shape)
    vel[..., :20] = 1.5
    vel[..., 20:] = 2.5
    _, _, ref, plan, rec, u, _, _ = _forward_both(shape, 10.0, 20, 4, 400, vel=vel, f0=0.01)
    assert rel_l2(rec, ref["smp"]) <= 1e-4 and rel_l2(u, ref["final"]) <= 1e-4
    plan.close()


def test_tile_shapes_agree_bitwise():
    model, geom = make_problem([40, 36, 44], 10.0, 8, 8, 40)
    plan = make_plan(model, geom, 8)
    base, _ = plan.forward(geom.src)
    u0 = plan.wavefield(geom.nt - 1)
    for tile in [(16, 16, 8), (32, 8, 7), (16, 32, 7), (32, 16, 7), (16, 16, -3), (16, 16, -4), (32, 8, -3), (16, 16, -103)]:
        for chunk in (0, 7, 60):
            plan.set_tile(*tile, chunk)
            rec, _ = plan.forward(geom.src)
            assert np.array_equal(rec, base)
            assert np.array_equal(plan.wavefield(geom.nt - 1), u0)
    plan.close()


def test_dense_and_separable_damping_agree():
    from paper_1808_01995_b200 import capi
    model, geom = make_problem([40, 36, 44], 10.0, 8, 8, 60)
    plan = make_plan(model, geom, 8)
    assert plan.get_tile()["sep"] == 1  # build_damping is a sum of 1-D profiles
    rec_s, _ = plan.forward(geom.src)
    u_s = plan.wavefield(geom.nt - 1)
    plan.close()
    dense = capi.Plan(model.N, model.spacing, 8, geom.dt, geom.nt, dense_damping=True)
    dense.set_model(model.m, model.damp, model.v_max)
    dense.set_points(capi.CLOUD_SRC, geom.src_base, geom.src_w)
    dense.set_points(capi.CLOUD_REC, geom.rec_base, geom.rec_w)
    assert dense.get_tile()["sep"] == 0
    rec_d, _ = dense.forward(geom.src)
    ref = o.forward(model, geom, 8, want_final=True)
    assert rel_l2(rec_d, ref["smp"]) <= 1e-5 and rel_l2(dense.wavefield(geom.nt - 1), ref["final"]) <= 1e-5
    assert rel_l2(rec_s, rec_d) <= 1e-6 and rel_l2(u_s, dense.wavefield(geom.nt - 1)) <= 1e-6
    # a damping field that is not separable must fall back to the dense stream
    bumpy = model.damp.copy()
    bumpy[5, 7, 9] += 0.01
    dense.set_dense_damping(False)
    dense.set_model(model.m, bumpy, model.v_max)
    assert dense.get_tile()["sep"] == 0
    dense.close()


def test_autotune_keeps_results_and_picks_a_compiled_shape():
    model, geom = make_problem([40, 36, 44], 10.0, 8, 12, 30)
    plan = make_plan(model, geom, 12)
    base, _ = plan.forward(geom.src)
    t = plan.autotune(3)
    assert t["txv"] in (16, 32) and t["chunk"] >= 1
    rec, _ = plan.forward(geom.src)
    assert np.array_equal(rec, base)
    plan.close()


def test_zero_source_gives_zero_receivers():  # proj/tests/test_seismic.cpp:165-174
    model, geom = make_problem([24, 24, 24], 10.0, 6, 8, 50)
    plan = make_plan(model, geom, 8)
    rec, _ = plan.forward(np.zeros_like(geom.src))
    assert (rec == 0.0).all() and (plan.wavefield(geom.nt - 1) == 0.0).all()
    plan.close()


def test_adjoint_parity_and_dot_test():  # proj/src/verify.cpp:201-253
    model, geom = make_problem([36, 32, 40], 10.0, 8, 6, 120, f0=0.01, dt_frac=0.8)
    o.forward(model, geom, 6)
    ref = o.adjoint(model, geom, 6, want_final=True)
    plan = make_plan(model, geom, 6)
    rec, _ = plan.forward(geom.src)
    assert rel_l2(rec, geom.rec) <= 1e-5
    srca, _ = plan.adjoint(geom.rec)
    assert rel_l2(srca, ref["smp"]) <= 1e-4
    assert rel_l2(plan.wavefield(0), ref["final"]) <= 1e-4
    # <F q, d> vs <q, F^T d> with d = F q, all on the GPU path
    srca_gpu, _ = plan.adjoint(rec)
    fdot = float((rec ** 2).sum())
    adot = float((geom.src * srca_gpu).sum())
    assert fdot > 0 and abs(fdot - adot) / fdot <= 1e-4
    plan.close()


@pytest.mark.parametrize("save_every", [1, 4])
def test_gradient_parity(save_every):
    model, geom = make_problem([30, 28, 34], 10.0, 8, 8, 96, dt_frac=0.9)
    o.forward(model, geom, 8)
    rng = np.random.default_rng(5)
    observed = geom.rec + 0.1 * np.abs(geom.rec).max() * rng.standard_normal(geom.rec.shape)
    observed[[0, 1, geom.nt - 1]] = 0.0
    phi, gref, resid = o.fwi_gradient(model, geom, observed, 8, save_every)
    plan = make_plan(model, geom, 8)
    rec, _ = plan.forward(geom.src, save_every=save_every)
    g, rep = plan.gradient(rec - observed)
    gfold = o.fold_gradient(model, g)
    assert np.abs(gref).max() > 0
    assert rel_l2(gfold, gref) <= 1e-3
    assert o.objective(rec, observed) == pytest.approx(phi, rel=1e-4)
    plan.close()


@pytest.mark.parametrize("nt,C", [(96, 7), (96, 16), (50, 2), (41, 40), (30, 64)])
def test_checkpointed_gradient_equals_full_history(nt, C):
    # recompute strategy: same kernels in the same order, so the gradient is the full-history
    # (save_every = 1, the reference's imaging condition) gradient bit for bit
    model, geom = make_problem([30, 28, 34], 10.0, 8, 8, nt, dt_frac=0.9)
    rng = np.random.default_rng(5)
    plan = make_plan(model, geom, 8)
    rec, _ = plan.forward(geom.src, save_every=1)
    resid = rec + 0.1 * np.abs(rec).max() * rng.standard_normal(rec.shape)
    g_full, _ = plan.gradient(resid)
    rec_c, _ = plan.forward_checkpointed(geom.src, C)
    g_ck, rep = plan.gradient(resid)
    assert np.array_equal(rec_c, rec)
    assert np.abs(g_full).max() > 0
    assert np.array_equal(g_ck, g_full)
    assert rep.steps == geom.nt - 2
    # a second gradient from the same checkpoints, and a plain forward invalidates them
    g_again, _ = plan.gradient(0.5 * resid)
    assert rel_l2(g_again, 0.5 * g_full) <= 1e-6
    plan.forward(geom.src)
    from paper_1808_01995_b200 import capi
    with pytest.raises(capi.SfbError):
        plan.gradient(resid)
    plan.close()


@pytest.mark.parametrize("order", [12, 14, 16])
def test_patch_kernel_agrees_bitwise_with_the_dual_stream_kernel(order):
    """acoustic_patch_kernel.cuh (2 x 2 nodes per thread, queue window slid by two planes) and
    acoustic_tall_kernel.cuh (2 x 4 nodes per thread) keep the arithmetic and its order per node: forward with snapshots, adjoint and the
    gradient with fused imaging equal the dual-stream kernel bit for bit, separable and dense
    damping, ragged extents, several d0 chunks."""
    from paper_1808_01995_b200 import capi
    model, geom = make_problem([75, 53, 67], 10.0, 9, order, 30, dt_frac=0.9, n_rec_line=40)
    data = np.random.default_rng(2).standard_normal((geom.nt, geom.n_rec)) * np.hanning(geom.nt)[:, None]
    for dense in (False, True):
        plan = capi.Plan(model.N, model.spacing, order, geom.dt, geom.nt, dense_damping=dense)
        plan.set_model(model.m, model.damp, model.v_max)
        plan.set_points(capi.CLOUD_SRC, geom.src_base, geom.src_w)
        plan.set_points(capi.CLOUD_REC, geom.rec_base, geom.rec_w)
        out = {}
        rows = 14 if order >= 14 else 16
        tiles = [("dual", (16, rows, -4)), ("patch", (16, 14, -204)), ("slide", (16, rows, -304))]
        if order >= 14:   # two rows of four nodes per thread (acoustic_tall_kernel.cuh)
            tiles += [("tall", (16, 28, -404))]
        for name, tile in tiles:
            for chunk in (0, 11):
                plan.set_tile(*tile, chunk)
                assert plan.get_tile()["stages"] == tile[2]
                rec, _ = plan.forward(geom.src, save_every=2)
                u = plan.wavefield(geom.nt - 1)
                g, _ = plan.gradient(data)
                srca, _ = plan.adjoint(data)
                out[(name, chunk)] = (rec, u, g, srca, plan.wavefield(0))
        ref = out[("dual", 0)]
        assert np.abs(ref[0]).max() > 0 and np.abs(ref[2]).max() > 0
        for key, val in out.items():
            for a, b in zip(val, ref):
                assert np.array_equal(a, b), (order, dense, key)
        plan.close()


@pytest.mark.parametrize("order,tile", [(8, None), (8, (16, 16, -3)), (12, None), (4, None),
                                        (16, (16, 14, -204))])
def test_gradient_runs_are_bitwise_repeatable(order, tile):
    """Regression for a pipeline race found at sizes that fill the SMs with several blocks:
    a stage was released to the TMA producer while a warp's shared-memory loads were still
    in flight, so single rows of a plane came out one pipeline round too new, differently
    from run to run, once the imaging traffic stretched the warps apart.  A dense carpet of
    injection points and six repeats expose it (tools/probe_determinism4.py)."""
    shape, h = [560, 128, 96], 10.0
    ii, jj = np.meshgrid(np.arange(0, shape[0] - 1, 2), np.arange(0, shape[1] - 1, 2), indexing="ij")
    rec = np.stack([ii.ravel() * h + 0.3 * h, jj.ravel() * h + 0.4 * h,
                    np.full(ii.size, 4.5 * h)], axis=1)
    model, geom = make_problem(shape, h, 8, order, 6, dt_frac=0.9, rec=rec)
    plan = make_plan(model, geom, order)
    if tile:
        plan.set_tile(*tile)
    rec_tr, _ = plan.forward(geom.src, save_every=1)
    resid = np.random.default_rng(5).standard_normal(rec_tr.shape)
    g0, _ = plan.gradient(resid)
    v0 = plan.wavefield(0)
    assert np.abs(g0).max() > 0
    for _ in range(5):
        g, _ = plan.gradient(resid)
        assert np.array_equal(plan.wavefield(0), v0)
        assert np.array_equal(g, g0)
    plan.close()


def test_checkpoint_interval_is_checked():
    from paper_1808_01995_b200 import capi
    model, geom = make_problem([20, 20, 20], 10.0, 6, 8, 20)
    plan = make_plan(model, geom, 8)
    with pytest.raises(capi.SfbError) as e:
        plan.forward_checkpointed(geom.src, 1)
    assert e.value.code == capi.ERR_PARAMETER
    plan.close()


def test_zero_residual_gives_zero_gradient():  # proj/tests/test_seismic.cpp:247-260
    model, geom = make_problem([20, 20, 20], 10.0, 6, 8, 40)
    plan = make_plan(model, geom, 8)
    rec, _ = plan.forward(geom.src, save_every=1)
    g, _ = plan.gradient(np.zeros_like(rec))
    assert (g == 0.0).all()
    plan.close()


def test_gradient_requires_history():  # proj/src/seismic_ops.cpp:113-114
    from paper_1808_01995_b200 import capi
    model, geom = make_problem([20, 20, 20], 10.0, 6, 8, 10)
    plan = make_plan(model, geom, 8)
    plan.forward(geom.src)
    with pytest.raises(capi.SfbError) as e:
        plan.gradient(np.zeros((geom.nt, geom.n_rec)))
    assert e.value.code == capi.ERR_PARAMETER
    plan.close()


def test_unstable_dt_and_nan_guard():
    from paper_1808_01995_b200 import capi
    model, geom = make_problem([20, 20, 20], 10.0, 6, 8, 60)
    plan = capi.Plan(model.N, model.spacing, 8, geom.dt * 1.5, geom.nt)
    with pytest.raises(capi.SfbError) as e:  # check_cfl, seismic_ops.cpp:15-22
        plan.set_model(model.m, model.damp, model.v_max)
    assert e.value.code == capi.ERR_STABILITY
    # with the gate skipped the run itself blows up and the NaN guard fires
    plan2 = capi.Plan(model.N, model.spacing, 8, geom.dt * 4.0, 400)
    plan2.set_model(model.m, model.damp, 0.0)
    plan2.set_points(capi.CLOUD_SRC, geom.src_base, geom.src_w)
    plan2.set_points(capi.CLOUD_REC, geom.rec_base, geom.rec_w)
    with pytest.raises(capi.SfbError) as e:
        plan2.forward(np.ones((400, 1)))
    assert e.value.code == capi.ERR_STABILITY
    plan.close()
    plan2.close()


def _run_slabs(model, geom, order, cuts, op=None, save_every=0, inj=None, prior_forward=False,
               fused=False, pushed=False, stall=None, single_launch=False):
    """N plans on one device stepping in lockstep with device-to-device ghost copies:
    the single-GPU emulation of the multi-GPU slab protocol.  Returns the summed sampled
    traces, the assembled last level and (gradient) the assembled grad."""
    from paper_1808_01995_b200 import capi
    op = capi.OP_FORWARD if op is None else op
    backward = op != capi.OP_FORWARD
    plans = [make_plan(model, geom, order, slab=(cuts[i], cuts[i + 1])) for i in range(len(cuts) - 1)]
    if pushed:   # fused halo push: boundary planes go straight into the neighbours' ghosts
        for i, p in enumerate(plans):
            p.link_peers(plans[i - 1] if i > 0 else None, plans[i + 1] if i + 1 < len(plans) else None)

    def sweep(o, traces_cloud, traces, se):
        for p in plans:
            p.upload_traces(traces_cloud, traces)
            p.step_begin(o, se)
        ts = range(geom.nt - 2, 0, -1) if o != capi.OP_FORWARD else range(1, geom.nt - 1)
        for t in ts:
            if pushed:   # no copies and no host synchronisation: events order the slabs
                for i, p in enumerate(plans):
                    if single_launch:   # sfb_step_slab_fused: one update launch per step
                        if stall and i == stall[0]:
                            p.debug_stall(0, stall[1])
                        p.step_slab_fused(o, t)
                        continue
                    p.step_slab_boundary(o, t)
                    if stall and i == stall[0]:   # hold this slab's main stream back
                        p.debug_stall(0, stall[1])
                    p.step_slab_interior(o, t)
                for i, p in enumerate(plans):
                    if i > 0:
                        p.peer_wait(plans[i - 1])
                    if i + 1 < len(plans):
                        p.peer_wait(plans[i + 1])
                continue
            for p in plans:
                if fused:   # the two native half-step calls of slabs.PlanEngine
                    p.step_slab_boundary(o, t)
                    p.step_slab_interior(o, t)
                    continue
                p.step_compute(o, t, capi.PART_LOW)
                p.step_compute(o, t, capi.PART_HIGH)
                p.step_points(o, t, capi.PART_LOW)
                p.step_compute(o, t, capi.PART_INTERIOR)
                p.step_points(o, t, capi.PART_INTERIOR)
            for p in plans:
                p.sync()
            for i in range(len(plans) - 1):
                a, b = plans[i].halo_blocks(o, t), plans[i + 1].halo_blocks(o, t)
                plans[i + 1].copy_halo(b["recv_lo"], a["send_hi"], a["count"])
                plans[i].copy_halo(a["recv_hi"], b["send_lo"], a["count"])
            for p in plans:
                p.sync()
        for p in plans:
            p.step_end(o)

    if prior_forward:  # the gradient sweep images against each slab's own saved history
        sweep(capi.OP_FORWARD, capi.CLOUD_SRC, geom.src, save_every)
    sweep(op, capi.CLOUD_REC if backward else capi.CLOUD_SRC, geom.src if inj is None else inj,
          save_every)
    smp_cloud = capi.CLOUD_SRC if backward else capi.CLOUD_REC
    n_smp = geom.n_src if backward else geom.n_rec
    rec = np.zeros((geom.nt, n_smp))
    u = np.zeros(model.N)
    grad = np.zeros(model.N)
    for p in plans:
        if op != capi.OP_GRADIENT:
            rec += p.download_traces(smp_cloud)
        p.wavefield(0 if backward else geom.nt - 1, out=u)
        if op == capi.OP_GRADIENT:
            import ctypes as C
            p._chk(capi.lib.sfb_get_gradient(p.h, C.byref(capi._view(grad))))
        p.close()
    return rec, u, grad


@pytest.mark.parametrize("single_launch", [False, True])
@pytest.mark.parametrize("order,shape,nslab", [(8, [48, 30, 34], 3), (16, [64, 30, 34], 2),
                                               (12, [64, 30, 34], 2), (4, [70, 30, 34], 3)])
def test_fused_halo_push_matches_single_domain_bitwise(order, shape, nslab, single_launch):
    """sfb_link_peers: the boundary kernels store their planes (and the point kernel its
    injected nodes) directly into the neighbours' ghost planes; slabs are ordered by events
    only.  Forward, adjoint and gradient equal the single-domain run bit for bit (ring
    kernel at order 8, dual-stream kernels with 16- and 14-row tiles above)."""
    from paper_1808_01995_b200 import capi
    model, geom = make_problem(shape, 10.0, 8, order, 50)
    rng = np.random.default_rng(9)
    data = rng.standard_normal((geom.nt, geom.n_rec)) * np.hanning(geom.nt)[:, None]
    plan = make_plan(model, geom, order)
    rec1, _ = plan.forward(geom.src)
    u1 = plan.wavefield(geom.nt - 1)
    srca1, _ = plan.adjoint(data)
    v1 = plan.wavefield(0)
    plan.forward(geom.src, save_every=2)
    g1, _ = plan.gradient(data)
    plan.close()
    n0 = model.N[0]
    src_plane = int(geom.src_base[0][0])
    cuts = [0, 20, src_plane + 1, n0] if nslab == 3 else [0, src_plane + 1, n0]   # source on a cut
    sl = dict(pushed=True, single_launch=single_launch)
    rec3, u3, _ = _run_slabs(model, geom, order, cuts, **sl)
    assert np.array_equal(rec3, rec1) and np.array_equal(u3, u1)
    srca3, v3, _ = _run_slabs(model, geom, order, cuts, op=capi.OP_ADJOINT, inj=data, **sl)
    assert np.array_equal(srca3, srca1) and np.array_equal(v3, v1)
    _, _, g3 = _run_slabs(model, geom, order, cuts, op=capi.OP_GRADIENT, save_every=2, inj=data,
                          prior_forward=True, **sl)
    assert np.abs(g1).max() > 0 and np.array_equal(g3, g1)


@pytest.mark.parametrize("single_launch", [False, True])
@pytest.mark.parametrize("slow_slab", [0, 1])
def test_fused_halo_push_waits_for_the_ghost_plane_readers(slow_slab, single_launch):
    """A receiver cell that straddles a slab cut is gathered by the slab below, which reads
    its high ghost plane in the interior half-step.  The neighbour's next boundary half-step
    overwrites that plane, so it must wait for the gather, not only for the boundary
    half-step (round-1 advisor finding): one slab's main stream is held back 300 us every
    step, off-node receivers sit in the last plane below each cut."""
    from paper_1808_01995_b200 import capi
    shape, h, nbl = [48, 30, 34], 10.0, 8
    cuts = [0, 22, 43, shape[0] + 2 * nbl]
    rec = [[(c - 1 - nbl + 0.4) * h, 0.5 * (shape[1] - 1) * h, 4.5 * h] for c in cuts[1:-1]]
    rec += [[(c - nbl + 0.3) * h, 0.45 * (shape[1] - 1) * h, 3.2 * h] for c in cuts[1:-1]]
    model, geom = make_problem(shape, h, nbl, 8, 40, rec=rec)
    assert sorted(int(b[0]) for b in geom.rec_base)[:2] == [cuts[1] - 1, cuts[1]]
    plan = make_plan(model, geom, 8)
    rec1, _ = plan.forward(geom.src)
    u1 = plan.wavefield(geom.nt - 1)
    plan.close()
    assert np.abs(rec1).min(axis=0).max() >= 0 and (np.abs(rec1).max(axis=0) > 0).all()
    rec3, u3, _ = _run_slabs(model, geom, 8, cuts, pushed=True, stall=(slow_slab, 300),
                             single_launch=single_launch)
    assert np.array_equal(rec3, rec1) and np.array_equal(u3, u1)
    # the adjoint samples at the source cell: put it across the first cut as well
    src = [[(cuts[1] - 1 - nbl + 0.37) * h, 0.5 * (shape[1] - 1) * h, 2.13 * h]]
    model, geom = make_problem(shape, h, nbl, 8, 40, rec=rec, src=src)
    data = np.random.default_rng(3).standard_normal((geom.nt, geom.n_rec)) * np.hanning(geom.nt)[:, None]
    plan = make_plan(model, geom, 8)
    srca1, _ = plan.adjoint(data)
    plan.close()
    srca3, _, _ = _run_slabs(model, geom, 8, cuts, op=capi.OP_ADJOINT, inj=data, pushed=True,
                             stall=(slow_slab, 300), single_launch=single_launch)
    assert np.abs(srca1).max() > 0 and np.array_equal(srca3, srca1)


def test_link_peers_checks_the_neighbours():
    from paper_1808_01995_b200 import capi
    model, geom = make_problem([48, 30, 34], 10.0, 8, 8, 10)
    n0 = model.N[0]
    a = make_plan(model, geom, 8, slab=(0, 20))
    b = make_plan(model, geom, 8, slab=(20, 41))
    c = make_plan(model, geom, 8, slab=(41, n0))
    b.link_peers(a, c)
    with pytest.raises(capi.SfbError) as e:      # c is not the slab below b
        b.link_peers(c, a)
    assert e.value.code == capi.ERR_PARAMETER
    with pytest.raises(capi.SfbError):           # a does not touch c
        a.link_peers(None, c)
    b.link_peers(None, None)                      # unlink
    for p in (a, b, c):
        p.close()


@pytest.mark.parametrize("fused", [False, True])
def test_slab_decomposition_matches_single_domain_bitwise(fused):
    model, geom = make_problem([48, 30, 34], 10.0, 8, 8, 60)
    plan = make_plan(model, geom, 8)
    rec1, _ = plan.forward(geom.src)
    u1 = plan.wavefield(geom.nt - 1)
    plan.close()
    n0 = model.N[0]
    rec3, u3, _ = _run_slabs(model, geom, 8, [0, 20, 41, n0], fused=fused)
    assert np.array_equal(rec3, rec1) and np.array_equal(u3, u1)


def test_slab_decomposition_adjoint_and_gradient_bitwise():
    from paper_1808_01995_b200 import capi
    model, geom = make_problem([48, 30, 34], 10.0, 8, 8, 40)
    rng = np.random.default_rng(9)
    data = rng.standard_normal((geom.nt, geom.n_rec)) * np.hanning(geom.nt)[:, None]
    plan = make_plan(model, geom, 8)
    srca1, _ = plan.adjoint(data)
    v1 = plan.wavefield(0)
    plan.forward(geom.src, save_every=2)
    g1, _ = plan.gradient(data)
    plan.close()
    n0 = model.N[0]
    for fused in (False, True):
        srca3, v3, _ = _run_slabs(model, geom, 8, [0, 20, 41, n0], op=capi.OP_ADJOINT, inj=data,
                                  fused=fused)
        assert np.array_equal(srca3, srca1) and np.array_equal(v3, v1)
        _, _, g3 = _run_slabs(model, geom, 8, [0, 20, 41, n0], op=capi.OP_GRADIENT, save_every=2,
                              inj=data, prior_forward=True, fused=fused)
        assert np.abs(g1).max() > 0 and np.array_equal(g3, g1)


def test_step_loop_engine_on_one_rank_matches_forward():
    """slabs.step_loop + PlanEngine (the multi-GPU driver) with a single slab and no
    neighbours must reproduce sfb_forward exactly."""
    import torch
    from paper_1808_01995_b200 import capi, slabs
    model, geom = make_problem([40, 30, 34], 10.0, 8, 8, 50)
    plan = make_plan(model, geom, 8)
    rec1, _ = plan.forward(geom.src)
    u1 = plan.wavefield(geom.nt - 1)
    plan.close()

    plan = make_plan(model, geom, 8)
    plan.upload_traces(capi.CLOUD_SRC, geom.src)
    eng = slabs.PlanEngine(plan, capi.OP_FORWARD, 0)
    plan.step_begin(capi.OP_FORWARD)
    slabs.step_loop(eng, slabs.HaloExchanger(0, 1), 1, geom.nt - 1)
    torch.cuda.synchronize()
    plan.step_end(capi.OP_FORWARD)
    assert np.array_equal(plan.download_traces(capi.CLOUD_REC), rec1)
    assert np.array_equal(plan.wavefield(geom.nt - 1), u1)
    plan.close()


def test_streamed_traces_with_many_receivers():
    # enough receivers that the trace table leaves in several pinned chunks
    from paper_1808_01995_b200 import capi
    model, geom = make_problem([24, 24, 24], 10.0, 6, 4, 30)
    n = 36
    L = model.spacing[0] * (model.shape[0] - 1)
    xs = np.linspace(0.0, L, n)
    rec = np.array([[x, y, 25.0] for x in xs for y in xs] * 260)  # 336960 points
    geom2 = o.Geometry(model, geom.src_coords.ravel(), rec.ravel(), 0.0, geom.tn, geom.dt, geom.f0)
    ref = o.forward(model, geom2, 4)
    plan = make_plan(model, geom2, 4)
    got, _ = plan.forward(geom2.src)
    assert rel_l2(got, ref["smp"]) <= 1e-5
    assert (got[[0, geom2.nt - 1]] == 0.0).all()
    plan.upload_traces(capi.CLOUD_SRC, geom2.src)
    plan.run_resident(capi.OP_FORWARD)
    assert np.array_equal(plan.download_traces(capi.CLOUD_REC), got)
    plan.close()


def test_forward_parity_1d_and_tiny_grids():
    # rank-1 grids (the reference's Grid allows ranks 1-3, proj/include/sf/grid.hpp:34-35)
    _, _, ref, plan, rec, u, _, _ = _forward_both([60], 10.0, 12, 4, 90)
    assert np.abs(ref["smp"]).max() > 0
    assert rel_l2(rec, ref["smp"]) <= 1e-5 and rel_l2(u, ref["final"]) <= 1e-5
    plan.close()
    # grids smaller than one tile and than the stencil radius
    for shape, order in (([3, 2, 4], 2), ([2, 2], 2), ([5, 4, 3], 8), ([2], 16)):
        nd = len(shape)
        src = [0.3 * 10.0 * (s - 1) for s in shape]
        rec_c = [[0.0] * nd, [10.0 * (s - 1) for s in shape]]
        _, _, ref, plan, rec, u, _, _ = _forward_both(shape, 10.0, 1, order, 25, src=src, rec=rec_c)
        assert np.abs(ref["final"]).max() > 0
        assert rel_l2(rec, ref["smp"]) <= 1e-5 and rel_l2(u, ref["final"]) <= 1e-5
        plan.close()


def test_concurrent_plans_from_two_threads():
    """the C-ABI is re-entrant per plan (proj/tests/test_compiler.cpp:559-578 runs distinct
    operators concurrently; fwi calls fwi_gradient from several threads)"""
    import threading
    probs = [make_problem([30, 26, 34], 10.0, 8, 8, 60), make_problem([28, 32, 24], 12.5, 6, 4, 70)]
    orders = [8, 4]
    serial = []
    for (m, g), k in zip(probs, orders):
        p = make_plan(m, g, k)
        serial.append(p.forward(g.src)[0])
        p.close()
    out = [None, None]

    def work(i):
        m, g = probs[i]
        p = make_plan(m, g, orders[i])
        for _ in range(3):
            out[i] = p.forward(g.src)[0]
        p.close()

    th = [threading.Thread(target=work, args=(i,)) for i in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert np.array_equal(out[0], serial[0]) and np.array_equal(out[1], serial[1])


def test_step_entry_points_reject_bad_operators_with_a_status():
    """Round-1 advisor finding: stepping the gradient operator without a bound history
    divided by save_every = 0 (SIGFPE across the C ABI), and the acoustic step accepted the
    TTI operator id.  Both are parameter errors now."""
    from paper_1808_01995_b200 import capi
    model, geom = make_problem([24, 24, 24], 10.0, 6, 8, 10)
    plan = make_plan(model, geom, 8)
    plan.upload_traces(capi.CLOUD_SRC, geom.src)
    plan.upload_traces(capi.CLOUD_REC, geom.rec)
    plan.step_begin(capi.OP_FORWARD)
    for call in (lambda: plan.step_compute(capi.OP_GRADIENT, 3, capi.PART_ALL),
                 lambda: plan.step_points(capi.OP_GRADIENT, 3, capi.PART_ALL),
                 lambda: plan.run_steps(capi.OP_GRADIENT, 1, 3),
                 lambda: plan.time_stencil(capi.OP_GRADIENT, 1, 3),
                 lambda: plan.step_compute(capi.OP_TTI_FORWARD, 3, capi.PART_ALL),
                 lambda: plan.step_points(capi.OP_TTI_FORWARD, 3, capi.PART_ALL),
                 lambda: plan.step_slab_boundary(capi.OP_TTI_FORWARD, 3)):
        with pytest.raises(capi.SfbError) as e:
            call()
        assert e.value.code == capi.ERR_PARAMETER
    plan.autotune(2)   # zeroes save_every; the plan must still refuse, not crash
    with pytest.raises(capi.SfbError):
        plan.run_steps(capi.OP_GRADIENT, 1, 3)
    plan.close()


def test_fed_and_resident_trace_tables_agree():
    """sfb_adjoint / sfb_gradient feed the receiver table to the device chunk by chunk while the
    sweep runs; with the whole table uploaded first (sfb_upload_traces + sfb_run_resident) the
    results are the same bit for bit.  30 000 receivers: 8 rows per chunk, several chunks in
    both sweep directions."""
    from paper_1808_01995_b200 import capi
    shape, order, nsteps = [40, 36, 30], 8, 37
    rng = np.random.default_rng(5)
    L = [(s - 1) * 10.0 for s in shape]
    rec_xyz = rng.uniform(0.0, 1.0, size=(30000, 3)) * np.asarray(L)
    model, geom = make_problem(shape, 10.0, 6, order, nsteps, rec=rec_xyz)
    plan = make_plan(model, geom, order)
    data = rng.standard_normal((geom.nt, rec_xyz.shape[0]))
    data[[0, geom.nt - 1]] = 0.0
    srca_fed, _ = plan.adjoint(data)
    plan.upload_traces(capi.CLOUD_REC, data)
    plan.run_resident(capi.OP_ADJOINT)
    srca_res = plan.download_traces(capi.CLOUD_SRC)
    assert np.abs(srca_fed).max() > 0
    assert np.array_equal(srca_fed[1:-1], srca_res[1:-1])
    plan.forward(geom.src, save_every=1)
    grad_fed, _ = plan.gradient(data)
    plan.upload_traces(capi.CLOUD_REC, data)
    plan.run_resident(capi.OP_GRADIENT, 1)
    import ctypes as C
    grad_res = np.zeros(model.N)
    plan._chk(capi.lib.sfb_get_gradient(plan.h, C.byref(capi._view(grad_res))))
    assert np.abs(grad_fed).max() > 0
    assert np.array_equal(grad_fed, grad_res)
    plan.close()


def test_slab_run_of_a_single_slab_equals_the_whole_domain_calls():
    """sfb_slab_run on an unlinked plan (one slab = the whole domain): forward with the
    sampled rows streamed out and the adjoint with the receiver table fed in reproduce
    sfb_forward / sfb_adjoint bit for bit; a partial range leaves the other rows alone."""
    from paper_1808_01995_b200 import capi
    rng = np.random.default_rng(11)
    shape, order, nsteps = [40, 36, 30], 8, 37
    L = [(s - 1) * 10.0 for s in shape]
    rec_xyz = rng.uniform(0.0, 1.0, size=(30000, 3)) * np.asarray(L)
    model, geom = make_problem(shape, 10.0, 6, order, nsteps, rec=rec_xyz)
    plan = make_plan(model, geom, order)
    rec1, _ = plan.forward(geom.src)
    u1 = plan.wavefield(geom.nt - 1)
    data = rng.standard_normal((geom.nt, rec_xyz.shape[0]))
    data[[0, geom.nt - 1]] = 0.0
    srca1, _ = plan.adjoint(data)
    # forward, in two ranges
    plan.upload_traces(capi.CLOUD_SRC, geom.src)
    table = np.full((geom.nt, geom.n_rec), np.nan)
    plan.step_begin(capi.OP_FORWARD)
    plan.slab_run(capi.OP_FORWARD, 1, 15, smp=table)
    assert np.array_equal(table[1:15], rec1[1:15]) and np.isnan(table[15:geom.nt - 1]).all()
    plan.slab_run(capi.OP_FORWARD, 15, geom.nt - 1, smp=table)
    plan.step_end(capi.OP_FORWARD)
    assert np.array_equal(table, rec1)
    assert np.array_equal(plan.wavefield(geom.nt - 1), u1)
    # adjoint, the receiver table fed while the sweep runs
    out = np.full((geom.nt, 1), np.nan)
    plan.step_begin(capi.OP_ADJOINT)
    plan.slab_run(capi.OP_ADJOINT, 1, geom.nt - 1, inj=data, smp=out)
    plan.step_end(capi.OP_ADJOINT)
    assert np.abs(srca1).max() > 0 and np.array_equal(out, srca1)
    with pytest.raises(capi.SfbError):
        plan.slab_run(capi.OP_FORWARD, 0, 5)
    plan.close()


def test_slab_run_refuses_plans_linked_inside_one_process():
    """plans linked with sfb_link_peers are ordered by each other's events: every plan must
    make each call before any plan makes the next, so the per-plan loop is refused"""
    from paper_1808_01995_b200 import capi
    model, geom = make_problem([40, 24, 26], 10.0, 6, 8, 12)
    lo = make_plan(model, geom, 8, slab=(0, 26))
    hi = make_plan(model, geom, 8, slab=(26, model.N[0]))
    lo.link_peers(None, hi)
    hi.link_peers(lo, None)
    lo.upload_traces(capi.CLOUD_SRC, geom.src)
    lo.step_begin(capi.OP_FORWARD)
    with pytest.raises(capi.SfbError) as e:
        lo.slab_run(capi.OP_FORWARD, 1, 5)
    assert e.value.code == capi.ERR_CAPABILITY
    lo.link_peers(None, None)
    hi.link_peers(None, None)
    lo.close()
    hi.close()
