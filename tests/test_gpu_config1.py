"""BASELINE.json config 1 exactly (the reference's own CPU-runnable case): 101^3 physical,
h = 10 m, order 4, 40-node layer (181^3 computed), two layers 1.5 / 2.5 km/s split at z = 50,
one 10 Hz Ricker source at the centre at 20 m depth, 101 receivers on a line, dt = the
critical dt, 1000 ms (nt = 708).  GPU vs the f64 oracle: rel-L2 <= 1e-5 after 100 steps and
<= 1e-4 after the full run, traces and final wavefield (the oracle needs ~15 s on 16 cores)."""
import numpy as np
import pytest

from oracle import oracle as o
from tests.common import rel_l2

pytestmark = pytest.mark.gpu


def test_config1_forward_parity():
    from paper_1808_01995_b200 import capi
    from paper_1808_01995_b200 import synthetic as syn
    cfg = syn.config(1)
    model = o.Model(cfg["shape"], [cfg["h"]] * 3, [0.0] * 3, cfg["velocity"](), cfg["nbl"], cfg["order"])
    dt = model.critical_dt(cfg["order"])
    assert dt == pytest.approx(1.41421356, abs=1e-7) and model.N == [181, 181, 181]
    geom = o.Geometry(model, np.asarray(cfg["src"]).ravel(), cfg["rec"].ravel(), 0.0, cfg["tn"], dt,
                      cfg["f0"])
    assert geom.nt == 708 and geom.n_rec == 101

    def gpu_run(nt):
        plan = capi.Plan(model.N, model.spacing, cfg["order"], dt, nt)
        plan.set_model(model.m, model.damp, model.v_max)
        plan.set_points(capi.CLOUD_SRC, geom.src_base, geom.src_w)
        plan.set_points(capi.CLOUD_REC, geom.rec_base, geom.rec_w)
        rec, rep = plan.forward(geom.src[:nt])
        u = plan.wavefield(nt - 1)
        plan.close()
        return rec, u, rep

    # 100-step checkpoint (level 101)
    ref100 = o.forward(model, geom, cfg["order"], want_final=True, nt=102)
    rec100, u100, _ = gpu_run(102)
    assert np.abs(ref100["final"]).max() > 0
    assert rel_l2(rec100, ref100["smp"]) <= 1e-5 and rel_l2(u100, ref100["final"]) <= 1e-5
    # full run
    ref = o.forward(model, geom, cfg["order"], want_final=True)
    rec, u, rep = gpu_run(geom.nt)
    assert rep.steps == 706
    assert rel_l2(rec, ref["smp"]) <= 1e-4 and rel_l2(u, ref["final"]) <= 1e-4
