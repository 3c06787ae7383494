"""Golden vectors produced by the reference itself (tests/golden/reference_outputs.npz,
generator oracle/make_golden.py).  CPU: the oracle must reproduce them to f64 round-off.
GPU: the CUDA path must reproduce them within BASELINE.json's fp32 tolerances -- these
tests need neither /root/reference nor oracle/_ref at run time."""
import os

import numpy as np
import pytest

from oracle import oracle as o
from tests import golden_cases as gc
from tests.common import rel_l2

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "reference_outputs.npz"))


def build(c):
    m = o.Model(c["shape"], c["spacing"], c["origin"], c["velocity"], c["nbl"], c["order"])
    g = o.Geometry(m, c["src"].ravel(), c["rec"].ravel(), 0.0, c["tn"], c["dt"], c["f0"])
    return m, g


@pytest.mark.parametrize("name", list(gc.CASES))
def test_oracle_reproduces_reference_outputs(name):
    c = gc.CASES[name]()
    m, g = build(c)
    assert g.nt == int(GOLD[f"{name}.nt"]) and c["dt"] == float(GOLD[f"{name}.dt"])
    f = o.forward(m, g, c["order"], want_final=True)
    rec = GOLD[f"{name}.rec"]
    assert np.abs(f["smp"] - rec).max() <= 1e-12 * np.abs(rec).max()
    fs = GOLD[f"{name}.final_sub"]
    assert np.abs(f["final"][gc.SUB[m.ndim]] - fs).max() <= 1e-12 * np.abs(fs).max()
    a = o.adjoint(m, g, c["order"], rec=rec)
    sa = GOLD[f"{name}.srca"]
    assert np.abs(a["smp"] - sa).max() <= 1e-12 * np.abs(sa).max()
    if c.get("gradient"):
        m0 = o.Model(c["shape"], c["spacing"], c["origin"], c["velocity0"], c["nbl"], c["order"])
        phi, grad, _ = o.fwi_gradient(m0, g, rec * 0.6, c["order"])
        assert phi == pytest.approx(float(GOLD[f"{name}.phi"]), rel=1e-12)
        gg = GOLD[f"{name}.grad"]
        assert np.abs(grad - gg).max() <= 1e-11 * np.abs(gg).max()


@pytest.mark.gpu
@pytest.mark.parametrize("name", list(gc.CASES))
def test_gpu_reproduces_reference_outputs(name):
    from paper_1808_01995_b200 import _sfb_host as H
    c = gc.CASES[name]()
    model = H.SeismicModel(c["shape"], c["spacing"], c["origin"], c["velocity"], c["nbl"], c["order"])
    geom = H.AcquisitionGeometry(model, c["src"].ravel(), c["rec"].ravel(), 0.0, c["tn"], c["dt"], c["f0"])
    assert geom.nt == int(GOLD[f"{name}.nt"])
    w = H.forward_operator(model, geom, c["order"])
    H.run_wave(w)
    rec = GOLD[f"{name}.rec"]
    assert rel_l2(geom.rec.traces, rec) <= 1e-4            # full run (BASELINE.json)
    u = w.wavefield.array()[(geom.nt - 1) % 3]
    assert rel_l2(u[gc.SUB[len(c["shape"])]], GOLD[f"{name}.final_sub"]) <= 1e-4
    geom.rec.traces[:] = rec                                 # adjoint of the reference's data
    a = H.adjoint_operator(model, geom, c["order"])
    H.run_wave(a)
    assert rel_l2(a.smp.traces, GOLD[f"{name}.srca"]) <= 1e-4
    if c.get("gradient"):
        model0 = H.SeismicModel(c["shape"], c["spacing"], c["origin"], c["velocity0"], c["nbl"], c["order"])
        geom0 = H.AcquisitionGeometry(model0, c["src"].ravel(), c["rec"].ravel(), 0.0, c["tn"], c["dt"], c["f0"])
        res = H.fwi_gradient(model0, geom0, rec * 0.6, c["order"])
        assert res.objective == pytest.approx(float(GOLD[f"{name}.phi"]), rel=1e-4)
        assert rel_l2(res.gradient, GOLD[f"{name}.grad"].ravel()) <= 1e-3
