"""Repeat gradient runs and report where repeated results differ."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
from common import make_problem, make_plan

shape, nt = [592, 160, 192], 40
model, geom = make_problem(shape, 10.0, 8, 8, nt, dt_frac=0.9)
plan = make_plan(model, geom, 8)
if len(sys.argv) > 1:
    plan.set_tile(*[int(a) for a in sys.argv[1:4]])
rec, _ = plan.forward(geom.src, save_every=1)
rng = np.random.default_rng(5)
resid = rec + 0.1 * np.abs(rec).max() * rng.standard_normal(rec.shape)
gs, vs = [], []
mode = os.environ.get("PROBE_MODE", "gradient")
for _ in range(6):
    if mode == "adjoint":
        plan.adjoint(resid)
        gs.append(plan.wavefield(1))
    else:
        gs.append(plan.gradient(resid)[0])
    vs.append((plan.wavefield(1), plan.wavefield(0)))
print(json.dumps({"tile": plan.get_tile(), "src_base": np.asarray(geom.src_base).tolist(),
                  "rec_base0": np.asarray(geom.rec_base)[:3].tolist()}))
for i in range(1, 6):
    d = np.abs(gs[i] - gs[0])
    idx = np.argwhere(d > 0)
    info = {"run": i, "ndiff": int(len(idx)), "maxdiff": float(d.max()),
            "v1_equal": bool(np.array_equal(vs[i][0], vs[0][0])), "v0_equal": bool(np.array_equal(vs[i][1], vs[0][1])),
            "eq_prev": bool(np.array_equal(gs[i], gs[i - 1]))}
    if len(idx):
        rel = d[d > 0] / np.maximum(np.abs(gs[0][d > 0]), 1e-300)
        info["rel_max"] = float(rel.max()); info["rel_med"] = float(np.median(rel))
        info["d0"] = [int(idx[:, 0].min()), int(idx[:, 0].max())]
        info["d1"] = [int(idx[:, 1].min()), int(idx[:, 1].max())]
        info["d2"] = [int(idx[:, 2].min()), int(idx[:, 2].max())]
        j = idx[d[d > 0].argmax()]
        info["worst"] = [int(v) for v in j]; info["worst_vals"] = [float(gs[0][tuple(j)]), float(gs[i][tuple(j)])]
    print(json.dumps(info), flush=True)
plan.close()
