"""Locate run-to-run differences of the adjoint wavefield inside gradient runs."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
from common import make_problem, make_plan

shape = [592, 160, 192]
for nt in (12,):
    model, geom = make_problem(shape, 10.0, 8, 8, nt, dt_frac=0.9)
    plan = make_plan(model, geom, 8)
    if len(sys.argv) > 1:
        plan.set_tile(*[int(a) for a in sys.argv[1:5]])
    rec, _ = plan.forward(geom.src, save_every=1)
    rng = np.random.default_rng(5)
    resid = rng.standard_normal(rec.shape)
    vs = []
    for _ in range(8):
        plan.gradient(resid)
        vs.append(plan.wavefield(1))
    print(json.dumps({"nt": geom.nt, "tile": plan.get_tile()}))
    for i in range(1, 8):
        d = np.abs(vs[i] - vs[0])
        idx = np.argwhere(d > 0)
        info = {"run": i, "ndiff": int(len(idx))}
        if len(idx):
            info["maxdiff"] = float(d.max()); info["absmax"] = float(np.abs(vs[0]).max())
        print(json.dumps(info), flush=True)
    plan.close()
