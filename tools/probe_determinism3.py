"""Smallest failing case: few backward steps, report the geometry of the differing nodes."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
from common import make_problem, make_plan

shape = [592, 160, 192]
nt = int(sys.argv[1]) if len(sys.argv) > 1 else 3
model, geom = make_problem(shape, 10.0, 8, 8, nt, dt_frac=0.9)
plan = make_plan(model, geom, 8)
rec, _ = plan.forward(geom.src, save_every=1)
rng = np.random.default_rng(5)
resid = rng.standard_normal(rec.shape)
vs = []
for _ in range(12):
    plan.gradient(resid)
    vs.append((plan.wavefield(1), plan.wavefield(0)))
print(json.dumps({"nt": geom.nt, "tile": plan.get_tile()}))
# majority reference
for i in range(1, 12):
    for lvl in (0, 1):
        d = np.abs(vs[i][lvl] - vs[0][lvl])
        idx = np.argwhere(d > 0)
        if not len(idx):
            continue
        info = {"run": i, "level": 1 - lvl, "ndiff": int(len(idx)), "maxdiff": float(d.max())}
        planes = sorted(set(int(v) for v in idx[:, 0]))
        info["planes"] = planes[:30]
        for pz in planes[:3]:
            sub = idx[idx[:, 0] == pz]
            info[f"p{pz}"] = {"d1": sorted(set(int(v) for v in sub[:, 1])), "d2": [int(sub[:, 2].min()), int(sub[:, 2].max())],
                              "n": int(len(sub))}
        print(json.dumps(info), flush=True)
plan.close()
