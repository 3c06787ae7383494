"""Dense injection carpet: geometry of fresh run-to-run differences after the last step."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
from common import make_problem, make_plan

shape = [576, 144, 176]
nt = int(sys.argv[1]) if len(sys.argv) > 1 else 3
h = 10.0
ii, jj = np.meshgrid(np.arange(0, shape[0] - 1, 1), np.arange(0, shape[1] - 1, 1), indexing="ij")
rec = np.stack([ii.ravel() * h + 0.3 * h, jj.ravel() * h + 0.4 * h, np.full(ii.size, 4.5 * h)], axis=1)
model, geom = make_problem(shape, h, 8, 8, nt, dt_frac=0.9, rec=rec)
plan = make_plan(model, geom, 8)
rec_tr, _ = plan.forward(geom.src, save_every=1)
rng = np.random.default_rng(5)
resid = rng.standard_normal(rec_tr.shape)
vs = []
for _ in range(10):
    plan.gradient(resid)
    vs.append((plan.wavefield(1), plan.wavefield(0)))
print(json.dumps({"nt": geom.nt, "tile": plan.get_tile(), "nrec": len(rec)}))
for i in range(1, 10):
    d1 = np.abs(vs[i][0] - vs[0][0]) > 0
    d0 = np.abs(vs[i][1] - vs[0][1]) > 0
    info = {"run": i, "lvl1_ndiff": int(d1.sum()), "lvl0_ndiff": int(d0.sum())}
    if d0.any() and not d1.any():
        idx = np.argwhere(d0)
        planes = sorted(set(int(v) for v in idx[:, 0]))
        info["planes"] = planes[:20]
        for pz in planes[:4]:
            sub = idx[idx[:, 0] == pz]
            rows = sorted(set(int(v) for v in sub[:, 1]))
            info[f"p{pz}"] = {"rows": rows, "n": int(len(sub)),
                              "cols_by_row": {int(r): [int(sub[sub[:, 1] == r][:, 2].min()), int(sub[sub[:, 1] == r][:, 2].max()), int((sub[:, 1] == r).sum())] for r in rows[:6]}}
        pz = planes[0]; sub = idx[idx[:, 0] == pz]; r = int(sub[0, 1])
        c0, c1 = int(sub[sub[:, 1] == r][:, 2].min()), int(sub[sub[:, 1] == r][:, 2].max())
        sl = (pz, r, slice(max(c0 - 2, 0), c1 + 3))
        info["row"] = [pz, r, max(c0 - 2, 0)]
        info["L0_run0"] = [float(f"{v:.6g}") for v in vs[0][1][sl]]
        info["L0_runi"] = [float(f"{v:.6g}") for v in vs[i][1][sl]]
        info["L1"] = [float(f"{v:.6g}") for v in vs[0][0][sl]]
    print(json.dumps(info), flush=True)
plan.close()
