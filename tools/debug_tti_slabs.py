import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
from tests.test_gpu_tti import tti_problem, tti_fields, _run_tti_slabs
from tests.common import make_plan
order = int(sys.argv[1]); nsteps = int(sys.argv[2])
model, geom = tti_problem([48, 26, 30], order, nsteps)
fields = tti_fields(model.N, seed=3)
plan = make_plan(model, geom, order)
plan.set_model_tti(*fields)
rec1, _ = plan.tti_forward(geom.src)
p1 = plan.wavefield(geom.nt - 1, field=0); r1 = plan.wavefield(geom.nt - 1, field=1)
plan.close()
K = order // 2
n0 = model.N[0]
for cuts in ([0, 2 * K + 3, 2 * K + 3 + 2 * K + 5, n0], [0, 32, n0], [0, 20, 41, n0]):
    for parts in (False, True):
        rec3, p3, r3 = _run_tti_slabs(model, geom, order, fields, cuts, overlap_parts=parts)
        dp = np.abs(p3 - p1); dr = np.abs(r3 - r1)
        print(order, cuts, parts, "rec", float(np.abs(rec3 - rec1).max()), "p", float(dp.max()), "r", float(dr.max()),
              "planes", sorted(set(np.argwhere(dp > 0)[:, 0].tolist()))[:20], "absmax", float(np.abs(p1).max()), flush=True)
