"""One tile shape of the acoustic step on an n^3 grid for an ncu capture:
    python tools/ncu_case.py <n> <order> <txv> <ty> <stages> [steps] [dense]
(stages < 0: dual-stream, < -100 rotated, < -200 patch, < -300 sliding window, < -400 tall).  A trailing
"grad" runs forward (every level saved) and then the gradient sweep: the update launches
after the first `steps` are imaging launches.  Cheap random medium, no oracle."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1808_01995_b200 import capi

n, order, txv, ty, st = (int(a) for a in sys.argv[1:6])
steps = int(sys.argv[6]) if len(sys.argv) > 6 else 6
dense = "dense" in sys.argv[7:]
grad = "grad" in sys.argv[7:]
N, h, vmax = [n] * 3, 12.5, 4.5
rng = np.random.default_rng(1)
dt = capi.critical_dt([h] * 3, vmax, order)
m = (1.0 / rng.uniform(1.5, vmax, size=n * n).reshape(1, n, n) ** 2) * np.ones((n, 1, 1))
prof = np.zeros(n); prof[:40] = np.linspace(0.02, 0, 40) ** 2 * 50; prof[-40:] = prof[:40][::-1]
damp = prof[:, None, None] + prof[None, :, None] + prof[None, None, :]
plan = capi.Plan(N, [h] * 3, order, dt, steps + 4, dense_damping=dense)
plan.set_model(m, damp, vmax)
plan.set_points(capi.CLOUD_SRC, np.array([[n // 2, n // 2, 41]], dtype=np.int64), np.full((1, 8), 0.125))
plan.set_points(capi.CLOUD_REC, np.array([[n // 2, n // 2, 42]], dtype=np.int64), np.full((1, 8), 0.125))
plan.upload_traces(capi.CLOUD_SRC, np.sin(np.arange(steps + 4) * 0.1).reshape(-1, 1))
plan.set_tile(txv, ty, st, 0)
if grad:
    plan.upload_traces(capi.CLOUD_REC, np.cos(np.arange(steps + 4) * 0.1).reshape(-1, 1))
    plan.run_resident(capi.OP_FORWARD, 1)
    rep = plan.run_resident(capi.OP_GRADIENT)
else:
    plan.step_begin(capi.OP_FORWARD)
    rep = plan.run_steps(capi.OP_FORWARD, 1, 1 + steps)
print(plan.get_tile(), f"{rep.gpts_per_s:.1f} GPts/s")
plan.close()
