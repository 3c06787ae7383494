"""Full-size repeatability soak: every default kernel (and the autotuned one) run twice at
592^3 must give bit-identical traces, wavefields and gradients -- the check that exposed the
pipeline-release race."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1808_01995_b200 import capi

n = int(sys.argv[1]) if len(sys.argv) > 1 else 592
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 200
rng = np.random.default_rng(1)
N = [n, n, n]
h, vmax = 12.5, 4.5
m = (1.0 / rng.uniform(1.5, vmax, size=n * n).reshape(1, n, n) ** 2) * np.ones((n, 1, 1))
prof = np.zeros(n); prof[:40] = np.linspace(0.02, 0, 40) ** 2 * 50; prof[-40:] = prof[:40][::-1]
damp = prof[:, None, None] + prof[None, :, None] + prof[None, None, :]
nr = min(512, n - 82)
ii, jj = np.meshgrid(np.arange(nr) + 40, np.arange(nr) + 40, indexing="ij")
rb = np.stack([ii.ravel(), jj.ravel(), np.full(ii.size, 42)], 1).astype(np.int64)
rw = np.zeros((rb.shape[0], 8)); rw[:, 0] = 0.7; rw[:, 4] = 0.3
sb = np.array([[n // 2, n // 2, 41]], dtype=np.int64)
sw = np.full((1, 8), 0.125)
out = []
dump = os.environ.get("SOAK_DUMP")   # save the order-8 traces, to compare runs across launch modes
for order, tile in ((8, None), (8, (16, 16, -103)), (8, (16, 16, -3)), (12, None), (16, None), (4, None)):
    dt = capi.critical_dt([h] * 3, vmax, order)
    nt = steps + 2
    plan = capi.Plan(N, [h] * 3, order, dt, nt)
    plan.set_model(m, damp, vmax)
    plan.set_points(capi.CLOUD_SRC, sb, sw)
    plan.set_points(capi.CLOUD_REC, rb, rw)
    if tile:
        plan.set_tile(*tile)
    src = np.sin(np.arange(nt) * 0.21).reshape(nt, 1)
    res = {"order": order, "tile": plan.get_tile()}
    recs, lv = [], []
    for _ in range(2):
        rec, _ = plan.forward(src, save_every=8)
        recs.append(rec); lv.append(plan.wavefield(nt - 1))
    res["forward_equal"] = bool(np.array_equal(recs[0], recs[1]) and np.array_equal(lv[0], lv[1]))
    if dump and tile is None:
        np.save(f"{dump}_rec_so{order}.npy", recs[0].astype(np.float32))
    res["finite"] = bool(np.isfinite(lv[0]).all()); res["absmax"] = float(np.abs(lv[0]).max())
    resid = np.random.default_rng(3).standard_normal(rec.shape) * np.hanning(nt)[:, None]
    gs = [plan.gradient(resid)[0] for _ in range(2)]
    res["gradient_equal"] = bool(np.array_equal(gs[0], gs[1]))
    res["grad_absmax"] = float(np.abs(gs[0]).max())
    print(json.dumps(res), flush=True)
    out.append(res)
    plan.close()
# the TTI pair (order 12, cheap analytic Thomsen fields)
lin = np.linspace(0.0, 1.0, n)
ones = np.ones(N)
eps = 0.3 * lin[:, None, None] * ones
delta = 0.2 * lin[None, :, None] * lin[:, None, None] * ones
theta = (np.pi / 4) * lin[None, None, :] * ones
phi = (np.pi / 4) * lin[None, :, None] * ones
tsteps = min(steps, 60)
dt = 0.9 * capi.critical_dt([h] * 3, vmax, 12) / np.sqrt(1.6)
plan = capi.Plan(N, [h] * 3, 12, dt, tsteps + 2)
plan.set_model(m, damp, vmax)
plan.set_model_tti(eps, delta, theta, phi)
plan.set_points(capi.CLOUD_SRC, sb, sw)
plan.set_points(capi.CLOUD_REC, rb, rw)
src = np.sin(np.arange(tsteps + 2) * 0.21).reshape(-1, 1)
runs = []
for _ in range(2):
    rec, _ = plan.tti_forward(src)
    runs.append((rec, plan.wavefield(tsteps + 1, field=0), plan.wavefield(tsteps + 1, field=1)))
res = {"tti_order": 12, "equal": bool(all(np.array_equal(a, b) for a, b in zip(*runs))),
       "finite": bool(np.isfinite(runs[0][1]).all()), "absmax": float(np.abs(runs[0][1]).max())}
print(json.dumps(res), flush=True)
plan.close()
assert res["equal"] and res["finite"]
assert all(r["forward_equal"] and r["gradient_equal"] and r["finite"] for r in out)
print("soak ok")
