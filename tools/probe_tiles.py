"""GPU probe: time every compiled tile shape of the acoustic step on a config-2 sized grid
(performance only: a cheap random medium, no oracle)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1808_01995_b200 import capi

n = int(sys.argv[1]) if len(sys.argv) > 1 else 592
order = int(sys.argv[2]) if len(sys.argv) > 2 else 8
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 60
rng = np.random.default_rng(1)
N = [n, n, n]
h = 12.5
vmax = 4.5
dt = capi.critical_dt([h] * 3, vmax, order)
nt = steps + 12
t0 = time.time()
m = (1.0 / rng.uniform(1.5, vmax, size=n * n).reshape(1, n, n) ** 2) * np.ones((n, 1, 1))
damp = np.zeros(N)
damp[:40] += 0.01; damp[-40:] += 0.01
print("host arrays", time.time() - t0, flush=True)
dense = len(sys.argv) > 4 and sys.argv[4] == "dense"
plan = capi.Plan(N, [h] * 3, order, dt, nt, dense_damping=dense)
plan.set_model(m, damp, vmax)
print("model up", time.time() - t0, flush=True)
nr = min(512, n - 82)
ii, jj = np.meshgrid(np.arange(nr) + 40, np.arange(nr) + 40, indexing="ij")
rb = np.stack([ii.ravel(), jj.ravel(), np.full(ii.size, 42)], 1).astype(np.int64)
rw = np.zeros((rb.shape[0], 8)); rw[:, 0] = 1.0
sb = np.array([[n // 2, n // 2, 41]], dtype=np.int64)
sw = np.full((1, 8), 0.125)
plan.set_points(capi.CLOUD_SRC, sb, sw)
plan.set_points(capi.CLOUD_REC, rb, rw)
src = np.sin(np.arange(nt) * 0.1).reshape(nt, 1)
plan.upload_traces(capi.CLOUD_SRC, src)
print("points up", time.time() - t0, flush=True)
K = order // 2
tiles = [(16, 16, K + 3), (16, 16, K + 4), (32, 8, K + 3), (16, 32, K + 3), (32, 16, K + 3), (16, 16, -3), (16, 16, -4), (16, 14, -4), (32, 8, -3), (16, 16, -103), (16, 14, -204), (16, 14, -304), (16, 16, -304), (16, 28, -404)]
if len(sys.argv) > 5:   # only the listed stage codes
    keep = {int(c) for c in sys.argv[5].split(',')}
    tiles = [t for t in tiles if t[2] in keep]
for tile in tiles:
    for chunk in (0,):
        try:
            plan.set_tile(*tile, chunk)
        except capi.SfbError as e:
            print("skip", tile, e)
            continue
        plan.step_begin(capi.OP_FORWARD)
        plan.run_steps(capi.OP_FORWARD, 1, 11)
        rep = plan.run_steps(capi.OP_FORWARD, 11, 11 + steps)
        print(f"n={n} order={order} tile={tile} {plan.get_tile()} : {rep.seconds/rep.steps*1e3:.3f} ms/step "
              f"{rep.gpts_per_s:.1f} GPts/s  ({rep.gpts_per_s*20/1e3:.2f} TB/s algorithmic)", flush=True)
plan.close()
