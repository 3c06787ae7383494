"""GPU probe: TTI forward throughput at config-4 size (cheap synthetic medium)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1808_01995_b200 import capi

n = int(sys.argv[1]) if len(sys.argv) > 1 else 592
order = int(sys.argv[2]) if len(sys.argv) > 2 else 12
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 20
rng = np.random.default_rng(1)
N = [n, n, n]
h, vmax = 12.5, 4.5
m = (1.0 / rng.uniform(1.5, vmax, size=n * n).reshape(1, n, n) ** 2) * np.ones((n, 1, 1))
prof = np.zeros(n); prof[:40] = np.linspace(0.02, 0, 40) ** 2 * 50; prof[-40:] = prof[:40][::-1]
damp = prof[:, None, None] + prof[None, :, None] + prof[None, None, :]
lin = np.linspace(0, 1, n)
eps = 0.3 * lin[:, None, None] * np.ones(N)
delta = 0.2 * lin[None, :, None] * lin[:, None, None] * np.ones(N)
theta = (np.pi / 4) * lin[None, None, :] * np.ones(N)
phi = (np.pi / 4) * lin[None, :, None] * np.ones(N)
dt = 0.9 * capi.critical_dt([h] * 3, vmax, order) / np.sqrt(1.6)
nt = steps + 2
plan = capi.Plan(N, [h] * 3, order, dt, nt)
plan.set_model(m, damp, vmax)
t0 = time.time()
plan.set_model_tti(eps, delta, theta, phi)
print("tti model up", time.time() - t0, flush=True)
nr = min(512, n - 82)
ii, jj = np.meshgrid(np.arange(nr) + 40, np.arange(nr) + 40, indexing="ij")
rb = np.stack([ii.ravel(), jj.ravel(), np.full(ii.size, 42)], 1).astype(np.int64)
rw = np.zeros((rb.shape[0], 8)); rw[:, 0] = 1.0
plan.set_points(capi.CLOUD_SRC, np.array([[n // 2, n // 2, 41]], dtype=np.int64), np.full((1, 8), 0.125))
plan.set_points(capi.CLOUD_REC, rb, rw)
plan.upload_traces(capi.CLOUD_SRC, np.sin(np.arange(nt) * 0.1).reshape(nt, 1))
plan.run_resident(capi.OP_TTI_FORWARD)
rep = plan.run_resident(capi.OP_TTI_FORWARD)
print(f"TTI n={n} order={order}: {rep.seconds/rep.steps*1e3:.3f} ms/step {rep.gpts_per_s:.1f} GPts/s "
      f"({rep.gpts_per_s*48/1e3:.2f} TB/s algorithmic @48 B/node), {rep.gflops/1e3:.1f} TFLOP/s", flush=True)
plan.close()
