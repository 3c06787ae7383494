"""GPU probe: forward / adjoint / gradient throughput per space order on a config-2 sized
grid (cheap random medium; performance only)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1808_01995_b200 import capi

n = int(sys.argv[1]) if len(sys.argv) > 1 else 592
orders = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [4, 8, 12, 16]
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 40
se = int(sys.argv[4]) if len(sys.argv) > 4 else 4
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
for order in orders:
    dt = capi.critical_dt([h] * 3, vmax, order)
    nt = steps + 12
    plan = capi.Plan(N, [h] * 3, order, dt, nt)
    plan.set_model(m, damp, vmax)
    plan.set_points(capi.CLOUD_SRC, sb, sw)
    plan.set_points(capi.CLOUD_REC, rb, rw)
    plan.upload_traces(capi.CLOUD_SRC, np.sin(np.arange(nt) * 0.1).reshape(nt, 1))
    plan.upload_traces(capi.CLOUD_REC, rng.standard_normal((nt, rb.shape[0])) * 1e-3)
    res = {}
    for name, op, s in [("forward", capi.OP_FORWARD, 0), ("forward+save", capi.OP_FORWARD, se),
                        ("adjoint", capi.OP_ADJOINT, 0), ("gradient", capi.OP_GRADIENT, se)]:
        plan.step_begin(op, s)
        plan.run_steps(op, 1, 7) if op == capi.OP_FORWARD else plan.run_steps(op, nt - 7, nt - 1)
        if op == capi.OP_FORWARD:
            rep = plan.run_steps(op, 7, 7 + steps)
        else:
            rep = plan.run_steps(op, nt - 7 - steps, nt - 7)
        if op == capi.OP_FORWARD and s:
            plan.step_end(op)
        res[name] = rep.gpts_per_s
    t = plan.get_tile()
    print(f"n={n} order={order:2d} tile=({t['txv']},{t['ty']},{t['stages']}) chunk={t['chunk']} sep={t['sep']}  " +
          "  ".join(f"{k} {v:6.1f}" for k, v in res.items()) + "  GPts/s", flush=True)
    plan.close()
