"""Small-grid step time: full step (update + point launch) vs the update kernel alone."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1808_01995_b200 import capi
for n, order in ((181, 4), (128, 8), (256, 8)):
    N = [n] * 3
    h, vmax = 10.0, 2.5
    dt = capi.critical_dt([h] * 3, vmax, order)
    steps = 600
    nt = steps + 12
    rng = np.random.default_rng(1)
    m = np.full(N, 1 / 2.25)
    prof = np.zeros(n); prof[:40] = np.linspace(0.02, 0, 40) ** 2 * 50; prof[-40:] = prof[:40][::-1]
    damp = prof[:, None, None] + prof[None, :, None] + prof[None, None, :]
    plan = capi.Plan(N, [h] * 3, order, dt, nt)
    plan.set_model(m, damp, vmax)
    nr = min(101, n - 82)
    rb = np.stack([np.arange(nr) + 40, np.full(nr, n // 2), np.full(nr, 42)], 1).astype(np.int64)
    rw = np.zeros((nr, 8)); rw[:, 0] = 1.0
    plan.set_points(capi.CLOUD_SRC, np.array([[n // 2, n // 2, 42]], dtype=np.int64), np.full((1, 8), 0.125))
    plan.set_points(capi.CLOUD_REC, rb, rw)
    plan.upload_traces(capi.CLOUD_SRC, np.sin(np.arange(nt) * 0.1).reshape(nt, 1))
    F = capi.OP_FORWARD
    plan.step_begin(F)
    plan.run_steps(F, 1, 11)
    rep = plan.run_steps(F, 11, 11 + steps)
    st = plan.time_stencil(F, 11, 11 + steps)
    pts = float(n) ** 3
    print(f"n={n} order={order} tile={plan.get_tile()}: step {rep.seconds/steps*1e6:.2f} us ({rep.gpts_per_s:.0f} GPts/s), "
          f"update kernel alone {st.seconds/steps*1e6:.2f} us ({pts*steps/st.seconds/1e9:.0f} GPts/s)", flush=True)
    plan.close()
