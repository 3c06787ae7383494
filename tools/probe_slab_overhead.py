"""Cost of the slab protocol on one GPU: a middle slab of BASELINE.json config 5's 8-GPU run
(138 x 1104 x 1104 owned nodes, order 16) stepped as one launch (what a single-GPU run does)
and as the multi-GPU protocol does it -- LOW and HIGH boundary plane groups on the boundary
stream, their scatter, then the interior on the main stream -- without neighbours (ghost
planes stay zero: timing only).  The ratio bounds the parallel efficiency the decomposition
can reach when the exchange itself is hidden behind the interior update."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1808_01995_b200 import capi

order = int(sys.argv[1]) if len(sys.argv) > 1 else 16
n0_slab = int(sys.argv[2]) if len(sys.argv) > 2 else 138
n = int(sys.argv[3]) if len(sys.argv) > 3 else 1104
steps = 60
N = [3 * n0_slab, n, n]
h, vmax = 12.5, 4.5
rng = np.random.default_rng(1)
m = (1.0 / rng.uniform(1.5, vmax, size=n * n).reshape(1, n, n) ** 2) * np.ones((N[0], 1, 1))
prof = np.zeros(n); prof[:40] = np.linspace(0.02, 0, 40) ** 2 * 50; prof[-40:] = prof[:40][::-1]
p0 = np.zeros(N[0]); p0[:40] = prof[:40]; p0[-40:] = prof[-40:]
damp = p0[:, None, None] + prof[None, :, None] + prof[None, None, :]
dt = capi.critical_dt([h] * 3, vmax, order)
nt = steps + 12
plan = capi.Plan(N, [h] * 3, order, dt, nt, 0, (n0_slab, 2 * n0_slab))
plan.set_model(m, damp, vmax)
nr = n - 82
ii, jj = np.meshgrid(np.arange(n0_slab) + n0_slab, np.arange(nr) + 40, indexing="ij")
rb = np.stack([ii.ravel(), jj.ravel(), np.full(ii.size, 42)], 1).astype(np.int64)
rw = np.zeros((rb.shape[0], 8)); rw[:, 0] = 1.0
plan.set_points(capi.CLOUD_SRC, np.array([[n0_slab + 3, n // 2, 41]], dtype=np.int64), np.full((1, 8), 0.125))
plan.set_points(capi.CLOUD_REC, rb, rw)
plan.upload_traces(capi.CLOUD_SRC, np.sin(np.arange(nt) * 0.1).reshape(nt, 1))
F = capi.OP_FORWARD
pts = float(n0_slab) * n * n

def timed(fn):
    plan.step_begin(F)
    for t in range(1, 6):
        fn(t)
    plan.sync()
    t0 = time.perf_counter()
    for t in range(6, 6 + steps):
        fn(t)
    plan.sync()
    return (time.perf_counter() - t0) / steps

def whole(t):
    plan.step_compute(F, t, capi.PART_ALL)
    plan.step_points(F, t, capi.PART_ALL)

def parts(t):
    plan.step_slab_boundary(F, t)
    plan.step_slab_interior(F, t)

def fused(t):
    plan.step_slab_fused(F, t)

def only_boundary(t):
    plan.step_slab_boundary(F, t)

def only_interior(t):
    plan.step_slab_interior(F, t)

a = timed(whole)
b = timed(parts)
bnd_only = timed(only_boundary)
int_only = timed(only_interior)
# the same protocol with the fused halo push: neighbours on the same device stand in for the
# peers (their ghost planes receive this slab's boundary planes as they are computed)
def neighbour(lo, hi):
    q = capi.Plan(N, [h] * 3, order, dt, nt, 0, (lo, hi))
    q.set_model(m, damp, vmax)
    return q
below, above = neighbour(0, n0_slab), neighbour(2 * n0_slab, 3 * n0_slab)
plan.link_peers(below, above)
c = timed(parts)
d = timed(fused)      # single-launch slab step: first chunk up, last chunk down, pushes first
plan.link_peers(None, None)
below.close(); above.close()
K = order // 2
print(json.dumps({"slab": [n0_slab, n, n], "order": order, "tile": plan.get_tile(),
                  "whole_ms": a * 1e3, "parts_ms": b * 1e3, "whole_gpts": pts / a / 1e9,
                  "parts_gpts": pts / b / 1e9, "protocol_efficiency": a / b, "boundary_alone_ms": bnd_only * 1e3, "interior_alone_ms": int_only * 1e3, "pushed_ms": c * 1e3, "pushed_efficiency": a / c,
                  "single_launch_pushed_ms": d * 1e3, "single_launch_efficiency": a / d,
                  "halo_mb_per_neighbour": K * n * n * 4 / 1e6}))
plan.close()
