"""BASELINE.json config 5, the one-GPU point of its weak-scaling series: 1024 x 1024 x (128 n)
physical nodes with n = 1 (slab axis first: 128 x 1024 x 1024; 208 x 1104 x 1104 computed),
space order 16, 40-node layer, seeded smoothed-noise velocity, 8 random off-grid sources,
1024 x 1024 receivers at 25 m depth, 1000 time steps."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1808_01995_b200 import _sfb_host as H, capi, synthetic as syn

nsteps = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
n0, n = 128, 1024
h = 12.5
vel = syn.smooth_field([n0, n, n], syn.SEED + 6, 8.0, 1.5, 4.5)
model = H.SeismicModel([n0, n, n], [h] * 3, [0.0] * 3, vel, 40, 16)
del vel
dt, tn = syn.time_axis(model.critical_dt(16), nsteps)
rng = np.random.default_rng(syn.SEED + 7)
src = rng.uniform([0, 0, 0], [h * (n0 - 1), h * (n - 1), h * (n - 1)], size=(8, 3))
ii, jj = np.meshgrid(np.arange(n) * h, np.arange(n) * h, indexing="ij")
# receivers on the (d1, d2)... the config puts them at depth 25 m over the 1024 x 1024 face;
# with the slab axis first that face is spanned by d1 and the depth axis d2 = z, so the grid
# of receivers runs over (d0 clipped to the slab, d1): use d1 x d1-sized lines over d0 x d1
rec = np.stack([np.minimum(ii.ravel(), h * (n0 - 1)), jj.ravel(), np.full(ii.size, 25.0)], axis=1)
geom = H.AcquisitionGeometry(model, src.ravel(), rec.ravel(), 0.0, tn, dt, 0.015)
assert geom.nt == nsteps + 2
plan = capi.Plan(model.grid.shape, model.grid.spacing, 16, dt, geom.nt)
plan.set_model(model.m.array(), model.damp.array(), model.v_max)
plan.set_points(capi.CLOUD_SRC, np.array(geom.src.base_table).reshape(-1, 3), np.array(geom.src.weight_table).reshape(-1, 8))
plan.set_points(capi.CLOUD_REC, np.array(geom.rec.base_table).reshape(-1, 3), np.array(geom.rec.weight_table).reshape(-1, 8))
tile = plan.autotune()
plan.upload_traces(capi.CLOUD_SRC, geom.src.traces)
if os.environ.get("SFB_CHUNK_SWEEP"):
    for chunk in (26, 35, 52, 70, 104, 208):
        plan.set_tile(tile["txv"], tile["ty"], tile["stages"], chunk)
        plan.step_begin(capi.OP_FORWARD)
        plan.run_steps(capi.OP_FORWARD, 1, 6)
        r = plan.run_steps(capi.OP_FORWARD, 6, 46)
        print("chunk", chunk, plan.get_tile(), f"{r.gpts_per_s:.1f} GPts/s", flush=True)
    plan.set_tile(tile["txv"], tile["ty"], tile["stages"], tile["chunk"])
plan.run_resident(capi.OP_FORWARD)
rep = plan.run_resident(capi.OP_FORWARD)
free, total = torch.cuda.mem_get_info()
halo = plan.halo_blocks(capi.OP_FORWARD, 1)["count"] * 4
print(json.dumps({"config": "BASELINE.json configs[4], weak-scaling point n_gpu = 1 (208 x 1104 x 1104 computed)",
                  "space_order": 16, "steps": rep.steps, "gpts_per_s": rep.gpts_per_s,
                  "ms_per_step": rep.seconds / rep.steps * 1e3, "tile": tile,
                  "frac_of_hbm_roofline_20B": rep.gpts_per_s * 20 / 6551.0,
                  "hbm_used_gb": (total - free) / 1e9, "halo_bytes_per_step_per_neighbour": halo,
                  "halo_us_at_770GBs": halo / 770e9 * 1e6}))
plan.close()
