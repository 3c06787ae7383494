"""BASELINE.json config 3 at full size on one B200: two-layer medium at 592^3 computed nodes,
order 8, 500 steps; the forward pass keeps every 4th level in HBM (126 x 0.83 GB), the adjoint
sweep is driven by seeded random band-limited residuals at the 512 x 512 receivers, imaging
fused into the sweep.  Prints throughputs, memory use and the dot-product test."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1808_01995_b200 import _sfb_host as H, capi, synthetic as syn

nsteps = int(sys.argv[1]) if len(sys.argv) > 1 else 500
# optional second argument C: checkpointed run (state kept every C levels, segments recomputed,
# imaging at EVERY level = the reference's exact condition) instead of every-4th-level history
ckpt = int(sys.argv[2]) if len(sys.argv) > 2 else 0
cfg = syn.config(3, 512, nsteps)
model = H.SeismicModel(cfg["shape"], [12.5] * 3, [0.0] * 3, cfg["velocity"](), 40, 8)
dt, tn = syn.time_axis(model.critical_dt(8), nsteps)
geom = H.AcquisitionGeometry(model, np.asarray(cfg["src"]).ravel(), cfg["rec"].ravel(), 0.0, tn, dt, cfg["f0"])
plan = capi.Plan(model.grid.shape, model.grid.spacing, 8, dt, geom.nt)
plan.set_model(model.m.array(), model.damp.array(), model.v_max)
plan.set_points(capi.CLOUD_SRC, np.array(geom.src.base_table).reshape(-1, 3), np.array(geom.src.weight_table).reshape(-1, 8))
plan.set_points(capi.CLOUD_REC, np.array(geom.rec.base_table).reshape(-1, 3), np.array(geom.rec.weight_table).reshape(-1, 8))
src = np.ascontiguousarray(geom.src.traces)
t0 = time.time()
rec, rf = plan.forward_checkpointed(src, ckpt) if ckpt else plan.forward(src, save_every=4)
t_fwd = time.time() - t0
free, total = torch.cuda.mem_get_info()
hbm_fwd = (total - free) / 1e9
rng = np.random.default_rng(syn.SEED + 10)
wavelet = np.array([H.ricker_value(0.015, t * dt) for t in range(geom.nt)])
spec = np.fft.rfft(wavelet)[:, None]
resid = np.empty_like(rec)
for lo in range(0, geom.n_rec, 32768):  # N(0,1) noise convolved in time with the 15 Hz Ricker
    xi = rng.standard_normal((geom.nt, min(32768, geom.n_rec - lo)))
    resid[:, lo:lo + xi.shape[1]] = np.fft.irfft(np.fft.rfft(xi, axis=0) * spec, n=geom.nt, axis=0)
resid[[0, geom.nt - 1]] = 0.0
t0 = time.time()
g, rg = plan.gradient(resid)
t_grad = time.time() - t0
free, total = torch.cuda.mem_get_info()
# dot-product test <F x, y> vs <x, F^T y> on the same plan
xt, ra = plan.adjoint(resid)
lhs, rhs = float((rec * resid).sum()), float((src * xt).sum())
print(json.dumps({
    "config": "BASELINE.json configs[2] (acoustic FWI gradient, 592^3, order 8, "
              + (f"checkpoint every {ckpt} levels + recompute, imaging every level)" if ckpt
                 else "save every 4th level)"),
    "hbm_after_forward_gb": hbm_fwd,
    "steps": nsteps, "forward_with_save_gpts": rf.gpts_per_s, "gradient_sweep_gpts": rg.gpts_per_s,
    "adjoint_gpts": ra.gpts_per_s, "forward_call_s": t_fwd, "gradient_call_s": t_grad,
    "hbm_used_gb": (total - free) / 1e9, "saved_levels": (2 * ((geom.nt - 2) // ckpt + 2) + ckpt) if ckpt else (geom.nt - 1) // 4 + 1,
    "dot_test_rel": abs(lhs - rhs) / max(abs(lhs), abs(rhs)),
    "grad_absmax": float(np.abs(g).max()), "grad_finite": bool(np.isfinite(g).all())}))
plan.close()
