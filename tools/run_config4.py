"""BASELINE.json config 4 at full size on one B200: TTI forward, 512^3 physical + 40-node
layer (592^3 computed), order 12, seeded smooth v / epsilon / delta / theta / phi, one 15 Hz
source, 512 x 512 receivers, 500 steps.  Reports throughput against both rooflines and the
growth check (late-time trace amplitude vs peak)."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1808_01995_b200 import _sfb_host as H, capi, synthetic as syn

nsteps = int(sys.argv[1]) if len(sys.argv) > 1 else 500
n = int(sys.argv[2]) if len(sys.argv) > 2 else 512
cfg = syn.config(4, n, nsteps)
t0 = time.time()
model = H.SeismicModel(cfg["shape"], [cfg["h"]] * 3, [0.0] * 3, cfg["velocity"](), cfg["nbl"], cfg["order"])
eps, delta, theta, phi = (syn.extend(f, cfg["nbl"]) for f in cfg["tti"]())
dt = 0.9 * model.critical_dt(cfg["order"]) / np.sqrt(1.0 + 2.0 * float(eps.max()))
tn = (nsteps + 1.5) * dt
geom = H.AcquisitionGeometry(model, np.asarray(cfg["src"]).ravel(), cfg["rec"].ravel(), 0.0, tn, dt, cfg["f0"])
t_gen = time.time() - t0
plan = capi.Plan(model.grid.shape, model.grid.spacing, cfg["order"], dt, geom.nt)
plan.set_model(model.m.array(), model.damp.array(), model.v_max)
plan.set_model_tti(eps, delta, theta, phi)
plan.set_points(capi.CLOUD_SRC, np.array(geom.src.base_table).reshape(-1, 3), np.array(geom.src.weight_table).reshape(-1, 8))
plan.set_points(capi.CLOUD_REC, np.array(geom.rec.base_table).reshape(-1, 3), np.array(geom.rec.weight_table).reshape(-1, 8))
src = np.ascontiguousarray(geom.src.traces)
t0 = time.time()
rec, rep = plan.tti_forward(src)
t_call = time.time() - t0
p = plan.wavefield(geom.nt - 1, field=0)
amp = np.abs(rec).max(axis=1)
N = model.grid.shape
print(json.dumps({
    "config": f"BASELINE.json configs[3] (TTI forward, {N[0]}^3 computed, order {cfg['order']}, {nsteps} steps)",
    "dt_ms": dt, "steps": rep.steps, "gpts_per_s": rep.gpts_per_s, "ms_per_step": rep.seconds / rep.steps * 1e3,
    "frac_hbm_roofline_48B": rep.gpts_per_s * 48 / 6551.0, "tflops": rep.gflops / 1e3,
    "frac_fp32_roofline": rep.gflops / 1e3 / 72.0, "call_s": t_call, "input_generation_s": t_gen,
    "finite": bool(np.isfinite(rec).all() and np.isfinite(p).all()),
    "trace_peak": float(amp.max()), "trace_peak_step": int(amp.argmax()),
    "trace_amp_last_step": float(amp[-2]), "wavefield_absmax": float(np.abs(p).max())}))
plan.close()
