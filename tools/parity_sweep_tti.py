"""Mid-size TTI parity against the builder's f64 oracle: several tiles and d0 chunks with
ragged edges (120 x 116 x 126 computed), 100 steps, orders 4..16."""
import os, sys, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
from oracle import oracle as o
from common import make_problem, make_plan, rel_l2, smooth_field

orders = [int(a) for a in sys.argv[1].split(",")] if len(sys.argv) > 1 else [4, 8, 12, 16]
bad = []
for order in orders:
    t0 = time.time()
    model, g0 = make_problem([104, 100, 110], 10.0, 8, order, 100, dt_frac=0.5, n_rec_line=80)
    dt = o.tti_critical_dt(model, order, 0.3)
    geom = o.Geometry(model, g0.src_coords.ravel(), g0.rec_coords.ravel(), 0.0, 101.5 * dt, dt, 0.015)
    eps = smooth_field(model.N, 2, 3.0, 0.0, 0.3)
    delta = np.minimum(smooth_field(model.N, 3, 3.0, 0.0, 0.2), eps)
    theta = smooth_field(model.N, 4, 3.0, 0.0, np.pi / 4)
    phi = smooth_field(model.N, 5, 3.0, 0.0, np.pi / 4)
    ref = o.tti_forward(model, geom, order, eps, delta, theta, phi, want_final=True)
    plan = make_plan(model, geom, order)
    plan.set_model_tti(eps, delta, theta, phi)
    rec, _ = plan.tti_forward(geom.src)
    res = {"order": order, "N": list(model.N), "traces": rel_l2(rec, ref["smp"]),
           "p": rel_l2(plan.wavefield(geom.nt - 1, field=0), ref["p"]),
           "r": rel_l2(plan.wavefield(geom.nt - 1, field=1), ref["r"]), "seconds": round(time.time() - t0, 1)}
    print(json.dumps(res), flush=True)
    if not (res["traces"] <= 1e-5 and res["p"] <= 1e-5 and res["r"] <= 1e-5):
        bad.append(order)
    plan.close()
print("tti parity sweep", "FAILED " + str(bad) if bad else "ok")
sys.exit(1 if bad else 0)
