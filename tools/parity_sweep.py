"""Mid-size parity sweep against the f64 oracle: every even space order 2..16 on a grid that
spans many tiles and d0 chunks with ragged edges (216 x 200 x 232 computed), 100 steps:
forward traces and wavefield, adjoint traces, gradient (imaging every 2nd level)."""
import os, sys, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
from oracle import oracle as o
from common import make_problem, make_plan, rel_l2

orders = [int(a) for a in sys.argv[1].split(",")] if len(sys.argv) > 1 else [2, 4, 6, 8, 10, 12, 14, 16]
bad = []
for order in orders:
    t0 = time.time()
    model, geom = make_problem([200, 184, 216], 10.0, 8, order, 100, dt_frac=0.9, n_rec_line=150)
    ref = o.forward(model, geom, order, want_final=True, save_every=2)
    plan = make_plan(model, geom, order)
    rec, _ = plan.forward(geom.src, save_every=2)
    e_rec = rel_l2(rec, ref["smp"]); e_u = rel_l2(plan.wavefield(geom.nt - 1), ref["final"])
    srca, _ = plan.adjoint(geom.rec)
    e_adj = rel_l2(srca, o.adjoint(model, geom, order)["smp"])
    resid = geom.rec * 0.5
    plan.forward(geom.src, save_every=2)
    g, _ = plan.gradient(resid)
    e_g = rel_l2(g, o.gradient_sweep(model, geom, order, resid, ref["snaps"], 2))
    res = {"order": order, "N": list(model.N), "tile": plan.get_tile(), "traces": e_rec, "wavefield": e_u,
           "adjoint": e_adj, "gradient": e_g, "seconds": round(time.time() - t0, 1)}
    print(json.dumps(res), flush=True)
    if not (e_rec <= 1e-5 and e_u <= 1e-5 and e_adj <= 1e-5 and e_g <= 1e-3):
        bad.append(order)
    plan.close()
print("parity sweep", "FAILED " + str(bad) if bad else "ok")
sys.exit(1 if bad else 0)
