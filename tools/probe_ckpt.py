"""Checkpointed vs full-history gradient at sizes where the stencil grid is chunked along d0."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
from common import make_problem, make_plan

for shape, nt in ([60, 60, 60], 70), ([200, 120, 136], 70), ([592, 96, 128], 70), ([300, 300, 300], 70):
    model, geom = make_problem(shape, 10.0, 8, 8, nt, dt_frac=0.9)
    plan = make_plan(model, geom, 8)
    rec, _ = plan.forward(geom.src, save_every=1)
    rng = np.random.default_rng(5)
    resid = rec + 0.1 * np.abs(rec).max() * rng.standard_normal(rec.shape)
    g_full, _ = plan.gradient(resid)
    g_full2, _ = plan.gradient(resid)
    out = {"shape": shape, "nt": geom.nt, "tile": plan.get_tile() if hasattr(plan, "get_tile") else None,
           "full_repeat_equal": bool(np.array_equal(g_full, g_full2))}
    for C in (8, 16, 32):
        rec_c, _ = plan.forward_checkpointed(geom.src, C)
        g, _ = plan.gradient(resid)
        d = np.abs(g - g_full)
        out[f"C{C}"] = {"rec_equal": bool(np.array_equal(rec_c, rec)), "equal": bool(np.array_equal(g, g_full)),
                        "maxdiff": float(d.max()), "absmax": float(np.abs(g_full).max()),
                        "where": [int(i) for i in np.unravel_index(d.argmax(), d.shape)]}
    print(json.dumps(out), flush=True)
    plan.close()
