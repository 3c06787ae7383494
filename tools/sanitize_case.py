"""Tiny end-to-end case for compute-sanitizer (memcheck / racecheck): ring kernel, dual-stream
kernel, point kernel, gradient with snapshots, TTI kernels, slab parts."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import oracle as o
from paper_1808_01995_b200 import capi
from tests.common import make_plan, make_problem, smooth_field

for order in (4, 12):
    model, geom = make_problem([20, 18, 22], 10.0, 4, order, 12)
    plan = make_plan(model, geom, order)
    rec, _ = plan.forward(geom.src, save_every=2)
    plan.adjoint(rec)
    plan.gradient(rec * 0.5)
    plan.step_begin(capi.OP_FORWARD)
    plan.upload_traces(capi.CLOUD_SRC, geom.src)
    for part in (capi.PART_LOW, capi.PART_HIGH, capi.PART_INTERIOR):
        plan.step_compute(capi.OP_FORWARD, 1, part)
        plan.step_points(capi.OP_FORWARD, 1, part)
    plan.step_end(capi.OP_FORWARD)
    plan.close()
    print("acoustic order", order, "ok", flush=True)
model, geom0 = make_problem([18, 16, 20], 10.0, 4, 4, 10, dt_frac=0.5)
N = model.N
eps = smooth_field(N, 1, 2.0, 0, 0.3)
delta = np.minimum(smooth_field(N, 2, 2.0, 0, 0.2), eps)
plan = make_plan(model, geom0, 4)
plan.set_model_tti(eps, delta, smooth_field(N, 3, 2.0, 0, 0.7), smooth_field(N, 4, 2.0, 0, 0.7))
plan.tti_forward(geom0.src)
plan.close()
print("tti ok", flush=True)
