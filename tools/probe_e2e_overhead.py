"""Where the end-to-end time of a short sfb_forward call goes: configs[1] (592^3, order 8, 512 x
512 receivers) for K steps, wall clock of the C-ABI call with host f64 tables against the device
time of the stepping loop the call reports."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench

K = int(sys.argv[1]) if len(sys.argv) > 1 else 20
wl = bench.Workload(2, "forward", K)
plan = wl.make_plan(0)
plan.autotune()
rec = np.empty((wl.nt, wl.rec_base.shape[0]))
calls = []
for i in range(7):
    t0 = time.perf_counter()
    _, rep = plan.forward(wl.src, out=rec)
    t1 = time.perf_counter()
    calls.append({"wall_ms": round((t1 - t0) * 1e3, 3), "loop_ms": round(rep.seconds * 1e3, 3)})
pts = float(np.prod(wl.N)) * K
best = min(c["wall_ms"] for c in calls[1:])
print(json.dumps({"steps": K, "chunk_kb": os.environ.get("SFB_ROW_CHUNK_KB"), "calls": calls,
                  "e2e_gpts": pts / best / 1e6,
                  "overhead_ms": best - min(c["loop_ms"] for c in calls[1:])}))
plan.close()

# the pieces: zeroing (step_begin), the guard + download (step_end)
from paper_1808_01995_b200 import capi
plan = wl.make_plan(0)
plan.upload_traces(capi.CLOUD_SRC, wl.src)
parts = []
for i in range(4):
    plan.sync()
    t0 = time.perf_counter(); plan.step_begin(capi.OP_FORWARD); plan.sync(); t1 = time.perf_counter()
    plan.step_compute(capi.OP_FORWARD, 1, capi.PART_ALL); plan.step_points(capi.OP_FORWARD, 1, capi.PART_ALL); plan.sync()
    t2 = time.perf_counter(); plan.step_end(capi.OP_FORWARD); t3 = time.perf_counter()
    t4 = time.perf_counter(); plan.upload_traces(capi.CLOUD_SRC, wl.src); plan.sync(); t5 = time.perf_counter()
    parts.append({"begin_ms": round((t1 - t0) * 1e3, 3), "end_ms": round((t3 - t2) * 1e3, 3),
                  "upload_src_ms": round((t5 - t4) * 1e3, 3)})
print(json.dumps({"parts": parts}))
plan.close()
