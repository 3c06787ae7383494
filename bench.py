#!/usr/bin/env python
"""bench.py -- headline benchmark of the wave-propagator path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N ...

Metric (BASELINE.json): GPts/s = padded grid points x time steps / seconds of the stepping
loop, acoustic forward operator.  A "step" is one time step of the propagator (dense
update + source scatter + receiver gather).  Workload at every N: BASELINE.json configs[1]
(512^3 physical + 40-node layer = 592^3, space order 8, 512x512 receivers, one off-node
Ricker source, seeded smoothed-noise velocity); at N > 1 the same grid is cut into N slabs
along the slowest axis (strong scaling, as configs[1] asks) and ghost planes travel over
NCCL send/recv each step.

One JSON line on stdout (rank 0).  `value` is timed with CUDA events on the plan's own
stream with all inputs resident in HBM; `e2e` is the same metric through the C-ABI call
sfb_forward with host buffers (source traces H2D, receiver traces D2H inside the timed
region); `roofline` is the dense-update kernel alone; `cpu_baseline` is the f64 oracle on
the host cores.  `--impl reference` times the CPU implementation (oracle/_ref when the
reference's own sources were compiled here, else the oracle port).  At N = 1 the line also
carries `other_operators`: device-timed GPts/s of the adjoint, the gradient sweep and the TTI
forward operator on the same grid (extras, not the contract metric; --no-other-ops skips them),
and `value_runs`: three timed windows of exactly K steps each, of which `value` is the median.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

BYTES_PER_POINT = 20.0   # u[t], u[t-1], u[t+1], m, damp, one touch each
N_PHYS, ORDER, NBL, H = 512, 8, 40, 12.5


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ---- clocks ---------------------------------------------------------------------------

class ClockSampler:
    """nvidia-smi samples during the timed region (B200_PROFILING.md clocks line)."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.rows, self.proc, self.index = [], None, index

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-i", str(self.index), "-lms", "100"], stdout=subprocess.PIPE, text=True)
            self.th = threading.Thread(target=self._pump, daemon=True)
            self.th.start()
        except OSError:
            self.proc = None
        return self

    def _pump(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            self.th.join(timeout=2)

    def summary(self):
        sm, mx, reasons = [], 0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                mx = max(mx, float(r[1]))
                for n, v in zip(names, r[3:7]):
                    if v.lower().startswith("active"):
                        reasons.add(n)
            except (ValueError, IndexError):
                pass
        busy = [s for s in sm if s > 0.6 * mx] or sm
        return {"sm_mhz": float(np.median(busy)) if busy else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---- workload -------------------------------------------------------------------------

def build_workload(nsteps_total):
    """configs[1] through the C++ host layer (SeismicModel / AcquisitionGeometry)."""
    from paper_1808_01995_b200 import _sfb_host as Hst
    from paper_1808_01995_b200 import synthetic as syn
    cfg = syn.config(2, N_PHYS)
    t0 = time.time()
    vel = cfg["velocity"]()
    log(f"[bench] velocity {vel.shape} in {time.time() - t0:.1f}s "
        f"[{vel.min():.3f}, {vel.max():.3f}]")
    t0 = time.time()
    model = Hst.SeismicModel(cfg["shape"], [H] * 3, [0.0] * 3, vel, NBL, ORDER)
    del vel
    dt, tn = syn.time_axis(model.critical_dt(ORDER), nsteps_total)
    geom = Hst.AcquisitionGeometry(model, np.asarray(cfg["src"]).ravel(), cfg["rec"].ravel(),
                                   0.0, tn, dt, cfg["f0"])
    assert geom.nt == nsteps_total + 2, (geom.nt, nsteps_total)
    log(f"[bench] model + geometry in {time.time() - t0:.1f}s: N={model.grid.shape} dt={dt:.6f} "
        f"nt={geom.nt} n_rec={geom.n_rec}")
    return cfg, model, geom


def make_plan(model, geom, device=0, slab=None):
    from paper_1808_01995_b200 import capi
    plan = capi.Plan(model.grid.shape, model.grid.spacing, ORDER, geom.dt, geom.nt, device, slab)
    plan.set_model(model.m.array(), model.damp.array(), model.v_max)
    nd = 3
    plan.set_points(capi.CLOUD_SRC, np.array(geom.src.base_table).reshape(-1, nd),
                    np.array(geom.src.weight_table).reshape(-1, 8))
    plan.set_points(capi.CLOUD_REC, np.array(geom.rec.base_table).reshape(-1, nd),
                    np.array(geom.rec.weight_table).reshape(-1, 8))
    return plan


def other_operators(plan, geom, rec, model, device):
    """Device-timed throughput of the other operators of the path on the same grid (not part
    of the contract's metric; reported so that every operator has a number from this box):
    adjoint and FWI-gradient sweep at order 8 on the bench plan, TTI forward at order 12
    (config 4's size) on its own plan with cheap analytic Thomsen fields."""
    from paper_1808_01995_b200 import capi
    out = {"unit": "GPts/s", "grid": list(model.grid.shape)}
    try:
        plan.upload_traces(capi.CLOUD_REC, rec)
        out["adjoint_so8"] = plan.run_resident(capi.OP_ADJOINT).gpts_per_s
        se = max(4, -(-geom.nt // 100))
        f = plan.run_resident(capi.OP_FORWARD, se)
        g = plan.run_resident(capi.OP_GRADIENT)
        out["forward_saving_so8"] = f.gpts_per_s
        out["gradient_sweep_so8"] = g.gpts_per_s
        out["gradient_images_every"] = se
        out["gradient_roofline_28B"] = peaks()[0] / 28.0
    except Exception as e:  # never lose the contract line over an extra
        out["error_acoustic"] = repr(e)
    try:
        N = list(model.grid.shape)
        steps = 20
        lin = [np.linspace(0.0, 1.0, n) for n in N]
        ones = np.ones(N)
        eps = 0.3 * lin[0][:, None, None] * ones
        delta = 0.2 * lin[1][None, :, None] * lin[0][:, None, None] * ones
        theta = (np.pi / 4) * lin[2][None, None, :] * ones
        phi = (np.pi / 4) * lin[1][None, :, None] * ones
        dt = 0.9 * capi.critical_dt(list(model.grid.spacing), model.v_max, 12) / np.sqrt(1.6)
        tp = capi.Plan(N, model.grid.spacing, 12, dt, steps + 2, device)
        tp.set_model(model.m.array(), model.damp.array(), model.v_max)
        tp.set_model_tti(eps, delta, theta, phi)
        del eps, delta, theta, phi, ones
        tp.set_points(capi.CLOUD_SRC, np.array(geom.src.base_table).reshape(-1, 3),
                      np.array(geom.src.weight_table).reshape(-1, 8))
        tp.set_points(capi.CLOUD_REC, np.array(geom.rec.base_table).reshape(-1, 3),
                      np.array(geom.rec.weight_table).reshape(-1, 8))
        tp.upload_traces(capi.CLOUD_SRC, np.sin(np.arange(steps + 2) * 0.1).reshape(-1, 1))
        tp.run_resident(capi.OP_TTI_FORWARD)
        r = tp.run_resident(capi.OP_TTI_FORWARD)
        out["tti_forward_so12"] = r.gpts_per_s
        out["tti_roofline_48B"] = peaks()[0] / 48.0
        out["tti_tflops"] = r.gflops / 1e3
        tp.close()
    except Exception as e:
        out["error_tti"] = repr(e)
    return out


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ---- CPU arm ----------------------------------------------------------------------------

def cpu_run(model_shape, vmax_dt, steps, threads=None):
    """Oracle (f64 port of the reference's loop nest, all host threads) on the same 592^3
    order-8 dense update; returns (GPts/s, threads, seconds)."""
    from oracle import oracle as o
    if threads:
        o.set_num_threads(threads)
    N = model_shape
    rng = np.random.default_rng(7)

    class M:  # minimal stand-in carrying what dense_steps reads
        pass
    m = M()
    m.ndim, m.N, m.spacing = 3, list(N), [H] * 3
    m.m = np.full(N, 1.0 / 3.0 ** 2)
    m.m += 0.05 * rng.random(N[2])[None, None, :]
    m.damp = np.zeros(N)
    m.damp[:NBL] = 0.01
    cur = rng.standard_normal(N) * 1e-3
    old = cur.copy()
    t0 = time.time()
    o.dense_steps(m, ORDER, vmax_dt, steps, cur, old)
    sec = time.time() - t0
    return float(np.prod(N)) * steps / sec / 1e9, o.num_threads(), sec


def reference_cpu(n, steps):
    """The reference's OWN engines (oracle/_ref: its unmodified sources compiled in place) on
    the bare order-8 acoustic update of an n^3 grid -- the recipe of its `bench`
    (proj/src/verify.cpp:338-376).  Tries its default engine (emitted C, serial) and its
    threaded interpreter with every host thread, returns the faster."""
    from oracle import ref
    cores = os.cpu_count() or 1
    best = None
    trials = [("interpreter", ref.INTERPRETER, cores)]
    if ref.emit_available():
        trials.insert(0, ("emitted-C (cc -O2, serial: proj/src/emit.cpp:282-283)", ref.EMITTED, 1))
    for name, be, thr in trials:
        sec, _ = ref.dense_bench(n, ORDER, steps, be, thr)
        g = float(n) ** 3 * steps / sec / 1e9
        if best is None or g > best[0]:
            best = (g, thr, sec, name)
    return best


def reference_arm(args):
    """`--impl reference`: the CPU implementation of the path on this box's host cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    n = N_PHYS + 2 * NBL
    from oracle import ref
    from paper_1808_01995_b200 import capi
    if ref.available():
        kind = "reference"
        g1, thr, s1, name = reference_cpu(n, 1)          # calibration (also warms the C cache)
        k = max(1, min(args.steps, int(20.0 / max(s1, 1e-3))))
        gpts, cores, sec, name = reference_cpu(n, k)
        sample = (f"{k} dense time steps of the full 592^3 order-8 grid on the reference's own "
                  f"engine ({name}, {cores} thread(s)), f64")
        w = 1
    else:
        kind = "port"
        dt = capi.critical_dt([H] * 3, 4.5, ORDER)
        gpts, cores, sec = cpu_run([n] * 3, dt, 1)
        k = max(1, min(args.steps, int(25.0 / max(sec, 1e-3))))
        w = 1
        gpts, cores, sec = cpu_run([n] * 3, dt, k)
        sample = (f"{k} dense time steps of the full 592^3 order-8 grid (f64 oracle port, "
                  f"OpenMP, {cores} threads)")
    line = {
        "impl": "reference", "metric": "acoustic_forward_gpts_per_s", "value": gpts,
        "unit": "GPts/s", "n_gpus": args.gpus, "steps": k, "warmup": w,
        "ms_per_step": sec / k * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args.gpus),
        "cpu_baseline": {"value": gpts, "unit": "GPts/s", "cores": cores, "kind": kind,
                         "sample": sample},
        "e2e": {"value": gpts, "unit": "GPts/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


def workload_config(n_gpus):
    return {"workload": "BASELINE.json configs[1]: acoustic forward, 512^3 physical + 40-node "
                        "absorbing layer (592^3 computed), space order 8, fp32, 1 Ricker source, "
                        "512x512 receivers, seeded smoothed-noise velocity in [1.5,4.5] km/s",
            "grid": [N_PHYS + 2 * NBL] * 3, "space_order": ORDER,
            "decomposition": f"{n_gpus} slab(s) along the slowest axis",
            "l2": "every field (0.83 GB) is larger than the 126 MB L2: no flush needed"}


# ---- our arm -----------------------------------------------------------------------------

def ours(args):
    import torch
    from paper_1808_01995_b200 import capi
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if not torch.cuda.is_available() or capi.device_count() < 1:
        raise SystemExit("bench.py needs a CUDA device: there is no CPU fallback")
    K, W = args.steps, max(args.warmup, 3)
    if world > 1 or os.environ.get("SFB_BENCH_FORCE_DIST"):
        from paper_1808_01995_b200 import slabs
        return slabs.bench_distributed(args, K, W, build_workload, workload_config,
                                       BYTES_PER_POINT, peaks)
    torch.cuda.set_device(local)
    cfg, model, geom = build_workload(W + K)
    N = model.grid.shape
    pts = float(np.prod(N))
    t0 = time.time()
    plan = make_plan(model, geom, local)
    tile = plan.autotune()   # as in the paper, timing starts after the tile-shape autotuning
    log(f"[bench] plan + uploads in {time.time() - t0:.1f}s, tile {tile}")
    src = geom.src.traces
    plan.upload_traces(capi.CLOUD_SRC, src)

    # --- value: K steps after W warm-up steps, inputs resident, device-timed ------------
    F = capi.OP_FORWARD
    plan.step_begin(F)
    plan.run_steps(F, 1, 1 + W)
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        rep = plan.run_steps(F, 1 + W, 1 + W + K)
        torch.cuda.synchronize()
        # two more windows of exactly K steps each ("median of >= 3"); the
        # line's value is the median window, all three are listed in `value_runs`
        windows = [rep]
        for _ in range(2):
            plan.step_begin(F)
            plan.run_steps(F, 1, 1 + W)
            windows.append(plan.run_steps(F, 1 + W, 1 + W + K))
            torch.cuda.synchronize()
        windows.sort(key=lambda r: r.seconds)
        value_runs = [pts * K / r.seconds / 1e9 for r in windows]
        rep = windows[1]
        # --- roofline: the dense-update kernel alone over the same K steps ----------------
        plan.step_begin(F)
        plan.run_steps(F, 1, 1 + W)
        st = plan.time_stencil(F, 1 + W, 1 + W + K)
    clocks = clk.summary()
    plan.step_end(F)
    value = pts * K / rep.seconds / 1e9
    kern_s = st.seconds / st.steps
    peak, peak_kind = peaks()
    achieved = BYTES_PER_POINT * pts / kern_s / 1e9
    traffic = None
    tf = os.path.join(ROOT, "profiles", "r01_traffic.json")
    if os.path.exists(tf):
        with open(tf) as f:
            traffic = json.load(f).get("dram_bytes_per_launch")

    # --- e2e: the C-ABI call with host buffers, K steps ---------------------------------
    plan.close()
    from paper_1808_01995_b200 import _sfb_host as Hst
    from paper_1808_01995_b200 import synthetic as syn
    dt, tn = syn.time_axis(model.critical_dt(ORDER), K)
    geom2 = Hst.AcquisitionGeometry(model, np.asarray(cfg["src"]).ravel(), cfg["rec"].ravel(),
                                    0.0, tn, dt, cfg["f0"])
    plan2 = make_plan(model, geom2, local)
    src2 = np.ascontiguousarray(geom2.src.traces)
    # the caller owns the receiver table (as geom.rec()->traces() in the reference): one
    # buffer, touched by the warm-up pass, filled again by the timed call
    rec = np.empty((geom2.nt, geom2.n_rec))
    plan2.forward(src2[:], out=rec)  # warm-up pass (allocations, first touch of every buffer)
    t0 = time.perf_counter()
    rec, rep2 = plan2.forward(src2, out=rec)
    e2e_s = time.perf_counter() - t0
    e2e = pts * K / e2e_s / 1e9
    assert np.isfinite(rec).all() and float(np.abs(rec).max()) > 0.0
    other = None
    if not args.no_other_ops:
        other = other_operators(plan2, geom2, rec, model, local)
    plan2.close()

    # --- CPU baseline on this box's host cores (bounded sample) -------------------------
    cpu = None
    if not args.no_cpu:
        g1, cores, s1 = cpu_run(N, geom.dt, 1)
        n = max(2, min(40, int(10.0 / max(s1, 1e-3))))
        g, cores, s = cpu_run(N, geom.dt, n)
        cpu = {"value": g, "unit": "GPts/s", "cores": cores, "kind": "port",
               "sample": f"{n} dense time steps of the same 592^3 order-8 grid, f64 oracle "
                         f"(oracle/sf_oracle.c, gcc -O3 -fopenmp), {s:.1f} s"}
        from oracle import ref
        if ref.available():
            rg, rthr, rs, rname = reference_cpu(N[0], 2)
            cpu = {"value": rg, "unit": "GPts/s", "cores": rthr, "kind": "reference",
                   "sample": f"2 dense time steps of the same 592^3 order-8 grid on the "
                             f"reference's own engine ({rname}), {rs:.1f} s; the OpenMP oracle "
                             f"port reaches {g:.3f} GPts/s on {cores} threads"}

    line = {
        "metric": "acoustic_forward_gpts_per_s", "value": value, "unit": "GPts/s", "n_gpus": 1,
        "steps": K, "warmup": W, "ms_per_step": rep.seconds / K * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": workload_config(1),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "peak_kind": peak_kind,
                     "kernel": ("acoustic_step_dual_kernel" if tile["stages"] < 0
                                else "acoustic_step_kernel"), "kernel_ms": kern_s * 1e3,
                     "algorithmic_bytes_per_launch": BYTES_PER_POINT * pts,
                     "tile": tile},
        "cpu_baseline": cpu,
        "e2e": {"value": e2e, "unit": "GPts/s", "h2d_bytes_per_step": int(geom2.n_src * 8),
                "d2h_bytes_per_step": int(geom2.n_rec * 8), "seconds": e2e_s,
                "device_seconds": rep2.seconds},
        "gpu_launches": int(rep.kernel_launches),
        "clocks": clocks,
        "value_runs": value_runs,
    }
    if other is not None:
        line["other_operators"] = other
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-other-ops", action="store_true",
                    help="skip the adjoint / gradient / TTI extras of the JSON line")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    args = ap.parse_args()
    if args.impl == "reference":
        return reference_arm(args)
    return ours(args)


if __name__ == "__main__":
    main()
