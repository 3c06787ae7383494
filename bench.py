#!/usr/bin/env python
"""bench.py -- benchmark of the wave-propagator path (BASELINE.json metric: GPts/s per operator
at 1/2/4/8 B200 and the fraction of the HBM roofline).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config 2|3|4|5] [--op forward|adjoint|gradient|tti] [--scaling strong|weak]
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N ...

GPts/s = computed (padded) grid nodes x time steps / seconds of the stepping loop.  A "step" is
one time step of the operator: dense update + point scatter + point gather (+ imaging for the
gradient sweep; two launches for the TTI pair).

Workloads (--config is BASELINE.json's 1-based numbering; default 2 = configs[1], the
configuration the metric is quoted on):
  2  acoustic forward, 592^3 computed nodes, order 8, 1 source, 512 x 512 receivers
  3  acoustic FWI gradient sweep on the two-layer medium, 592^3, order 8, every 4th level saved
  4  TTI forward, 592^3, order 12, seeded smooth Thomsen fields (delta clipped to epsilon:
     the builder's pseudo-acoustic system is ill-posed otherwise)
  5  large-domain acoustic forward, order 16, 8 off-node sources, 1024 x 1024 receivers; weak
     scaling (default): 1024 x 1024 x (128 N) physical nodes, slab axis first
At N > 1 the grid is cut into N slabs along the slowest axis; ghost planes are pushed into the
neighbours' memory by the update kernels (CUDA IPC) with NCCL send/recv as the fallback
(SFB_HALO=nccl forces it).  Every operator runs there: --op adjoint on config 2, --config 3
(the gradient sweep against a history that a forward slab run of the same plans saved),
--config 4 (the TTI pair pushes g, then the new p and r).

One JSON line on stdout (rank 0).  `value`: device-timed (CUDA events on the plan's stream,
max over ranks), inputs resident in HBM.  `e2e`: the same metric through the C-ABI with HOST
buffers, host<->device copies inside the timed region.  `roofline`: the dominant kernel alone
(N = 1) against MEASURED_PEAKS.json.  `cpu_baseline` / `--impl reference`: the reference's own
CPU engine (oracle/_ref) or the oracle port on the host cores, bounded sample.  The default
N = 1 line also carries `operators`: adjoint, gradient sweep and TTI forward on the same
grid, each with its own roofline and e2e (--no-other-ops skips them).
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

NBL, H = 40, 12.5
CONFIGS = {
    2: dict(key="configs[1]", op="forward", order=8, n=512, scaling="strong"),
    3: dict(key="configs[2]", op="gradient", order=8, n=512, scaling="strong"),
    4: dict(key="configs[3]", op="tti", order=12, n=512, scaling="strong"),
    5: dict(key="configs[4]", op="forward", order=16, n=1024, scaling="weak", per_rank=128),
}
# contract bytes per node-step and what the kernels really have to move
CONTRACT_BYTES = {"forward": 20.0, "adjoint": 20.0, "gradient": 28.0, "tti": 48.0}
METRIC = {"forward": "acoustic_forward_gpts_per_s", "adjoint": "acoustic_adjoint_gpts_per_s",
          "gradient": "acoustic_gradient_gpts_per_s", "tti": "tti_forward_gpts_per_s"}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def actual_bytes(op, sep, images_every=1):
    """Bytes a node-step must move with this build's data layout: the separable-damping kernel
    rebuilds damp from three 1-D profiles (16 B instead of 20); the gradient sweep adds the
    grad read-modify-write and the snapshot read on imaging steps only; the TTI pair streams
    a, b, c for theta, phi."""
    base = 16.0 if sep else 20.0
    if op == "gradient":
        return base + 12.0 / max(images_every, 1)
    if op == "tti":
        return 48.0 if sep else 52.0
    return base


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


# ---- workloads ------------------------------------------------------------------------

def grid_of(config, world, scaling):
    """computed (padded) extents and physical extents of a configuration at `world` GPUs"""
    c = CONFIGS[config]
    if config == 5 and scaling == "weak":
        phys = [c["per_rank"] * world, c["n"], c["n"]]
    else:
        phys = [c["n"]] * 3
    return [p + 2 * NBL for p in phys], phys


def workload_config(config, op, world, scaling, extra=None):
    c = CONFIGS[config]
    N, phys = grid_of(config, world, scaling)
    what = {
        2: "acoustic forward, 1 off-node 15 Hz Ricker source, 512x512 receivers at 25 m, seeded "
           "smoothed-noise velocity (sigma 8) in [1.5,4.5] km/s",
        3: "acoustic FWI gradient sweep (forward history every 4th level in HBM, residual traces at "
           "512x512 receivers, imaging fused into the sweep), two-layer medium 1.5/2.5 km/s",
        4: "TTI forward (rotated first-derivative pairs, coupled p/r), seeded smooth fields: v in "
           "[1.5,4.5], epsilon in [0,0.3], delta in [0,0.2] clipped to delta <= epsilon (deviation "
           "from BASELINE: the builder's system is ill-posed for epsilon < delta), theta, phi in "
           "[0,pi/4]; 1 source, 512x512 receivers",
        5: "large-domain acoustic forward, 8 seeded off-node sources, 1024x1024 receivers at 25 m, "
           "seeded smoothed-noise velocity in [1.5,4.5] km/s generated per slab",
    }[config]
    if op != c["op"]:
        what = f"{op} operator on the grid and medium of: " + what
    cfg = {"workload": f"BASELINE.json {c['key']}: {what}; {phys[0]}x{phys[1]}x{phys[2]} physical + "
                       f"{NBL}-node absorbing layer = {N[0]}x{N[1]}x{N[2]} computed nodes, space order "
                       f"{c['order']}, fp32",
           "grid": N, "space_order": c["order"], "operator": op,
           "decomposition": f"{world} slab(s) along the slowest axis",
           "l2": f"every field ({np.prod(N) * 4 / world / 1e9:.2f} GB per GPU) is larger than the "
                 "126 MB L2: no flush needed"}
    if extra:
        cfg.update(extra)
    return cfg


class Workload:
    """One configuration's host-side inputs for one rank."""

    def __init__(self, config, op, nsteps, rank=0, world=1, scaling="strong"):
        from paper_1808_01995_b200 import capi, slabs
        from paper_1808_01995_b200 import synthetic as syn
        self.config, self.op, self.rank, self.world = config, op, rank, world
        c = CONFIGS[config]
        self.order = c["order"]
        self.N, self.phys = grid_of(config, world, scaling)
        self.bounds = slabs.split_slabs(self.N[0], world, self.order // 2)
        self.slab = self.bounds[rank] if world > 1 else None
        self.tti = None
        t0 = time.time()
        if config == 5:
            self._build_slab_local(nsteps, syn, capi)
        else:
            self._build_global(nsteps, syn)
        if world > 1:
            # a point is sampled by the rank that owns its base plane: a rank binds -- and later
            # downloads -- only its own receivers (the record is the concatenation over ranks)
            lo, hi = self.slab
            own = (self.rec_base[:, 0] >= lo) & (self.rec_base[:, 0] < hi)
            self.n_rec_global = int(self.rec_base.shape[0])
            self.rec_base, self.rec_w = self.rec_base[own], self.rec_w[own]
            if self.rec_base.shape[0] == 0:   # keep the cloud non-empty: one receiver of the rank below
                self.rec_base = np.array([[lo, 0, 0]], dtype=np.int64)
                self.rec_w = np.zeros((1, 8))
        log(f"[bench] rank {rank}: workload {config} built in {time.time() - t0:.1f}s: N={self.N} "
            f"dt={self.dt:.6f} nt={self.nt} n_src={self.src_base.shape[0]} n_rec={self.rec_base.shape[0]}")

    def _build_global(self, nsteps, syn):
        from paper_1808_01995_b200 import _sfb_host as Hst
        cfg = syn.config(self.config, CONFIGS[self.config]["n"])
        self.vel_phys = cfg["velocity"]()
        model = Hst.SeismicModel(cfg["shape"], [H] * 3, [0.0] * 3, self.vel_phys, NBL, self.order)
        crit = model.critical_dt(self.order)
        if self.op == "tti":
            eps, delta, theta, phi = cfg["tti"]() if "tti" in cfg else syn.tti_fields(cfg["shape"])
            self.tti = [syn.extend(f, NBL) for f in (eps, delta, theta, phi)]
            crit = 0.9 * crit / np.sqrt(1.0 + 2.0 * float(eps.max()))
        dt, tn = syn.time_axis(crit, nsteps)
        # the geometry checks dt against the acoustic limit only; the TTI limit is smaller
        geom = Hst.AcquisitionGeometry(model, np.asarray(cfg["src"]).ravel(), cfg["rec"].ravel(),
                                       0.0, tn, dt, cfg["f0"])
        assert geom.nt == nsteps + 2, (geom.nt, nsteps)
        self.model, self.geom = model, geom
        self.dt, self.nt, self.v_max = dt, geom.nt, model.v_max
        self.src_base = np.array(geom.src.base_table).reshape(-1, 3)
        self.src_w = np.array(geom.src.weight_table).reshape(-1, 8)
        self.rec_base = np.array(geom.rec.base_table).reshape(-1, 3)
        self.rec_w = np.array(geom.rec.weight_table).reshape(-1, 8)
        self.src = np.ascontiguousarray(geom.src.traces)
        self.m = lambda: model.m.array()
        self.damp = lambda: model.damp.array()

    def _build_slab_local(self, nsteps, syn, capi):
        """configs[4]: no rank holds a global field (1104^3 in f64 is 10.8 GB per field)."""
        from paper_1808_01995_b200 import _sfb_host as Hst
        self.v_max = 4.5
        self.dt = capi.critical_dt([H] * 3, self.v_max, self.order)
        self.nt = nsteps + 2
        lo, hi = self.slab if self.slab else (0, self.N[0])
        self._m, self._damp = syn.slab_model(
            self.phys, NBL, [H] * 3, lo, hi,
            lambda a, b: syn.smooth_slab(self.phys, a, b, syn.SEED + 6, 8.0, 1.5, 4.5), self.v_max)
        ext = [H * (p - 1) for p in self.phys]
        src = np.random.default_rng(syn.SEED + 7).uniform([0, 0, 0], ext, size=(8, 3))
        n = CONFIGS[5]["n"]
        ii, jj = np.meshgrid(np.linspace(0.0, ext[0], n), np.arange(n) * H, indexing="ij")
        rec = np.stack([ii.ravel(), jj.ravel(), np.full(ii.size, 25.0)], axis=1)
        org = [-NBL * H] * 3
        self.src_base, self.src_w = capi.locate(self.N, [H] * 3, org, src)
        self.rec_base, self.rec_w = capi.locate(self.N, [H] * 3, org, rec)
        wavelet = np.asarray(Hst.ricker(0.015, 0.0, self.dt, self.nt))
        self.src = np.repeat(wavelet[:, None], 8, axis=1).copy()
        self.m = self.damp = None

    def make_plan(self, device, dense_damping=False):
        from paper_1808_01995_b200 import capi
        plan = capi.Plan(self.N, [H] * 3, self.order, self.dt, self.nt, device, self.slab,
                         dense_damping=dense_damping)
        if self.m is None:
            plan.set_model_slab(self._m, self._damp, self.v_max)
        else:
            plan.set_model(self.m(), self.damp(), self.v_max)
        plan.set_points(capi.CLOUD_SRC, self.src_base, self.src_w)
        plan.set_points(capi.CLOUD_REC, self.rec_base, self.rec_w)
        if self.tti is not None:
            plan.set_model_tti(*self.tti)
        return plan

    def residual_traces(self):
        """configs[2]: N(0,1) noise per receiver convolved in time with the 15 Hz Ricker"""
        from paper_1808_01995_b200 import _sfb_host as Hst
        from paper_1808_01995_b200 import synthetic as syn
        n_rec = self.rec_base.shape[0]
        spec = np.fft.rfft(np.asarray(Hst.ricker(0.015, 0.0, self.dt, self.nt)))[:, None]
        rng = np.random.default_rng(syn.SEED + 10)
        out = np.empty((self.nt, n_rec))
        for lo in range(0, n_rec, 65536):
            xi = rng.standard_normal((self.nt, min(65536, n_rec - lo)))
            out[:, lo:lo + xi.shape[1]] = np.fft.irfft(np.fft.rfft(xi, axis=0) * spec, n=self.nt, axis=0)
        out[[0, self.nt - 1]] = 0.0
        return out


# ---- one operator on one GPU ------------------------------------------------------------

def op_ids(op):
    from paper_1808_01995_b200 import capi
    return {"forward": capi.OP_FORWARD, "adjoint": capi.OP_ADJOINT, "gradient": capi.OP_GRADIENT,
            "tti": capi.OP_TTI_FORWARD}[op]


def windows(plan, op, nt, W, K, runs=3, stencil_only=False):
    """`runs` windows of exactly K steps, each after W untimed warm-up steps from a zeroed
    state; device-timed by the engine (CUDA events on the plan's stream).  Sorted by time."""
    import torch
    oid = op_ids(op)
    fn = plan.time_stencil if stencil_only else plan.run_steps
    out = []
    for _ in range(runs):
        plan.step_begin(oid)
        if op in ("adjoint", "gradient"):      # descending: window [a, b) runs t = b-1 .. a
            top = nt - 1
            plan.run_steps(oid, top - W, top)
            out.append(fn(oid, top - W - K, top - W))
        else:
            plan.run_steps(oid, 1, 1 + W)
            out.append(fn(oid, 1 + W, 1 + W + K))
        torch.cuda.synchronize()
    return sorted(out, key=lambda r: r.seconds)


def roofline_of(op, pts, kernel_s, sep, images_every, tile, K_half, clocks, grid=None):
    """`achieved` uses the bytes this build's kernels must move per node-step (see
    actual_bytes); the SURVEY.md 8(d) contract figure is carried beside it."""
    peak, kind = peaks()
    b = actual_bytes(op, sep, images_every)
    cb = CONTRACT_BYTES[op]
    r = {"bound": "hbm", "achieved": b * pts / kernel_s / 1e9, "peak": peak, "unit": "GB/s",
         "frac": b * pts / kernel_s / 1e9 / peak, "peak_kind": kind,
         "frac_actual_bytes": b * pts / kernel_s / 1e9 / peak,     # the same figure, named as in VERDICT r1
         "basis_bytes_per_point": b, "algorithmic_bytes_per_launch": b * pts,
         "contract_bytes_per_point": cb, "achieved_contract": cb * pts / kernel_s / 1e9,
         "frac_contract": cb * pts / kernel_s / 1e9 / peak,
         "basis": ("bytes the kernel must move with this build's layout (separable damping "
                   "rebuilt from 1-D profiles: 16 B; the SURVEY.md 8(d) contract figure of "
                   f"{cb:.0f} B is in *_contract)"),
         "kernel_ms": kernel_s * 1e3, "tile": tile}
    if op == "tti":
        r["kernel"] = "tti_rot_kernel + tti_div_update_kernel (two launches per step)"
        flops = 57.0 * K_half + 29.0          # reference accounting, engine_tti.cu
        sm_mhz = (clocks or {}).get("sm_mhz") or 1965.0
        fp32_peak = 148 * 128 * 2 * sm_mhz * 1e6 / 1e12
        r["fp32"] = {"flops_per_point": flops, "achieved_tflops": flops * pts / kernel_s / 1e12,
                     "peak_tflops": fp32_peak, "frac": flops * pts / kernel_s / 1e12 / fp32_peak}
    else:
        r["kernel"] = "acoustic_step_dual_kernel" if tile.get("stages", 0) < 0 else "acoustic_step_kernel"
    if op == "gradient":
        r["images_every"] = images_every
    r.update(static_traffic(op, sep, grid, 2 * K_half))
    return r


def static_traffic(op, sep, grid, order):
    """DRAM bytes per launch from the committed ncu --set full capture of the same kernel on
    the same grid (profiles/r02_traffic.json, written by tools/ncu_summary.py); it cannot be
    measured inside an unprofiled run, and there is a capture for the 592^3 grid only."""
    path = os.path.join(ROOT, "profiles", "r02_traffic.json")
    key = {"forward": "acoustic_sep" if sep else "acoustic_dense", "adjoint": "acoustic_sep" if sep else "acoustic_dense",
           "gradient": "gradient", "tti": "tti"}[op]
    if list(grid or []) != [592, 592, 592] or order != (12 if op == "tti" else 8):
        return {"traffic": None, "traffic_source": "no ncu capture committed for this grid / order"}
    try:
        with open(path) as f:
            d = json.load(f)
        return {"traffic": d[key]["dram_bytes_per_launch"],
                "traffic_source": f"static: {d[key]['source']} (ncu --set full, dram__bytes_read.sum + "
                                  "dram__bytes_write.sum per launch)"}
    except Exception:
        return {"traffic": None, "traffic_source": "no ncu capture committed for this kernel"}


def measure_op(wl, op, K, W, device, want_e2e=True):
    """value / roofline / e2e of one operator on one GPU; returns a dict (no `metric` keys)."""
    import torch
    from paper_1808_01995_b200 import capi
    pts = float(np.prod(wl.N))
    plan = wl.make_plan(device)
    tile = plan.autotune() if op != "tti" else {}
    sep = bool(plan.get_tile()["sep"])
    images_every = 1
    plan.upload_traces(capi.CLOUD_SRC, wl.src)
    data = None
    if op in ("adjoint", "gradient"):
        data = wl.residual_traces()
        plan.upload_traces(capi.CLOUD_REC, data)
    if op == "gradient":
        images_every = 4                       # configs[2]: every 4th level saved in HBM
        plan.run_resident(capi.OP_FORWARD, images_every)
    with ClockSampler(device) as clk:
        ws = windows(plan, op, wl.nt, W, K)
        st = windows(plan, op, wl.nt, W, K, runs=1, stencil_only=True)[0]
    clocks = clk.summary()
    rep = ws[len(ws) // 2]
    res = {"value": pts * K / rep.seconds / 1e9, "unit": "GPts/s", "ms_per_step": rep.seconds / K * 1e3,
           "value_runs": [pts * K / r.seconds / 1e9 for r in ws], "gpu_launches": int(rep.kernel_launches),
           "clocks": clocks,
           "roofline": roofline_of(op, pts, st.seconds / st.steps, sep, images_every,
                                   plan.get_tile() if op != "tti" else {}, wl.order // 2, clocks, wl.N)}
    if want_e2e:
        # the C-ABI call with HOST buffers over exactly K steps: a plan with nt = K + 2
        plan.close()
        wk = wl_with_steps(wl, K)
        p2 = wk.make_plan(device)
        if tile:
            p2.set_tile(tile["txv"], tile["ty"], tile["stages"], 0)
        n_src, n_rec = wk.src_base.shape[0], wk.rec_base.shape[0]
        if op == "forward":
            rec = np.empty((wk.nt, n_rec))
            call = lambda: p2.forward(wk.src, out=rec)[0]          # noqa: E731
            h2d, d2h = n_src * 8, n_rec * 8
        elif op == "tti":
            call = lambda: p2.tti_forward(wk.src)[0]               # noqa: E731
            h2d, d2h = n_src * 8, n_rec * 8
        elif op == "adjoint":
            d2 = wk.residual_traces()
            call = lambda: p2.adjoint(d2)[0]                       # noqa: E731
            h2d, d2h = n_rec * 8, n_src * 8
        else:
            d2 = wk.residual_traces()
            p2.forward(wk.src, save_every=images_every)            # the history the sweep images against
            gbuf = np.zeros(wk.N)                                  # the caller owns the gradient array
            call = lambda: p2.gradient(d2, out=gbuf)[0]            # noqa: E731
            h2d, d2h = n_rec * 8, int(pts * 8 / K)                 # grad (f64, padded grid) comes back once
        call()                                                     # warm-up: allocations, first touch
        t0 = time.perf_counter()
        out = call()
        sec = time.perf_counter() - t0
        assert np.isfinite(out).all()
        if wl.config != 5:    # configs[4]'s random sources may sit far from the receiver plane
            assert float(np.abs(out).max()) > 0.0
        res["e2e"] = {"value": pts * K / sec / 1e9, "unit": "GPts/s", "h2d_bytes_per_step": int(h2d),
                      "d2h_bytes_per_step": int(d2h), "seconds": sec,
                      "call": {"forward": "sfb_forward", "adjoint": "sfb_adjoint",
                               "gradient": "sfb_gradient (history of a prior sfb_forward resident)",
                               "tti": "sfb_tti_forward"}[op]}
        p2.close()
    else:
        plan.close()
    torch.cuda.synchronize()
    return res


def wl_with_steps(wl, nsteps):
    """the same configuration over `nsteps` steps: only the time axis shrinks (the Ricker
    source table of a shorter run is a prefix of the longer one's)"""
    if wl.nt == nsteps + 2:
        return wl
    assert nsteps + 2 <= wl.nt
    w2 = object.__new__(Workload)
    w2.__dict__.update(wl.__dict__)
    w2.nt = nsteps + 2
    w2.src = np.ascontiguousarray(wl.src[: w2.nt])
    return w2


def cheap_tti_fields(N):
    """analytic Thomsen fields for the TTI extra of the default line (the seeded config-4 fields
    take a minute of host filtering; --op tti / --config 4 uses them)"""
    lin = [np.linspace(0.0, 1.0, n) for n in N]
    ones = np.ones(N)
    eps = 0.3 * lin[0][:, None, None] * ones
    delta = 0.2 * lin[1][None, :, None] * lin[0][:, None, None] * ones
    theta = (np.pi / 4) * lin[2][None, None, :] * ones
    phi = (np.pi / 4) * lin[1][None, :, None] * ones
    return [eps, delta, theta, phi]


# ---- CPU legs ---------------------------------------------------------------------------

def oracle_dense(N, order, dt, steps, threads=None):
    """f64 oracle port (oracle/sf_oracle.c, OpenMP) on the dense update of an N grid."""
    from oracle import oracle as o
    if threads:
        o.set_num_threads(threads)
    rng = np.random.default_rng(7)

    class M:
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
    o.dense_steps(m, order, dt, steps, cur, old)
    sec = time.time() - t0
    return float(np.prod(N)) * steps / sec / 1e9, o.num_threads(), sec


def oracle_tti(planes, order, nsteps):
    """The builder's f64 TTI restatement (oracle/sf_oracle.c, OpenMP) on a planes x 592 x 592
    cut of configs[3]'s grid with analytic Thomsen fields; returns (GPts/s, threads, seconds).
    The reference has no TTI operator: this port is the only CPU implementation there is."""
    from oracle import oracle as o
    n = CONFIGS[4]["n"]
    phys = [max(planes - 2 * NBL, 16), n, n]
    om = o.Model(phys, [H] * 3, [0.0] * 3, np.full(phys, 3.0), NBL, order)
    dt = o.tti_critical_dt(om, order, 0.3)
    c = H * (n - 1) / 2.0 + H / 4.0
    og = o.Geometry(om, [H * (phys[0] - 1) / 2.0, c, 18.75], [[0.0, c, 25.0]], 0.0, (nsteps + 1.5) * dt,
                    dt, 0.015)
    eps, delta, theta, phi = cheap_tti_fields(om.N)
    t0 = time.time()
    o.tti_forward(om, og, order, eps, delta, theta, phi)
    sec = time.time() - t0
    return float(np.prod(om.N)) * nsteps / sec / 1e9, o.num_threads(), sec, om.N


def reference_inputs(config, planes, vel=None):
    """configs[1] / configs[4] inputs cut to `planes` physical planes along the slowest axis
    (the whole workload when planes = the configuration's extent)"""
    from paper_1808_01995_b200 import synthetic as syn
    c = CONFIGS[config]
    n = c["n"]
    shape = [planes, n, n]
    ext0 = H * (planes - 1)
    if config == 5:
        if vel is None:
            vel = syn.smooth_slab([n, n, n], 0, planes, syn.SEED + 6, 8.0, 1.5, 4.5)
        src = np.random.default_rng(syn.SEED + 7).uniform([0, 0, 0], [ext0, H * (n - 1), H * (n - 1)], size=(8, 3))
        ii, jj = np.meshgrid(np.linspace(0.0, ext0, n), np.arange(n) * H, indexing="ij")
        rec = np.stack([ii.ravel(), jj.ravel(), np.full(ii.size, 25.0)], axis=1)
    else:
        cfg = syn.config(2, n)
        if vel is None:
            vel = cfg["velocity"]()
        vel = vel[:planes]
        src = np.asarray(cfg["src"], dtype=float).copy()
        src[:, 0] = np.minimum(src[:, 0], 0.5 * ext0 + H / 4)
        rec = cfg["rec"][cfg["rec"][:, 0] <= ext0]
    return shape, np.ascontiguousarray(vel), src, rec


def reference_forward(config, inputs, nsteps, threads):
    """The reference's OWN forward_operator + run_wave (proj/src/seismic_ops.cpp:58-82,137-141)
    through oracle/_ref, threaded interpreter engine; returns (seconds of its stepping loop,
    computed nodes)."""
    from oracle import oracle as o
    from oracle import ref
    shape, vel, src, rec = inputs
    order = CONFIGS[config]["order"]
    w = o.second_derivative_weights(order)
    sum_abs = float(abs(w[0]) + 2 * np.abs(w[1:]).sum())
    dt = H / 4.5 / np.sqrt(3 * sum_abs / 2.0) * (1.0 - 1e-9)          # critical dt at v_max <= 4.5
    p = ref.Problem(shape, [H] * 3, [0.0] * 3, vel, NBL, order, order, src, rec,
                    0.0, (nsteps + 1.5) * dt, dt, 0.015)
    out = p.forward(backend=ref.INTERPRETER, nthreads=threads, levels=False)
    assert out["nt"] == nsteps + 2, (out["nt"], nsteps)
    return out["seconds"], float(np.prod([x + 2 * NBL for x in shape]))


def reference_arm(args):
    """`--impl reference`: the reference's CPU implementation of the path on this box's host
    cores -- its own forward_operator through oracle/_ref when that was built (kind
    "reference"), else the oracle port (kind "port") -- W warm-up steps, then K timed steps,
    on a sample of the workload bounded to about 150 s of CPU work."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    config, op = args.config, args.op
    K, W = args.steps, max(args.warmup, 1)
    cores = os.cpu_count() or 1
    c = CONFIGS[config]
    order, n1 = c["order"], c["n"] + 2 * NBL
    N, phys = grid_of(config, args.gpus, args.scaling)
    budget = 150.0
    from oracle import ref
    if op == "forward" and config in (2, 5) and ref.available():
        kind = "reference"
        s1, pts1 = reference_forward(config, reference_inputs(config, 48), 2, cores)
        rate = pts1 * 2 / s1                                          # node-steps per second
        total = int(min(N[0], budget * rate / (K + W) / (n1 * n1), 4.0e8 / (n1 * n1)))
        planes = max(48, min(phys[0], total - 2 * NBL))
        inputs = reference_inputs(config, planes)
        reference_forward(config, inputs, W, cores)                   # W untimed warm-up steps
        sec, pts = reference_forward(config, inputs, K, cores)
        gpts = pts * K / sec / 1e9
        sample = (f"the reference's own forward_operator + run_wave (threaded interpreter engine, "
                  f"{cores} threads, f64) on {c['key']}'s inputs"
                  + ("" if planes == phys[0] else f", {planes} of {phys[0]} physical planes along the "
                     "slowest axis (bounded sample)")
                  + f": {K} time steps incl. source injection and receiver sampling, order {order}")
    elif op == "tti":
        kind = "port"
        g1, cores, s1, N1 = oracle_tti(96, order, 1)
        rate = float(np.prod(N1)) / s1
        planes = int(max(96, min(N[0], budget * rate / (K + W) / (n1 * n1), 2.5e8 / (n1 * n1))))
        oracle_tti(planes, order, W)
        gpts, cores, sec, Nt = oracle_tti(planes, order, K)
        sample = (f"{K} time steps of the builder's f64 TTI restatement (oracle/sf_oracle.c, OpenMP, "
                  f"{cores} threads) on {Nt[0]}x{Nt[1]}x{Nt[2]} computed nodes (configs[3]: 592^3), order {order}, "
                  "analytic Thomsen fields; the reference itself has no TTI operator")
    else:
        kind = "port"
        from paper_1808_01995_b200 import capi
        dt = capi.critical_dt([H] * 3, 4.5, order)
        g, cores, s = oracle_dense([64, n1, n1], order, dt, 1)
        rate = 64.0 * n1 * n1 / s
        planes = int(max(64, min(N[0], budget * rate / (K + W) / (n1 * n1), 4.0e8 / (n1 * n1))))
        oracle_dense([planes, n1, n1], order, dt, W)
        gpts, cores, sec = oracle_dense([planes, n1, n1], order, dt, K)
        why = {"forward": "", "adjoint": "; the adjoint and gradient sweeps run this same dense update",
               "gradient": "; the adjoint and gradient sweeps run this same dense update",
               "tti": "; the reference has no TTI operator: the acoustic update at the same order stands in"}[op]
        sample = (f"{K} dense time steps of a {planes}x{n1}x{n1} grid, order {order}, f64 oracle port "
                  f"(oracle/sf_oracle.c, OpenMP, {cores} threads){why}")
    line = {
        "impl": "reference", "metric": METRIC[op], "value": gpts, "unit": "GPts/s",
        "n_gpus": args.gpus, "steps": K, "warmup": W, "ms_per_step": sec / K * 1e3,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": workload_config(config, op, args.gpus, args.scaling),
        "cpu_baseline": {"value": gpts, "unit": "GPts/s", "cores": cores, "kind": kind, "sample": sample},
        "e2e": {"value": gpts, "unit": "GPts/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


def cpu_baseline_leg(config, vel=None):
    """bounded CPU sample beside the GPU line (rank 0): the reference's own engine when
    oracle/_ref exists, with the oracle port's figure quoted in the sample text"""
    from paper_1808_01995_b200 import capi
    c = CONFIGS[config]
    order, n1 = c["order"], c["n"] + 2 * NBL
    dt = capi.critical_dt([H] * 3, 4.5, order)
    if config == 4:   # the TTI pair: the builder's f64 restatement is the only CPU implementation
        g, cores, s, Nt = oracle_tti(176, order, 3)
        return {"value": g, "unit": "GPts/s", "cores": cores, "kind": "port",
                "sample": f"3 time steps of the f64 TTI restatement (oracle/sf_oracle.c, OpenMP) on "
                          f"{Nt[0]}x{Nt[1]}x{Nt[2]} computed nodes, order {order}, {s:.1f} s; the reference "
                          "has no TTI operator"}
    planes, nst = (336, 10) if config != 5 else (96, 10)
    oracle_dense([planes, n1, n1], order, dt, 1)            # first touch of the oracle's buffers
    g, cores, s = oracle_dense([planes, n1, n1], order, dt, nst)
    cpu = {"value": g, "unit": "GPts/s", "cores": cores, "kind": "port",
           "sample": f"{nst} dense time steps of a {planes}x{n1}x{n1} grid (order {order}), f64 oracle port "
                     f"(oracle/sf_oracle.c, gcc -O3 -fopenmp), {s:.1f} s"}
    from oracle import ref
    if ref.available() and config in (2, 5):
        threads = os.cpu_count() or 1
        pl, rst = (256, 8) if config != 5 else (64, 8)
        sec, pts = reference_forward(config, reference_inputs(config, pl, vel), rst, threads)
        cpu = {"value": pts * rst / sec / 1e9, "unit": "GPts/s", "cores": threads, "kind": "reference",
               "sample": f"{rst} time steps of the reference's own forward_operator (threaded interpreter, "
                         f"f64) on {c['key']}'s inputs, {pl} of {c['n']} physical planes along the slowest "
                         f"axis, {sec:.1f} s; the OpenMP oracle port reaches {g:.3f} GPts/s on {cores} threads"}
    return cpu


# ---- our arm, one GPU -------------------------------------------------------------------

def single_gpu(args):
    import torch
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    K, W = args.steps, max(args.warmup, 3)
    config, op = args.config, args.op
    wl = Workload(config, op, W + K, scaling=args.scaling)
    main = measure_op(wl, op, K, W, local)
    line = {"metric": METRIC[op], "value": main["value"], "unit": "GPts/s", "n_gpus": 1, "steps": K,
            "warmup": W, "ms_per_step": main["ms_per_step"], "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": workload_config(config, op, 1, args.scaling),
            "roofline": main["roofline"], "cpu_baseline": None, "e2e": main["e2e"],
            "gpu_launches": main["gpu_launches"], "clocks": main["clocks"],
            "value_runs": main["value_runs"]}
    if op == "forward" and config == 2 and not args.no_other_ops:
        # the dense-damping build of the same kernel really streams the contract's 20 B
        try:
            from paper_1808_01995_b200 import capi
            pd = wl.make_plan(local, dense_damping=True)
            pd.autotune()
            pd.upload_traces(capi.CLOUD_SRC, wl.src)
            st = windows(pd, "forward", wl.nt, W, K, runs=1, stencil_only=True)[0]
            pts = float(np.prod(wl.N))
            ks = st.seconds / st.steps
            line["roofline"]["dense_damping_build"] = {
                "kernel_ms": ks * 1e3, "bytes_per_point": 20.0, "achieved": 20.0 * pts / ks / 1e9,
                "frac": 20.0 * pts / ks / 1e9 / peaks()[0], "tile": pd.get_tile()}
            pd.close()
        except Exception as e:
            line["roofline"]["dense_damping_build"] = {"error": repr(e)}
        ops = {}
        for other in ("adjoint", "gradient"):
            try:
                ops[other] = measure_op(wl, other, K, W, local)
            except Exception as e:  # never lose the contract line over an extra
                ops[other] = {"error": repr(e)}
        try:
            wt = object.__new__(Workload)
            wt.__dict__.update(wl.__dict__)
            wt.config, wt.op, wt.order = 2, "tti", 12
            wt.tti = cheap_tti_fields(wl.N)
            from paper_1808_01995_b200 import capi
            wt.dt = 0.9 * capi.critical_dt([H] * 3, wl.v_max, 12) / np.sqrt(1.6)
            wt.src = np.sin(np.arange(wl.nt) * 0.1).reshape(-1, 1) * np.ones((1, wl.src.shape[1]))
            ops["tti"] = measure_op(wt, "tti", K, W, local, want_e2e=False)
            ops["tti"]["note"] = ("order 12 on the 592^3 grid with analytic Thomsen fields; "
                                  "`--config 4` runs BASELINE.json configs[3] with its seeded fields")
        except Exception as e:
            ops["tti"] = {"error": repr(e)}
        line["operators"] = ops
    if not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline_leg(config, getattr(wl, "vel_phys", None))
    print(json.dumps(line), flush=True)


# ---- our arm, N GPUs ----------------------------------------------------------------------

class SlabJob:
    """bench_core job over one capi.Plan on one GPU: forward (acoustic, TTI), adjoint, or the
    gradient sweep against a history that a forward slab run of the same plans saved."""

    def __init__(self, wl, plan, op, device, rank, world, comm, resid=None, images_every=4):
        import torch
        from paper_1808_01995_b200 import capi, slabs
        self.torch, self.capi, self.wl, self.plan, self.op = torch, capi, wl, plan, op
        self.oid = op_ids(op)
        self.backward = op in ("adjoint", "gradient")
        lo, hi = wl.bounds[rank]
        self.points_owned = float(hi - lo) * wl.N[1] * wl.N[2]
        self.halo = "none (one GPU)"
        self.drv = None
        # injected table (caller input) and sampled table (caller-owned output; written once
        # here so that its pages exist, as those of a long-lived buffer do)
        self.inj = resid if self.backward else wl.src
        self.c_inj = capi.CLOUD_REC if self.backward else capi.CLOUD_SRC
        self.c_smp = capi.CLOUD_SRC if self.backward else capi.CLOUD_REC
        self.rec = None
        if op != "gradient":
            n_smp = wl.src_base.shape[0] if self.backward else wl.rec_base.shape[0]
            self.rec = np.empty((wl.nt, n_smp))
            self.rec.fill(0.0)
        self.grad = None
        ex = slabs.HaloExchanger(rank, world)
        push = os.environ.get("SFB_HALO", "push") == "push"
        if op == "tti":
            self.eng = slabs.TtiPlanEngine(plan, device)
            self._loop = lambda a, b: slabs.tti_step_loop(self.eng, ex, a, b)     # noqa: E731
            make = lambda w: slabs.TtiPeerPushDriver(plan, rank, w)               # noqa: E731
            names = ("nccl send/recv (two exchanges per step: g, then p and r)",
                     "fused peer push (CUDA IPC stores from both passes: g, then the new p and r)")
        else:
            self.eng = slabs.PlanEngine(plan, self.oid, device)
            self._loop = lambda a, b: slabs.step_loop(self.eng, ex, a, b,         # noqa: E731
                                                      backward=self.backward)
            make = lambda w: slabs.PeerPushDriver(plan, self.oid, rank, w)        # noqa: E731
            names = ("nccl send/recv", "fused peer push (CUDA IPC stores from the boundary kernels)")
        if world > 1:
            self.halo = names[0]
        if push:   # world 1: one slab = the whole domain, same single-launch step and tables
            try:
                self.drv = make(world)
                self._loop = lambda a, b: self.drv.run(a, b, backward=self.backward)   # noqa: E731
                if world > 1:
                    self.halo = names[1]
            except RuntimeError as e:
                if rank == 0:
                    log(f"[bench] {e}; falling back to NCCL send/recv")
        if op == "gradient":
            # the history the sweep images against: a forward slab run of the same plans that
            # keeps every images_every-th level in HBM (configs[2])
            F = capi.OP_FORWARD
            plan.upload_traces(capi.CLOUD_SRC, wl.src)
            plan.step_begin(F, images_every)
            self.sync()
            comm.barrier()
            if self.drv is not None:
                self.drv.op = F
                self.drv.run(1, wl.nt - 1)
                self.drv.op = self.oid
            else:
                fwd = slabs.PlanEngine(plan, F, device)
                slabs.step_loop(fwd, ex, 1, wl.nt - 1)
                self.eng = slabs.PlanEngine(plan, self.oid, device)   # streams of the sweep
            plan.step_end(F)
            self.sync()
            comm.barrier()
            self.grad = np.empty(wl.N)
            self.grad.fill(0.0)
        self.e0 = torch.cuda.Event(enable_timing=True)
        self.e1 = torch.cuda.Event(enable_timing=True)

    def steps(self, a, b):
        """bench_core counts steps upwards from 1; a backward sweep starts at the top level"""
        return (self.wl.nt - b, self.wl.nt - a) if self.backward else (a, b)

    def begin(self):
        self.plan.step_begin(self.oid)

    def loop(self, a, b):
        self._loop(*self.steps(a, b))

    def sync(self):
        self.torch.cuda.synchronize()

    def start(self):
        e = self.eng
        e.s_main.wait_stream(e.s_bnd)
        with self.torch.cuda.stream(e.s_main):
            self.e0.record()
        e.s_bnd.wait_stream(e.s_main)

    def stop(self):
        e = self.eng
        e.s_main.wait_stream(e.s_bnd)
        with self.torch.cuda.stream(e.s_main):
            self.e1.record()
        self.torch.cuda.synchronize()
        return self.e0.elapsed_time(self.e1) * 1e-3

    def launches(self):
        return self.plan.launch_count()

    def upload(self):
        if self.drv is not None and self.backward:
            return 0.0      # the receiver table is fed while the sweep runs (run_e2e counts it)
        self.plan.upload_traces(self.c_inj, self.inj)
        return float(self.inj.nbytes)

    def download(self):
        if self.op == "gradient":
            import ctypes as C
            self.plan._chk(self.capi.lib.sfb_get_gradient(self.plan.h, C.byref(self.capi._view(self.grad))))
            return self.points_owned * 8.0
        self.rec = self.plan.download_traces(self.c_smp)
        return float(self.rec.nbytes)

    def run_e2e(self, a, b):
        """the K steps with the trace tables moving while they run (sfb_slab_run): sampled
        rows into the host table, the receiver table of a backward sweep to the device; the
        send/recv fallback steps from Python and moves the tables before / afterwards"""
        if self.drv is None:
            self.loop(a, b)
            return self.download()
        lo, hi = self.steps(a, b)
        self.drv.run_tables(lo, hi, inj=self.inj if self.backward else None, smp=self.rec)
        moved = float((b - a) * self.rec.shape[1] * 8) if self.rec is not None else 0.0
        if self.backward:
            self.fed = float((b - a) * self.inj.shape[1] * 8)
        if self.op == "gradient":
            moved += self.download()
        return moved

    def result(self):
        return self.grad if self.op == "gradient" else self.rec


def multi_gpu(args):
    import torch
    import torch.distributed as dist
    from paper_1808_01995_b200 import capi, slabs
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    # SFB_BENCH_DEVICE / SFB_BENCH_BACKEND=gloo: functional check of this code path with several
    # ranks sharing ONE device (CUDA IPC works between contexts on a device, NCCL does not
    # accept it); a number measured that way means nothing
    local = int(os.environ.get("SFB_BENCH_DEVICE", os.environ.get("LOCAL_RANK", rank)))
    backend = os.environ.get("SFB_BENCH_BACKEND", "nccl")
    torch.cuda.set_device(local)
    # NCCL prints its banner (and, with NCCL_DEBUG=INFO, its communicator lines) on stdout;
    # the contract is ONE JSON line there, so stdout is parked on stderr until the line is ready
    sys.stdout.flush()
    saved_stdout = os.dup(1)
    os.dup2(2, 1)
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29577")
    os.environ.setdefault("NCCL_DEBUG", "INFO")          # communicator lines -> stderr
    os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    if world > 1 or os.environ.get("SFB_BENCH_INIT_PG"):
        if backend == "nccl":
            dist.init_process_group("nccl", rank=rank, world_size=world,
                                    device_id=torch.device(f"cuda:{local}"))
        else:
            dist.init_process_group(backend, rank=rank, world_size=world)
    K, W = args.steps, max(args.warmup, 3)
    config, op = args.config, args.op
    wl = Workload(config, op, W + K, rank, world, args.scaling)
    plan = wl.make_plan(local)
    tile = plan.autotune() if op != "tti" else {}
    sep = bool(plan.get_tile()["sep"])
    comm = slabs.Comm(rank, world, torch.device(f"cuda:{local}") if backend == "nccl" else None)
    resid = None
    if op in ("adjoint", "gradient"):
        resid = wl.residual_traces()           # of the rank's own receivers
        plan.upload_traces(capi.CLOUD_REC, resid)
    else:
        plan.upload_traces(capi.CLOUD_SRC, wl.src)
    job = SlabJob(wl, plan, op, local, rank, world, comm, resid)
    with ClockSampler(local) as clk:
        meas = slabs.bench_core(comm, job, K, W)
    clocks = clk.summary()
    plan.step_end(op_ids(op))
    assert np.isfinite(job.result()).all()
    log(f"[bench] rank {rank}: {meas['per_rank_ms_per_step'][rank]:.4f} ms/step on its slab "
        f"{wl.bounds[rank]}, halo: {job.halo}")
    halo_bytes = int(plan.halo_blocks(capi.OP_FORWARD, 1)["count"] * 4) * (4 if op == "tti" else 1)
    cpu = None
    if rank == 0 and not args.no_cpu:
        cpu = cpu_baseline_leg(config)
    sys.stdout.flush()
    os.dup2(saved_stdout, 1)
    os.close(saved_stdout)
    if rank == 0:
        peak, kind = peaks()
        line = slabs.scaling_line(
            meas, metric=METRIC[op], world=world, K=K, W=W, scaling=args.scaling,
            config=workload_config(config, op, world, args.scaling, {"tile": tile or None}),
            bytes_per_point=actual_bytes(op, sep, 4), contract_bytes=CONTRACT_BYTES[op], peak=peak,
            peak_kind=kind, halo=job.halo, halo_bytes=halo_bytes,
            extra={"cpu_baseline": cpu, "clocks": clocks})
        print(json.dumps(line), flush=True)
    plan.close()
    if dist.is_initialized():
        dist.barrier()
        dist.destroy_process_group()


def ours(args):
    import torch
    from paper_1808_01995_b200 import capi
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if not torch.cuda.is_available() or capi.device_count() < 1:
        raise SystemExit("bench.py needs a CUDA device: there is no CPU fallback")
    if world > 1 or os.environ.get("SFB_BENCH_FORCE_DIST"):
        return multi_gpu(args)
    return single_gpu(args)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2, choices=sorted(CONFIGS),
                    help="BASELINE.json configuration, 1-based (default 2 = configs[1])")
    ap.add_argument("--op", default=None, choices=["forward", "adjoint", "gradient", "tti"],
                    help="operator (default: the configuration's own)")
    ap.add_argument("--scaling", default=None, choices=["strong", "weak"])
    ap.add_argument("--no-other-ops", action="store_true",
                    help="skip the adjoint / gradient / TTI extras of the default line")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    args = ap.parse_args()
    args.op = args.op or CONFIGS[args.config]["op"]
    args.scaling = args.scaling or CONFIGS[args.config]["scaling"]
    if args.scaling == "weak" and args.config != 5:
        raise SystemExit("weak scaling is defined for --config 5 only")
    if (args.op == "tti") != (args.config == 4):
        raise SystemExit("the TTI operator is --config 4, and --config 4 is the TTI operator")
    if args.impl == "reference":
        return reference_arm(args)
    return ours(args)


if __name__ == "__main__":
    main()
