"""Parity of the CUDA path against the f64 oracle at BASELINE.json's headline sizes
(SURVEY.md section 8(d) "parity gates").

  config2   configs[1] exactly: seeded sigma-8 medium, 592^3 computed nodes, order 8,
            500 steps, one off-node 15 Hz source, 512 x 512 receivers.  Traces and the
            wavefield after 100 steps (gate 1e-5) and after the full run (gate 1e-4).
  config3   configs[2]: two-layer medium at 592^3, order 8, forward keeping every 4th level
            in HBM, gradient sweep driven by seeded random band-limited residuals at all
            262 144 receivers, over a window of `--grad-steps` steps (default 64) against
            the oracle's gradient sweep with the same save_every rule (gate 1e-3).
  config5   configs[4] on a reduced grid (208 x 256 x 256 computed nodes, order 16, 8 random
            off-node sources, 176 x 176 receivers, 1000 steps): gates as config2.

The oracle is test infrastructure (oracle/sf_oracle.c); everything on the GPU side goes
through the C-ABI (ctypes on include/sfb200.h).  Writes one JSON record per case; the
pytest wrapper is tests/test_gpu_parity_fullsize.py.

    python tools/parity_fullsize.py [config2] [config3] [config5] [--steps N] [--out FILE]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

H = 12.5
NBL = 40


def rel_l2(a, b):
    num = den = 0.0
    # chunked: the operands are GB-sized, avoid f64 temporaries of the whole array
    a2 = a.reshape(a.shape[0], -1)
    b2 = b.reshape(b.shape[0], -1)
    for i in range(a2.shape[0]):
        d = a2[i].astype(np.float64) - b2[i]
        num += float(d @ d)
        den += float(b2[i].astype(np.float64) @ b2[i].astype(np.float64))
    return float(np.sqrt(num) / (np.sqrt(den) if den > 0 else 1.0))


def gpu_plan(om, og, order):
    from paper_1808_01995_b200 import capi
    plan = capi.Plan(om.N, om.spacing, order, og.dt, og.nt)
    plan.set_model(om.m, om.damp, om.v_max)
    plan.set_points(capi.CLOUD_SRC, og.src_base, og.src_w)
    plan.set_points(capi.CLOUD_REC, og.rec_base, og.rec_w)
    return plan


def forward_case(name, shape, order, vel, src, rec, nsteps, early=100):
    """Forward run: GPU vs oracle at level `early` (traces rows <= early, wavefield level
    `early`) and at the end.  One oracle run serves both gates (levels t % early == 0 kept)."""
    from oracle import oracle as o
    om = o.Model(shape, [H] * 3, [0.0] * 3, vel, NBL, order)
    dt = om.critical_dt(order)
    og = o.Geometry(om, np.asarray(src, dtype=float).ravel(), np.asarray(rec, dtype=float).ravel(),
                    0.0, (nsteps + 1.5) * dt, dt, 0.015)
    assert og.nt == nsteps + 2
    early = min(early, nsteps)
    plan = gpu_plan(om, og, order)
    t0 = time.time()
    grec, rep = plan.forward(og.src, save_every=early)
    g_early = plan.wavefield(early)
    g_final = plan.wavefield(og.nt - 1)
    tile = plan.get_tile()
    plan.close()
    t_gpu = time.time() - t0
    t0 = time.time()
    ref = o.forward(om, og, order, want_final=True, save_every=early)
    t_cpu = time.time() - t0
    out = {
        "case": name, "computed_nodes": list(om.N), "space_order": order, "steps": nsteps,
        "dt_ms": dt, "n_src": og.n_src, "n_rec": og.n_rec, "tile": tile,
        "gpu_gpts_per_s": rep.gpts_per_s, "oracle_seconds": t_cpu, "oracle_threads": o.num_threads(),
        "oracle_gpts_per_s": float(np.prod(om.N)) * nsteps / t_cpu / 1e9, "gpu_call_seconds": t_gpu,
        "early_level": early,
        "traces_rel_l2_early": rel_l2(grec[: early + 1], ref["smp"][: early + 1]),
        "wavefield_rel_l2_early": rel_l2(g_early, ref["snaps"][1]),
        "traces_rel_l2_full": rel_l2(grec, ref["smp"]),
        "wavefield_rel_l2_full": rel_l2(g_final, ref["final"]),
        "traces_absmax": float(np.abs(ref["smp"]).max()),
        "wavefield_absmax": float(np.abs(ref["final"]).max()),
        "gates": {"early": 1e-5, "full": 1e-4},
    }
    out["pass"] = bool(out["traces_absmax"] > 0 and out["wavefield_absmax"] > 0
                       and out["traces_rel_l2_early"] <= 1e-5 and out["wavefield_rel_l2_early"] <= 1e-5
                       and out["traces_rel_l2_full"] <= 1e-4 and out["wavefield_rel_l2_full"] <= 1e-4)
    return out


def config2(nsteps=500, n=512):
    from paper_1808_01995_b200 import synthetic as syn
    cfg = syn.config(2, n, nsteps)
    return forward_case("config2", cfg["shape"], 8, cfg["velocity"](), cfg["src"], cfg["rec"], nsteps)


def config5_reduced(nsteps=1000):
    """configs[4] shrunk to 208 x 256 x 256 computed nodes (128 x 176 x 176 physical): same
    order, layer, medium recipe, 8 random off-node sources, receiver lattice at 25 m."""
    from paper_1808_01995_b200 import synthetic as syn
    shape = [128, 176, 176]
    vel = syn.smooth_field(shape, syn.SEED + 6, 8.0, 1.5, 4.5)
    rng = np.random.default_rng(syn.SEED + 7)
    src = rng.uniform([0, 0, 0], [H * (s - 1) for s in shape], size=(8, 3))
    rec = syn.receiver_grid(shape[0], shape[1], H, 25.0)
    return forward_case("config5_reduced", shape, 16, vel, src, rec, nsteps)


def residual_traces(nt, n_rec, dt, seed):
    """per-receiver N(0,1) noise convolved in time with the 15 Hz
    Ricker, rows 0 and nt-1 zeroed."""
    from oracle import oracle as o
    spec = np.fft.rfft(o.ricker(0.015, 0.0, dt, nt))[:, None]
    rng = np.random.default_rng(seed)
    out = np.empty((nt, n_rec))
    for lo in range(0, n_rec, 32768):
        xi = rng.standard_normal((nt, min(32768, n_rec - lo)))
        out[:, lo:lo + xi.shape[1]] = np.fft.irfft(np.fft.rfft(xi, axis=0) * spec, n=nt, axis=0)
    out[[0, nt - 1]] = 0.0
    return out


def config3(nsteps=64, n=512, save_every=4):
    from oracle import oracle as o
    from paper_1808_01995_b200 import synthetic as syn
    cfg = syn.config(3, n, nsteps)
    om = o.Model(cfg["shape"], [H] * 3, [0.0] * 3, cfg["velocity"](), NBL, 8)
    dt = om.critical_dt(8)
    og = o.Geometry(om, np.asarray(cfg["src"]).ravel(), cfg["rec"].ravel(), 0.0,
                    (nsteps + 1.5) * dt, dt, 0.015)
    resid = residual_traces(og.nt, og.n_rec, dt, syn.SEED + 10)
    plan = gpu_plan(om, og, 8)
    grec, rf = plan.forward(og.src, save_every=save_every)
    gg, rg = plan.gradient(resid)
    # dot test on the same window: <F x, y> vs <x, F^T y>
    xt, _ = plan.adjoint(resid)
    lhs, rhs = float((grec * resid).sum()), float((og.src * xt).sum())
    plan.close()
    t0 = time.time()
    ref = o.forward(om, og, 8, save_every=save_every)
    og_ = o.gradient_sweep(om, og, 8, resid, ref["snaps"], save_every)
    t_cpu = time.time() - t0
    out = {
        "case": "config3", "computed_nodes": list(om.N), "space_order": 8, "steps": nsteps,
        "save_every": save_every, "n_rec": og.n_rec, "oracle_seconds": t_cpu,
        "forward_with_save_gpts": rf.gpts_per_s, "gradient_sweep_gpts": rg.gpts_per_s,
        "traces_rel_l2": rel_l2(grec, ref["smp"]),
        "gradient_rel_l2": rel_l2(gg, og_),
        "gradient_absmax": float(np.abs(og_).max()),
        "dot_test_rel": abs(lhs - rhs) / max(abs(lhs), abs(rhs)),
        "gates": {"gradient": 1e-3, "dot_test": 1e-4},
    }
    out["pass"] = bool(out["gradient_absmax"] > 0 and out["gradient_rel_l2"] <= 1e-3
                       and out["dot_test_rel"] <= 1e-4 and out["traces_rel_l2"] <= 1e-5)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cases", nargs="*", default=["config2", "config3", "config5"])
    ap.add_argument("--steps", type=int, default=0, help="override the step count of config2/config5")
    ap.add_argument("--grad-steps", type=int, default=64)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    results = []
    for c in a.cases:
        t0 = time.time()
        if c == "config2":
            r = config2(a.steps or 500)
        elif c == "config3":
            r = config3(a.grad_steps)
        elif c == "config5":
            r = config5_reduced(a.steps or 1000)
        else:
            raise SystemExit(f"unknown case {c}")
        r["case_seconds"] = time.time() - t0
        print(json.dumps(r), flush=True)
        results.append(r)
    if a.out:
        with open(a.out, "w") as f:
            json.dump(results, f, indent=1)
    return 0 if all(r["pass"] for r in results) else 1


if __name__ == "__main__":
    sys.exit(main())
