"""Seeded synthetic inputs of BASELINE.json's configurations.

The reference uses no public dataset and BASELINE.json names none: every benchmark and
full-size test runs on the generators below (numpy default_rng(seed) + a separable
Gaussian blur), which stand in for no external data.  Host-side input generation only --
nothing here is on the propagator path.
"""
from __future__ import annotations

import numpy as np

SEED = 18080199  # base seed; +i per field


def smooth_field(shape, seed, sigma, lo, hi, dtype=np.float32):
    """Gaussian blur (sigma in cells, periodic so the statistics are uniform) of N(0,1)
    noise, mapped linearly to [lo, hi]."""
    from scipy.ndimage import gaussian_filter1d
    g = np.random.default_rng(seed).standard_normal(shape, dtype=dtype)
    for ax in range(len(shape)):
        g = gaussian_filter1d(g, float(sigma), axis=ax, mode="wrap", truncate=3.0)
    gmin, gmax = float(g.min()), float(g.max())
    return (lo + (hi - lo) * (g.astype(np.float64) - gmin) / (gmax - gmin))


def two_layer(shape, split, v_top=1.5, v_bottom=2.5):
    """Two layers split on the depth (last, contiguous) axis (proj/src/verify.cpp:210-213)."""
    v = np.empty(shape, dtype=np.float64)
    v[..., :split] = v_top
    v[..., split:] = v_bottom
    return v


def receiver_grid(n0, n1, h, depth):
    """n0 x n1 receivers on the lattice at fixed depth: (h*i, h*j, depth)."""
    ii, jj = np.meshgrid(np.arange(n0) * h, np.arange(n1) * h, indexing="ij")
    return np.stack([ii.ravel(), jj.ravel(), np.full(ii.size, float(depth))], axis=1)


def config(number: int, n: int | None = None, nsteps: int | None = None):
    """Parameters of BASELINE.json config `number` (1-based), optionally shrunk to n^3
    physical nodes / nsteps time steps for parity tests.  Returns a dict; velocity is
    generated lazily by the caller via the 'velocity' callable."""
    if number == 1:
        n = n or 101
        return dict(name="cfg1_acoustic_so4_101", shape=[n, n, n], h=10.0, nbl=40, order=4,
                    f0=0.010, velocity=lambda: two_layer([n, n, n], n // 2 if n != 101 else 50),
                    src=[[(n - 1) * 5.0, (n - 1) * 5.0, 20.0]],
                    rec=np.array([[10.0 * i, (n - 1) * 5.0, 20.0] for i in range(n)]),
                    tn=1000.0, nsteps=nsteps)
    if number in (2, 3):
        n = n or 512
        h = 12.5
        c = h * (n - 1) / 2.0 + h / 4.0  # off-node, centre of the grid (3193.75 at n=512)
        vel = (lambda: smooth_field([n, n, n], SEED, 8.0, 1.5, 4.5)) if number == 2 else \
              (lambda: two_layer([n, n, n], n // 2))
        return dict(name=f"cfg{number}_acoustic_so8_{n}", shape=[n, n, n], h=h, nbl=40, order=8,
                    f0=0.015, velocity=vel, src=[[c, c, 18.75]],
                    rec=receiver_grid(n, n, h, 25.0), tn=None, nsteps=nsteps or 500)
    if number == 5:
        n = n or 1024
        h = 12.5
        rng = np.random.default_rng(SEED + 7)
        src = rng.uniform(0.0, h * (n - 1), size=(8, 3))
        return dict(name=f"cfg5_acoustic_so16_{n}", shape=[n, n, n], h=h, nbl=40, order=16,
                    f0=0.015, velocity=lambda: smooth_field([n, n, n], SEED + 6, 8.0, 1.5, 4.5),
                    src=src, rec=receiver_grid(n, n, h, 25.0), tn=None, nsteps=nsteps or 1000)
    if number == 4:
        n = n or 512
        h = 12.5
        c = h * (n - 1) / 2.0 + h / 4.0
        return dict(name=f"cfg4_tti_so12_{n}", shape=[n, n, n], h=h, nbl=40, order=12, f0=0.015,
                    velocity=lambda: smooth_field([n, n, n], SEED + 1, 8.0, 1.5, 4.5),
                    tti=lambda: tti_fields([n, n, n]), src=[[c, c, 18.75]],
                    rec=receiver_grid(n, n, h, 25.0), tn=None, nsteps=nsteps or 500)
    raise ValueError(f"no config {number}")


def tti_fields(shape, sigma=8.0):
    """Config 4's Thomsen parameters and angles: independent smooth
    fields, epsilon in [0, 0.3], delta in [0, 0.2] clipped to delta <= epsilon (the
    pseudo-acoustic system is ill-posed otherwise), tilt and azimuth
    in [0, pi/4].  Physical extent; the caller extends them over the absorbing layer."""
    eps = smooth_field(shape, SEED + 2, sigma, 0.0, 0.3)
    delta = np.minimum(smooth_field(shape, SEED + 3, sigma, 0.0, 0.2), eps)
    theta = smooth_field(shape, SEED + 4, sigma, 0.0, np.pi / 4)
    phi = smooth_field(shape, SEED + 5, sigma, 0.0, np.pi / 4)
    return eps, delta, theta, phi


def extend(field, nbl):
    """Edge-clamped extension over the absorbing layer (the rule of proj/src/model.cpp:92-100)."""
    return np.pad(field, nbl, mode="edge")


def time_axis(critical_dt, nsteps=None, tn=None):
    """dt = the CFL critical dt; tn chosen so that floor(tn/dt)+1 = nsteps+2 robustly
    (SURVEY.md section 8d), unless the config fixes tn."""
    dt = critical_dt
    if tn is None or nsteps is not None:
        tn = (nsteps + 1.5) * dt
    return dt, tn


# ---- slab-local generators (multi-GPU weak scaling: no rank ever holds a global field) ------

def damping_profiles(N, nbl, spacing, v_max):
    """The three 1-D profiles whose sum is build_damping's field (proj/src/model.cpp:35-56,
    quadratic ramp): eta_d w^2 with w = (nbl - dist)/nbl for dist = min(i, N-1-i) < nbl,
    eta_d = v_max ln(1000) / (nbl h_d).  Checked against the host SeismicModel in
    tests/test_host_cpu.py."""
    out = []
    for n, h in zip(N, spacing):
        i = np.arange(n)
        dist = np.minimum(i, n - 1 - i)
        w = np.where(dist < nbl, (nbl - dist) / float(nbl), 0.0)
        out.append((v_max * np.log(1000.0) / (nbl * h)) * w * w)
    return out


def smooth_slab(shape, lo, hi, seed, sigma, vlo, vhi, spread=4.2):
    """Planes [lo, hi) of axis 0 of a seeded smoothed-noise field over `shape`, computable by
    a rank that owns only those planes: white noise is drawn per global plane (seed + plane),
    blurred in-plane (periodic) and along axis 0 over a 3-sigma window of neighbouring planes
    (periodic), normalised by its analytic standard deviation and mapped linearly, clipped at
    `spread` standard deviations, to [vlo, vhi].  Any two ranks produce identical values for a
    plane they both generate.  Same value range and correlation length as smooth_field."""
    from scipy.ndimage import gaussian_filter1d
    n0, n1, n2 = shape
    R = int(3.0 * sigma + 0.5)
    k = np.exp(-0.5 * (np.arange(-R, R + 1) / float(sigma)) ** 2)
    k /= k.sum()
    planes = {}
    for z in range(lo - R, hi + R):
        zz = z % n0
        if zz in planes:
            continue
        g = np.random.default_rng([seed, zz]).standard_normal((n1, n2), dtype=np.float32)
        for ax in (0, 1):
            g = gaussian_filter1d(g, float(sigma), axis=ax, mode="wrap", truncate=3.0)
        planes[zz] = g
    out = np.empty((hi - lo, n1, n2), dtype=np.float64)
    for z in range(lo, hi):
        acc = np.zeros((n1, n2), dtype=np.float64)
        for j in range(-R, R + 1):
            acc += k[j + R] * planes[(z + j) % n0]
        out[z - lo] = acc
    std = float(np.sqrt((k ** 2).sum()) ** 3)   # unit white noise through three 1-D kernels
    mid, half = 0.5 * (vlo + vhi), 0.5 * (vhi - vlo)
    return mid + half * np.clip(out / (spread * std), -1.0, 1.0)


def slab_model(phys_shape, nbl, spacing, z_lo, z_hi, velocity_planes, v_max):
    """m = 1/v^2 and damp on padded planes [z_lo, z_hi) of axis 0 (edge-clamped extension,
    proj/src/model.cpp:92-100; damping as a sum of the three profiles).  velocity_planes(lo,
    hi) returns physical planes [lo, hi) of the velocity."""
    N = [s + 2 * nbl for s in phys_shape]
    p_lo = min(max(z_lo - nbl, 0), phys_shape[0] - 1)
    p_hi = min(max(z_hi - 1 - nbl, 0), phys_shape[0] - 1) + 1
    v = velocity_planes(p_lo, p_hi)
    idx = np.clip(np.arange(z_lo, z_hi) - nbl, 0, phys_shape[0] - 1) - p_lo
    v = np.pad(v, ((0, 0), (nbl, nbl), (nbl, nbl)), mode="edge")[idx]
    m = 1.0 / (v * v)
    dz, dy, dx = damping_profiles(N, nbl, spacing, v_max)
    damp = dz[z_lo:z_hi, None, None] + dy[None, :, None] + dx[None, None, :]
    return m, np.ascontiguousarray(damp)
