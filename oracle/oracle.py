"""ctypes/numpy front end of the CPU oracle (oracle/sf_oracle.c).

TEST INFRASTRUCTURE ONLY -- see the header of sf_oracle.c.  Imported by tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs, never by
the product package.

The exact-rational finite-difference weights follow the reference's
src/fdcoeff.cpp:60-95 (moment system solved exactly; here with fractions.Fraction
instead of Boost cpp_rational) and are pinned against tests/test_symbolic.cpp:52-97.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from fractions import Fraction
from math import factorial

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_lib = None


def _cpu_key() -> str:
    """-march=native objects must not travel between hosts: key the build by CPU flags."""
    import hashlib
    try:
        with open("/proc/cpuinfo") as f:
            flags = next((ln for ln in f if ln.startswith("flags")), "")
    except OSError:
        flags = ""
    return hashlib.md5(flags.encode()).hexdigest()[:10]


_LIB_PATH = os.path.join(_HERE, "_build", f"libsf_oracle_{_cpu_key()}.so")


def build(force: bool = False) -> str:
    """Compile sf_oracle.c -> oracle/_build/libsf_oracle.so (gcc -O3 -fopenmp)."""
    src = os.path.join(_HERE, "sf_oracle.c")
    if (not force and os.path.exists(_LIB_PATH)
            and os.path.getmtime(_LIB_PATH) >= os.path.getmtime(src)):
        return _LIB_PATH
    os.makedirs(os.path.dirname(_LIB_PATH), exist_ok=True)
    cmd = ["gcc", "-O3", "-march=native", "-fopenmp", "-fPIC", "-shared", "-std=c11",
           "-o", _LIB_PATH, src, "-lm"]
    subprocess.check_call(cmd)
    return _LIB_PATH


class _Grid(C.Structure):
    _fields_ = [("ndim", C.c_int), ("n", C.c_long * 3), ("h", C.c_double * 3),
                ("space_order", C.c_int), ("dt", C.c_double), ("nt", C.c_long),
                ("w2", C.POINTER(C.c_double))]


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = C.CDLL(_LIB_PATH)
        _lib.sfo_critical_dt.restype = C.c_double
        _lib.sfo_objective.restype = C.c_double
        _lib.sfo_locate.restype = C.c_long
        _lib.sfo_num_samples.restype = C.c_long
        _lib.sfo_num_samples.argtypes = [C.c_double, C.c_double, C.c_double]
    return _lib


def _p(a, t=C.c_double):
    return a.ctypes.data_as(C.POINTER(t)) if a is not None else None


# ---- FD weights: src/fdcoeff.cpp:12-18, 60-95 ---------------------------------------

def centered_offsets(order: int):
    if order <= 0 or order % 2:
        raise ValueError("centered stencils require a positive even accuracy order")
    return list(range(-order // 2, order // 2 + 1))


def fd_weights_exact(deriv_order: int, offsets):
    """Exact weights solving sum_j w_j o_j^p = p! [p == deriv_order], p = 0..n-1."""
    n = len(offsets)
    if deriv_order < 1 or n < deriv_order + 1 or len(set(offsets)) != n:
        raise ValueError("bad stencil request")
    a = [[Fraction(o) ** p for o in offsets] for p in range(n)]
    b = [Fraction(0)] * n
    b[deriv_order] = Fraction(factorial(deriv_order))
    for col in range(n):
        piv = next(r for r in range(col, n) if a[r][col] != 0)
        a[col], a[piv] = a[piv], a[col]
        b[col], b[piv] = b[piv], b[col]
        for r in range(col + 1, n):
            if a[r][col] == 0:
                continue
            f = a[r][col] / a[col][col]
            for c in range(col, n):
                a[r][c] -= f * a[col][c]
            b[r] -= f * b[col]
    x = [Fraction(0)] * n
    for ri in range(n - 1, -1, -1):
        s = b[ri] - sum(a[ri][c] * x[c] for c in range(ri + 1, n))
        x[ri] = s / a[ri][ri]
    return x


def second_derivative_weights(order: int) -> np.ndarray:
    """w_0..w_K (centre first) as correctly rounded doubles."""
    ws = fd_weights_exact(2, centered_offsets(order))
    K = order // 2
    return np.array([float(ws[K + j]) for j in range(K + 1)], dtype=np.float64)


def first_derivative_weights(order: int) -> np.ndarray:
    """w_1..w_K of the centred first derivative (antisymmetric, w_0 = 0)."""
    ws = fd_weights_exact(1, centered_offsets(order))
    K = order // 2
    return np.array([float(ws[K + j]) for j in range(1, K + 1)], dtype=np.float64)


# ---- model / geometry helpers -------------------------------------------------------

class Model:
    """Restates SeismicModel (src/model.cpp:58-111): padded grid, m, damp, CFL."""

    def __init__(self, shape, spacing, origin, velocity, nbl, space_order=8, linear=False):
        self.ndim = len(shape)
        self.shape = [int(s) for s in shape]
        self.spacing = [float(s) for s in spacing]
        self.nbl = int(nbl)
        self.space_order = int(space_order)
        self.linear = bool(linear)
        self.origin = [float(o) - self.nbl * float(h) for o, h in zip(origin, spacing)]
        self.N = [s + 2 * self.nbl for s in self.shape]
        self.set_velocity(velocity)
        self.damp = np.empty(self.N, dtype=np.float64)
        rc = lib().sfo_build_damping(C.c_int(self.ndim), (C.c_long * 3)(*self.N),
                                     (C.c_double * 3)(*self.spacing), C.c_long(self.nbl),
                                     C.c_double(self.v_max), C.c_int(int(self.linear)),
                                     _p(self.damp))
        if rc:
            raise ValueError("build_damping: nbl must be < min(shape)/2")

    def set_velocity(self, velocity):
        vel = np.ascontiguousarray(velocity, dtype=np.float64).reshape(self.shape)
        self.m = np.empty(self.N, dtype=np.float64)
        vmin, vmax = C.c_double(), C.c_double()
        rc = lib().sfo_pad_slowness(C.c_int(self.ndim), (C.c_long * 3)(*self.shape),
                                    C.c_long(self.nbl), _p(vel), _p(self.m),
                                    C.byref(vmin), C.byref(vmax))
        if rc:
            raise ValueError("velocity must be positive")
        self.v_min, self.v_max = vmin.value, vmax.value

    def physical_m(self):
        sl = tuple(slice(self.nbl, self.nbl + s) for s in self.shape)
        return np.ascontiguousarray(self.m[sl])

    def set_physical_m(self, m_phys):
        mp = np.ascontiguousarray(m_phys, dtype=np.float64).reshape(self.shape)
        if not (mp > 0).all():
            raise ValueError("m must be positive")
        v = 1.0 / np.sqrt(mp)
        self.v_min, self.v_max = float(v.min()), float(v.max())
        self.m = np.empty(self.N, dtype=np.float64)
        lib().sfo_pad_m(C.c_int(self.ndim), (C.c_long * 3)(*self.shape), C.c_long(self.nbl),
                        _p(mp), _p(self.m))

    def critical_dt(self, space_order=None, gamma=1.0):
        k = self.space_order if space_order is None else int(space_order)
        w2 = second_derivative_weights(k)
        return lib().sfo_critical_dt(C.c_int(self.ndim), (C.c_double * 3)(*self.spacing),
                                     C.c_double(self.v_max), C.c_int(k), _p(w2),
                                     C.c_double(gamma))


def locate(model: Model, coords):
    """src/sparse.cpp:36-70.  Returns (base int64 [np][ndim], w f64 [np][2^ndim])."""
    coords = np.ascontiguousarray(coords, dtype=np.float64).reshape(-1, model.ndim)
    npnt = coords.shape[0]
    base = np.zeros((npnt, model.ndim), dtype=np.int64)
    w = np.zeros((npnt, 1 << model.ndim), dtype=np.float64)
    rc = lib().sfo_locate(C.c_int(model.ndim), (C.c_long * 3)(*model.N),
                          (C.c_double * 3)(*model.spacing), (C.c_double * 3)(*model.origin),
                          C.c_long(npnt), _p(coords), _p(base, C.c_long), _p(w))
    if rc:
        raise ValueError(f"point {rc - 1} outside domain")  # LocationError
    return base, w


def ricker(f0, t0, dt, nt):
    out = np.empty(nt, dtype=np.float64)
    lib().sfo_ricker(C.c_double(f0), C.c_double(t0), C.c_double(dt), C.c_long(nt), _p(out))
    return out


def num_samples(t0, tn, dt):
    return int(lib().sfo_num_samples(t0, tn, dt))


class Geometry:
    """Restates AcquisitionGeometry (src/geometry.cpp:10-34)."""

    def __init__(self, model: Model, src_coords, rec_coords, t0, tn, dt, f0):
        if not (dt > 0.0) or not (tn > t0):
            raise ValueError("bad time axis")
        if dt > model.critical_dt() * (1.0 + 1e-12):
            raise ArithmeticError("dt exceeds the stable limit")  # StabilityError
        self.t0, self.tn, self.dt, self.f0 = float(t0), float(tn), float(dt), float(f0)
        self.nt = num_samples(t0, tn, dt)
        self.src_base, self.src_w = locate(model, src_coords)
        self.rec_base, self.rec_w = locate(model, rec_coords)
        self.n_src, self.n_rec = self.src_base.shape[0], self.rec_base.shape[0]
        self.src_coords = np.asarray(src_coords, dtype=np.float64).reshape(-1, model.ndim)
        self.rec_coords = np.asarray(rec_coords, dtype=np.float64).reshape(-1, model.ndim)
        wv = ricker(f0, t0, dt, self.nt)
        self.src = np.repeat(wv[:, None], self.n_src, axis=1).copy()
        self.rec = np.zeros((self.nt, self.n_rec), dtype=np.float64)


def _grid(model: Model, space_order, dt, nt, w2):
    g = _Grid()
    g.ndim = model.ndim
    for a in range(3):
        g.n[a] = model.N[a] if a < model.ndim else 1
        g.h[a] = model.spacing[a] if a < model.ndim else 1.0
    g.space_order = int(space_order)
    g.dt = float(dt)
    g.nt = int(nt)
    g.w2 = _p(w2)
    return g


def check_cfl(model: Model, dt, space_order):
    """src/seismic_ops.cpp:15-22"""
    if dt > model.critical_dt(space_order) * (1.0 + 1e-12):
        raise ArithmeticError("dt exceeds the stable limit")


def propagate(model: Model, space_order, dt, nt, direction, inj_base, inj_w, inj_tr,
              smp_base, smp_w, want_final=False, save_every=0):
    """Forward (direction=+1) or adjoint (-1) sweep; returns dict with 'smp' traces and
    optionally 'final' (last level written), 'prev', 'snaps'."""
    check_cfl(model, dt, space_order)
    w2 = second_derivative_weights(space_order)
    g = _grid(model, space_order, dt, nt, w2)
    inj_tr = np.ascontiguousarray(inj_tr, dtype=np.float64)
    smp = np.zeros((nt, smp_base.shape[0]), dtype=np.float64)
    fa = np.empty(model.N) if want_final else None
    fb = np.empty(model.N) if want_final else None
    snaps = None
    if save_every and direction > 0:
        snaps = np.empty([(nt - 1) // save_every + 1] + list(model.N), dtype=np.float64)
    rc = lib().sfo_propagate(C.byref(g), C.c_int(direction), _p(model.m), _p(model.damp),
                             C.c_long(inj_base.shape[0]), _p(inj_base, C.c_long), _p(inj_w),
                             _p(inj_tr), C.c_long(smp_base.shape[0]), _p(smp_base, C.c_long),
                             _p(smp_w), _p(smp), _p(fa), _p(fb), _p(snaps),
                             C.c_long(max(save_every, 1)))
    if rc == 2:
        raise ArithmeticError("field went non-finite")  # StabilityError
    if rc:
        raise MemoryError("oracle allocation failed")
    out = {"smp": smp}
    if want_final:
        out["final"], out["prev"] = fa, fb
    if snaps is not None:
        out["snaps"] = snaps
    return out


def forward(model, geom, space_order, want_final=False, save_every=0, src=None, nt=None):
    """forward_operator + run_wave (src/seismic_ops.cpp:58-82,137-141).  Writes geom.rec."""
    nt = geom.nt if nt is None else nt
    src = geom.src if src is None else src
    r = propagate(model, space_order, geom.dt, nt, +1, geom.src_base, geom.src_w, src[:nt],
                  geom.rec_base, geom.rec_w, want_final, save_every)
    if nt == geom.nt:
        geom.rec = r["smp"]
    return r


def adjoint(model, geom, space_order, rec=None, want_final=False):
    """adjoint_operator + run_wave (src/seismic_ops.cpp:84-107).  Returns srca traces."""
    rec = geom.rec if rec is None else rec
    return propagate(model, space_order, geom.dt, geom.nt, -1, geom.rec_base, geom.rec_w, rec,
                     geom.src_base, geom.src_w, want_final)


def gradient_sweep(model, geom, space_order, resid, snaps, save_every=1):
    check_cfl(model, geom.dt, space_order)
    w2 = second_derivative_weights(space_order)
    g = _grid(model, space_order, geom.dt, geom.nt, w2)
    resid = np.ascontiguousarray(resid, dtype=np.float64)
    snaps = np.ascontiguousarray(snaps, dtype=np.float64)
    grad = np.empty(model.N, dtype=np.float64)
    rc = lib().sfo_gradient(C.byref(g), _p(model.m), _p(model.damp), C.c_long(geom.n_rec),
                            _p(geom.rec_base, C.c_long), _p(geom.rec_w), _p(resid), _p(snaps),
                            C.c_long(save_every), _p(grad))
    if rc == 2:
        raise ArithmeticError("field went non-finite")
    if rc:
        raise MemoryError("oracle allocation failed")
    return grad


def objective(pred, observed):
    pred = np.ascontiguousarray(pred, dtype=np.float64)
    observed = np.ascontiguousarray(observed, dtype=np.float64)
    if pred.size != observed.size:
        raise ValueError("objective: observed trace shape mismatch")
    return lib().sfo_objective(C.c_long(pred.size), _p(pred), _p(observed))


def fold_gradient(model: Model, grad_padded):
    out = np.empty(model.shape, dtype=np.float64)
    gp = np.ascontiguousarray(grad_padded, dtype=np.float64)
    lib().sfo_fold_gradient(C.c_int(model.ndim), (C.c_long * 3)(*model.shape),
                            C.c_long(model.nbl), _p(gp), _p(out))
    return out


def fwi_gradient(model, geom, observed, space_order, save_every=1):
    """src/seismic_ops.cpp:197-216.  Returns (objective, gradient[physical], residual)."""
    r = forward(model, geom, space_order, save_every=save_every)
    observed = np.asarray(observed, dtype=np.float64).reshape(geom.nt, geom.n_rec)
    phi = objective(geom.rec, observed)
    resid = geom.rec - observed
    g = gradient_sweep(model, geom, space_order, resid, r["snaps"], save_every)
    return phi, fold_gradient(model, g), resid


def dense_steps(model, space_order, dt, steps, cur, old):
    """Bare dense stepping (CPU throughput baseline).  cur/old updated in place."""
    w2 = second_derivative_weights(space_order)
    g = _grid(model, space_order, dt, steps + 2, w2)
    rc = lib().sfo_dense_steps(C.byref(g), _p(model.m), _p(model.damp), C.c_long(steps),
                               _p(cur), _p(old))
    if rc:
        raise MemoryError("oracle allocation failed")


class _Tti(C.Structure):
    _fields_ = [("eps", C.POINTER(C.c_double)), ("delta", C.POINTER(C.c_double)),
                ("theta", C.POINTER(C.c_double)), ("phi", C.POINTER(C.c_double)),
                ("w1", C.POINTER(C.c_double))]


def tti_critical_dt(model: Model, space_order, eps_max):
    """The builder's TTI time-step bound: the acoustic CFL rule
    (src/model.cpp:103-111) evaluated with v_max*sqrt(1 + 2 eps_max), times 0.9 because the
    rotated operator applies first-derivative stencils twice."""
    return 0.9 * model.critical_dt(space_order) / np.sqrt(1.0 + 2.0 * eps_max)


def tti_forward(model: Model, geom, space_order, eps, delta, theta, phi, src=None,
                want_final=False, want_energy=False):
    """Builder-defined TTI forward operator (no reference counterpart: parity unpinned)."""
    w2 = second_derivative_weights(space_order)
    w1 = first_derivative_weights(space_order)
    g = _grid(model, space_order, geom.dt, geom.nt, w2)
    fields = [np.ascontiguousarray(np.broadcast_to(np.asarray(f, dtype=np.float64), model.N))
              for f in (eps, delta, theta, phi)]
    t = _Tti(*[_p(f) for f in fields], _p(w1))
    src = np.ascontiguousarray(geom.src if src is None else src, dtype=np.float64)
    rec = np.zeros((geom.nt, geom.n_rec))
    fp = np.empty(model.N) if want_final else None
    fr = np.empty(model.N) if want_final else None
    en = np.zeros(geom.nt) if want_energy else None
    rc = lib().sfo_tti_forward(C.byref(g), C.byref(t), _p(model.m), _p(model.damp),
                               C.c_long(geom.n_src), _p(geom.src_base, C.c_long), _p(geom.src_w),
                               _p(src), C.c_long(geom.n_rec), _p(geom.rec_base, C.c_long),
                               _p(geom.rec_w), _p(rec), _p(fp), _p(fr), _p(en))
    if rc == 2:
        raise ArithmeticError("field went non-finite")
    if rc:
        raise MemoryError("oracle allocation failed")
    out = {"smp": rec}
    if want_final:
        out["p"], out["r"] = fp, fr
    if want_energy:
        out["energy"] = en
    return out


def num_threads():
    return int(lib().sfo_num_threads())


def set_num_threads(n):
    lib().sfo_set_num_threads(C.c_int(int(n)))
