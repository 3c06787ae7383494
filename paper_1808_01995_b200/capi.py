"""ctypes binding of include/sfb200.h (libsfb200.so).  Thin: no arithmetic happens here."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libsfb200.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
        "g.build()'` (nvcc, sm_100a).  There is no CPU fallback.")

lib = C.CDLL(LIB_PATH)

OK, ERR_PARAMETER, ERR_STABILITY, ERR_LOCATION, ERR_CAPABILITY, ERR_BINDING, ERR_CUDA, ERR_ORDER = range(8)
CLOUD_SRC, CLOUD_REC = 0, 1
OP_FORWARD, OP_ADJOINT, OP_GRADIENT, OP_TTI_FORWARD = 0, 1, 2, 3
TTI_HALO_G_P, TTI_HALO_G_R, TTI_HALO_P, TTI_HALO_R = 0, 1, 2, 3
PART_ALL, PART_LOW, PART_HIGH, PART_INTERIOR = 0, 1, 2, 3


class PlanDesc(C.Structure):
    _fields_ = [("ndim", C.c_int32), ("shape", C.c_int64 * 3), ("spacing", C.c_double * 3),
                ("space_order", C.c_int32), ("dt", C.c_double), ("nt", C.c_int64),
                ("device", C.c_int32), ("slab_lo", C.c_int64), ("slab_hi", C.c_int64)]


class FieldView(C.Structure):
    _fields_ = [("ptr", C.c_void_p), ("stride", C.c_int64 * 3)]


class Report(C.Structure):
    _fields_ = [("seconds", C.c_double), ("flops", C.c_longlong), ("gflops", C.c_double),
                ("steps", C.c_long), ("gpts_per_s", C.c_double), ("kernel_launches", C.c_long)]


# every symbol include/sfb200.h declares (tests/test_capi_cpu.py checks the list against
# the header)
SYMBOLS = [
    "sfb_abi_version", "sfb_last_error", "sfb_device_count", "sfb_plan_create",
    "sfb_plan_destroy", "sfb_fd_weights", "sfb_critical_dt", "sfb_set_model", "sfb_set_model_slab",
    "sfb_set_model_tti", "sfb_set_points", "sfb_locate", "sfb_forward", "sfb_forward_checkpointed", "sfb_adjoint",
    "sfb_gradient", "sfb_tti_forward", "sfb_get_wavefield", "sfb_upload_traces",
    "sfb_download_traces", "sfb_run_resident", "sfb_run_steps", "sfb_time_stencil", "sfb_step_begin", "sfb_step_compute",
    "sfb_step_points", "sfb_step_slab_boundary", "sfb_step_slab_interior", "sfb_step_slab_fused", "sfb_step_end", "sfb_tti_step_rot", "sfb_tti_step_update", "sfb_tti_step_rot_fused", "sfb_tti_peer_wait_g", "sfb_tti_peer_wait_g_ipc", "sfb_tti_step_update_fused", "sfb_slab_run", "sfb_tti_halo_blocks", "sfb_link_peers", "sfb_peer_wait", "sfb_peer_export", "sfb_link_peers_ipc", "sfb_peer_wait_ipc", "sfb_put_history", "sfb_get_gradient", "sfb_halo_blocks", "sfb_stream_sync", "sfb_streams",
    "sfb_set_streams", "sfb_copy_halo", "sfb_set_tile", "sfb_get_tile",
    "sfb_set_dense_damping", "sfb_launch_count", "sfb_autotune", "sfb_debug_stall",
]

lib.sfb_last_error.restype = C.c_char_p
lib.sfb_last_error.argtypes = [C.c_void_p]
lib.sfb_plan_create.argtypes = [C.POINTER(PlanDesc), C.POINTER(C.c_void_p)]
lib.sfb_plan_destroy.argtypes = [C.c_void_p]
lib.sfb_set_model.argtypes = [C.c_void_p, C.POINTER(FieldView), C.POINTER(FieldView), C.c_double]
lib.sfb_set_model_slab.argtypes = lib.sfb_set_model.argtypes
lib.sfb_set_model_tti.argtypes = [C.c_void_p] + [C.POINTER(FieldView)] * 4
lib.sfb_tti_forward.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(Report)]
lib.sfb_set_points.argtypes = [C.c_void_p, C.c_int, C.c_int64, C.c_void_p, C.c_void_p]
lib.sfb_forward.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.POINTER(Report)]
lib.sfb_forward_checkpointed.argtypes = lib.sfb_forward.argtypes
lib.sfb_adjoint.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(Report)]
lib.sfb_gradient.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(FieldView), C.POINTER(Report)]
lib.sfb_get_wavefield.argtypes = [C.c_void_p, C.c_int, C.c_int64, C.POINTER(FieldView)]
lib.sfb_upload_traces.argtypes = [C.c_void_p, C.c_int, C.c_void_p]
lib.sfb_download_traces.argtypes = [C.c_void_p, C.c_int, C.c_void_p]
lib.sfb_run_resident.argtypes = [C.c_void_p, C.c_int, C.c_int64, C.POINTER(Report)]
lib.sfb_run_steps.argtypes = [C.c_void_p, C.c_int, C.c_int64, C.c_int64, C.POINTER(Report)]
lib.sfb_time_stencil.argtypes = lib.sfb_run_steps.argtypes
lib.sfb_step_begin.argtypes = [C.c_void_p, C.c_int, C.c_int64]
lib.sfb_step_compute.argtypes = [C.c_void_p, C.c_int, C.c_int64, C.c_int]
lib.sfb_step_points.argtypes = [C.c_void_p, C.c_int, C.c_int64, C.c_int]
lib.sfb_step_end.argtypes = [C.c_void_p, C.c_int]
lib.sfb_step_slab_boundary.argtypes = [C.c_void_p, C.c_int, C.c_int64]
lib.sfb_step_slab_interior.argtypes = [C.c_void_p, C.c_int, C.c_int64]
lib.sfb_step_slab_fused.argtypes = [C.c_void_p, C.c_int, C.c_int64]
lib.sfb_put_history.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.POINTER(FieldView)]
lib.sfb_get_gradient.argtypes = [C.c_void_p, C.POINTER(FieldView)]
lib.sfb_halo_blocks.argtypes = [C.c_void_p, C.c_int, C.c_int64] + [C.POINTER(C.c_void_p)] * 4 + [C.POINTER(C.c_int64)]
lib.sfb_tti_step_rot.argtypes = [C.c_void_p, C.c_int64, C.c_int]
lib.sfb_tti_step_update.argtypes = [C.c_void_p, C.c_int64, C.c_int]
lib.sfb_tti_halo_blocks.argtypes = lib.sfb_halo_blocks.argtypes
lib.sfb_tti_step_rot_fused.argtypes = [C.c_void_p, C.c_int64]
lib.sfb_tti_step_update_fused.argtypes = [C.c_void_p, C.c_int64]
lib.sfb_slab_run.argtypes = [C.c_void_p, C.c_int, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p]
lib.sfb_tti_peer_wait_g.argtypes = [C.c_void_p, C.c_void_p]
lib.sfb_tti_peer_wait_g_ipc.argtypes = [C.c_void_p]
lib.sfb_link_peers.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
lib.sfb_peer_wait.argtypes = [C.c_void_p, C.c_void_p]
lib.sfb_peer_export.argtypes = [C.c_void_p, C.c_void_p]
lib.sfb_link_peers_ipc.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
lib.sfb_peer_wait_ipc.argtypes = [C.c_void_p]
PEER_BLOB_BYTES = 1024
lib.sfb_stream_sync.argtypes = [C.c_void_p]
lib.sfb_debug_stall.argtypes = [C.c_void_p, C.c_int, C.c_int64]
lib.sfb_streams.argtypes = [C.c_void_p, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p)]
lib.sfb_set_streams.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
lib.sfb_copy_halo.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64]
lib.sfb_set_tile.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int]
lib.sfb_get_tile.argtypes = [C.c_void_p] + [C.POINTER(C.c_int)] * 5
lib.sfb_set_dense_damping.argtypes = [C.c_void_p, C.c_int]
lib.sfb_autotune.argtypes = [C.c_void_p, C.c_int]
lib.sfb_launch_count.argtypes = [C.c_void_p, C.POINTER(C.c_int64)]
lib.sfb_fd_weights.argtypes = [C.c_int, C.c_int, C.c_void_p]
lib.sfb_critical_dt.argtypes = [C.c_int, C.c_void_p, C.c_double, C.c_int, C.POINTER(C.c_double)]
lib.sfb_locate.argtypes = [C.POINTER(PlanDesc), C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p]


class SfbError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[sfb {code}] {msg}")
        self.code = code


def _view(a: np.ndarray) -> FieldView:
    assert a.dtype == np.float64 and 1 <= a.ndim <= 3
    v = FieldView()
    v.ptr = a.ctypes.data
    for d in range(a.ndim):
        v.stride[d] = a.strides[d] // 8
    return v


def fd_weights(deriv, order):
    out = np.zeros(order // 2 + 1)
    rc = lib.sfb_fd_weights(deriv, order, out.ctypes.data)
    if rc:
        raise SfbError(rc, lib.sfb_last_error(None).decode())
    return out


def critical_dt(spacing, v_max, order):
    h = np.asarray(spacing, dtype=np.float64)
    out = C.c_double()
    rc = lib.sfb_critical_dt(len(h), h.ctypes.data, v_max, order, C.byref(out))
    if rc:
        raise SfbError(rc, lib.sfb_last_error(None).decode())
    return out.value


def locate(shape, spacing, origin, coords):
    """SparseFunction::locate on a padded grid (sfb_locate): base int64 [np][ndim], weights
    f64 [np][2^ndim].  `origin` is the origin of the padded grid."""
    nd = len(shape)
    d = PlanDesc()
    d.ndim = nd
    for a in range(nd):
        d.shape[a] = int(shape[a])
        d.spacing[a] = float(spacing[a])
    d.space_order = 2
    d.dt, d.nt = 1.0, 3
    org = np.asarray(origin, dtype=np.float64)
    co = np.ascontiguousarray(coords, dtype=np.float64).reshape(-1, nd)
    base = np.zeros((co.shape[0], nd), dtype=np.int64)
    w = np.zeros((co.shape[0], 1 << nd))
    rc = lib.sfb_locate(C.byref(d), org.ctypes.data, co.shape[0], co.ctypes.data,
                        base.ctypes.data, w.ctypes.data)
    if rc:
        raise SfbError(rc, lib.sfb_last_error(None).decode())
    return base, w


def device_count():
    n = C.c_int()
    lib.sfb_device_count(C.byref(n))
    return n.value


class Plan:
    """One operator context on one device (sfb_plan)."""

    def __init__(self, shape, spacing, space_order, dt, nt, device=0, slab=None,
                 dense_damping=False):
        d = PlanDesc()
        d.ndim = len(shape)
        for a in range(len(shape)):
            d.shape[a] = int(shape[a])
            d.spacing[a] = float(spacing[a])
        d.space_order = int(space_order)
        d.dt = float(dt)
        d.nt = int(nt)
        d.device = int(device)
        if slab is not None:
            d.slab_lo, d.slab_hi = int(slab[0]), int(slab[1])
        self.desc = d
        self.shape = [int(s) for s in shape]
        self.nt = int(nt)
        self.h = C.c_void_p()
        rc = lib.sfb_plan_create(C.byref(d), C.byref(self.h))
        if rc:
            raise SfbError(rc, lib.sfb_last_error(None).decode())
        self.np = [0, 0]
        if dense_damping:
            self.set_dense_damping(True)

    def _chk(self, rc):
        if rc:
            raise SfbError(rc, lib.sfb_last_error(self.h).decode())

    def close(self):
        if self.h:
            lib.sfb_plan_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_model(self, m, damp, v_max=0.0):
        m = np.asarray(m, dtype=np.float64)
        damp = np.asarray(damp, dtype=np.float64)
        self._chk(lib.sfb_set_model(self.h, C.byref(_view(m)), C.byref(_view(damp)), float(v_max)))

    def set_model_slab(self, m_slab, damp_slab, v_max=0.0):
        """m and damp over the plan's own planes only (a rank of a decomposed run)."""
        m = np.asarray(m_slab, dtype=np.float64)
        damp = np.asarray(damp_slab, dtype=np.float64)
        self._chk(lib.sfb_set_model_slab(self.h, C.byref(_view(m)), C.byref(_view(damp)), float(v_max)))

    def set_model_tti(self, epsilon, delta, theta, phi):
        arrs = [np.asarray(f, dtype=np.float64) for f in (epsilon, delta, theta, phi)]
        views = [_view(a) for a in arrs]   # FieldView.ptr is a bare address: arrs must outlive the call
        self._chk(lib.sfb_set_model_tti(self.h, *[C.byref(v) for v in views]))
        del arrs

    def tti_forward(self, src):
        src = np.ascontiguousarray(src, dtype=np.float64)
        rec = np.empty((self.nt, self.np[CLOUD_REC]))
        rep = Report()
        self._chk(lib.sfb_tti_forward(self.h, src.ctypes.data, rec.ctypes.data, C.byref(rep)))
        return rec, rep

    def set_points(self, cloud, base, w):
        base = np.ascontiguousarray(base, dtype=np.int64)
        w = np.ascontiguousarray(w, dtype=np.float64)
        self.np[cloud] = base.shape[0]
        self._chk(lib.sfb_set_points(self.h, cloud, base.shape[0], base.ctypes.data, w.ctypes.data))

    def forward(self, src, save_every=0, out=None):
        """out: optional C-contiguous f64 [nt][n_rec] table to fill (the reference's callers
        own their trace tables, proj/include/sf/sparse.hpp:46-49); allocated when omitted."""
        src = np.ascontiguousarray(src, dtype=np.float64)
        rec = np.empty((self.nt, self.np[CLOUD_REC])) if out is None else out
        if rec.shape != (self.nt, self.np[CLOUD_REC]) or rec.dtype != np.float64 \
                or not rec.flags.c_contiguous:
            raise ValueError("out must be a C-contiguous float64 [nt][n_rec] array")
        rep = Report()
        self._chk(lib.sfb_forward(self.h, src.ctypes.data, rec.ctypes.data, save_every, C.byref(rep)))
        return rec, rep

    def forward_checkpointed(self, src, checkpoint_every):
        src = np.ascontiguousarray(src, dtype=np.float64)
        rec = np.empty((self.nt, self.np[CLOUD_REC]))
        rep = Report()
        self._chk(lib.sfb_forward_checkpointed(self.h, src.ctypes.data, rec.ctypes.data,
                                               checkpoint_every, C.byref(rep)))
        return rec, rep

    def adjoint(self, rec):
        rec = np.ascontiguousarray(rec, dtype=np.float64)
        srca = np.empty((self.nt, self.np[CLOUD_SRC]))
        rep = Report()
        self._chk(lib.sfb_adjoint(self.h, rec.ctypes.data, srca.ctypes.data, C.byref(rep)))
        return srca, rep

    def gradient(self, resid, out=None):
        """out: optional f64 array of the padded grid shape to fill (the reference's callers own
        the gradient Function, proj/include/sf/seismic_ops.hpp:49-58); allocated when omitted."""
        resid = np.ascontiguousarray(resid, dtype=np.float64)
        grad = np.zeros(self.shape) if out is None else out
        if tuple(grad.shape) != tuple(self.shape) or grad.dtype != np.float64:
            raise ValueError("out must be a float64 array of the padded grid shape")
        rep = Report()
        self._chk(lib.sfb_gradient(self.h, resid.ctypes.data, C.byref(_view(grad)), C.byref(rep)))
        return grad, rep

    def wavefield(self, level, out=None, field=0):
        out = np.zeros(self.shape) if out is None else out
        self._chk(lib.sfb_get_wavefield(self.h, field, level, C.byref(_view(out))))
        return out

    def upload_traces(self, cloud, tr):
        tr = np.ascontiguousarray(tr, dtype=np.float64)
        self._chk(lib.sfb_upload_traces(self.h, cloud, tr.ctypes.data))

    def download_traces(self, cloud):
        out = np.empty((self.nt, self.np[cloud]))
        self._chk(lib.sfb_download_traces(self.h, cloud, out.ctypes.data))
        return out

    def run_resident(self, op, save_every=0):
        rep = Report()
        self._chk(lib.sfb_run_resident(self.h, op, save_every, C.byref(rep)))
        return rep

    def run_steps(self, op, t_from, t_to):
        rep = Report()
        self._chk(lib.sfb_run_steps(self.h, op, t_from, t_to, C.byref(rep)))
        return rep

    def time_stencil(self, op, t_from, t_to):
        rep = Report()
        self._chk(lib.sfb_time_stencil(self.h, op, t_from, t_to, C.byref(rep)))
        return rep

    def set_tile(self, txv, ty, stages=0, chunk=0):
        self._chk(lib.sfb_set_tile(self.h, txv, ty, stages, chunk))

    def get_tile(self):
        v = [C.c_int() for _ in range(5)]
        self._chk(lib.sfb_get_tile(self.h, *[C.byref(x) for x in v]))
        return dict(zip(["txv", "ty", "stages", "chunk", "sep"], [x.value for x in v]))

    def autotune(self, steps=0):
        self._chk(lib.sfb_autotune(self.h, steps))
        return self.get_tile()

    def launch_count(self):
        n = C.c_int64()
        self._chk(lib.sfb_launch_count(self.h, C.byref(n)))
        return n.value

    def set_dense_damping(self, on=True):
        self._chk(lib.sfb_set_dense_damping(self.h, int(on)))

    # slab stepping
    def step_begin(self, op, save_every=0):
        self._chk(lib.sfb_step_begin(self.h, op, save_every))

    def step_compute(self, op, t, part):
        self._chk(lib.sfb_step_compute(self.h, op, t, part))

    def step_points(self, op, t, part):
        self._chk(lib.sfb_step_points(self.h, op, t, part))

    def step_slab_boundary(self, op, t):
        self._chk(lib.sfb_step_slab_boundary(self.h, op, t))

    def step_slab_interior(self, op, t):
        self._chk(lib.sfb_step_slab_interior(self.h, op, t))

    def step_slab_fused(self, op, t):
        self._chk(lib.sfb_step_slab_fused(self.h, op, t))

    def step_end(self, op):
        self._chk(lib.sfb_step_end(self.h, op))

    def halo_blocks(self, op, t):
        p = [C.c_void_p() for _ in range(4)]
        n = C.c_int64()
        self._chk(lib.sfb_halo_blocks(self.h, op, t, *[C.byref(x) for x in p], C.byref(n)))
        return dict(send_lo=p[0].value, send_hi=p[1].value, recv_lo=p[2].value,
                    recv_hi=p[3].value, count=n.value)

    def tti_step_rot(self, t, part):
        self._chk(lib.sfb_tti_step_rot(self.h, t, part))

    def tti_step_update(self, t, part):
        self._chk(lib.sfb_tti_step_update(self.h, t, part))

    def tti_step_rot_fused(self, t):
        self._chk(lib.sfb_tti_step_rot_fused(self.h, t))

    def tti_step_update_fused(self, t):
        self._chk(lib.sfb_tti_step_update_fused(self.h, t))

    def slab_run(self, op, t_from, t_to, inj=None, smp=None):
        """Steps [t_from, t_to) of this rank's slab in one call (sfb_slab_run); `smp`: f64
        [nt][np] table of the sampled cloud filled while the loop runs, `inj`: f64 [nt][np]
        table of the injected cloud fed while the loop runs (None: the uploaded one)."""
        def table(a, cloud_np):
            if a is None:
                return None
            if a.dtype != np.float64 or not a.flags.c_contiguous or a.shape[0] != self.nt \
                    or a.size != self.nt * cloud_np:
                raise ValueError("trace tables are C-contiguous float64 [nt][np] arrays")
            return a.ctypes.data
        backward = op in (OP_ADJOINT, OP_GRADIENT)
        c_inj = CLOUD_REC if backward else CLOUD_SRC
        c_smp = CLOUD_SRC if backward else CLOUD_REC
        self._chk(lib.sfb_slab_run(self.h, op, t_from, t_to, table(inj, self.np[c_inj]),
                                   table(smp, self.np[c_smp])))
        return smp

    def tti_peer_wait_g(self, neighbour):
        self._chk(lib.sfb_tti_peer_wait_g(self.h, neighbour.h))

    def tti_peer_wait_g_ipc(self):
        self._chk(lib.sfb_tti_peer_wait_g_ipc(self.h))

    def tti_halo_blocks(self, which, t):
        p = [C.c_void_p() for _ in range(4)]
        n = C.c_int64()
        self._chk(lib.sfb_tti_halo_blocks(self.h, which, t, *[C.byref(x) for x in p], C.byref(n)))
        return dict(send_lo=p[0].value, send_hi=p[1].value, recv_lo=p[2].value,
                    recv_hi=p[3].value, count=n.value)

    def link_peers(self, lo=None, hi=None):
        self._chk(lib.sfb_link_peers(self.h, lo.h if lo else None, hi.h if hi else None))

    def peer_export(self):
        blob = C.create_string_buffer(PEER_BLOB_BYTES)
        self._chk(lib.sfb_peer_export(self.h, blob))
        return blob.raw

    def link_peers_ipc(self, lo_blob=None, hi_blob=None):
        self._chk(lib.sfb_link_peers_ipc(self.h, lo_blob, hi_blob))

    def peer_wait_ipc(self):
        self._chk(lib.sfb_peer_wait_ipc(self.h))

    def peer_wait(self, neighbour):
        self._chk(lib.sfb_peer_wait(self.h, neighbour.h))

    def copy_halo(self, dst, src, count):
        self._chk(lib.sfb_copy_halo(self.h, dst, src, count))

    def debug_stall(self, boundary_stream, microseconds):
        self._chk(lib.sfb_debug_stall(self.h, int(boundary_stream), int(microseconds)))

    def sync(self):
        self._chk(lib.sfb_stream_sync(self.h))
