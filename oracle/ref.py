"""ctypes front end of oracle/_ref/libsf_ref.so: the REFERENCE's own sources, compiled in
place by oracle/Makefile against the Boost stand-in (oracle/ref_shim), driven through its
public API by oracle/ref_driver.cpp.

TEST INFRASTRUCTURE ONLY (see oracle/sf_oracle.c).  Used to (1) validate the oracle
restatement against the real reference, (2) generate the golden fixtures under
tests/golden/ (oracle/make_golden.py), (3) time the reference's own CPU engines in
bench.py --impl reference.  /root/reference is not needed at run time, only the built .so.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "libsf_ref.so")
INTERPRETER, EMITTED, AUTO = 0, 1, 2
_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


class _Problem(C.Structure):
    _fields_ = [("ndim", C.c_int), ("shape", C.c_void_p), ("spacing", C.c_void_p),
                ("origin", C.c_void_p), ("velocity", C.c_void_p), ("nbl", C.c_long),
                ("model_order", C.c_int), ("op_order", C.c_int), ("nsrc", C.c_long),
                ("nrec", C.c_long), ("src_coords", C.c_void_p), ("rec_coords", C.c_void_p),
                ("t0", C.c_double), ("tn", C.c_double), ("dt", C.c_double), ("f0", C.c_double)]


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(LIB_PATH)
        _lib.sfr_last_error.restype = C.c_char_p
    return _lib


class RefError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[reference {code}] {msg}")
        self.code = code


def _chk(rc):
    if rc:
        raise RefError(rc, lib().sfr_last_error().decode())


class Problem:
    """Inputs of one reference run (SeismicModel + AcquisitionGeometry arguments)."""

    def __init__(self, shape, spacing, origin, velocity, nbl, model_order, op_order, src, rec,
                 t0, tn, dt, f0):
        self.ndim = len(shape)
        self.shape = np.array(shape, dtype=np.int64)
        self.spacing = np.array(spacing, dtype=np.float64)
        self.origin = np.array(origin, dtype=np.float64)
        self.velocity = np.ascontiguousarray(velocity, dtype=np.float64).ravel()
        self.src = np.ascontiguousarray(src, dtype=np.float64).reshape(-1, self.ndim)
        self.rec = np.ascontiguousarray(rec, dtype=np.float64).reshape(-1, self.ndim)
        self.N = [int(s) + 2 * int(nbl) for s in shape]
        p = _Problem()
        p.ndim = self.ndim
        p.shape, p.spacing, p.origin = (a.ctypes.data for a in (self.shape, self.spacing, self.origin))
        p.velocity = self.velocity.ctypes.data
        p.nbl, p.model_order, p.op_order = int(nbl), int(model_order), int(op_order)
        p.nsrc, p.nrec = self.src.shape[0], self.rec.shape[0]
        p.src_coords, p.rec_coords = self.src.ctypes.data, self.rec.ctypes.data
        p.t0, p.tn, p.dt, p.f0 = float(t0), float(tn), float(dt), float(f0)
        self.c = p

    def model(self):
        m, d = np.empty(self.N), np.empty(self.N)
        crit = C.c_double()
        _chk(lib().sfr_model(C.byref(self.c), m.ctypes.data_as(C.c_void_p),
                             d.ctypes.data_as(C.c_void_p), C.byref(crit)))
        return m, d, crit.value

    def geometry(self):
        nt = C.c_long()
        nc = 1 << self.ndim
        sb = np.zeros((self.c.nsrc, self.ndim), dtype=np.int64)
        rb = np.zeros((self.c.nrec, self.ndim), dtype=np.int64)
        sw, rw = np.zeros((self.c.nsrc, nc)), np.zeros((self.c.nrec, nc))
        _chk(lib().sfr_geometry(C.byref(self.c), C.byref(nt), None, None, None, None, None))
        tr = np.zeros((nt.value, self.c.nsrc))
        _chk(lib().sfr_geometry(C.byref(self.c), C.byref(nt), sb.ctypes.data_as(C.c_void_p),
                                sw.ctypes.data_as(C.c_void_p), rb.ctypes.data_as(C.c_void_p),
                                rw.ctypes.data_as(C.c_void_p), tr.ctypes.data_as(C.c_void_p)))
        return dict(nt=nt.value, src_base=sb, src_w=sw, rec_base=rb, rec_w=rw, src=tr)

    def nt(self):
        nt = C.c_long()
        _chk(lib().sfr_geometry(C.byref(self.c), C.byref(nt), None, None, None, None, None))
        return nt.value

    def forward(self, src_traces=None, backend=AUTO, nthreads=1, levels=True):
        nt = self.nt()
        rec = np.zeros((nt, self.c.nrec))
        a = np.empty(self.N) if levels else None
        b = np.empty(self.N) if levels else None
        sec = C.c_double()
        st = None if src_traces is None else np.ascontiguousarray(src_traces, dtype=np.float64)
        _chk(lib().sfr_forward(C.byref(self.c), None if st is None else st.ctypes.data_as(C.c_void_p),
                               backend, nthreads, rec.ctypes.data_as(C.c_void_p),
                               None if a is None else a.ctypes.data_as(C.c_void_p),
                               None if b is None else b.ctypes.data_as(C.c_void_p), C.byref(sec)))
        return dict(rec=rec, final=a, prev=b, seconds=sec.value, nt=nt)

    def adjoint(self, rec_in, backend=AUTO, nthreads=1):
        nt = self.nt()
        rec_in = np.ascontiguousarray(rec_in, dtype=np.float64)
        srca = np.zeros((nt, self.c.nsrc))
        lvl = np.empty(self.N)
        _chk(lib().sfr_adjoint(C.byref(self.c), rec_in.ctypes.data_as(C.c_void_p), backend, nthreads,
                               srca.ctypes.data_as(C.c_void_p), lvl.ctypes.data_as(C.c_void_p)))
        return dict(srca=srca, level0=lvl)

    def fwi_gradient(self, observed, backend=AUTO):
        nt = self.nt()
        observed = np.ascontiguousarray(observed, dtype=np.float64)
        phi = C.c_double()
        g = np.zeros([int(s) for s in self.shape])
        r = np.zeros((nt, self.c.nrec))
        _chk(lib().sfr_fwi_gradient(C.byref(self.c), observed.ctypes.data_as(C.c_void_p), backend,
                                    C.byref(phi), g.ctypes.data_as(C.c_void_p),
                                    r.ctypes.data_as(C.c_void_p)))
        return phi.value, g, r


def dense_bench(n, order, steps, backend=EMITTED, nthreads=1):
    """Seconds the reference's own engine needs for `steps` bare acoustic updates of n^3."""
    sec, fpp = C.c_double(), C.c_double()
    _chk(lib().sfr_dense_bench(C.c_long(n), order, C.c_long(steps), backend, nthreads,
                               C.byref(sec), C.byref(fpp)))
    return sec.value, fpp.value


def emit_available():
    return bool(lib().sfr_emit_available())


def write_grid(path, data):
    data = np.ascontiguousarray(data, dtype=np.float64)
    shape = (C.c_long * data.ndim)(*data.shape)
    _chk(lib().sfr_write_grid(path.encode(), data.ndim, shape, data.ctypes.data_as(C.c_void_p)))


def read_grid(path, capacity=1 << 24):
    nd = C.c_int()
    shape = (C.c_long * 8)()
    buf = np.zeros(capacity)
    _chk(lib().sfr_read_grid(path.encode(), C.byref(nd), shape, buf.ctypes.data_as(C.c_void_p),
                             C.c_long(capacity)))
    sh = [shape[i] for i in range(nd.value)]
    return buf[: int(np.prod(sh))].reshape(sh).copy()


def write_traces_table(path, traces, t0, dt):
    tr = np.ascontiguousarray(traces, dtype=np.float64)
    _chk(lib().sfr_write_traces_table(path.encode(), C.c_long(tr.shape[0]), C.c_long(tr.shape[1]),
                                      tr.ctypes.data_as(C.c_void_p), C.c_double(t0), C.c_double(dt)))


def write_cloud_csv(traces_path, coords_path, ndim, n, coords, traces, times):
    co = np.ascontiguousarray(coords, dtype=np.float64)
    tr = np.ascontiguousarray(traces, dtype=np.float64)
    tm = np.ascontiguousarray(times, dtype=np.float64)
    _chk(lib().sfr_write_cloud_csv(traces_path.encode(), coords_path.encode(), ndim, C.c_long(n),
                                   C.c_long(tr.shape[1]), C.c_long(tr.shape[0]),
                                   co.ctypes.data_as(C.c_void_p), tr.ctypes.data_as(C.c_void_p),
                                   tm.ctypes.data_as(C.c_void_p)))
