"""Host layer (C++ mirror of the reference's model/geometry/sparse/function interface),
CPU-only part: the reference's own unit tests for these classes, restated
(proj/tests/test_seismic.cpp:29-114, proj/tests/test_symbolic.cpp:252-315,
proj/tests/test_verify.cpp:30-52), plus agreement with the oracle."""
import numpy as np
import pytest

from oracle import oracle as o
from paper_1808_01995_b200 import _sfb_host as H


def constant_model(n, h, c, nbl, order=8):
    return H.SeismicModel([n, n], [h, h], [0.0, 0.0], np.full(n * n, c), nbl, order)


def test_damping_vanishes_inside_and_peaks_at_edge():  # test_seismic.cpp:29-46
    m = constant_model(21, 10.0, 1.5, 6)
    d = m.damp.array()
    n = 21 + 12
    assert d.shape == (n, n)
    assert (d[6:n - 6, 6:n - 6] == 0.0).all()
    mid, prev = n // 2, 0.0
    for i in range(5, -1, -1):
        assert d[i, mid] > prev
        prev = d[i, mid]
    edge = d[0, mid]
    assert (d <= 2.0 * edge + 1e-18).all()
    assert d[0, 0] == pytest.approx(2.0 * edge, rel=1e-12)


def test_nbl_zero_leaves_no_layer():  # test_seismic.cpp:48-54
    m = constant_model(15, 10.0, 2.0, 0)
    assert (m.damp.array() == 0.0).all() and m.grid.shape[0] == 15


def test_critical_dt():  # test_seismic.cpp:56-60
    m = constant_model(15, 10.0, 2.0, 0)
    assert m.critical_dt(2) == pytest.approx(10.0 / 4.0, rel=1e-14)
    assert m.critical_dt(8) < m.critical_dt(2)


def test_velocity_edge_extension():  # test_seismic.cpp:62-75
    n, nbl = 9, 5
    vel = np.array([[1.0 + 0.1 * i + 0.01 * j for j in range(n)] for i in range(n)])
    m = H.SeismicModel([n, n], [10.0, 10.0], [0.0, 0.0], vel, nbl, 4)
    mm = m.m.array()
    slow = lambda v: 1.0 / (v * v)
    assert mm[0, 0] == pytest.approx(slow(vel[0, 0]), rel=1e-14)
    assert mm[nbl, nbl] == pytest.approx(slow(vel[0, 0]), rel=1e-14)
    assert mm[nbl + n - 1 + nbl, nbl] == pytest.approx(slow(vel[n - 1, 0]), rel=1e-14)
    assert mm[nbl + 3, 0] == pytest.approx(slow(vel[3, 0]), rel=1e-14)


def test_physical_m_roundtrip():  # test_seismic.cpp:77-83
    m = constant_model(11, 10.0, 1.5, 4)
    vals = m.physical_m()
    vals = vals + 0.001 * (np.arange(vals.size) % 7)
    m.set_physical_m(vals)
    assert (m.physical_m() == vals).all()


def test_geometry_time_axis_and_ricker():  # test_seismic.cpp:85-106
    m = constant_model(21, 10.0, 1.5, 4)
    g = H.AcquisitionGeometry(m, [100.0, 100.0], [50.0, 50.0, 150.0, 50.0], 0.0, 101.0, 2.0, 0.01)
    assert g.nt == 51 and g.n_src == 1 and g.n_rec == 2
    tr = g.src.traces[:, 0]
    assert tr.max() == pytest.approx(1.0, rel=1e-9)
    assert abs(int(tr.argmax()) * 2.0 - 100.0) <= 2.0
    assert (g.rec.traces == 0.0).all()


def test_geometry_rejects_unstable_dt():  # test_seismic.cpp:108-114
    m = constant_model(21, 10.0, 1.5, 4)
    with pytest.raises(H.StabilityError):
        H.AcquisitionGeometry(m, [100.0, 100.0], [50.0, 50.0], 0.0, 100.0, m.critical_dt() * 1.5, 0.01)


def test_operator_rejects_unstable_dt():  # seismic_ops.cpp:15-22: before touching a device
    m = constant_model(21, 10.0, 1.5, 4, order=2)
    g = H.AcquisitionGeometry(m, [100.0, 100.0], [50.0, 50.0], 0.0, 50.0, 0.99 * m.critical_dt(2), 0.01)
    with pytest.raises(H.StabilityError):
        H.forward_operator(m, g, 16)
    with pytest.raises(H.OrderError):
        H.forward_operator(m, g, 3)


def test_wavelets():  # test_verify.cpp:30-52
    w = H.ricker(0.01, 0.0, 0.5, 401)
    assert w[200] == pytest.approx(1.0, rel=1e-14) and np.abs(w).max() == pytest.approx(1.0, rel=1e-14)
    assert abs(w[0]) < 1e-3 and abs(H.dgauss4_value(0.01, 0.0)) < abs(w[0])
    with pytest.raises(H.ParameterError):
        H.ricker(0.0, 0.0, 0.5, 10)
    with pytest.raises(H.ParameterError):
        H.ricker(0.01, 0.0, -1.0, 10)
    fp = 0.045
    assert H.dgauss4_value(fp, 2.0 / fp) == pytest.approx(1.0, rel=1e-14)
    assert abs(H.dgauss4_value(fp, 0.0)) < 1e-5


def test_field_storage_halos_and_strides():  # test_symbolic.cpp:252-263
    g = H.Grid([11, 11], [1.0, 1.0], [0.0, 0.0])
    f = H.Function.create("f", g, 4)
    assert f.padded_extent(0) == 15 and f.storage_size == 15 * 15
    f.set([0, 0], 7.0)
    f.set([10, 10], -3.0)
    a = f.array()
    assert a[0, 0] == 7.0 and a[10, 10] == -3.0 and a.strides == (15 * 8, 8)
    assert np.count_nonzero(a) == 2


def test_time_function_slot_policies():  # test_symbolic.cpp:265-276
    g = H.Grid([8], [1.0], [0.0])
    u = H.TimeFunction.create("u", g, 2, 2)
    assert u.time_buffered and u.time_slots == 3
    s = H.TimeFunction.create("s", g, 2, 2, 12)
    assert (not s.time_buffered) and s.time_slots == 12
    with pytest.raises(H.ParameterError):
        H.TimeFunction.create("bad", g, 2, 2, 2)
    with pytest.raises(H.OrderError):
        H.TimeFunction.create("bad", g, 3, 2)
    with pytest.raises(H.OrderError):
        H.Function.create("bad", g, 0)
    with pytest.raises(H.ParameterError):
        H.Grid([1, 5], [1.0, 1.0], [0.0, 0.0])


def test_sparse_locate():  # test_symbolic.cpp:278-315
    g = H.Grid([11, 11], [1.0, 1.0], [0.0, 0.0])
    sp = H.SparseFunction.create("src", g, np.array([0.3, 0.7]), 5)
    sp.locate()
    assert np.allclose(sp.weight_table, [0.21, 0.09, 0.49, 0.21], rtol=1e-12)
    assert sp.base_table == [0, 0]
    far = H.SparseFunction.create("r", g, np.array([10.0, 10.0]), 1)
    far.locate()
    assert far.base_table == [9, 9] and far.weight_table[3] == pytest.approx(1.0)
    with pytest.raises(H.LocationError):
        H.SparseFunction.create("bad", g, np.array([11.0, 5.0]), 1).locate()
    with pytest.raises(H.LocationError):
        H.SparseFunction.create("neg", g, np.array([-0.5, 5.0]), 1).locate()
    node = H.SparseFunction.create("s", g, np.array([4.0, 6.0]), 1)
    node.locate()
    assert node.base_table == [4, 6] and node.weight_table == [1.0, 0.0, 0.0, 0.0]


@pytest.mark.parametrize("ndim", [1, 2, 3])
def test_model_and_geometry_match_oracle(ndim):
    rng = np.random.default_rng(3)
    shape = [13, 9, 11][:ndim]
    h = [10.0, 7.5, 12.5][:ndim]
    vel = rng.uniform(1.5, 4.0, size=shape)
    om = o.Model(shape, h, [5.0] * ndim, vel, 4, 6)
    hm = H.SeismicModel(shape, h, [5.0] * ndim, vel, 4, 6)
    assert np.array_equal(hm.m.array(), om.m) and np.array_equal(hm.damp.array(), om.damp)
    assert hm.critical_dt(6) == om.critical_dt(6) and hm.v_max == om.v_max
    L = [(s - 1) * x for s, x in zip(shape, h)]
    src = [5.0 + 0.37 * x for x in L]
    rec = np.array([[5.0 + f * x for x in L] for f in (0.0, 0.21, 0.5, 1.0)]).ravel()
    dt = 0.7 * om.critical_dt()
    og = o.Geometry(om, src, rec, 0.0, 40.0, dt, 0.02)
    hg = H.AcquisitionGeometry(hm, src, rec, 0.0, 40.0, dt, 0.02)
    assert hg.nt == og.nt
    assert np.array_equal(np.array(hg.rec.base_table).reshape(-1, ndim), og.rec_base)
    assert np.array_equal(np.array(hg.rec.weight_table).reshape(-1, 1 << ndim), og.rec_w)
    assert np.array_equal(hg.src.traces, og.src)


def test_objective_shape_check():  # seismic_ops.cpp:151-152
    g = H.Grid([5, 5], [10.0, 10.0], [0.0, 0.0])
    s = H.SparseFunction.create("s", g, np.array([5.0, 5.0, 35.0, 12.0]), 6)
    with pytest.raises(H.ParameterError):
        H.objective(s, np.zeros(5))
    s.traces[:] = 2.0
    assert H.objective(s, np.zeros(12)) == pytest.approx(0.5 * 4.0 * 12)


def test_no_cpu_fallback_without_a_device():
    """On a box without a GPU every operator build must fail loudly (CapabilityError),
    never run on the host."""
    from paper_1808_01995_b200 import capi
    if capi.device_count() > 0:
        pytest.skip("a CUDA device is present")
    m = constant_model(21, 10.0, 1.5, 4)
    g = H.AcquisitionGeometry(m, [100.0, 100.0], [50.0, 50.0], 0.0, 50.0, 0.9 * m.critical_dt(), 0.01)
    with pytest.raises(H.CapabilityError):
        H.forward_operator(m, g, 8)
    with pytest.raises(capi.SfbError) as e:
        capi.Plan([21, 21], [10.0, 10.0], 8, 1.0, 10)
    assert e.value.code == capi.ERR_CAPABILITY


def test_loglog_fit():  # proj/tests/test_verify.cpp:13-28
    x = [1.0, 2.0, 4.0, 8.0]
    f = H.fit_loglog(x, [3.5 * v ** 2.25 for v in x])
    assert f.slope == pytest.approx(2.25, rel=1e-12)
    assert f.intercept == pytest.approx(np.log(3.5), rel=1e-12) and f.residual <= 1e-12
    for bad in ([[1.0, 2.0], [1.0, 2.0]], [[1.0, 2.0, 2.0], [1.0, 2.0, 3.0]],
                [[1.0, 2.0, 3.0], [1.0, -2.0, 3.0]], [[1.0, 3.0, 2.0], [1.0, 2.0, 3.0]]):
        with pytest.raises(H.ParameterError):
            H.fit_loglog(*bad)
