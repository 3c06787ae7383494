"""Wire formats next to the propagator path: SFGD grid container and
trace / coordinate CSV tables.  Round trips restate proj/tests/test_seismic.cpp:315-350;
byte-level identity is checked against files written by the reference itself (oracle/_ref)."""
import numpy as np
import pytest

from oracle import ref
from paper_1808_01995_b200 import _sfb_host as H


def test_grid_container_and_trace_csv_roundtrip_exactly(tmp_path):  # test_seismic.cpp:315-350
    rng = np.random.default_rng(7)
    data = rng.uniform(-1.0, 1.0, size=(3, 4))
    path = str(tmp_path / "roundtrip_test.sfgd")
    H.write_grid(path, [3, 4], data)
    back = H.read_grid(path)
    assert back.shape == (3, 4) and np.array_equal(back, data)

    g = H.Grid([5, 5], [10.0, 10.0], [0.0, 0.0])
    s = H.SparseFunction.create("s", g, np.array([5.0, 5.0, 35.0, 12.0]), 6)
    times = [0.5 * t for t in range(6)]
    s.traces[:] = rng.uniform(-1.0, 1.0, size=(6, 2))
    saved = s.traces.copy()
    csv = str(tmp_path / "roundtrip_test.csv")
    H.write_traces_csv(csv, s, times)
    s.traces[:] = 0.0
    assert H.read_traces_csv(csv, s) == times
    assert np.array_equal(s.traces, saved)
    coords = str(tmp_path / "coords.csv")
    H.write_coords_csv(coords, s)
    assert H.read_coords_csv(coords, 2) == [5.0, 5.0, 35.0, 12.0]


def test_format_errors(tmp_path):
    bad = tmp_path / "bad.sfgd"
    bad.write_bytes(b"NOPE" + bytes(12))
    with pytest.raises(H.ParameterError):
        H.read_grid(str(bad))
    with pytest.raises(H.ParameterError):
        H.write_grid(str(tmp_path / "x.sfgd"), [2, 3], np.zeros(5))
    trunc = tmp_path / "trunc.sfgd"
    H.write_grid(str(trunc), [4], np.arange(4.0))
    trunc.write_bytes(trunc.read_bytes()[:-8])
    with pytest.raises(H.ParameterError):
        H.read_grid(str(trunc))
    g = H.Grid([5, 5], [10.0, 10.0], [0.0, 0.0])
    s = H.SparseFunction.create("s", g, np.array([5.0, 5.0]), 3)
    with pytest.raises(H.ParameterError):
        H.write_traces_csv(str(tmp_path / "t.csv"), s, [0.0, 1.0])


@pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")
def test_files_are_byte_identical_to_the_reference(tmp_path):
    rng = np.random.default_rng(3)
    data = rng.standard_normal((5, 3, 7)) * 1e3
    a, b = str(tmp_path / "ours.sfgd"), str(tmp_path / "ref.sfgd")
    H.write_grid(a, list(data.shape), data)
    ref.write_grid(b, data)
    assert open(a, "rb").read() == open(b, "rb").read()
    assert np.array_equal(ref.read_grid(a), data) and np.array_equal(H.read_grid(b), data)

    tr = rng.standard_normal((9, 4)) * np.array([1e-12, 1.0, 1e6, 1e300])
    a, b = str(tmp_path / "ours.csv"), str(tmp_path / "ref.csv")
    H.write_traces_table(a, tr, 0.25, 1.7)
    ref.write_traces_table(b, tr, 0.25, 1.7)
    assert open(a).read() == open(b).read()

    coords = rng.uniform(0.0, 7.0, size=(4, 3))
    times = np.arange(9) * 0.1
    g = H.Grid([8, 8, 8], [1.0] * 3, [0.0] * 3)
    s = H.SparseFunction.create("s", g, coords, 9)
    s.traces[:] = tr
    ta, ca = str(tmp_path / "t_ours.csv"), str(tmp_path / "c_ours.csv")
    tb, cb = str(tmp_path / "t_ref.csv"), str(tmp_path / "c_ref.csv")
    H.write_traces_csv(ta, s, list(times))
    H.write_coords_csv(ca, s)
    ref.write_cloud_csv(tb, cb, 3, 8, coords, tr, times)
    assert open(ta).read() == open(tb).read() and open(ca).read() == open(cb).read()
