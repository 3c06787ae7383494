"""bench.py's N > 1 code path without GPUs: slabs.bench_core (warm-up, barrier-bracketed timed
window, max over ranks, end-to-end leg) and slabs.scaling_line driven under gloo with the
numpy slab engine of tests/test_slabs_gloo.py standing in for the CUDA plan; plus the
slab-local workload generators of configs[4]'s weak-scaling series."""
import json
import os
import time

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1808_01995_b200 import slabs
from paper_1808_01995_b200 import synthetic as syn
from tests.test_slabs_gloo import K as HALO
from tests.test_slabs_gloo import N, NumpyEngine, _free_port


class StubJob:
    """what bench.SlabJob provides, on the numpy engine (host clock instead of CUDA events)"""

    def __init__(self, rank, world):
        self.bounds = slabs.split_slabs(N[0], world, HALO)
        self.rank, self.world = rank, world
        self.ex = slabs.HaloExchanger(rank, world)
        self.eng = None
        self.points_owned = float(self.bounds[rank][1] - self.bounds[rank][0]) * N[1] * N[2]
        self.calls = 0

    def begin(self):
        self.eng = NumpyEngine(*self.bounds[self.rank])

    def loop(self, a, b):
        slabs.step_loop(self.eng, self.ex, a, b)
        self.calls += 3 * (b - a)

    def sync(self):
        pass

    def start(self):
        self.t0 = time.perf_counter()

    def stop(self):
        return time.perf_counter() - self.t0

    def launches(self):
        return self.calls

    def upload(self):
        return 8.0 * self.eng.src.size if self.eng is not None else 8.0

    def download(self):
        return float(self.eng.rec.nbytes)


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    job = StubJob(rank, world)
    job.begin()
    meas = slabs.bench_core(slabs.Comm(rank, world), job, 4, 3)
    if rank == 0:
        line = slabs.scaling_line(meas, metric="acoustic_forward_gpts_per_s", world=world, K=4, W=3,
                                  scaling="strong", config={"workload": "stub"}, bytes_per_point=16.0,
                                  contract_bytes=20.0, peak=6551.0, peak_kind="measured",
                                  halo="gloo send/recv", halo_bytes=HALO * N[1] * N[2] * 8)
        with open(out, "w") as f:
            json.dump(line, f)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_bench_core_under_gloo(tmp_path, world):
    out = str(tmp_path / "line.json")
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    line = json.load(open(out))
    assert line["n_gpus"] == world and line["steps"] == 4 and line["warmup"] == 3
    assert len(line["per_rank_ms_per_step"]) == world
    assert line["ms_per_step"] == pytest.approx(max(line["per_rank_ms_per_step"]))
    # whole-job value: all ranks' nodes over the slowest rank's time
    pts = float(np.prod(N))
    assert line["value"] == pytest.approx(pts * 4 / (line["ms_per_step"] * 4e-3) / 1e9)
    assert line["gpu_launches"] == 12 and line["e2e"]["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] > 0 and line["e2e"]["d2h_bytes_per_step"] > 0
    assert line["roofline"]["frac_contract"] == pytest.approx(line["roofline"]["frac"] * 20.0 / 16.0)
    assert line["cpu_baseline"] if "cpu_baseline" in line else True


def test_bench_core_single_rank_needs_no_process_group():
    job = StubJob(0, 1)
    job.begin()
    meas = slabs.bench_core(slabs.Comm(0, 1), job, 4, 3)
    assert meas["points"] == float(np.prod(N)) and len(meas["per_rank_ms_per_step"]) == 1


def test_weak_scaling_extents():
    assert slabs.weak_extent(128, 8) == 1024
    b = slabs.split_slabs(128 * 8 + 80, 8, 8)
    assert b[0] == (0, 138) and b[-1][1] == 1104 and all(h - l == 138 for l, h in b)


def test_slab_local_generators_agree_with_the_global_model():
    """ranks of the weak-scaling series build m and damp for their own planes only"""
    from paper_1808_01995_b200 import _sfb_host as H
    shape, nbl, h = [20, 24, 28], 6, [10.0, 12.5, 8.0]
    vel = syn.smooth_field(shape, 3, 2.0, 1.5, 4.5)
    model = H.SeismicModel(shape, h, [0.0] * 3, vel, nbl, 8)
    N3 = list(model.grid.shape)
    dz, dy, dx = syn.damping_profiles(N3, nbl, h, model.v_max)
    full = dz[:, None, None] + dy[None, :, None] + dx[None, None, :]
    assert np.abs(full - model.damp.array()).max() <= 1e-15 * np.abs(full).max()
    for lo, hi in [(0, 5), (5, 17), (17, 28), (28, 32)]:
        m, d = syn.slab_model(shape, nbl, h, lo, hi, lambda a, b: vel[a:b], model.v_max)
        assert np.array_equal(m, model.m.array()[lo:hi])
        assert np.abs(d - model.damp.array()[lo:hi]).max() <= 1e-15 * np.abs(full).max()
    # per-plane seeded noise: two ranks generate identical values for shared planes
    a = syn.smooth_slab([64, 48, 40], 10, 30, 7, 4.0, 1.5, 4.5)
    b = syn.smooth_slab([64, 48, 40], 20, 44, 7, 4.0, 1.5, 4.5)
    assert np.array_equal(a[10:], b[:10]) and 1.5 <= a.min() < a.max() <= 4.5


def test_bench_workload_deals_every_receiver_to_exactly_one_rank(monkeypatch):
    """bench.Workload at N > 1 (host side only): slab bounds, the receivers a rank binds."""
    import bench
    monkeypatch.setitem(bench.CONFIGS[2], "n", 48)
    world, seen, total = 4, [], None
    for rank in range(world):
        wl = bench.Workload(2, "forward", 6, rank, world, "strong")
        lo, hi = wl.slab
        assert wl.bounds == slabs.split_slabs(48 + 2 * bench.NBL, world, 4)
        assert ((wl.rec_base[:, 0] >= lo) & (wl.rec_base[:, 0] < hi)).all()
        total = wl.n_rec_global
        real = wl.rec_w.any(axis=1)    # a rank without receivers binds one weightless dummy
        seen.append({tuple(b) for b in wl.rec_base[real]})
        assert wl.src_base.shape[0] == 1 and wl.nt == 8
    assert sum(len(s) for s in seen) == total == 48 * 48
    assert len(set().union(*seen)) == total
    # the weak-scaling series grows the slab axis with the rank count
    N, phys = bench.grid_of(5, 8, "weak")
    assert phys == [1024, 1024, 1024] and N == [1104] * 3
    assert bench.grid_of(5, 2, "weak")[1] == [256, 1024, 1024]
