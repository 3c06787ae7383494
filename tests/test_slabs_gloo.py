"""Multi-rank host logic on CPU (gloo, world_size 2): the slab protocol of
paper_1808_01995_b200/slabs.py -- bounds, neighbour exchange of ghost planes, ownership of
scattered nodes and sampled points, step order -- driven through the same step_loop the GPU
path uses, with a small numpy engine standing in for the CUDA plan.  The decomposed run must
equal the single-domain run bit for bit."""
import contextlib
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1808_01995_b200 import slabs

K = 2                       # order-4 star stencil
W = np.array([-2.5, 4.0 / 3.0, -1.0 / 12.0])
N = (23, 9, 11)
NT = 14


class NumpyEngine:
    """Slab engine with the interface step_loop expects (ghost offset K on axis 0)."""

    def __init__(self, lo, hi):
        self.lo, self.hi, self.n0 = lo, hi, hi - lo
        self.u = [np.zeros((self.n0 + 2 * K, N[1], N[2])) for _ in range(2)]
        rng = np.random.default_rng(11)
        self.r = 0.05 + 0.01 * rng.random(N)          # same field on every rank
        self.src_cell = (11, 4, 5)                     # plane 11 is the last plane of rank 0
        self.src = np.sin(0.7 * np.arange(NT))
        self.rec_base = [(z, 3, 4) for z in range(0, N[0] - 1)]   # cells straddle the cut
        self.rec_w = np.array([0.4, 0.6])              # weights of planes z, z+1
        self.rec = np.zeros((NT, len(self.rec_base)))

    boundary = interior = staticmethod(contextlib.nullcontext)

    def _planes(self, part):
        if part == "low":
            return range(0, min(K, self.n0))
        if part == "high":
            return range(max(self.n0 - K, K), self.n0)
        if part == "interior":
            return range(K, max(self.n0 - K, K))
        return range(0, self.n0)

    def update(self, part, t):
        cur, new = self.u[t & 1], self.u[(t + 1) & 1]
        p = np.pad(cur, ((0, 0), (K, K), (K, K)))
        for z in self._planes(part):
            c = z + K
            lap = 3 * W[0] * cur[c]
            for j in (1, 2):
                lap = lap + W[j] * (cur[c - j] + cur[c + j])
                lap = lap + W[j] * (p[c, K - j:K - j + N[1], K:K + N[2]] + p[c, K + j:K + j + N[1], K:K + N[2]])
                lap = lap + W[j] * (p[c, K:K + N[1], K - j:K - j + N[2]] + p[c, K:K + N[1], K + j:K + j + N[2]])
            new[c] = 2 * cur[c] + self.r[self.lo + z] * lap - new[c]

    def scatter(self, part, t):
        z = self.src_cell[0] - self.lo
        planes = self._planes("low" if part == "boundary" else "interior")
        hit = z in planes or (part == "boundary" and z in self._planes("high"))
        if hit:
            self.u[(t + 1) & 1][z + K, self.src_cell[1], self.src_cell[2]] += self.src[t] * self.r[self.src_cell]

    def gather(self, t):
        cur = self.u[t & 1]
        for i, (z, y, x) in enumerate(self.rec_base):
            if self.lo <= z < self.hi:                 # owner of the base plane samples
                c = z - self.lo + K
                self.rec[t, i] = self.rec_w[0] * cur[c, y, x] + self.rec_w[1] * cur[c + 1, y, x]

    def blocks(self, t):
        u = self.u[(t + 1) & 1]
        n0 = self.n0
        f = torch.from_numpy
        return f(u[K:2 * K]), f(u[n0:n0 + K]), f(u[0:K]), f(u[n0 + K:n0 + 2 * K])


def serial_run():
    e = NumpyEngine(0, N[0])
    slabs.step_loop(e, slabs.HaloExchanger(0, 1), 1, NT - 1)
    return e.rec, e.u[(NT - 1) & 1][K:K + N[0]]


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    bounds = slabs.split_slabs(N[0], world, K)
    e = NumpyEngine(*bounds[rank])
    slabs.step_loop(e, slabs.HaloExchanger(rank, world), 1, NT - 1)
    rec = torch.from_numpy(e.rec.copy())
    dist.all_reduce(rec)  # non-owners hold zeros: the sum is the record
    field = torch.zeros(N, dtype=torch.float64)
    field[bounds[rank][0]:bounds[rank][1]] = torch.from_numpy(e.u[(NT - 1) & 1][K:K + e.n0])
    dist.all_reduce(field)
    if rank == 0:
        np.save(out + "_rec.npy", rec.numpy())
        np.save(out + "_u.npy", field.numpy())
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2, 3])
def test_decomposed_run_equals_serial_run(tmp_path, world):
    out = str(tmp_path / "slab")
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    rec, u = serial_run()
    assert np.abs(rec).max() > 0
    assert np.array_equal(np.load(out + "_rec.npy"), rec)
    assert np.array_equal(np.load(out + "_u.npy"), u)


def test_split_slabs_and_ownership():
    b = slabs.split_slabs(592, 8, 4)
    assert b[0] == (0, 74) and b[-1] == (518, 592) and all(h - l == 74 for l, h in b)
    b = slabs.split_slabs(23, 3, 2)
    assert [h - l for l, h in b] == [8, 8, 7] and b[0][0] == 0 and b[-1][1] == 23
    assert slabs.owner_of_plane(b, 7) == 0 and slabs.owner_of_plane(b, 8) == 1
    assert slabs.neighbours(0, 3) == (None, 1) and slabs.neighbours(2, 3) == (1, None)
    with pytest.raises(ValueError):
        slabs.split_slabs(20, 4, 4)  # 5-plane slabs cannot hold two 4-plane boundary groups
    with pytest.raises(ValueError):
        slabs.owner_of_plane(b, 23)


# ---- the two-pass (TTI) protocol: one extra exchange of the intermediate per step ----------

D1 = np.array([0.0, 2.0 / 3.0, -1.0 / 12.0])   # order-4 first-derivative weights


class TwoPassEngine:
    """Numpy stand-in with the dependency structure of the TTI operator: pass 1 makes
    g = a * D0 f from two fields (needs their ghost planes), pass 2 differentiates g along
    d0 again (needs ITS ghost planes) and updates both fields in place; injection into both."""

    def __init__(self, lo, hi):
        self.lo, self.hi, self.n0 = lo, hi, hi - lo
        shape = (self.n0 + 2 * K, N[1], N[2])
        self.f = {k: [np.zeros(shape), np.zeros(shape)] for k in ("p", "r")}
        self.g = {k: np.zeros(shape) for k in ("p", "r")}
        rng = np.random.default_rng(5)
        self.a = 0.5 + rng.random(N)
        self.c = 0.02 + 0.01 * rng.random(N)
        self.src_cell = (11, 4, 5)
        self.src = np.sin(0.7 * np.arange(NT))
        self.rec_base = [(z, 4, 5) for z in range(0, N[0] - 1)]   # the source's column
        self.rec = np.zeros((NT, len(self.rec_base)))
        self.log = []

    boundary = interior = staticmethod(contextlib.nullcontext)
    _planes = NumpyEngine._planes

    def join(self, first, then):
        self.log.append((first, then))

    def rot(self, t):
        for k in ("p", "r"):
            cur = self.f[k][t & 1]
            for z in range(self.n0):
                c = z + K
                d = sum(D1[j] * (cur[c + j] - cur[c - j]) for j in (1, 2))
                self.g[k][c] = self.a[self.lo + z] * d

    def update(self, part, t):
        for z in self._planes(part):
            c = z + K
            hz = {k: sum(D1[j] * (self.g[k][c + j] - self.g[k][c - j]) for j in (1, 2)) for k in ("p", "r")}
            for k, mix in (("p", hz["p"] + 0.5 * hz["r"]), ("r", 0.5 * hz["p"] + hz["r"])):
                cur, new = self.f[k][t & 1], self.f[k][(t + 1) & 1]
                new[c] = 2 * cur[c] + self.c[self.lo + z] * mix - new[c]
        if part != "low":   # "high" carries the point work of both boundary groups
            z = self.src_cell[0] - self.lo
            planes = (list(self._planes("interior")) if part == "interior"
                      else list(self._planes("low")) + list(self._planes("high")))
            if z in planes:
                for k in ("p", "r"):
                    self.f[k][(t + 1) & 1][z + K, self.src_cell[1], self.src_cell[2]] += self.src[t]
        if part == "interior":
            cur = self.f["p"][t & 1]
            for i, (z, y, x) in enumerate(self.rec_base):
                if self.lo <= z < self.hi:
                    c = z - self.lo + K
                    self.rec[t, i] = 0.4 * cur[c, y, x] + 0.6 * cur[c + 1, y, x]

    def blocks(self, which, t):
        u = self.g[which[2:]] if which.startswith("g_") else self.f[which][(t + 1) & 1]
        n0 = self.n0
        f = torch.from_numpy
        return f(u[K:2 * K]), f(u[n0:n0 + K]), f(u[0:K]), f(u[n0 + K:n0 + 2 * K])


def _two_pass_result(e):
    return e.rec, e.f["p"][(NT - 1) & 1][K:K + e.n0], e.f["r"][(NT - 1) & 1][K:K + e.n0]


def _tti_worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    bounds = slabs.split_slabs(N[0], world, K)
    e = TwoPassEngine(*bounds[rank])
    slabs.tti_step_loop(e, slabs.HaloExchanger(rank, world), 1, NT - 1)
    rec, p, r = _two_pass_result(e)
    rec = torch.from_numpy(rec.copy())
    dist.all_reduce(rec)
    fields = torch.zeros((2,) + N, dtype=torch.float64)
    fields[0, bounds[rank][0]:bounds[rank][1]] = torch.from_numpy(p)
    fields[1, bounds[rank][0]:bounds[rank][1]] = torch.from_numpy(r)
    dist.all_reduce(fields)
    if rank == 0:
        np.save(out + "_rec.npy", rec.numpy())
        np.save(out + "_f.npy", fields.numpy())
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_two_pass_protocol_equals_serial_run(tmp_path, world):
    out = str(tmp_path / "tti")
    mp.spawn(_tti_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    e = TwoPassEngine(0, N[0])
    slabs.tti_step_loop(e, slabs.HaloExchanger(0, 1), 1, NT - 1)
    rec, p, r = _two_pass_result(e)
    assert np.abs(rec).max() > 0 and np.abs(r).max() > 0
    assert np.array_equal(np.load(out + "_rec.npy"), rec)
    f = np.load(out + "_f.npy")
    assert np.array_equal(f[0], p) and np.array_equal(f[1], r)
    # every step joins the streams in both directions (pass 1 + exchange before the
    # boundary update; the received ghost planes before the next pass 1)
    assert e.log[:2] == [("interior", "boundary"), ("boundary", "interior")]
