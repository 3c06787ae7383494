"""Slab domain decomposition across the GPUs of one box.

One process per GPU.  The slowest axis d0 of the padded grid is cut into contiguous slabs;
each rank owns one slab plus K = space_order/2 ghost planes per side and, every time step,
ships its K boundary planes to each neighbour (torch.distributed isend/irecv: NCCL over
NVLink on GPUs, gloo in the CPU tests).  There is no other communication on the path: no
all-reduce, no gather inside the loop.  The reference has no counterpart (it is a single
address space); the protocol below is what keeps the decomposed run
bit-identical to the single-domain one:

    step t:   boundary stream : update LOW planes, update HIGH planes, scatter into them
              exchange        : send boundary planes of level t+1, receive ghost planes
              main stream     : update INTERIOR planes, scatter into them, gather level t

A node is injected by the rank that owns its plane (before that plane is shipped); a point
is sampled by the rank that owns its base plane, reading its ghost plane when the cell
straddles the cut.  Sampled traces are zero on non-owners, so the global record is the sum
over ranks.
"""
from __future__ import annotations

import json
import os
import time

import numpy as np


def split_slabs(n0: int, world: int, halo: int):
    """Balanced contiguous split of [0, n0) into `world` slabs; every slab must hold at
    least 2*halo planes (a slab's two boundary groups may not overlap)."""
    if world < 1 or n0 < 1:
        raise ValueError("bad decomposition request")
    base, extra = divmod(n0, world)
    bounds, lo = [], 0
    for r in range(world):
        hi = lo + base + (1 if r < extra else 0)
        bounds.append((lo, hi))
        lo = hi
    if world > 1 and min(h - l for l, h in bounds) < 2 * halo:
        raise ValueError(f"slabs of {base} planes are thinner than 2*{halo} halo planes")
    return bounds


def neighbours(rank: int, world: int):
    """(rank owning the planes below, rank owning the planes above); None at outer faces,
    which keep the zero (Dirichlet) ghost planes."""
    return (rank - 1 if rank > 0 else None, rank + 1 if rank < world - 1 else None)


def owner_of_plane(bounds, z: int) -> int:
    for r, (lo, hi) in enumerate(bounds):
        if lo <= z < hi:
            return r
    raise ValueError(f"plane {z} outside the grid")


class HaloExchanger:
    """Neighbour exchange of the four ghost/boundary blocks of one time level."""

    def __init__(self, rank: int, world: int, group=None):
        self.rank, self.world, self.group = rank, world, group
        self.lo, self.hi = neighbours(rank, world)
        self.dist = None
        if world > 1:
            import torch.distributed as dist
            self.dist = dist

    def start(self, send_lo, send_hi, recv_lo, recv_hi):
        """Post all sends/receives of this step; returns the outstanding requests."""
        if self.lo is None and self.hi is None:
            return []
        d = self.dist
        ops = []
        if self.lo is not None:
            ops.append(d.P2POp(d.isend, send_lo, self.lo, self.group))
            ops.append(d.P2POp(d.irecv, recv_lo, self.lo, self.group))
        if self.hi is not None:
            ops.append(d.P2POp(d.isend, send_hi, self.hi, self.group))
            ops.append(d.P2POp(d.irecv, recv_hi, self.hi, self.group))
        return d.batch_isend_irecv(ops) if ops else []

    @staticmethod
    def finish(reqs):
        for r in reqs:
            r.wait()


def step_loop(engine, exchanger: HaloExchanger, t_from: int, t_to: int, backward=False):
    """The per-step protocol, engine-agnostic (the GPU plan below, or the numpy engine of
    tests/test_slabs_gloo.py).  `engine` provides update(part, t), scatter(part, t),
    gather(t), blocks(t) -> (send_lo, send_hi, recv_lo, recv_hi), and the context managers
    boundary() / interior() that select where the work is queued."""
    steps = range(t_to - 1, t_from - 1, -1) if backward else range(t_from, t_to)
    fused = hasattr(engine, "boundary_step")  # one native call per half step
    for t in steps:
        with engine.boundary():
            if fused:
                engine.boundary_step(t)
            else:
                engine.update("low", t)
                engine.update("high", t)
                engine.scatter("boundary", t)
            reqs = exchanger.start(*engine.blocks(t))
        with engine.interior():
            if fused:
                engine.interior_step(t)
            else:
                engine.update("interior", t)
                engine.scatter("interior", t)
                engine.gather(t)
        with engine.boundary():
            exchanger.finish(reqs)


def tti_step_loop(engine, exchanger: HaloExchanger, t_from: int, t_to: int):
    """Per-step protocol of the two-pass TTI operator (include/sfb200.h, "TTI slab
    stepping"): the second pass differentiates the intermediate a*g along d0, so its K
    boundary planes are exchanged between the passes -- SURVEY.md 8e's "extra exchange of
    the intermediate" -- and the new p and r levels are exchanged at the end of the step,
    overlapped with the interior update as in the acoustic loop.

    `engine` provides rot(t) (first pass on every owned plane: the exchange that follows
    needs all of it), update(part, t) with part in low/high/interior (update
    "high" also does the point work of both boundary groups), blocks(which, t) for which in
    ("g_p", "g_r", "p", "r"), the stream contexts boundary() / interior(), and
    join(first, then): make stream `then` wait for the work queued on `first`."""
    for t in range(t_from, t_to):
        with engine.interior():
            engine.rot(t)
            for which in ("g_p", "g_r"):
                exchanger.finish(exchanger.start(*engine.blocks(which, t)))
        engine.join("interior", "boundary")
        with engine.boundary():
            engine.update("low", t)
            engine.update("high", t)
            reqs = exchanger.start(*engine.blocks("p", t)) + exchanger.start(*engine.blocks("r", t))
        with engine.interior():
            engine.update("interior", t)
        with engine.boundary():
            exchanger.finish(reqs)
        engine.join("boundary", "interior")


class _DeviceFloats:
    """Zero-copy torch view of `count` floats at a raw device pointer."""

    def __init__(self, ptr, count):
        self.__cuda_array_interface__ = {"shape": (int(count),), "typestr": "<f4",
                                         "data": (int(ptr), False), "version": 2}


class PlanEngine:
    """step_loop engine over one capi.Plan; the plan launches on two torch streams so that
    NCCL orders against them."""

    def __init__(self, plan, op, device):
        import torch
        from . import capi
        self.torch, self.capi, self.plan, self.op, self.device = torch, capi, plan, op, device
        self.s_main = torch.cuda.Stream(device=device)
        self.s_bnd = torch.cuda.Stream(device=device, priority=-1)
        plan._chk(capi.lib.sfb_set_streams(plan.h, self.s_main.cuda_stream, self.s_bnd.cuda_stream))
        self._views = {}

    def boundary(self):
        return self.torch.cuda.stream(self.s_bnd)

    def interior(self):
        return self.torch.cuda.stream(self.s_main)

    def update(self, part, t):
        c = self.capi
        self.plan.step_compute(self.op, t, {"low": c.PART_LOW, "high": c.PART_HIGH,
                                            "interior": c.PART_INTERIOR}[part])

    def scatter(self, part, t):
        c = self.capi
        self.plan.step_points(self.op, t, c.PART_LOW if part == "boundary" else c.PART_INTERIOR)

    def gather(self, t):
        pass  # fused into the interior point launch

    def boundary_step(self, t):
        self.plan.step_slab_boundary(self.op, t)

    def interior_step(self, t):
        self.plan.step_slab_interior(self.op, t)

    def blocks(self, t):
        key = (t + 1) & 1
        if key not in self._views:
            b = self.plan.halo_blocks(self.op, t)
            dev = f"cuda:{self.device}"
            self._views[key] = tuple(
                self.torch.as_tensor(_DeviceFloats(b[k], b["count"]), device=dev)
                for k in ("send_lo", "send_hi", "recv_lo", "recv_hi"))
        return self._views[key]


class TtiPlanEngine:
    """tti_step_loop engine over one capi.Plan with the TTI fields bound."""

    def __init__(self, plan, device):
        import torch
        from . import capi
        self.torch, self.capi, self.plan, self.device = torch, capi, plan, device
        self.s_main = torch.cuda.Stream(device=device)
        self.s_bnd = torch.cuda.Stream(device=device, priority=-1)
        plan._chk(capi.lib.sfb_set_streams(plan.h, self.s_main.cuda_stream, self.s_bnd.cuda_stream))
        self._views = {}
        self._part = {"low": capi.PART_LOW, "high": capi.PART_HIGH, "interior": capi.PART_INTERIOR}
        self._which = {"g_p": capi.TTI_HALO_G_P, "g_r": capi.TTI_HALO_G_R,
                       "p": capi.TTI_HALO_P, "r": capi.TTI_HALO_R}

    def boundary(self):
        return self.torch.cuda.stream(self.s_bnd)

    def interior(self):
        return self.torch.cuda.stream(self.s_main)

    def join(self, first, then):
        a = self.s_main if first == "interior" else self.s_bnd
        b = self.s_main if then == "interior" else self.s_bnd
        b.wait_stream(a)

    def rot(self, t):
        self.plan.tti_step_rot(t, self.capi.PART_ALL)

    def update(self, part, t):
        self.plan.tti_step_update(t, self._part[part])

    def blocks(self, which, t):
        key = (which, (t + 1) & 1 if which in ("p", "r") else 0)
        if key not in self._views:
            b = self.plan.tti_halo_blocks(self._which[which], t)
            dev = f"cuda:{self.device}"
            self._views[key] = tuple(
                self.torch.as_tensor(_DeviceFloats(b[k], b["count"]), device=dev)
                for k in ("send_lo", "send_hi", "recv_lo", "recv_hi"))
        return self._views[key]


class PeerPushDriver:
    """The slab loop with the fused halo push between processes (one per GPU): instead of
    send/recv, every boundary half-step stores its planes straight into the neighbours'
    ghost planes, which are mapped through CUDA IPC; the ranks are ordered on the device by
    the plans' step counters (stream memory operations), not by the host.  torch.distributed
    is used once, to hand the IPC blobs to the neighbours."""

    def __init__(self, plan, op, rank: int, world: int, group=None):
        self.plan, self.op = plan, op
        if world > 1:
            import torch.distributed as dist
            blobs = [None] * world
            dist.all_gather_object(blobs, plan.peer_export(), group=group)
            err = None
            try:
                plan.link_peers_ipc(blobs[rank - 1] if rank > 0 else None,
                                    blobs[rank + 1] if rank < world - 1 else None)
            except Exception as e:  # e.g. no peer access between two of the devices
                err = repr(e)
            # every rank has mapped its neighbours before any push -- or nobody pushes
            errs = [None] * world
            dist.all_gather_object(errs, err, group=group)
            if any(errs):
                plan.link_peers_ipc(None, None)
                raise RuntimeError("peer linking failed on rank(s) " +
                                   ", ".join(f"{i}: {e}" for i, e in enumerate(errs) if e))

    def run(self, t_from: int, t_to: int, backward=False):
        """One update launch + one point launch per step (sfb_step_slab_fused: the first d0
        chunk sweeps up, the last one down, so both boundary plane groups are computed and
        pushed first), the whole range in one library call (sfb_slab_run);
        SFB_SLAB_PROTOCOL=split runs the boundary / interior half-steps on two streams instead
        (the protocol the NCCL fallback uses), call by call."""
        from . import capi
        assert backward == (self.op in (capi.OP_ADJOINT, capi.OP_GRADIENT))
        if os.environ.get("SFB_SLAB_PROTOCOL", "fused") != "split":
            self.plan.slab_run(self.op, t_from, t_to)   # the loop inside the library
            return
        steps = range(t_to - 1, t_from - 1, -1) if backward else range(t_from, t_to)
        for t in steps:
            self.plan.step_slab_boundary(self.op, t)
            self.plan.step_slab_interior(self.op, t)
            self.plan.peer_wait_ipc()


    def run_tables(self, t_from: int, t_to: int, inj=None, smp=None):
        """The same loop inside the library (sfb_slab_run): one call per range of steps, the
        sampled rows leave the device -- and the injected rows reach it -- while it runs."""
        return self.plan.slab_run(self.op, t_from, t_to, inj=inj, smp=smp)


class TtiPeerPushDriver(PeerPushDriver):
    """The TTI pair with the fused halo push between processes: link after
    sfb_set_model_tti (the blob then carries the handles of g(p), g(r) and r as well); each pass
    of a step is one launch per slab that pushes its boundary planes, the ranks are ordered by
    three device-side counters (first pass done / pushes landed / ghost readers done)."""

    def __init__(self, plan, rank: int, world: int, group=None):
        from . import capi
        super().__init__(plan, capi.OP_TTI_FORWARD, rank, world, group)

    def run(self, t_from: int, t_to: int, backward=False):
        assert not backward, "the TTI operator is forward-only"
        if os.environ.get("SFB_SLAB_PROTOCOL", "fused") != "percall":
            self.plan.slab_run(self.op, t_from, t_to)
            return
        for t in range(t_from, t_to):   # the same four calls per step, made from here
            self.plan.tti_step_rot_fused(t)
            self.plan.tti_peer_wait_g_ipc()
            self.plan.tti_step_update_fused(t)
            self.plan.peer_wait_ipc()


# ---- bench.py at N > 1 ----------------------------------------------------------------------

def weak_extent(per_rank: int, world: int) -> int:
    """Slab-axis extent of a weak-scaling run (BASELINE.json configs[4]: 128 physical planes
    per GPU)."""
    return per_rank * world


class Comm:
    """The few collectives the bench needs, over torch.distributed (nccl on GPUs, gloo in the
    CPU test).  None of them is on the data path."""

    def __init__(self, rank, world, device=None):
        self.rank, self.world, self.device = rank, world, device
        import torch
        self.torch = torch
        self.dist = torch.distributed if world > 1 else None

    def barrier(self):
        if self.dist:
            self.dist.barrier()

    def gather_floats(self, x):
        """every rank's value of x, on every rank"""
        if not self.dist:
            return [float(x)]
        t = self.torch.tensor([float(x)], dtype=self.torch.float64, device=self.device)
        out = [self.torch.zeros_like(t) for _ in range(self.world)]
        self.dist.all_gather(out, t)
        return [float(o.item()) for o in out]


def bench_core(comm: Comm, job, K: int, W: int):
    """The timed region of one slab benchmark, backend-agnostic: W untimed warm-up steps, then
    exactly K steps bracketed by a barrier and a device synchronisation on both sides, device
    time per rank, MAX over ranks; then the end-to-end leg (upload of the injected traces,
    K steps, download of the rank's sampled rows) by wall clock, max over ranks.

    `job` provides begin(), loop(t_from, t_to), sync(), start()/stop() -> seconds of the
    queued work on the device, points_owned, launches(), upload(), download() -> bytes moved,
    and optionally run_e2e(t_from, t_to) -> bytes moved (the loop with the sampled rows
    streaming out while it runs, instead of loop() + download()).
    Returns the measurements every rank agrees on."""
    import time as _time
    job.begin()
    job.sync()
    comm.barrier()   # nobody pushes into a neighbour that is still zeroing its fields
    job.loop(1, 1 + W)
    job.sync()
    launches0 = job.launches()
    comm.barrier()
    job.start()
    job.loop(1 + W, 1 + W + K)
    sec_rank = job.stop()
    job.sync()
    comm.barrier()
    launches = job.launches() - launches0
    per_rank = comm.gather_floats(sec_rank)
    pts = sum(comm.gather_floats(job.points_owned))
    # end to end: host buffers in, host buffers out, every copy inside the timed region; one
    # untimed pass first (pinned staging buffers, copy stream), as the one-GPU line does
    for _pass in range(2):
        comm.barrier()
        t0 = _time.perf_counter()
        h2d = job.upload()
        job.begin()
        job.sync()
        comm.barrier()   # as above: no push may land in a field its owner is still zeroing
        if hasattr(job, "run_e2e"):     # loop and table traffic in one library call per rank
            d2h = job.run_e2e(1, 1 + K)
            h2d += getattr(job, "fed", 0.0)   # injected rows fed while the loop ran
        else:
            job.loop(1, 1 + K)
            d2h = job.download()
        job.sync()
        e2e_rank = _time.perf_counter() - t0
        comm.barrier()
    e2e = comm.gather_floats(e2e_rank)
    return {"seconds": max(per_rank), "per_rank_ms_per_step": [s / K * 1e3 for s in per_rank],
            "points": pts, "launches": int(launches), "e2e_seconds": max(e2e),
            "h2d_bytes_per_step": sum(comm.gather_floats(h2d)) / K,
            "d2h_bytes_per_step": sum(comm.gather_floats(d2h)) / K}


def scaling_line(meas, *, metric, world, K, W, scaling, config, bytes_per_point, contract_bytes,
                 peak, peak_kind, halo, halo_bytes, dtype="f32", extra=None):
    """The JSON line of an N-GPU run from bench_core's measurements (rank 0 prints it)."""
    sec, pts = meas["seconds"], meas["points"]
    value = pts * K / sec / 1e9
    per_gpu_gbs = bytes_per_point * pts * K / sec / 1e9 / world
    line = {
        "metric": metric, "value": value, "unit": "GPts/s", "n_gpus": world, "steps": K,
        "warmup": W, "ms_per_step": sec / K * 1e3, "higher_is_better": True, "scaling": scaling,
        "vs_baseline": None, "dtype": dtype, "data": "synthetic", "config": config,
        "roofline": {"bound": "hbm", "achieved": per_gpu_gbs, "peak": peak, "unit": "GB/s",
                     "frac": per_gpu_gbs / peak, "traffic": None, "peak_kind": peak_kind,
                     "basis_bytes_per_point": bytes_per_point,
                     "frac_contract": contract_bytes * pts * K / sec / 1e9 / world / peak,
                     "contract_bytes_per_point": contract_bytes,
                     "note": "per-GPU figure of the whole slab step (update + point work + "
                             "exchange), not of one kernel"},
        "e2e": {"value": pts * K / meas["e2e_seconds"] / 1e9, "unit": "GPts/s",
                "h2d_bytes_per_step": meas["h2d_bytes_per_step"],
                "d2h_bytes_per_step": meas["d2h_bytes_per_step"],
                "seconds": meas["e2e_seconds"],
                "how": "per rank: upload of the injected trace table from host memory, K slab "
                       "steps, the rank's sampled rows into host memory (streamed while the loop "
                       "runs by sfb_slab_run with the fused push; downloaded after it with "
                       "send/recv); wall clock between barriers, max over ranks"},
        "gpu_launches": meas["launches"],
        "per_rank_ms_per_step": meas["per_rank_ms_per_step"],
        "halo": halo, "halo_bytes_per_step_per_neighbour": halo_bytes,
    }
    if extra:
        line.update(extra)
    return line
