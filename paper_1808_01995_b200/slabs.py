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
        steps = range(t_to - 1, t_from - 1, -1) if backward else range(t_from, t_to)
        for t in steps:
            self.plan.step_slab_boundary(self.op, t)
            self.plan.step_slab_interior(self.op, t)
            self.plan.peer_wait_ipc()


def bench_distributed(args, K, W, build_workload, workload_config, bytes_per_point, peaks):
    """bench.py at N > 1: configs[1] cut into N slabs (strong scaling), NCCL halo exchange,
    device time = max over ranks between barriers."""
    import torch
    import torch.distributed as dist
    from . import capi
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    # NCCL prints its version banner on stdout; the contract is ONE JSON line there, so
    # stdout is parked on stderr until the line is ready
    import sys
    sys.stdout.flush()
    saved_stdout = os.dup(1)
    os.dup2(2, 1)
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29577")
    dist.init_process_group("nccl", rank=rank, world_size=world,
                            device_id=torch.device(f"cuda:{local}"))
    cfg, model, geom = build_workload(W + K)
    N = model.grid.shape
    order = model.space_order
    bounds = split_slabs(N[0], world, order // 2)
    plan = capi.Plan(N, model.grid.spacing, order, geom.dt, geom.nt, local, bounds[rank])
    plan.set_model(model.m.array(), model.damp.array(), model.v_max)
    plan.set_points(capi.CLOUD_SRC, np.array(geom.src.base_table).reshape(-1, 3),
                    np.array(geom.src.weight_table).reshape(-1, 8))
    plan.set_points(capi.CLOUD_REC, np.array(geom.rec.base_table).reshape(-1, 3),
                    np.array(geom.rec.weight_table).reshape(-1, 8))
    plan.upload_traces(capi.CLOUD_SRC, geom.src.traces)
    eng = PlanEngine(plan, capi.OP_FORWARD, local)
    ex = HaloExchanger(rank, world)
    # the exchange: fused halo push over peer memory (default), NCCL send/recv as the fallback
    halo = "nccl send/recv"
    loop = lambda a, b: step_loop(eng, ex, a, b)   # noqa: E731
    if world > 1 and os.environ.get("SFB_HALO", "push") == "push":
        try:
            drv = PeerPushDriver(plan, capi.OP_FORWARD, rank, world)
            loop = drv.run
            halo = "fused peer push (CUDA IPC stores from the boundary kernels)"
        except RuntimeError as e:
            if rank == 0:
                print(f"[bench] {e}; falling back to NCCL send/recv", file=sys.stderr)
    plan.step_begin(capi.OP_FORWARD)
    torch.cuda.synchronize()
    dist.barrier()   # nobody pushes into a neighbour that is still zeroing its fields
    loop(1, 1 + W)
    torch.cuda.synchronize()
    launches0 = plan.launch_count()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    eng.s_main.wait_stream(eng.s_bnd)
    with torch.cuda.stream(eng.s_main):
        e0.record()
    eng.s_bnd.wait_stream(eng.s_main)
    loop(1 + W, 1 + W + K)
    eng.s_main.wait_stream(eng.s_bnd)
    with torch.cuda.stream(eng.s_main):
        e1.record()
    torch.cuda.synchronize()
    dist.barrier()
    ms = torch.tensor([e0.elapsed_time(e1)], device=f"cuda:{local}")
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    plan.step_end(capi.OP_FORWARD)
    pts = float(np.prod(N))
    sec = float(ms.item()) * 1e-3
    sys.stdout.flush()
    os.dup2(saved_stdout, 1)
    os.close(saved_stdout)
    if rank == 0:
        peak, kind = peaks()
        line = {
            "metric": "acoustic_forward_gpts_per_s", "value": pts * K / sec / 1e9,
            "unit": "GPts/s", "n_gpus": world, "steps": K, "warmup": W,
            "ms_per_step": sec / K * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": workload_config(world),
            "roofline": {"bound": "hbm", "achieved": bytes_per_point * pts * K / sec / 1e9 / world,
                         "peak": peak, "unit": "GB/s",
                         "frac": bytes_per_point * pts * K / sec / 1e9 / world / peak,
                         "traffic": None, "peak_kind": kind,
                         "note": "per-GPU figure of the whole step (update + exchange)"},
            "cpu_baseline": None,
            "e2e": None,
            "gpu_launches": int(plan.launch_count() - launches0),
            "halo_bytes_per_step_per_neighbour": int(plan.halo_blocks(capi.OP_FORWARD, 1)["count"] * 4),
            "halo": halo,
        }
        print(json.dumps(line), flush=True)
    plan.close()
    dist.destroy_process_group()
