"""The fused halo push between PROCESSES (CUDA IPC + stream memory operations): two ranks,
each with its own CUDA context and one slab plan -- both on cuda:0 here, which CUDA IPC
allows -- reproduce the single-domain forward run bit for bit.  torch.distributed (gloo) only
carries the IPC blobs and the final gather."""
import os
import socket

import numpy as np
import pytest

from tests.common import make_plan, make_problem

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(300)]

SHAPE, ORDER, NSTEPS = [44, 30, 34], 8, 40


def _worker(rank, world, port, out, streamed=False):
    import torch
    import torch.distributed as dist
    from paper_1808_01995_b200 import capi, slabs
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    model, geom = make_problem(SHAPE, 10.0, 8, ORDER, NSTEPS)
    bounds = slabs.split_slabs(model.N[0], world, ORDER // 2)
    plan = make_plan(model, geom, ORDER, slab=bounds[rank])
    plan.upload_traces(capi.CLOUD_SRC, geom.src)
    drv = slabs.PeerPushDriver(plan, capi.OP_FORWARD, rank, world)
    plan.step_begin(capi.OP_FORWARD)
    dist.barrier()   # nobody pushes into a neighbour that is still zeroing its fields
    if streamed:   # the loop inside the library, sampled rows streaming into the host table
        table = np.full((geom.nt, geom.n_rec), np.nan)
        drv.run_tables(1, geom.nt - 1, smp=table)
        plan.step_end(capi.OP_FORWARD)
        assert np.array_equal(table, plan.download_traces(capi.CLOUD_REC))
        rec = torch.from_numpy(table)
    else:
        drv.run(1, geom.nt - 1)
        plan.step_end(capi.OP_FORWARD)
        rec = torch.from_numpy(plan.download_traces(capi.CLOUD_REC))
    u = np.zeros(model.N)
    plan.wavefield(geom.nt - 1, out=u)
    u = torch.from_numpy(u)
    dist.all_reduce(rec)
    dist.all_reduce(u)
    dist.barrier()   # keep every mapping alive until all ranks are done
    if rank == 0:
        np.save(out + "_rec.npy", rec.numpy())
        np.save(out + "_u.npy", u.numpy())
    plan.close()
    dist.destroy_process_group()


def _adjoint_data(geom):
    rng = np.random.default_rng(21)
    data = rng.standard_normal((geom.nt, geom.n_rec)) * np.hanning(geom.nt)[:, None]
    data[[0, geom.nt - 1]] = 0.0
    return data


def _adjoint_worker(rank, world, port, out):
    """the backward sweep of each rank as one sfb_slab_run: receiver table fed while it runs,
    source-side trace streamed out"""
    import torch
    import torch.distributed as dist
    from paper_1808_01995_b200 import capi, slabs
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    model, geom = make_problem(SHAPE, 10.0, 8, ORDER, NSTEPS)
    data = _adjoint_data(geom)
    bounds = slabs.split_slabs(model.N[0], world, ORDER // 2)
    plan = make_plan(model, geom, ORDER, slab=bounds[rank])
    drv = slabs.PeerPushDriver(plan, capi.OP_ADJOINT, rank, world)
    plan.step_begin(capi.OP_ADJOINT)
    plan.sync()
    dist.barrier()
    table = np.full((geom.nt, geom.n_src), np.nan)
    drv.run_tables(1, geom.nt - 1, inj=data, smp=table)
    plan.step_end(capi.OP_ADJOINT)
    srca = torch.from_numpy(table)
    v = np.zeros(model.N)
    plan.wavefield(0, out=v)
    v = torch.from_numpy(v)
    dist.all_reduce(srca)
    dist.all_reduce(v)
    dist.barrier()
    if rank == 0:
        np.save(out + "_srca.npy", srca.numpy())
        np.save(out + "_v.npy", v.numpy())
    plan.close()
    dist.destroy_process_group()


def _gradient_worker(rank, world, port, out):
    """forward slab run that keeps every 2nd level, then the gradient sweep as one
    sfb_slab_run per rank with the residual table fed while it runs"""
    import ctypes as C
    import torch
    import torch.distributed as dist
    from paper_1808_01995_b200 import capi, slabs
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    model, geom = make_problem(SHAPE, 10.0, 8, ORDER, NSTEPS)
    data = _adjoint_data(geom)
    bounds = slabs.split_slabs(model.N[0], world, ORDER // 2)
    plan = make_plan(model, geom, ORDER, slab=bounds[rank])
    plan.upload_traces(capi.CLOUD_SRC, geom.src)
    drv = slabs.PeerPushDriver(plan, capi.OP_FORWARD, rank, world)
    plan.step_begin(capi.OP_FORWARD, 2)
    plan.sync()
    dist.barrier()
    drv.run(1, geom.nt - 1)
    plan.step_end(capi.OP_FORWARD)
    plan.sync()
    dist.barrier()
    drv.op = capi.OP_GRADIENT
    plan.step_begin(capi.OP_GRADIENT)
    plan.sync()
    dist.barrier()
    drv.run_tables(1, geom.nt - 1, inj=data)
    plan.step_end(capi.OP_GRADIENT)
    grad = np.zeros(model.N)
    plan._chk(capi.lib.sfb_get_gradient(plan.h, C.byref(capi._view(grad))))
    grad = torch.from_numpy(grad)
    dist.all_reduce(grad)
    dist.barrier()
    if rank == 0:
        np.save(out + "_grad.npy", grad.numpy())
    plan.close()
    dist.destroy_process_group()


def _tti_inputs():
    from tests.test_gpu_tti import tti_fields, tti_problem
    model, geom = tti_problem([44, 26, 30], 8, 30)
    return model, geom, tti_fields(model.N, seed=3)


def _tti_worker(rank, world, port, out, streamed=False):
    import torch
    import torch.distributed as dist
    from paper_1808_01995_b200 import capi, slabs
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    model, geom, fields = _tti_inputs()
    bounds = slabs.split_slabs(model.N[0], world, 4)
    plan = make_plan(model, geom, 8, slab=bounds[rank])
    plan.set_model_tti(*fields)
    plan.upload_traces(capi.CLOUD_SRC, geom.src)
    drv = slabs.TtiPeerPushDriver(plan, rank, world)
    plan.step_begin(capi.OP_TTI_FORWARD)
    plan.sync()
    dist.barrier()
    if streamed:
        table = np.full((geom.nt, geom.n_rec), np.nan)
        drv.run_tables(1, geom.nt - 1, smp=table)
        plan.step_end(capi.OP_TTI_FORWARD)
        rec = torch.from_numpy(table)
    else:
        drv.run(1, geom.nt - 1)
        plan.step_end(capi.OP_TTI_FORWARD)
        rec = torch.from_numpy(plan.download_traces(capi.CLOUD_REC))
    p, r = np.zeros(model.N), np.zeros(model.N)
    plan.wavefield(geom.nt - 1, out=p, field=0)
    plan.wavefield(geom.nt - 1, out=r, field=1)
    p, r = torch.from_numpy(p), torch.from_numpy(r)
    for x in (rec, p, r):
        dist.all_reduce(x)
    dist.barrier()
    if rank == 0:
        np.save(out + "_rec.npy", rec.numpy())
        np.save(out + "_p.npy", p.numpy())
        np.save(out + "_r.npy", r.numpy())
    plan.close()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world,streamed", [(2, False), (3, False), (3, True)])
def test_peer_push_between_processes_matches_single_domain(tmp_path, world, streamed):
    import torch.multiprocessing as mp
    model, geom = make_problem(SHAPE, 10.0, 8, ORDER, NSTEPS)
    plan = make_plan(model, geom, ORDER)
    rec1, _ = plan.forward(geom.src)
    u1 = plan.wavefield(geom.nt - 1)
    plan.close()
    out = str(tmp_path / "ipc")
    mp.spawn(_worker, args=(world, _free_port(), out, streamed), nprocs=world, join=True)
    assert np.abs(rec1).max() > 0
    assert np.array_equal(np.load(out + "_rec.npy"), rec1)
    assert np.array_equal(np.load(out + "_u.npy"), u1)


@pytest.mark.parametrize("world,streamed", [(2, False), (3, False), (2, True)])
def test_tti_peer_push_between_processes_matches_single_domain(tmp_path, world, streamed):
    import torch.multiprocessing as mp
    model, geom, fields = _tti_inputs()
    plan = make_plan(model, geom, 8)
    plan.set_model_tti(*fields)
    rec1, _ = plan.tti_forward(geom.src)
    p1 = plan.wavefield(geom.nt - 1, field=0)
    r1 = plan.wavefield(geom.nt - 1, field=1)
    plan.close()
    out = str(tmp_path / "ipc_tti")
    mp.spawn(_tti_worker, args=(world, _free_port(), out, streamed), nprocs=world, join=True)
    assert np.abs(rec1).max() > 0
    assert np.array_equal(np.load(out + "_rec.npy"), rec1)
    assert np.array_equal(np.load(out + "_p.npy"), p1) and np.array_equal(np.load(out + "_r.npy"), r1)


def test_adjoint_sweep_with_streamed_tables_between_processes(tmp_path):
    import torch.multiprocessing as mp
    model, geom = make_problem(SHAPE, 10.0, 8, ORDER, NSTEPS)
    data = _adjoint_data(geom)
    plan = make_plan(model, geom, ORDER)
    srca1, _ = plan.adjoint(data)
    v1 = plan.wavefield(0)
    plan.close()
    out = str(tmp_path / "ipc_adj")
    mp.spawn(_adjoint_worker, args=(3, _free_port(), out), nprocs=3, join=True)
    assert np.abs(srca1).max() > 0
    assert np.array_equal(np.load(out + "_srca.npy"), srca1)
    assert np.array_equal(np.load(out + "_v.npy"), v1)


def test_gradient_sweep_between_processes_matches_single_domain(tmp_path):
    import torch.multiprocessing as mp
    model, geom = make_problem(SHAPE, 10.0, 8, ORDER, NSTEPS)
    data = _adjoint_data(geom)
    plan = make_plan(model, geom, ORDER)
    plan.forward(geom.src, save_every=2)
    g1, _ = plan.gradient(data)
    plan.close()
    out = str(tmp_path / "ipc_grad")
    mp.spawn(_gradient_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    assert np.abs(g1).max() > 0
    assert np.array_equal(np.load(out + "_grad.npy"), g1)
