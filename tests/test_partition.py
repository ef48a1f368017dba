"""Domain decomposition host logic (CPU): partition, ghost layers, exchange maps,
D4 self-consistency, and a world_size-2 gloo run of the halo exchanges and
distributed reductions the multi-GPU path performs."""

import os
import socket

import numpy as np
import pytest

from oracle.solver import OracleSolver, roe_jacobian
from paper_2304_09485_b200.mesh import generate_box_mesh
from paper_2304_09485_b200.meshgen import generate_sphere_mesh
from paper_2304_09485_b200.partition import (LocalMesh, build_domains, partition_cells, stencil_closure_ok)
from paper_2304_09485_b200.stencils import build_stencils


def meshes():
    return {
        "tet4p": generate_box_mesh((1, 1, 1), (4, 4, 4), split="tet", periodic=("x", "y", "z")),
        "tet4j": generate_box_mesh((1, 1, 1), (4, 4, 4), split="tet", perturb=0.15, seed=3),
        "sphere": generate_sphere_mesh(2, far=4.0, nr=5),
    }


@pytest.fixture(scope="module", params=["tet4p", "tet4j", "sphere"])
def mesh(request):
    return meshes()[request.param]


@pytest.mark.parametrize("nparts", [2, 3, 4])
def test_partition_balanced_and_complete(mesh, nparts):
    part = partition_cells(mesh, nparts)
    counts = np.bincount(part, minlength=nparts)
    assert counts.sum() == mesh.ncells and counts.max() - counts.min() <= 1


@pytest.mark.parametrize("layers", [2, 3])
def test_ghost_maps_self_consistent(mesh, layers):
    part = partition_cells(mesh, 3)
    doms, g2l = build_domains(mesh, part, layers)
    st = build_stencils(mesh)
    union = np.zeros(mesh.ncells, dtype=np.int64)
    for d in doms:
        union[d.cells[: d.n_owned]] += 1
        assert np.all(part[d.cells[: d.n_owned]] == d.rank)
        # every face of an owned cell is local with both cells local
        LocalMesh(mesh, d, g2l[d.rank])
        if layers == 3:
            assert stencil_closure_ok(st, d, g2l[d.rank])
        # exchange maps: what s sends is exactly what r receives (global ids)
        for peer, recv in d.q_recv.items():
            sent = doms[peer].q_send[d.rank]
            assert np.array_equal(doms[peer].cells[sent], d.cells[recv])
            assert np.all(doms[peer].owner_rank[sent] == peer)
        for peer, recv in d.x_recv.items():
            assert np.all(recv < d.n_recon)
    assert np.all(union == 1)


def test_owned_residual_depends_only_on_local_cells(mesh):
    """Replacing every non-local cell state by another valid state leaves the
    owned-cell residual bit-identical (the local set is closed)."""
    from paper_2304_09485_b200.boundary import PatchSpec
    from paper_2304_09485_b200.kinetic import primitive_to_conserved

    ref = np.array([1.0, 0.4, 0.05, -0.02, 1 / 1.4])
    patches = {"sphere": PatchSpec("sphere", "wall_slip_adiabatic")}
    for n in mesh.patch_names:
        patches.setdefault(n, PatchSpec(n, "farfield_riemann", reference=ref))
    o = OracleSolver(mesh, patches=patches)
    rng = np.random.default_rng(1)
    w = np.tile([1.0, 0.4, 0.05, -0.02, 0.7], (mesh.ncells, 1))
    w *= 1 + 0.02 * rng.normal(size=w.shape)
    q = primitive_to_conserved(w)
    dt = o.local_dt(q)
    full, _ = o.residual(q, None, dt)
    A_full = roe_jacobian(mesh, q, dt, o.ghosts(q))
    x = rng.normal(size=q.shape)
    y_full = A_full.mv(x)
    part = partition_cells(mesh, 2)
    doms, g2l = build_domains(mesh, part, 3)
    for d in doms:
        local = np.zeros(mesh.ncells, dtype=bool)
        local[d.cells] = True
        q2 = q.copy()
        q2[~local] = primitive_to_conserved(np.array([0.9, -0.1, 0.2, 0.0, 0.6]))
        dt2 = dt.copy()
        dt2[~local] = 1e-3
        res2, _ = o.residual(q2, None, dt2)
        own = d.cells[: d.n_owned]
        assert np.array_equal(res2[own], full[own])
        # spmv rows of owned cells only need x on layer-1 ghosts
        x2 = x.copy()
        far = np.ones(mesh.ncells, dtype=bool)
        far[d.cells[: d.n_recon]] = False
        x2[far] = 7.0
        assert np.array_equal(A_full.mv(x2)[own], y_full[own])


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mesh = generate_box_mesh((1, 1, 1), (4, 4, 4), split="tet", perturb=0.1, seed=5)
        part = partition_cells(mesh, world)
        doms, g2l = build_domains(mesh, part, 3)
        d = doms[rank]
        rng = np.random.default_rng(7)
        qg = rng.normal(size=(mesh.ncells, 5))
        # local state: owned cells filled, ghosts garbage, then the halo exchange
        ql = np.full((d.n_local, 5), np.nan)
        ql[: d.n_owned] = qg[d.cells[: d.n_owned]]

        def exchange(arr, send, recv):
            reqs = []
            bufs = {}
            for peer, ids in sorted(send.items()):
                reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(arr[ids])), dst=peer))
            for peer, ids in sorted(recv.items()):
                bufs[peer] = torch.empty((len(ids),) + arr.shape[1:], dtype=torch.float64)
                reqs.append(dist.irecv(bufs[peer], src=peer))
            for r in reqs:
                r.wait()
            for peer, ids in recv.items():
                arr[ids] = bufs[peer].numpy()

        exchange(ql, d.q_send, d.q_recv)
        ok_q = bool(np.array_equal(ql, qg[d.cells]))
        # distributed dot product == global
        loc = torch.tensor([float(np.sum(ql[: d.n_owned] * ql[: d.n_owned]))], dtype=torch.float64)
        dist.all_reduce(loc)
        ok_dot = abs(loc.item() - float(np.sum(qg * qg))) <= 1e-12 * float(np.sum(qg * qg))
        # layer-1 exchange for Krylov vectors
        xl = np.full((d.n_local, 5), np.nan)
        xl[: d.n_owned] = qg[d.cells[: d.n_owned]]
        exchange(xl, d.x_send, d.x_recv)
        ok_x = bool(np.array_equal(xl[: d.n_recon], qg[d.cells[: d.n_recon]]))
        res = torch.tensor([float(ok_q and ok_dot and ok_x)], dtype=torch.float64)
        dist.all_reduce(res, op=dist.ReduceOp.MIN)
        out.put((rank, res.item(), ok_q, ok_dot, ok_x))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_halo_and_reductions():
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(r[1] == 1.0 for r in results), results
