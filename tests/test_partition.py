"""Domain decomposition host logic (CPU): canonical order, partition,
ghost layers, exchange maps, per-rank native setup (bit-identical to the
global build), the partition-invariant reduction fold, and world_size-2 gloo
runs in which every rank builds only its own domain."""

import os
import socket

import numpy as np
import pytest

from oracle.solver import OracleSolver, roe_jacobian
from paper_2304_09485_b200.mesh import generate_box_mesh
from paper_2304_09485_b200.meshgen import generate_sphere_mesh
from paper_2304_09485_b200.partition import (Decomposition, LocalMesh, SetupMesh, build_domain, build_domains,
                                             canonical_order, partition_bounds, reduction_granule,
                                             stencil_closure_ok)
from paper_2304_09485_b200.stencils import build_stencils

import _fold


def meshes():
    return {
        "tet12p": generate_box_mesh((1, 1, 1), (12, 12, 12), split="tet", periodic=("x", "y", "z")),
        "tet10j": generate_box_mesh((1, 1, 1), (10, 10, 10), split="tet", perturb=0.15, seed=3),
        "sphere": generate_sphere_mesh(3, far=4.0, nr=6),
    }


_MESHES = {}


@pytest.fixture(scope="module", params=["tet12p", "tet10j", "sphere"])
def mesh(request):
    if not _MESHES:
        _MESHES.update(meshes())
    return _MESHES[request.param]


def test_granule_matches_library():
    from paper_2304_09485_b200 import _native as N

    lib = N.load()
    for nc in (1, 767, 768, 5000, 786432, 786433, 10_000_000):
        assert lib.gks_reduction_granularity(nc) == reduction_granule(nc) == 768 * _fold.group_segments(nc)


@pytest.mark.parametrize("nranks", [1, 2, 3, 4])
def test_partition_aligned_complete_rcb(mesh, nranks):
    canon = canonical_order(mesh)
    assert np.array_equal(np.sort(canon.perm), np.arange(mesh.ncells))
    b = partition_bounds(canon, nranks)
    g = reduction_granule(mesh.ncells)
    assert b[0] == 0 and b[-1] == mesh.ncells and np.all(np.diff(b) > 0)
    assert np.all(b[:-1] % g == 0)
    dec = Decomposition.build(mesh, nranks, canon)
    counts = np.bincount(dec.part, minlength=nranks)
    assert np.array_equal(counts, np.diff(b))
    if nranks in (2, 4):
        # power-of-two ranks: exactly the RCB parts (spatially separated along one axis at level 1)
        assert list(b) == canon.levels[nranks.bit_length() - 1]
        if nranks == 2:
            c0 = mesh.cell_centroid[dec.part == 0]
            c1 = mesh.cell_centroid[dec.part == 1]
            ax = int(np.argmax(mesh.cell_centroid.max(0) - mesh.cell_centroid.min(0)))
            assert c0[:, ax].max() <= c1[:, ax].min() or c1[:, ax].max() <= c0[:, ax].min()


@pytest.mark.parametrize("layers", [2, 3])
def test_ghost_maps_self_consistent(mesh, layers):
    dec = Decomposition.build(mesh, 3)
    doms = build_domains(mesh, dec, layers)
    st = build_stencils(mesh)
    union = np.zeros(mesh.ncells, dtype=np.int64)
    for d in doms:
        union[d.cells[: d.n_owned]] += 1
        assert np.all(dec.part[d.cells[: d.n_owned]] == d.rank)
        # owned cells are the rank's contiguous canonical range, in canonical order
        assert np.array_equal(dec.canon.pos[d.cells[: d.n_owned]], np.arange(dec.bounds[d.rank], dec.bounds[d.rank + 1]))
        g2l = d.g2l(mesh.ncells)
        # every face of an owned cell is local with both cells local
        LocalMesh(mesh, d, g2l)
        if layers == 3:
            assert stencil_closure_ok(st, d, g2l)
        # exchange maps: what s sends is exactly what r receives (reference ids)
        for peer, recv in d.q_recv.items():
            sent = doms[peer].q_send[d.rank]
            assert np.array_equal(doms[peer].cells[sent], d.cells[recv])
            assert np.all(doms[peer].owner_rank[sent] == peer)
        for peer, recv in d.x_recv.items():
            assert np.all(recv < d.n_recon)
            assert np.array_equal(doms[peer].cells[doms[peer].x_send[d.rank]], d.cells[recv])
    assert np.all(union == 1)


def test_local_mesh_orders_and_ranks(mesh):
    dec = Decomposition.build(mesh, 2)
    d = build_domain(mesh, dec, 1, 3)
    lm = LocalMesh(mesh, d)
    # faces sorted by local owner; face_rank / fq_rank are the reference order among local faces
    assert np.all(np.diff(lm.face_owner) >= 0)
    assert np.array_equal(np.sort(lm.face_rank), np.arange(lm.nfaces))
    assert np.all(np.diff(lm.faces[np.argsort(lm.face_rank)]) > 0)
    assert np.array_equal(np.sort(lm.fq_rank), np.arange(len(lm.fq_face)))
    assert np.all(np.diff(lm.fq_global[np.argsort(lm.fq_rank)]) > 0)
    assert np.array_equal(lm.cell_rank, d.cells)
    np.testing.assert_array_equal(lm.fq_point, mesh.fq_point[lm.fq_global])


def test_per_rank_setup_bit_identical_to_global(mesh):
    """Stencils and operators of every reconstructed cell, built from the
    rank's own cells (SetupMesh), equal the global build bit for bit."""
    from paper_2304_09485_b200 import _native as N

    gs = N.NativeSetup(mesh, schemes=3)
    dec = Decomposition.build(mesh, 3)
    for r in range(3):
        d = build_domain(mesh, dec, r, 3)
        sm = SetupMesh(mesh, d)
        ls = N.NativeSetup(sm, schemes=3)
        rc = d.cells[: d.n_recon]
        sub = sm.local_to_sub[: d.n_recon]
        for name in ("avg0", "beta_mat", "weno_big_degree", "weno_sub_active", "hweno_big_degree",
                     "hweno_sub_active", "weno_fallback", "hweno_fallback", "hweno_big_ncols"):
            assert np.array_equal(gs.array(name)[rc], ls.array(name)[sub]), name
        for op, gather in (("weno_big_op", "weno_big_gather"), ("hweno_big_grad_scale", "hweno_big_grad_gather")):
            a, b = gs.array(op)[rc], ls.array(op)[sub]
            w = min(a.shape[-1], b.shape[-1])  # widths are padded to each build's maximum
            assert np.array_equal(a[..., :w], b[..., :w]) and not np.any(a[..., w:]) and not np.any(b[..., w:]), op
            ga, gb = gs.array(gather)[rc][:, :w], ls.array(gather)[sub][:, :w]
            used = np.any(a[..., :w] != 0, axis=tuple(range(1, a.ndim - 1))) if a.ndim > 2 else a[..., :w] != 0
            ref_b = d.cells[sm.sub_to_local[gb]]
            assert np.array_equal(ga[used], ref_b[used]), gather
        a, b = gs.array("weno_sub_op")[rc], ls.array("weno_sub_op")[sub]
        m, s = min(a.shape[1], b.shape[1]), min(a.shape[3], b.shape[3])
        assert np.array_equal(a[:, :m, :, :s], b[:, :m, :, :s])
        ga, gb = gs.array("weno_sub_gather")[rc][:, :m, :s], ls.array("weno_sub_gather")[sub][:, :m, :s]
        act = gs.array("weno_sub_active")[rc][:, :m].astype(bool)
        assert np.array_equal(ga[act], d.cells[sm.sub_to_local[gb]][act])
        a, b = gs.array("hweno_big_op")[rc], ls.array("hweno_big_op")[sub]
        assert a.shape == b.shape and np.array_equal(a, b)


def test_owned_residual_depends_only_on_local_cells():
    """Replacing every non-local cell state by another valid state leaves the
    owned-cell residual bit-identical (the local set is closed)."""
    from paper_2304_09485_b200.boundary import PatchSpec
    from paper_2304_09485_b200.kinetic import primitive_to_conserved

    mesh = generate_sphere_mesh(2, far=4.0, nr=8)
    ref = np.array([1.0, 0.4, 0.05, -0.02, 1 / 1.4])
    patches = {"sphere": PatchSpec("sphere", "wall_slip_adiabatic"),
               "farfield": PatchSpec("farfield", "farfield_riemann", reference=ref)}
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
    dec = Decomposition.build(mesh, 2)
    for d in build_domains(mesh, dec, 3):
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


def test_fold_partition_invariant():
    """The reduction tree of the device, restated in numpy: summing the group
    partials of any partition into whole groups reproduces the 1-rank sum
    bit for bit (and it is a good sum)."""
    rng = np.random.default_rng(5)
    for nc in (1000, 23040, 800_000):
        x = rng.normal(size=(nc, 5)) * np.exp(rng.normal(size=(nc, 1)) * 3)
        y = rng.normal(size=(nc, 5))
        p = (x * y).ravel()
        one = _fold.total(_fold.cell_sum(p, 5, nc), nc)
        gcells = 768 * _fold.group_segments(nc)
        ngr = -(-nc // gcells)
        for nranks in (2, 3, 5):
            if nranks > ngr:
                continue
            b = [min(nc, round(r * ngr / nranks) * gcells) for r in range(nranks)] + [nc]
            groups = {}
            for r in range(nranks):
                groups.update(_fold.cell_sum(p[b[r] * 5:b[r + 1] * 5], 5, nc, b[r]))
            assert _fold.total(groups, nc) == one
        assert abs(one - float(np.sum(p))) <= 1e-12 * float(np.sum(np.abs(p)))


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
        mesh = generate_box_mesh((1, 1, 1), (10, 10, 10), split="tet", perturb=0.1, seed=5)
        dec = Decomposition.build(mesh, world)
        d = build_domain(mesh, dec, rank, 3)  # this rank only: maps derived locally
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
        # distributed dot: group partials of the owned rows, exchanged (sum of
        # zero-padded arrays, exact), then the common final fold == 1-rank fold
        nc = mesh.ncells
        ng = -(-nc // (768 * _fold.group_segments(nc)))
        mine = _fold.cell_sum((ql[: d.n_owned] * ql[: d.n_owned]).ravel(), 5, nc, d.owned_offset)
        arr = torch.zeros(ng, dtype=torch.float64)
        for k, v in mine.items():
            arr[k] = v
        dist.all_reduce(arr)
        tot = _fold.fold(arr.numpy())
        canon_q = qg[dec.canon.perm]
        one = _fold.dot(canon_q, canon_q)
        ok_dot = tot == one
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
    results = [q.get(timeout=180) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(r[1] == 1.0 for r in results), results
