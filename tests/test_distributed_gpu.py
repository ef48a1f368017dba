"""Partitioned (multi-GPU) device path on ONE GPU.

* Rank-local handles driven with their ghost layers uploaded from the global
  state (no communicator): the owned-cell residual is bitwise the global
  handle's -- pins the local meshes, the per-rank native setup (stencils and
  operators built from the rank's own cells), the owned / reconstructed
  kernel ranges and the owned-row Jacobian.
* The in-process loopback transport (csrc/gks_comm.cu) steps 2 and 4
  rank-local handles of one mesh concurrently through the real pack /
  exchange / unpack code and the group-partial reductions: their step
  histories and fields are bitwise those of the 1-rank canonical run
  (partition-invariant reductions, csrc/gks_reduce.cuh), and within 1e-10 of
  the plain single-domain Solver.
* A 1-rank NCCL communicator runs the NCCL legs (group-partial allreduce,
  captured in the step graph) bitwise against the communicator-free run.
"""

import dataclasses

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def setup_case(kind, n=3):
    from paper_2304_09485_b200.boundary import PatchSpec
    from paper_2304_09485_b200.kinetic import primitive_to_conserved
    from paper_2304_09485_b200.meshgen import generate_sphere_mesh
    from paper_2304_09485_b200.stepping import SolverOptions

    mesh = generate_sphere_mesh(n, far=4.0, nr=6) if n == 3 else generate_sphere_mesh(n)
    rng = np.random.default_rng(2)
    if kind == "c3":
        # C3 physics (cases/sphere_re118_ma0p2535.ini): viscous HWENO, no-slip wall
        ma = 0.2535
        ref = np.array([1.0, ma, 0.0, 0.0, 1 / 1.4])
        patches = {"sphere": PatchSpec("sphere", "wall_noslip_adiabatic"),
                   "farfield": PatchSpec("farfield", "farfield_riemann", reference=ref)}
        opts = SolverOptions(scheme="hweno_gmres", model="viscous", mu=0.0021483, weights="linear",
                             patches=patches)
        w = np.tile([1.0, ma, 0.0, 0.0, 0.7], (mesh.ncells, 1))
    else:
        ref = np.array([1.0, 0.5, 0.02, -0.01, 1 / 1.4])
        patches = {"sphere": PatchSpec("sphere", "wall_slip_adiabatic"),
                   "farfield": PatchSpec("farfield", "farfield_riemann", reference=ref)}
        scheme = "hweno_gmres" if kind == "hweno" else "weno_gmres"
        opts = SolverOptions(scheme=scheme, patches=patches)
        w = np.tile([1.0, 0.5, 0.02, -0.01, 0.7], (mesh.ncells, 1))
    w *= 1 + 0.02 * rng.normal(size=w.shape)
    q = primitive_to_conserved(w)
    grad = 0.05 * rng.normal(size=(mesh.ncells, 3, 5)) if opts.scheme.startswith("hweno") else None
    return mesh, opts, q, grad


@pytest.mark.parametrize("kind", ["weno", "hweno"])
def test_rank_local_residual_bitwise(kind):
    from paper_2304_09485_b200.distributed import DistributedSolver
    from paper_2304_09485_b200.partition import Decomposition
    from paper_2304_09485_b200.stepping import SolutionField, Solver

    mesh, opts, q, grad = setup_case(kind)
    full = Solver(mesh, opts)
    fld = SolutionField(q, grad)
    dt = full.local_time_step(fld)
    res, gnew = full.residual(fld, dt)
    dec = Decomposition.build(mesh, 3)
    for rank in range(3):
        # 3-way topology driven in one process without a communicator: the
        # ghost layers come from the uploaded global state
        ds = DistributedSolver(mesh, opts, rank=rank, nranks=3, dec=dec)
        cells = ds.dom.cells
        assert ds.dom.n_owned < len(cells)
        r, g = ds.residual_local(q[cells], None if grad is None else grad[cells], dt[cells],
                                 with_gradients=grad is not None)
        own = cells[: ds.dom.n_owned]
        assert np.array_equal(r, res[own])
        if grad is not None:
            assert np.array_equal(g, gnew[own])
        ds.close()


def _run_ranks(mesh, opts, q, grad, nranks, steps):
    from paper_2304_09485_b200.distributed import DistributedSolver, LoopbackGroup, gather_owned
    from paper_2304_09485_b200.partition import Decomposition
    from paper_2304_09485_b200.stepping import SolutionField

    dec = Decomposition.build(mesh, nranks)
    grp = LoopbackGroup(nranks) if nranks > 1 else None
    ss = [DistributedSolver(mesh, opts, rank=r, nranks=nranks, dec=dec, loopback=grp) for r in range(nranks)]
    for s in ss:
        s.upload(SolutionField(q, grad))
    hist = []
    for _ in range(steps):
        infos = grp.advance_all(ss) if grp else [ss[0].advance_resident()]
        # every rank reports the same (global) norms
        assert len({(i.res_rho_l1, i.res_l2, i.dt_min, i.solver_cycles, i.matvecs) for i in infos}) == 1
        hist.append(infos[0])
    qq, gg = gather_owned([s.download_owned() for s in ss], mesh.ncells, compact=grad is not None)
    if grp:
        grp.close()
    else:
        ss[0].close()
    return hist, qq, gg


@pytest.mark.parametrize("kind,jac,n", [("weno", "roe", 4), ("weno", "frechet", 4), ("c3", "roe", 4)])
def test_loopback_ranks_bitwise_equal_one_rank(kind, jac, n):
    from paper_2304_09485_b200.stepping import SolutionField, Solver

    mesh, opts, q, grad = setup_case(kind, n)
    opts = dataclasses.replace(opts, jacobian=jac)
    steps = 5
    h1, q1, g1 = _run_ranks(mesh, opts, q, grad, 1, steps)
    for nranks in (2, 4):
        hn, qn, gn = _run_ranks(mesh, opts, q, grad, nranks, steps)
        for a, b in zip(h1, hn):
            assert (a.res_rho_l1, a.res_l2, a.dt_min, a.solver_cycles, a.matvecs) == \
                (b.res_rho_l1, b.res_l2, b.dt_min, b.solver_cycles, b.matvecs), (nranks, a, b)
        assert np.array_equal(qn, q1), nranks
        if grad is not None:
            assert np.array_equal(gn, g1), nranks
    # the canonical run vs the plain single-domain solver: same scheme, other
    # summation trees (reference cell order) -> rounding-level agreement
    # (Frechet: rounding amplified by the finite-difference step, ~1/sigma)
    tol = 1e-10 if jac == "roe" else 1e-7
    s = Solver(mesh, opts)
    s.upload(SolutionField(q, grad))
    for a in h1:
        b = s.advance_resident()
        assert abs(a.res_rho_l1 - b.res_rho_l1) <= tol * abs(b.res_rho_l1)
        assert a.solver_cycles == b.solver_cycles
    qs = s.download().q
    assert np.max(np.abs(qs - q1)) <= tol * np.max(np.abs(qs))


@pytest.mark.parametrize("kind,jac", [("weno", "roe"), ("weno", "frechet"), ("hweno", "roe")])
def test_one_rank_nccl_communicator_matches(kind, jac):
    from paper_2304_09485_b200.distributed import DistributedSolver
    from paper_2304_09485_b200.stepping import SolutionField

    # Three steps: the second and third replay the captured step graph (with
    # the NCCL group-partial allreduces inside it).
    mesh, opts, q, grad = setup_case(kind)
    opts = dataclasses.replace(opts, jacobian=jac)
    ref = DistributedSolver(mesh, opts, rank=0, nranks=1)
    ref.upload(SolutionField(q, grad))
    ds = DistributedSolver(mesh, opts, rank=0, nranks=1, comm_id=DistributedSolver.unique_id())
    ds.upload(SolutionField(q, grad))
    for _ in range(3):
        a = ref.advance_resident()
        b = ds.advance_resident()
        assert a.res_rho_l1 == b.res_rho_l1 and a.res_l2 == b.res_l2 and a.solver_cycles == b.solver_cycles
    assert np.array_equal(ds.download_owned()[1], ref.download_owned()[1])
    ds.close()
    ref.close()


def test_loopback_retry_and_failure_agree_across_ranks():
    """An impossible CFL makes the update unphysical: every rank must take
    the dt-halving branch together and raise the same SteppingError naming
    reference cell ids (stepping.py:286-296)."""
    from paper_2304_09485_b200.distributed import DistributedSolver, LoopbackGroup
    from paper_2304_09485_b200.partition import Decomposition
    from paper_2304_09485_b200.stepping import SolutionField, SteppingError

    mesh, opts, q, grad = setup_case("weno", 4)
    opts = dataclasses.replace(opts, cfl=1e6)
    dec = Decomposition.build(mesh, 2)
    grp = LoopbackGroup(2)
    ss = [DistributedSolver(mesh, opts, rank=r, nranks=2, dec=dec, loopback=grp) for r in range(2)]
    for s in ss:
        s.upload(SolutionField(q, grad))
    one = DistributedSolver(mesh, opts, rank=0, nranks=1)
    one.upload(SolutionField(q, grad))
    try:
        ref = one.advance_resident()
        ref_err = None
    except SteppingError as e:
        ref, ref_err = None, str(e)
    try:
        got = grp.advance_all(ss)
        err = None
    except SteppingError as e:
        got, err = None, str(e)
    if ref_err is None:
        assert err is None and got[0].retried == ref.retried and got[0].res_rho_l1 == ref.res_rho_l1
    else:
        assert err is not None and "dt halving" in err
    grp.close()
    one.close()


@pytest.mark.parametrize("nc", [1000, 23040, 400_000])
def test_device_dot_is_the_specified_fold(nc):
    """gks_blocksys_dot (the GMRES reduction) equals the numpy statement of
    the partition-invariant fold bit for bit (tests/_fold.py)."""
    import ctypes as C

    import _fold
    from paper_2304_09485_b200 import _native as N

    lib = N.load()
    rng = np.random.default_rng(nc)
    diag = np.tile(np.eye(5), (nc, 1, 1))
    rowptr = np.zeros(nc + 1, dtype=np.int64)
    h = C.c_void_p()
    N.check(lib.gks_blocksys_create(nc, 0, N.dptr(diag.reshape(-1)), None, None, N.iptr(rowptr), 0, C.byref(h)))
    x = rng.normal(size=(nc, 5)) * np.exp(3 * rng.normal(size=(nc, 1)))
    y = rng.normal(size=(nc, 5))
    out = C.c_double()
    N.check(lib.gks_blocksys_dot(h, N.dptr(x), N.dptr(y), C.byref(out)))
    lib.gks_blocksys_destroy(h)
    assert out.value == _fold.dot(x, y)


@pytest.mark.parametrize("jac", ["roe", "frechet"])
def test_cgs2_multidot_gmres(jac):
    """ortho="cgs2": three fused multi-dot passes per Arnoldi column.  Same
    step results as the reference MGS to rounding, partition-invariant
    (2-rank loopback bitwise equal to the canonical 1-rank run)."""
    from paper_2304_09485_b200.stepping import SolutionField, Solver

    mesh, opts, q, grad = setup_case("weno", 4)
    mgs = dataclasses.replace(opts, jacobian=jac)
    cgs = dataclasses.replace(opts, jacobian=jac, ortho="cgs2")
    a, b = Solver(mesh, mgs), Solver(mesh, cgs)
    a.upload(SolutionField(q, grad))
    b.upload(SolutionField(q, grad))
    tol = 1e-9 if jac == "roe" else 1e-6
    for _ in range(4):
        ia, ib = a.advance_resident(), b.advance_resident()
        assert ia.solver_cycles == ib.solver_cycles and ia.matvecs == ib.matvecs
        assert abs(ia.res_rho_l1 - ib.res_rho_l1) <= tol * abs(ia.res_rho_l1)
    assert np.max(np.abs(a.download().q - b.download().q)) <= tol * np.max(np.abs(a.download().q))
    h1, q1, _ = _run_ranks(mesh, cgs, q, grad, 1, 3)
    h2, q2, _ = _run_ranks(mesh, cgs, q, grad, 2, 3)
    assert [(x.res_rho_l1, x.res_l2) for x in h1] == [(x.res_rho_l1, x.res_l2) for x in h2]
    assert np.array_equal(q1, q2)


@pytest.mark.parametrize("kind", ["weno", "c3"])
def test_loopback_host_array_steps_equal_resident(kind):
    """The bench's end-to-end path on rank-local handles: gks_advance from
    each rank's host field (H2D, step with device halo exchanges, D2H) on 2
    loopback ranks reproduces the 1-rank resident run bit for bit."""
    from paper_2304_09485_b200.distributed import DistributedSolver, LoopbackGroup
    from paper_2304_09485_b200.partition import Decomposition

    mesh, opts, q, grad = setup_case(kind, 4)
    steps = 3
    h1, q1, g1 = _run_ranks(mesh, opts, q, grad, 1, steps)
    dec = Decomposition.build(mesh, 2)
    grp = LoopbackGroup(2)
    ss = [DistributedSolver(mesh, opts, rank=r, nranks=2, dec=dec, loopback=grp) for r in range(2)]
    fq = [np.ascontiguousarray(q[s.dom.cells]) for s in ss]
    fg = [None if grad is None else np.ascontiguousarray(grad[s.dom.cells]) for s in ss]
    for k in range(steps):
        infos = grp.advance_all(ss, step=lambda r, s: s.advance_inplace(fq[r], fg[r]))
        assert infos[0].res_rho_l1 == h1[k].res_rho_l1 and infos[0].solver_cycles == h1[k].solver_cycles
    for r, s in enumerate(ss):
        n = s.dom.n_owned
        own = s.dom.cells[:n]
        assert np.array_equal(fq[r][:n], q1[own])
        if grad is not None:
            assert np.array_equal(fg[r][:n], g1[own])
    grp.close()
