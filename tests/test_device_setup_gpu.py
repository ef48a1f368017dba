"""Device-side setup (csrc/gks_setup_dev.cu) against the host native setup
(csrc/gks_setup.cpp): stencil selection, reconstruction geometry and the
WENO / HWENO operators of stencils.py:72-192, recon.py:60-274 and
hweno.py:45-137, built per cell on the GPU from the shared per-cell code
(csrc/gks_setup_cell.cuh).  Every padded record the reconstruction kernels
read must be BITWISE the host build's (both compiled without FP
contraction); the host build itself is pinned to the reference's goldens
(tests/test_setup.py), so the device build inherits that parity.
"""

import ctypes as C

import numpy as np
import pytest

from paper_2304_09485_b200 import _native as N
from paper_2304_09485_b200 import meshgen as MG
from paper_2304_09485_b200.boundary import PatchSpec
from paper_2304_09485_b200.mesh import generate_box_mesh
from paper_2304_09485_b200.stepping import SolutionField, Solver, SolverOptions, initial_field

pytestmark = pytest.mark.gpu

GAMMA = 1.4
REF = np.array([1.0, 0.5, 0.1, 0.0, 1.0 / GAMMA])

MESHES = {
    "sphere2": lambda: MG.generate_sphere_mesh(2, radius=0.5, far=10.0),
    "wing8": lambda: MG.generate_swept_wing_mesh(8),
    "tetbox_perturbed": lambda: generate_box_mesh((1, 1, 1), (4, 3, 5), split="tet", perturb=0.15, seed=11),
    "hexbox": lambda: generate_box_mesh((1, 2, 1), (4, 3, 5), split="hex"),
    "hexbox_periodic": lambda: generate_box_mesh((1, 1, 1), (4, 4, 4), split="hex", periodic=("x", "y", "z")),
    "tetbox_periodic": lambda: generate_box_mesh((1, 1, 1), (3, 3, 3), split="tet", periodic=("x", "z")),
}

WENO_ARRAYS = ["avg0", "beta", "big_op", "big_gather", "sub_op", "sub_gather", "sub_active"]
HWENO_ARRAYS = ["avg0", "beta", "big_op", "avg_gather", "grad_gather", "grad_scale", "sub_op", "sub_gather",
                "sub_active"]


def handle_array(solver, name):
    lib = N.load()
    nb = C.c_int64(0)
    N.check(lib.gks_handle_array(solver._handle, name.encode(), None, C.byref(nb)))
    out = np.empty(nb.value, dtype=np.uint8)
    N.check(lib.gks_handle_array(solver._handle, name.encode(), out.ctypes.data_as(C.c_void_p), C.byref(nb)))
    return out


def make(mesh, scheme, setup, reorder="none"):
    patches = {n: PatchSpec(n, "farfield_riemann", reference=REF) for n in mesh.patch_names}
    return Solver(mesh, SolverOptions(scheme=scheme, patches=patches, setup=setup, reorder=reorder))


def info(solver, k):
    return int(N.load().gks_handle_info(solver._handle, k))


@pytest.mark.parametrize("scheme", ["weno_gmres", "hweno_gmres"])
@pytest.mark.parametrize("name", list(MESHES))
def test_device_setup_records_bitwise_equal_host(name, scheme):
    mesh = MESHES[name]()
    dev = make(mesh, scheme, "device")
    host = make(mesh, scheme, "host")
    for k in (6, 7, 8):  # reference widths (K, M, S) / (HA + 3 HG, HM, 7)
        assert info(dev, k) == info(host, k), k
    for arr in (HWENO_ARRAYS if scheme == "hweno_gmres" else WENO_ARRAYS):
        a, b = handle_array(dev, arr), handle_array(host, arr)
        assert a.shape == b.shape, arr
        assert np.array_equal(a, b), (arr, int(np.count_nonzero(a != b)))
    # and the residual the records produce
    q = initial_field(mesh, REF).q * (1.0 + 0.01 * np.sin(np.arange(mesh.ncells)))[:, None]
    grad = 0.01 * np.cos(np.arange(mesh.ncells * 15)).reshape(-1, 3, 5) if scheme == "hweno_gmres" else None
    fld = SolutionField(q, grad)
    dt = host.local_time_step(fld)
    r1, _ = dev.residual(fld, dt)
    r2, _ = host.residual(fld, dt)
    assert np.array_equal(r1, r2)


@pytest.mark.parametrize("scheme", ["weno_gmres", "hweno_gmres"])
@pytest.mark.parametrize("reorder", ["rcm", "morton"])
def test_device_setup_on_renumbered_mesh(reorder, scheme):
    """A renumbered handle builds its stencils on the permuted mesh: the
    enlarged tet members sort by the reference id (cell_rank), so the
    records equal the host setup restricted to the permutation."""
    mesh = MG.generate_sphere_mesh(2, radius=0.5, far=10.0)
    dev = make(mesh, scheme, "device", reorder)
    host = make(mesh, scheme, "host", reorder)
    for arr in (HWENO_ARRAYS if scheme == "hweno_gmres" else WENO_ARRAYS):
        assert np.array_equal(handle_array(dev, arr), handle_array(host, arr)), arr


def test_device_setup_default_and_c2_size():
    """The default path builds on the device; at C2 n=8 (184k cells) the
    device build equals the host build too."""
    assert SolverOptions().setup == "device"
    mesh = MG.generate_sphere_mesh(8, radius=0.5, far=20.0)
    dev = make(mesh, "weno_gmres", "device")
    host = make(mesh, "weno_gmres", "host")
    for arr in WENO_ARRAYS:
        assert np.array_equal(handle_array(dev, arr), handle_array(host, arr)), arr


@pytest.mark.parametrize("scheme", ["weno_gmres", "hweno_gmres"])
def test_device_setup_rank_local_handles(scheme):
    """Rank-local handles (DistributedSolver, no communicator) build on
    their SetupMesh on the device and place the records in local order:
    equal to the host per-rank setup + gks_setup_subset path."""
    from paper_2304_09485_b200.distributed import DistributedSolver
    from paper_2304_09485_b200.partition import Decomposition

    mesh = MG.generate_sphere_mesh(4, radius=0.5, far=10.0)
    patches = {n: PatchSpec(n, "farfield_riemann", reference=REF) for n in mesh.patch_names}
    dec = Decomposition.build(mesh, 3)
    arrays = HWENO_ARRAYS if scheme == "hweno_gmres" else WENO_ARRAYS
    for rank in range(3):
        d = DistributedSolver(mesh, SolverOptions(scheme=scheme, patches=patches, setup="device"), rank=rank,
                              nranks=3, dec=dec)
        h = DistributedSolver(mesh, SolverOptions(scheme=scheme, patches=patches, setup="host"), rank=rank,
                              nranks=3, dec=dec)
        for k in (6, 7, 8):
            assert info(d, k) == info(h, k), (rank, k)
        for arr in arrays:
            assert np.array_equal(handle_array(d, arr), handle_array(h, arr)), (rank, arr)
