"""Locality renumbering (reorder.py) on the CPU: the permuted mesh is a
consistent relabelling of the reference mesh, and the permuted native setup
is exactly the reference's operators moved to the new numbering."""

import numpy as np
import pytest

from paper_2304_09485_b200 import _native as N
from paper_2304_09485_b200.mesh import generate_box_mesh
from paper_2304_09485_b200.meshgen import generate_sphere_mesh
from paper_2304_09485_b200.reorder import PermutedMesh, cell_order


def meshes():
    return {
        "tet4p": generate_box_mesh((1, 1, 1), (4, 4, 4), split="tet", periodic=("x", "y", "z")),
        "hex3": generate_box_mesh((1, 1, 1), (3, 3, 3)),
        "sphere": generate_sphere_mesh(2, far=4.0, nr=5),
    }


@pytest.fixture(scope="module", params=["tet4p", "hex3", "sphere"])
def mesh(request):
    return meshes()[request.param]


@pytest.mark.parametrize("method", ["rcm", "morton"])
def test_permuted_mesh_is_a_relabelling(mesh, method):
    perm = cell_order(mesh, method)
    assert np.array_equal(np.sort(perm), np.arange(mesh.ncells))
    pm = PermutedMesh(mesh, perm)
    inv = pm.inv
    fr = pm.face_rank
    assert np.array_equal(np.sort(fr), np.arange(mesh.nfaces))
    # faces sorted by new owner
    assert np.all(np.diff(pm.face_owner) >= 0)
    assert np.array_equal(pm.face_owner, inv[mesh.face_owner[fr]])
    nb = mesh.face_neighbor[fr]
    assert np.array_equal(pm.face_neighbor, np.where(nb >= 0, inv[np.maximum(nb, 0)], -1))
    for k in ("face_area", "face_normal", "face_frame", "face_shift", "face_patch"):
        assert np.array_equal(getattr(pm, k), getattr(mesh, k)[fr]), k
    # face points follow their faces; fq_rank is the reference index
    assert np.array_equal(np.sort(pm.fq_rank), np.arange(len(mesh.fq_face)))
    assert np.array_equal(fr[pm.fq_face], mesh.fq_face[pm.fq_rank])
    assert np.array_equal(pm.fq_point, mesh.fq_point[pm.fq_rank])
    # cell -> face lists in each cell's own order
    for c in range(0, mesh.ncells, max(1, mesh.ncells // 50)):
        old = mesh.cell_face_list[mesh.cell_face_start[perm[c]]: mesh.cell_face_start[perm[c] + 1]]
        new = pm.cell_face_list[pm.cell_face_start[c]: pm.cell_face_start[c + 1]]
        assert np.array_equal(fr[new], old)
    assert np.allclose(pm.cq_weight.sum(), mesh.cq_weight.sum(), rtol=0, atol=1e-12)


def test_permuted_setup_equals_reference_operators(mesh):
    import ctypes as C

    perm = cell_order(mesh, "rcm")
    inv = np.empty_like(perm)
    inv[perm] = np.arange(len(perm))
    gs = N.NativeSetup(mesh, schemes=3)
    lib = N.load()
    sub = C.c_void_p()
    N.check(lib.gks_setup_subset(gs.handle, N.iptr(perm), mesh.ncells, N.iptr(inv), mesh.ncells, C.byref(sub)))

    def arr(name):
        dt, nd = C.c_int(), C.c_int()
        shape = (C.c_int64 * 4)()
        N.check(lib.gks_setup_query(sub, name.encode(), C.byref(dt), C.byref(nd), shape))
        out = np.empty(tuple(shape[i] for i in range(nd.value)), dtype=N._DTYPES[dt.value])
        N.check(lib.gks_setup_copy(sub, name.encode(), out.ctypes.data_as(C.c_void_p), out.nbytes))
        return out

    try:
        for k in ("weno_big_op", "weno_sub_op", "hweno_big_op", "hweno_sub_op", "avg0", "beta_mat",
                  "weno_sub_active", "hweno_sub_active", "hweno_big_grad_scale"):
            assert np.array_equal(arr(k), gs.array(k)[perm]), k
        for k in ("weno_big_gather", "weno_sub_gather", "hweno_big_avg_gather", "hweno_big_grad_gather",
                  "hweno_sub_gather"):
            ref = gs.array(k)[perm]
            got = arr(k)
            # gathers point at the same cells, renumbered (padding slots stay padding)
            assert np.array_equal(got, inv[ref]), k
    finally:
        lib.gks_setup_free(sub)
