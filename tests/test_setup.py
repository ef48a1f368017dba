"""Native setup (C++) vs reference goldens: mesh, stencils (bit-exact), operators.

CPU-only: runs the host mesh builder and the native setup library, no GPU.
"""

import importlib.util
from pathlib import Path

import numpy as np
import pytest

from paper_2304_09485_b200 import _native as N
from paper_2304_09485_b200.mesh import generate_box_mesh
from paper_2304_09485_b200.stencils import build_stencils

_spec = importlib.util.spec_from_file_location("make_golden", Path(__file__).parent / "golden" / "make_golden.py")
MG = importlib.util.module_from_spec(_spec)
_spec.loader.exec_module(MG)

CASES = list(MG.MESH_CASES)
INT_MESH = ("cell_kind", "cell_nodes", "face_nodes", "face_owner", "face_neighbor", "face_patch", "fq_face",
            "face_fq_start", "cell_cq_start")
GEO_MESH = ("cell_volume", "cell_centroid", "cell_h", "face_area", "face_normal", "face_frame", "face_shift",
            "fq_point", "fq_weight", "cq_point", "cq_weight")


@pytest.fixture(scope="module", params=CASES)
def case(request, golden):
    name = request.param
    mesh = generate_box_mesh(**MG.MESH_CASES[name])
    return name, mesh, golden(f"mesh_{name}")


def test_mesh_connectivity_bit_exact(case):
    _, mesh, g = case
    for k in INT_MESH:
        assert np.array_equal(getattr(mesh, k), g[f"mesh_{k}"]), k
    assert np.array_equal(mesh.cell_face_list, g["mesh_cell_face_list"])


def test_mesh_geometry(case):
    _, mesh, g = case
    for k in GEO_MESH:
        assert np.allclose(getattr(mesh, k), g[f"mesh_{k}"], rtol=0, atol=1e-15), k


def test_stencils_bit_exact(case):
    _, mesh, g = case
    st = build_stencils(mesh)
    nf = g["st_nbr_ids"].shape[1]
    assert np.array_equal(st.nbr_ids[:, :nf], g["st_nbr_ids"])
    assert np.array_equal(st.nbr_shift[:, :nf], g["st_nbr_shift"])
    for k in ("big_start", "big_ids", "sub_cell_start", "sub_member_start", "sub_ids"):
        assert np.array_equal(getattr(st, k), g[f"st_{k}"]), k
    for k in ("big_shift", "sub_shift"):
        assert np.array_equal(getattr(st, k).reshape(-1, 3), g[f"st_{k}"].reshape(-1, 3)), k
    assert np.array_equal(st.weno_fallback, g["st_weno_fallback"].astype(bool))
    assert np.array_equal(st.hweno_fallback, g["st_hweno_fallback"].astype(bool))


OPS_INT = ("weno_big_gather", "weno_big_degree", "weno_sub_gather", "weno_sub_active", "hweno_big_avg_gather",
           "hweno_big_grad_gather", "hweno_big_ncols", "hweno_big_degree", "hweno_sub_gather", "hweno_sub_active")
OPS_F = ("avg0", "beta_mat", "weno_big_op", "weno_sub_op", "hweno_big_op", "hweno_big_grad_scale", "hweno_sub_op")


def test_operators(case):
    _, mesh, g = case
    s = N.NativeSetup(mesh, schemes=3)
    for k in OPS_INT:
        assert np.array_equal(s.array(k), g[k].astype(s.array(k).dtype)), k
    for k in OPS_F:
        ref = g[k]
        got = s.array(k)
        assert got.shape == ref.shape, k
        # pseudo-inverses are unpinned bitwise (SVD backend); agree to rounding
        scale = max(float(np.max(np.abs(ref))), 1e-300)
        assert float(np.max(np.abs(got - ref))) <= 1e-12 * scale, k


def test_setup_rejects_bad_name(case):
    _, mesh, _ = case
    s = N.NativeSetup(mesh, schemes=1)
    with pytest.raises(N.GksError):
        s.array("no_such_array")
