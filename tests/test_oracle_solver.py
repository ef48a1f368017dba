"""Oracle pinning (CPU): the numpy solver restatement vs reference goldens."""

import numpy as np
import pytest

from oracle.solver import OracleSolver, gmres, roe_jacobian
from test_solver_gpu import CASES, MG, relmax


def build_oracle(name):
    from paper_2304_09485_b200.boundary import PatchSpec
    from paper_2304_09485_b200.mesh import generate_box_mesh

    case = MG.SOLVER_CASES[name]
    mesh = generate_box_mesh(**MG.MESH_CASES[case["mesh"]])
    ref = np.array(case.get("reference", (1.0, 0.5, 0.0, 0.0, 1.0 / 1.4)))
    patches = {}
    kinds = case.get("patches", {})
    for n in mesh.patch_names:
        spec = kinds.get(n, kinds.get("*"))
        if spec is None:
            continue
        kind, kw = spec
        kw = dict(kw)
        if kind in ("farfield_riemann", "supersonic_inlet") and "reference" not in kw:
            kw["reference"] = ref
        patches[n] = PatchSpec(n, kind, **kw)
    return mesh, OracleSolver(mesh, scheme=case["scheme"], model=case.get("model", "inviscid"),
                              mu=case.get("mu", 0.0), weights=case.get("weights", "nonlinear"), patches=patches)


@pytest.fixture(scope="module", params=CASES)
def ocase(request, golden):
    mesh, s = build_oracle(request.param)
    return mesh, s, golden(f"solver_{request.param}")


def test_dt_residual_ghosts(ocase):
    mesh, s, g = ocase
    grad = g["grad"] if s.compact else None
    assert relmax(s.local_dt(g["q"]), g["dt"]) < 1e-14
    res, gnew = s.residual(g["q"], grad, g["dt"])
    assert relmax(res, g["res"]) < 1e-12
    if s.compact:
        assert relmax(gnew, g["grad_new"]) < 1e-12
    gh = s.ghosts(g["q"])
    if gh is not None:
        assert relmax(gh, g["ghosts"]) < 1e-13


def test_jacobian_and_gmres(ocase):
    mesh, s, g = ocase
    A = roe_jacobian(mesh, g["q"], g["dt"], g["ghosts"] if len(g["ghosts"]) else None)
    assert relmax(A.diag, g["jac_diag"]) < 1e-13
    assert np.array_equal(A.row, g["jac_off_row"]) and np.array_equal(A.col, g["jac_off_col"])
    assert relmax(A.off, g["jac_off"]) < 1e-13
    x, cyc, nmv = gmres(A, g["res"])
    assert nmv == int(g["gmres_matvecs"])
    assert relmax(x, g["gmres_x"]) < 1e-9


def test_frechet_and_advance(ocase):
    mesh, s, g = ocase
    grad = g["grad"] if s.compact else None
    fm = s.frechet(g["q"], grad, g["frechet_v"], g["dt"])
    assert relmax(fm, g["frechet"]) < 1e-6
    q, gr = g["q"], grad
    for k in range(2):
        q, gr, info = s.advance(q, gr)
        assert info["res_rho_l1"] == pytest.approx(g["hist"][k][0], rel=1e-8, abs=1e-13)
        assert relmax(q, g["q_after"][k]) < 1e-9
