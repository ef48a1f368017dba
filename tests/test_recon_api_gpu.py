"""The reference's reconstruction API (recon.py / hweno.py), device-backed:
combined coefficients through the solver's own k_recon_* kernels, candidate
coefficients, combine_candidates and evaluate_faces as device batches --
against the oracle (oracle/recon.py, pinned to the reference) and against
the reference's padded-operator formulas evaluated here on the API's own
operator arrays.
"""

import numpy as np
import pytest

from oracle import recon as OR
from paper_2304_09485_b200 import hweno as HW
from paper_2304_09485_b200 import recon as R
from paper_2304_09485_b200.mesh import generate_box_mesh
from paper_2304_09485_b200.stencils import build_stencils

pytestmark = pytest.mark.gpu

MESHES = {
    "tet": lambda: generate_box_mesh((1, 1, 1), (3, 3, 3), split="tet", perturb=0.12, seed=42),
    "hex": lambda: generate_box_mesh((1, 1, 1), (4, 4, 4), split="hex"),
    "hex_periodic": lambda: generate_box_mesh((1, 1, 1), (4, 3, 4), split="hex", periodic=("x", "z")),
}


def relmax(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def fields(mesh, m, seed=3):
    rng = np.random.default_rng(seed)
    x = mesh.cell_centroid
    q = np.stack([np.sin(2.0 * x[:, 0] + k) + 0.3 * x[:, 1] * x[:, 2] + 0.05 * rng.normal(size=len(x))
                  for k in range(m)], axis=1)
    g = 0.2 * rng.normal(size=(len(x), 3, m))
    return q, g


@pytest.mark.parametrize("name", list(MESHES))
@pytest.mark.parametrize("compact", [False, True])
def test_combined_coeffs_match_oracle(name, compact):
    mesh = MESHES[name]()
    geom = R.ReconGeometry(mesh, build_stencils(mesh))
    q, g = fields(mesh, 7)  # 7 components: two device passes of 5
    orc = OR.Recon(mesh, OR.stencils(mesh), compact)
    if compact:
        got = HW.HwenoReconstructor(geom).combined_coeffs(q, g)
        ref = orc.coefficients(q, g)
    else:
        got = R.WenoReconstructor(geom).combined_coeffs(q)
        ref = orc.coefficients(q)
    assert got.shape == (mesh.ncells, 9, 7)
    assert relmax(got, ref) <= 1e-12


@pytest.mark.parametrize("compact", [False, True])
def test_candidates_and_combine(compact):
    mesh = MESHES["tet"]()
    geom = R.ReconGeometry(mesh, build_stencils(mesh))
    q, g = fields(mesh, 3)
    if compact:
        rec = HW.HwenoReconstructor(geom)
        c_big, b_sub = rec.candidate_coeffs(q, g)
        # hweno.py:139-160 on the API's own reference-layout operators
        nc = mesh.ncells
        ga = q[rec.big_avg_gather] - q[:, None, :]
        gg = (rec.big_grad_scale[:, :, None, None] * g[rec.big_grad_gather]).reshape(nc, -1, q.shape[1])
        amax = rec.big_avg_gather.shape[1]
        ref_big = np.einsum("cdk,ckm->cdm", rec.big_op[:, :, :amax], ga) + \
            np.einsum("cdk,ckm->cdm", rec.big_op[:, :, amax:], gg)
        sg = rec.sub_gather
        rhs = np.concatenate([(q[sg[:, :, 1]] - q[:, None, :])[:, :, None, :],
                              mesh.cell_h[sg[:, :, 0], None, None] * g[sg[:, :, 0]],
                              mesh.cell_h[sg[:, :, 1], None, None] * g[sg[:, :, 1]]], axis=2)
        ref_sub = np.einsum("cmds,cmsk->cmdk", rec.sub_op, rhs)
        combined = rec.combined_coeffs(q, g)
    else:
        rec = R.WenoReconstructor(geom)
        c_big, b_sub = rec.candidate_coeffs(q)
        ref_big = np.einsum("cdk,ckm->cdm", rec.big_op, q[rec.big_gather] - q[:, None, :])
        ref_sub = np.einsum("cmds,cmsk->cmdk", rec.sub_op, q[rec.sub_gather] - q[:, None, None, :])
        combined = rec.combined_coeffs(q)
    assert b_sub.shape == ref_sub.shape
    assert relmax(c_big, ref_big) <= 1e-12
    act = rec.sub_active
    assert relmax(b_sub[act], ref_sub[act]) <= 1e-12
    out, w0n, wmn = R.combine_candidates(c_big, b_sub, act, geom.beta_mat)
    assert relmax(out, combined) <= 1e-13
    # normalised weights sum to one; inactive slots carry none
    assert np.allclose(w0n + wmn.sum(axis=1), 1.0, rtol=0, atol=1e-14)
    assert np.all(wmn[~act] == 0.0)


def test_evaluate_faces_and_single_cell_views():
    mesh = MESHES["hex"]()
    geom = R.ReconGeometry(mesh, build_stencils(mesh))
    rec = R.WenoReconstructor(geom)
    q, _ = fields(mesh, 2)
    coef = rec.combined_coeffs(q)
    vo, go, vn, gn = R.evaluate_faces(geom, q, coef)
    own = geom.fq_owner
    nb = np.where(geom.fq_interior, geom.fq_neighbor, own)
    ref_vo = q[own] + np.einsum("fd,fdk->fk", geom.phi_owner, coef[own])
    ref_go = np.einsum("fxd,fdk->fxk", geom.dphi_owner, coef[own])
    ref_vn = np.where(geom.fq_interior[:, None], q[nb] + np.einsum("fd,fdk->fk", geom.phi_neighbor, coef[nb]), ref_vo)
    assert relmax(vo, ref_vo) <= 1e-12 and relmax(go, ref_go) <= 1e-11 and relmax(vn, ref_vn) <= 1e-12
    # single-cell views: every candidate keeps the cell average
    c = int(np.flatnonzero(rec.sub_active.sum(axis=1) == 8)[0])
    polys = [R.fit_big_polynomial(rec, c, q)] + R.fit_sub_polynomials(rec, c, q)
    assert len(polys) == 9
    for p in polys:
        assert np.allclose(p.cell_average(geom), q[c], rtol=0, atol=1e-13)
    betas = [R.smoothness_indicator(geom, p) for p in polys]
    x = mesh.fq_point[np.flatnonzero(own == c)[0]]
    val, grad = R.nonlinear_combine(polys[0], polys[1:], betas, R.LINEAR_WEIGHT, R.WENO_EPS, x)
    i = np.flatnonzero(own == c)[0]
    assert np.allclose(val, vo[i], rtol=1e-10, atol=1e-12)
    assert np.allclose(grad, go[i], rtol=1e-9, atol=1e-10)
