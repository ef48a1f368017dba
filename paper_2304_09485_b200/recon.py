"""Non-compact WENO reconstruction API (mirrors gks3d/recon.py).

The reference's public reconstruction objects, backed by the device:

* ``ReconGeometry`` (recon.py:104-164): the zero-mean basis offsets ``avg0``
  and smoothness matrices ``beta_mat`` of the native setup, plus the face
  tables of the face quadrature points;
* ``WenoReconstructor`` (recon.py:198-294): the operators of the native
  setup in the reference's padded layout; ``candidate_coeffs`` and
  ``combined_coeffs`` run on the GPU (gks_recon_candidates and the solver's
  own k_recon_weno through gks_recon_coeffs) on a cached handle of the mesh;
* ``combine_candidates`` (recon.py:167-195) and ``evaluate_faces``
  (recon.py:297-314): device batches (gks_combine_candidates,
  gks_face_values);
* the single-cell views ``fit_big_polynomial`` / ``fit_sub_polynomials``
  (recon.py:327-367) select one cell's device-computed candidates;
  ``ReconPolynomial``, ``smoothness_indicator`` and ``nonlinear_combine``
  (recon.py:73-101, 370-406) evaluate ONE polynomial / point on the host,
  as the reference's inspection helpers do.

Fields with any number of components are processed five at a time (the
device state width).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as N

NCOEF = 9
WENO_EPS = 1e-6
LINEAR_WEIGHT = 0.025
RANK_TOL = 1e-10

_MONO = ((0,), (1,), (2,), (0, 0), (0, 1), (0, 2), (1, 1), (1, 2), (2, 2))  # x y z xx xy xz yy yz zz


def monomial_rows(xt):
    """The nine basis monomials at scaled points: (..., 3) -> (..., 9)."""
    xt = np.asarray(xt, dtype=float)
    return np.stack([np.prod([xt[..., a] for a in idx], axis=0) for idx in _MONO], axis=-1)


def monomial_grad_rows(xt):
    """d monomial / d xt: (..., 3) -> (..., 3, 9)."""
    xt = np.asarray(xt, dtype=float)
    out = np.zeros(xt.shape[:-1] + (3, NCOEF))
    for d, idx in enumerate(_MONO):
        if len(idx) == 1:
            out[..., idx[0], d] = 1.0
        else:
            a, b = idx
            out[..., a, d] += xt[..., b]
            out[..., b, d] += xt[..., a]
    return out


@dataclass
class ReconPolynomial:
    """Q(x) = q0 + coeffs . (p(xt) - basis_offset), xt = (x - centroid) / h
    (recon.py:73-101): the zero-mean basis makes q0 the cell average."""

    cell: int
    q0: np.ndarray
    coeffs: np.ndarray
    degree: int
    centroid: np.ndarray
    h: float
    basis_offset: np.ndarray

    def _xt(self, x):
        return (np.asarray(x, dtype=float) - self.centroid) / self.h

    def value(self, x):
        return self.q0 + (monomial_rows(self._xt(x)) - self.basis_offset) @ self.coeffs

    def gradient(self, x):
        return (monomial_grad_rows(self._xt(x)) @ self.coeffs) / self.h

    def cell_average(self, geom):
        pts, w = geom.mesh.cell_quadrature_of(self.cell)
        return self.q0 + w @ ((monomial_rows(self._xt(pts)) - self.basis_offset) @ self.coeffs)


# -- device handles ------------------------------------------------------------

_HANDLES: dict = {}


def _handle(mesh, scheme, eps=WENO_EPS, lin_weight=LINEAR_WEIGHT):
    """A reconstruction handle of the mesh (cached: one per scheme / weights)."""
    from .boundary import PatchSpec
    from .stepping import Solver, SolverOptions

    key = (id(mesh), scheme, float(eps), float(lin_weight))
    s = _HANDLES.get(key)
    if s is None or s.mesh is not mesh:
        for k in [k for k, v in _HANDLES.items() if v.mesh is not mesh or k[0] != id(mesh)]:
            del _HANDLES[k]
        patches = {n: PatchSpec(n, "supersonic_outlet") for n in mesh.patch_names}
        s = Solver(mesh, SolverOptions(scheme=scheme, patches=patches, weno_eps=eps, linear_weight=lin_weight))
        _HANDLES[key] = s
    return s


def _field(field):
    field = np.asarray(field, dtype=float)
    return field[:, None] if field.ndim == 1 else field


def _chunks(m):
    for k0 in range(0, m, 5):
        yield slice(k0, min(k0 + 5, m)), min(5, m - k0)


def _pad5(a, sl, k):
    """Components sl of a (..., m) array, zero-padded to 5."""
    out = np.zeros(a.shape[:-1] + (5,))
    out[..., :k] = a[..., sl]
    return out


def _device_candidates(solver, field, grad=None):
    lib = N.load()
    h = solver._handle
    nc = solver.mesh.ncells
    M = int(lib.gks_handle_info(h, 7))
    m = field.shape[1]
    c_big = np.empty((nc, NCOEF, m))
    b_sub = np.empty((nc, M, 3, m))
    for sl, k in _chunks(m):
        q5 = _pad5(field, sl, k)
        g5 = None if grad is None else _pad5(grad, sl, k)
        cb = np.empty((nc, NCOEF, 5))
        bs = np.empty((nc, M, 3, 5))
        N.check(lib.gks_recon_candidates(h, N.dptr(q5), N.dptr(g5), N.dptr(cb), N.dptr(bs)))
        c_big[..., sl] = cb[..., :k]
        b_sub[..., sl] = bs[..., :k]
    return c_big, b_sub


def _device_combined(solver, field, grad, linear):
    lib = N.load()
    nc = solver.mesh.ncells
    m = field.shape[1]
    out = np.empty((nc, NCOEF, m))
    for sl, k in _chunks(m):
        q5 = _pad5(field, sl, k)
        g5 = None if grad is None else _pad5(grad, sl, k)
        co = np.empty((nc, NCOEF, 5))
        N.check(lib.gks_recon_coeffs(solver._handle, N.dptr(q5), N.dptr(g5), int(linear), N.dptr(co)))
        out[..., sl] = co[..., :k]
    return out


# -- geometry ---------------------------------------------------------------------


class ReconGeometry:
    """Basis offsets, smoothness matrices and face tables (recon.py:104-164)."""

    def __init__(self, mesh, stencils):
        self.mesh = mesh
        self.stencils = stencils
        setup = getattr(stencils, "setup", None)
        if setup is None:
            setup = N.NativeSetup(mesh, schemes=0)
        self._setup = setup
        self.avg0 = np.array(setup.array("avg0"))
        self.beta_mat = np.array(setup.array("beta_mat"))
        self.fq_owner = mesh.face_owner[mesh.fq_face]
        self.fq_neighbor = mesh.face_neighbor[mesh.fq_face]
        self.fq_interior = self.fq_neighbor >= 0
        self._tables = None

    def member_rows(self, c, ids, shifts):
        """Cell-average basis rows of stencil members ids[1:] in the chart of c."""
        mesh = self.mesh
        rows = np.empty((len(ids) - 1, NCOEF))
        for r, (j, s) in enumerate(zip(ids[1:], shifts[1:])):
            pts, w = mesh.cell_quadrature_of(int(j), s)
            rows[r] = w @ monomial_rows((pts - mesh.cell_centroid[c]) / mesh.cell_h[c]) - self.avg0[c]
        return rows

    def _face_tables(self):
        if self._tables is None:
            mesh = self.mesh
            own = self.fq_owner
            nb = np.where(self.fq_interior, self.fq_neighbor, 0)
            xo = (mesh.fq_point - mesh.cell_centroid[own]) / mesh.cell_h[own, None]
            xn = (mesh.fq_point - mesh.face_shift[mesh.fq_face] - mesh.cell_centroid[nb]) / mesh.cell_h[nb, None]
            self._tables = (monomial_rows(xo) - self.avg0[own], monomial_grad_rows(xo) / mesh.cell_h[own, None, None],
                            monomial_rows(xn) - self.avg0[nb], monomial_grad_rows(xn) / mesh.cell_h[nb, None, None])
        return self._tables

    phi_owner = property(lambda self: self._face_tables()[0])
    dphi_owner = property(lambda self: self._face_tables()[1])
    phi_neighbor = property(lambda self: self._face_tables()[2])
    dphi_neighbor = property(lambda self: self._face_tables()[3])


# -- WENO ----------------------------------------------------------------------------


class WenoReconstructor:
    """Third-order simple WENO over the two-level stencil (recon.py:198-294);
    weights="linear" keeps the big polynomial."""

    def __init__(self, geom: ReconGeometry, eps=WENO_EPS, lin_weight=LINEAR_WEIGHT, weights="nonlinear"):
        if weights not in ("nonlinear", "linear"):
            raise ValueError(f"weights must be 'nonlinear' or 'linear', got {weights!r}")
        self.geom = geom
        self.eps = eps
        self.lin_weight = lin_weight
        self.weights = weights
        ops = N.NativeSetup(geom.mesh, schemes=1)
        self.big_op = np.array(ops.array("weno_big_op"))
        self.big_gather = np.array(ops.array("weno_big_gather"))
        self.big_degree = np.array(ops.array("weno_big_degree"))
        self.sub_op = np.array(ops.array("weno_sub_op"))
        self.sub_gather = np.array(ops.array("weno_sub_gather"))
        self.sub_active = np.array(ops.array("weno_sub_active")).astype(bool)

    def _solver(self):
        return _handle(self.geom.mesh, "weno_gmres", self.eps, self.lin_weight)

    def candidate_coeffs(self, field):
        """(c_big (nc, 9, m), b_sub (nc, M, 3, m)) of an (nc, m) field."""
        return _device_candidates(self._solver(), _field(field))

    def combined_coeffs(self, field):
        return _device_combined(self._solver(), _field(field), None, self.weights == "linear")


def combine_candidates(c_big, b_sub, active, beta_mat, eps=WENO_EPS, lin_weight=LINEAR_WEIGHT):
    """Nonlinear blend of candidate coefficients per cell and component
    (recon.py:167-195) -> (combined (n, 9, m), w0n (n, m), wmn (n, M, m))."""
    c_big = np.ascontiguousarray(c_big, dtype=float)
    n, _, m = c_big.shape
    if b_sub.shape[1] == 0:
        return c_big.copy(), np.ones((n, m)), np.zeros((n, 0, m))
    M = b_sub.shape[1]
    out = np.empty_like(c_big)
    w0n = np.empty((n, m))
    wmn = np.empty((n, M, m))
    act = np.ascontiguousarray(active, dtype=np.int8)
    N.check(N.load().gks_combine_candidates(
        n, m, M, N.dptr(c_big), N.dptr(np.ascontiguousarray(b_sub, dtype=float)),
        act.ctypes.data_as(C.c_void_p), N.dptr(np.ascontiguousarray(beta_mat, dtype=float)), float(eps),
        float(lin_weight), N.dptr(out), N.dptr(w0n), N.dptr(wmn)))
    return out, w0n, wmn


def evaluate_faces(geom: ReconGeometry, field, coeffs):
    """Face-point values and gradients of both sides (recon.py:297-314);
    boundary points repeat the owner side."""
    field = _field(field)
    coeffs = np.asarray(coeffs, dtype=float)
    s = _handle(geom.mesh, "weno_gmres")
    lib = N.load()
    nfq = geom.mesh.nfq
    m = field.shape[1]
    val_o, val_n = np.empty((nfq, m)), np.empty((nfq, m))
    grad_o, grad_n = np.empty((nfq, 3, m)), np.empty((nfq, 3, m))
    for sl, k in _chunks(m):
        q5, c5 = _pad5(field, sl, k), _pad5(coeffs, sl, k)
        vo, vn = np.empty((nfq, 5)), np.empty((nfq, 5))
        go, gn = np.empty((nfq, 3, 5)), np.empty((nfq, 3, 5))
        N.check(lib.gks_face_values(s._handle, N.dptr(q5), N.dptr(c5), N.dptr(vo), N.dptr(go), N.dptr(vn),
                                    N.dptr(gn)))
        val_o[:, sl], val_n[:, sl] = vo[:, :k], vn[:, :k]
        grad_o[..., sl], grad_n[..., sl] = go[..., :k], gn[..., :k]
    return val_o, grad_o, val_n, grad_n


# -- single-cell views ---------------------------------------------------------------


def _poly(geom, c, q0, coeffs, degree):
    mesh = geom.mesh
    return ReconPolynomial(cell=int(c), q0=q0, coeffs=coeffs, degree=int(degree), centroid=mesh.cell_centroid[c],
                           h=float(mesh.cell_h[c]), basis_offset=geom.avg0[c])


def _linear(b, m):
    coeffs = np.zeros((NCOEF, m))
    coeffs[:3] = b
    return coeffs


def fit_big_polynomial(recon: WenoReconstructor, c, field) -> ReconPolynomial:
    """The quadratic (or degenerate-stencil linear) candidate of cell c."""
    field = _field(field)
    c_big, _ = recon.candidate_coeffs(field)
    return _poly(recon.geom, c, field[c], c_big[c], recon.big_degree[c])


def fit_sub_polynomials(recon: WenoReconstructor, c, field) -> list[ReconPolynomial]:
    """The linear candidates of cell c, one per surviving sub-stencil."""
    field = _field(field)
    _, b_sub = recon.candidate_coeffs(field)
    return [_poly(recon.geom, c, field[c], _linear(b_sub[c, mm], field.shape[1]), 1)
            for mm in np.flatnonzero(recon.sub_active[c])]


def smoothness_indicator(geom: ReconGeometry, poly: ReconPolynomial):
    """beta of one candidate (recon.py:370-375): the cell's quadratic form on
    its coefficients; linear candidates reduce to |grad|^2 in the chart."""
    a = poly.coeffs
    if poly.degree == 1:
        return np.sum(a[:3] * a[:3], axis=0)
    return np.sum(a * (geom.beta_mat[poly.cell] @ a), axis=0)


def nonlinear_combine(p0, subs, betas, lin_weight, eps, point):
    """Value and gradient of the weighted candidate blend at one point
    (recon.py:378-406): w0 = g0 (1 + tau / (beta0 + eps)), w_m = g (1 + tau /
    (beta_m + eps)), tau = mean |beta0 - beta_m|; the big candidate enters
    as (p0 - g sum_m p_m) / g0."""
    m = len(subs)
    if m == 0:
        return p0.value(point), p0.gradient(point)
    b = [np.atleast_1d(np.asarray(x, dtype=float)) for x in betas]
    g0 = 1.0 - lin_weight * m
    tau = np.sum([np.abs(b[0] - bm) for bm in b[1:]], axis=0) / m
    w = np.array([g0 * (1.0 + tau / (b[0] + eps))] + [lin_weight * (1.0 + tau / (bm + eps)) for bm in b[1:]])
    w = w / np.sum(w, axis=0)

    def blend(f):
        vals = [f(p) for p in [p0] + list(subs)]
        big = (vals[0] - lin_weight * np.sum(vals[1:], axis=0)) / g0
        return w[0] * big + np.sum([wk * v for wk, v in zip(w[1:], vals[1:])], axis=0)

    return blend(lambda p: p.value(point)), blend(lambda p: p.gradient(point))
