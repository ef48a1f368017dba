"""Compact HWENO reconstruction API and gradient update (mirrors gks3d/hweno.py).

HwenoReconstructor (hweno.py:32-169): the operators of the native setup in
the reference's padded layout; candidate_coeffs / combined_coeffs run on the
GPU (gks_recon_candidates, and the solver's own k_recon_hweno through
gks_recon_coeffs).  fit_big_hermite / fit_sub_hermite (hweno.py:200-245)
select one cell's device-computed candidates.

update_gradients(mesh, point_values): cell-averaged gradients from the
interface point values by the Gauss theorem, |Omega| grad Q = sum over the
cell's face points of w S n Q_G (owner +, neighbour -).  Runs on the device
(gks_update_gradients: the assembly kernel of the residual pipeline with
zero flux contributions) on a cached handle of the mesh.  The HWENO
reconstruction operators themselves are built by the native setup
(csrc/gks_setup.cpp) and applied by k_recon_hweno.
"""

from __future__ import annotations

import numpy as np

from . import _native as N
from .kinetic import DEFAULT_GAMMA
from .recon import (LINEAR_WEIGHT, WENO_EPS, ReconGeometry, ReconPolynomial, _device_candidates, _device_combined,
                    _field, _handle, _linear, _poly)


def _grad(grad):
    grad = np.asarray(grad, dtype=float)
    return grad[:, :, None] if grad.ndim == 2 else grad


class HwenoReconstructor:
    """Compact reconstruction from averages and average gradients."""

    def __init__(self, geom: ReconGeometry, eps=WENO_EPS, lin_weight=LINEAR_WEIGHT, weights="nonlinear"):
        if weights not in ("nonlinear", "linear"):
            raise ValueError(f"weights must be 'nonlinear' or 'linear', got {weights!r}")
        self.geom = geom
        self.eps = eps
        self.lin_weight = lin_weight
        self.weights = weights
        ops = N.NativeSetup(geom.mesh, schemes=2)
        for name in ("big_op", "big_avg_gather", "big_grad_gather", "big_grad_scale", "big_ncols", "big_degree",
                     "sub_op", "sub_gather"):
            setattr(self, name, np.array(ops.array("hweno_" + name)))
        self.sub_active = np.array(ops.array("hweno_sub_active")).astype(bool)

    def _solver(self):
        return _handle(self.geom.mesh, "hweno_gmres", self.eps, self.lin_weight)

    def _grad_rows(self, c, ids, shifts):
        """h_j * cell-mean gradient rows of the basis over members (j, s),
        target included, in the chart of c (hweno.py:45-60): (3 len(ids), 9)."""
        from .recon import monomial_grad_rows

        mesh = self.geom.mesh
        h0 = mesh.cell_h[c]
        out = np.empty((3 * len(ids), 9))
        for r, (j, s) in enumerate(zip(ids, shifts)):
            pts, w = mesh.cell_quadrature_of(int(j), s)
            out[3 * r:3 * r + 3] = mesh.cell_h[j] * (np.tensordot(w, monomial_grad_rows((pts - mesh.cell_centroid[c]) / h0),
                                                                  axes=1) / h0)
        return out

    def candidate_coeffs(self, field, grad):
        """(c_big (nc, 9, m), b_sub (nc, M, 3, m)) from an (nc, m) field and its (nc, 3, m) gradients."""
        return _device_candidates(self._solver(), _field(field), _grad(grad))

    def combined_coeffs(self, field, grad):
        return _device_combined(self._solver(), _field(field), _grad(grad), self.weights == "linear")


def fit_big_hermite(recon: HwenoReconstructor, c, field, grad) -> ReconPolynomial:
    """The quadratic compact candidate of cell c."""
    field = _field(field)
    c_big, _ = recon.candidate_coeffs(field, grad)
    return _poly(recon.geom, c, field[c], c_big[c], recon.big_degree[c])


def fit_sub_hermite(recon: HwenoReconstructor, c, field, grad) -> list[ReconPolynomial]:
    """The linear two-cell candidates of cell c, one per surviving face neighbour."""
    field = _field(field)
    _, b_sub = recon.candidate_coeffs(field, grad)
    return [_poly(recon.geom, c, field[c], _linear(b_sub[c, mm], field.shape[1]), 1)
            for mm in np.flatnonzero(recon.sub_active[c])]


def update_gradients(mesh, point_values, gamma: float = DEFAULT_GAMMA):
    from .stepping import _jacobian_handle

    s = _jacobian_handle(mesh, gamma)  # reference numbering (no reorder)
    vals = np.asarray(point_values, dtype=float)
    nfq, m = vals.shape
    out = np.empty((mesh.ncells, 3, m))
    # the device assembles 5 components at a time (zero-padded)
    for c0 in range(0, m, 5):
        k = min(5, m - c0)
        qpt = np.zeros((nfq, 5))
        qpt[:, :k] = vals[:, c0:c0 + k]
        g = np.empty((mesh.ncells, 3, 5))
        N.check(N.load().gks_update_gradients(s._handle, N.dptr(qpt), N.dptr(g)))
        out[:, :, c0:c0 + k] = g[:, :, :k]
    return out
