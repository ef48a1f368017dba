"""Linear solvers on the device block system (mirrors gks3d/krylov.py).

gmres_solve runs the reference's left-preconditioned restarted GMRES
(krylov.py:55-140: Arnoldi MGS with one conditional re-orthogonalisation,
Givens rotations, happy-breakdown / early exit) entirely on the GPU with the
Hessenberg scalars kept in device memory; jacobi_precondition is the fixed
count block-Jacobi of krylov.py:24-34.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .jacobian import BlockJacobian

MAX_DIM = 64
MAX_RESTARTS = 64


class SolverError(RuntimeError):
    pass


class GksGmresInfo(C.Structure):
    _fields_ = [("ncycles", C.c_int), ("matvecs", C.c_int), ("breakdown", C.c_int), ("ortho_error", C.c_double),
                ("cycle_len", C.c_int * MAX_RESTARTS), ("norms", C.c_double * (MAX_RESTARTS * (MAX_DIM + 1)))]


@dataclass
class GmresInfo:
    """Per-cycle preconditioned residual norms and counters (krylov.py:37-52)."""

    cycle_residuals: list = field(default_factory=list)
    matvecs: int = 0
    breakdown: bool = False
    ortho_error: float = 0.0

    @property
    def initial_residual(self):
        return self.cycle_residuals[0][0] if self.cycle_residuals else 0.0

    @property
    def final_residual(self):
        return self.cycle_residuals[-1][-1] if self.cycle_residuals else 0.0

    @classmethod
    def from_c(cls, ci: GksGmresInfo):
        cyc = []
        for c in range(ci.ncycles):
            base = c * (MAX_DIM + 1)
            cyc.append([float(ci.norms[base + k]) for k in range(ci.cycle_len[c])])
        return cls(cyc, int(ci.matvecs), bool(ci.breakdown), float(ci.ortho_error))


def _raise_solver(rc):
    lib = N.load()
    msg = lib.gks_last_error().decode(errors="replace")
    if rc in (N.GKS_ERR_SINGULAR, N.GKS_ERR_NONFINITE):
        raise SolverError(msg)
    N.check(rc)


def jacobi_precondition(a: BlockJacobian, b, k_max: int = 2, diag_inv=None):
    """Fixed-count block-Jacobi approximation of A^-1 b (device)."""
    b = N.f64(b, (a.ncells, 5))
    z = np.empty_like(b)
    rc = N.load().gks_blocksys_jacobi(a._ptr, N.dptr(b), int(k_max), N.dptr(z))
    if rc:
        _raise_solver(rc)
    return z


def gmres_solve(a: BlockJacobian, b, m: int = 10, restarts: int = 3, k_max: int = 2,
                rtol: float = 0.0, atol: float = 0.0, check_orthogonality: bool = False):
    """Restarted GMRES with Jacobi preconditioning; returns (x, GmresInfo)."""
    if not 1 <= m <= MAX_DIM or not 1 <= restarts <= MAX_RESTARTS:
        raise ValueError(f"krylov_dim must be in [1, {MAX_DIM}] and restarts in [1, {MAX_RESTARTS}]")
    b = N.f64(b, (a.ncells, 5))
    x = np.zeros_like(b)
    info = GksGmresInfo()
    rc = N.load().gks_gmres(a._ptr, N.dptr(b), N.dptr(x), int(m), int(restarts), int(k_max), float(rtol),
                            float(atol), int(bool(check_orthogonality)), C.byref(info))
    if rc:
        _raise_solver(rc)
    return x, GmresInfo.from_c(info)


def lusgs_sweep(a, r):
    """The sequential LUSGS baseline (krylov.py:143-168) is not on the device path."""
    raise NotImplementedError("lusgs_sweep is the reference's sequential CPU baseline; "
                              "the B200 build solves with device GMRES (see DESIGN.md)")
