"""Boundary patch specifications (mirrors gks3d/boundary.py:18-48).

The ghost-state arithmetic itself (boundary.py:66-171) runs on the device,
fused into the face kernel (csrc/gks_solver.cuh: ghost_state /
ghost_gradients).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

WALL_KINDS = ("wall_noslip_isothermal", "wall_noslip_adiabatic", "wall_slip_adiabatic")
PATCH_KINDS = WALL_KINDS + ("farfield_riemann", "supersonic_inlet", "supersonic_outlet", "periodic")

# C ABI patch kind ids (include/gks.h GKS_PATCH_*)
KIND_ID = {
    "wall_noslip_isothermal": 0,
    "wall_noslip_adiabatic": 1,
    "wall_slip_adiabatic": 2,
    "farfield_riemann": 3,
    "supersonic_inlet": 4,
    "supersonic_outlet": 5,
}


class BoundaryError(ValueError):
    pass


@dataclass
class PatchSpec:
    """Configuration of one boundary patch."""

    name: str
    kind: str
    reference: np.ndarray | None = None  # (rho, U, V, W, p)
    lambda_wall: float | None = None
    velocity: np.ndarray = field(default_factory=lambda: np.zeros(3))
    mate: str | None = None

    def __post_init__(self):
        if self.kind not in PATCH_KINDS:
            raise BoundaryError(f"patch {self.name!r}: unknown kind {self.kind!r}")
        if self.kind in ("farfield_riemann", "supersonic_inlet") and self.reference is None:
            raise BoundaryError(f"patch {self.name!r}: kind {self.kind} needs a reference state")
        if self.kind == "wall_noslip_isothermal" and self.lambda_wall is None:
            raise BoundaryError(f"patch {self.name!r}: isothermal wall needs lambda_wall")
        if self.reference is not None:
            self.reference = np.asarray(self.reference, dtype=float)
            if self.reference[0] <= 0.0 or self.reference[4] <= 0.0:
                raise BoundaryError(f"patch {self.name!r}: invalid reference state")
        self.velocity = np.asarray(self.velocity, dtype=float)


def _patch_desc(spec: PatchSpec):
    from . import _native as N

    d = N.GksPatchDesc()
    d.kind = KIND_ID.get(spec.kind, -1)
    if spec.reference is not None:
        for k in range(5):
            d.reference[k] = float(spec.reference[k])
    else:
        d.reference[0], d.reference[4] = 1.0, 1.0
    d.lambda_wall = float(spec.lambda_wall) if spec.lambda_wall is not None else 0.0
    for k in range(3):
        d.velocity[k] = float(spec.velocity[k])
    return d


def _ghost_batch(q, grad, spec, normal, gamma):
    import ctypes as C

    from . import _native as N
    from .kinetic import UnphysicalStateError

    if spec.kind not in KIND_ID:
        raise BoundaryError(f"patch {spec.name!r}: kind {spec.kind} has no ghost state")
    n = q.shape[0]
    q_out = np.empty((n, 5))
    g_out = np.empty((n, 3, 5)) if grad is not None else None
    d = _patch_desc(spec)
    lib = N.load()
    rc = lib.gks_ghost_batch(n, C.byref(d), N.dptr(q), N.dptr(normal), N.dptr(grad), float(gamma), N.dptr(q_out),
                             N.dptr(g_out))
    if rc == N.GKS_ERR_UNPHYSICAL:
        raise UnphysicalStateError(lib.gks_last_error().decode())
    N.check(rc)
    return q_out, g_out


def ghost_state(q_interior, spec: PatchSpec, normal, gamma: float = 1.4):
    """Exterior conserved state across a boundary face (boundary.py:66-100),
    evaluated by the device ghost_state the face kernel fuses."""
    from . import _native as N

    shape = np.shape(q_interior)
    q = N.f64(np.atleast_2d(q_interior), (-1, 5))
    n = N.f64(np.broadcast_to(np.asarray(normal, dtype=float), (q.shape[0], 3)))
    return _ghost_batch(q, None, spec, n, gamma)[0].reshape(shape)


def ghost_gradients(grad_interior, spec: PatchSpec, normal):
    """Exterior gradients (boundary.py:144-171): interior copy, walls get the
    mirror-image field's (device ghost_gradients)."""
    from . import _native as N

    g = np.asarray(grad_interior, dtype=float)
    if spec.kind not in WALL_KINDS:
        return g.copy()
    shape = g.shape
    gg = N.f64(g.reshape(-1, 3, 5))
    n = N.f64(np.broadcast_to(np.asarray(normal, dtype=float), (gg.shape[0], 3)))
    # any physical interior state: only the gradient mirror is wanted
    q = np.tile([1.0, 0.0, 0.0, 0.0, 2.5], (gg.shape[0], 1))
    return _ghost_batch(q, gg, spec, n, 1.4)[1].reshape(shape)
