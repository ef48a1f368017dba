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
