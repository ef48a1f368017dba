"""Host-side kinetic constants, state conversions and exception types.

Mirrors the small host helpers of gks3d/kinetic.py (:17-87) that the case
API uses for setup (initial fields, patch references).  The per-point
moment engine itself only exists on the device (csrc/gks_kinetic.cuh).
"""

from __future__ import annotations

import numpy as np

DEFAULT_GAMMA = 1.4


class UnphysicalStateError(ValueError):
    """Raised when a state has non-positive density or internal energy (kinetic.py:26)."""


def internal_dof(gamma: float) -> float:
    return (5.0 - 3.0 * gamma) / (gamma - 1.0)


def conserved_to_primitive(q, gamma: float = DEFAULT_GAMMA):
    q = np.asarray(q, dtype=float)
    rho = q[..., 0]
    if np.any(rho <= 0.0) or not np.all(np.isfinite(rho)):
        raise UnphysicalStateError("non-positive density")
    vel = q[..., 1:4] / rho[..., None]
    e_int = q[..., 4] - 0.5 * np.sum(q[..., 1:4] * vel, axis=-1)
    if np.any(e_int <= 0.0) or not np.all(np.isfinite(e_int)):
        raise UnphysicalStateError("non-positive internal energy")
    out = np.empty_like(q)
    out[..., 0] = rho
    out[..., 1:4] = vel
    out[..., 4] = (internal_dof(gamma) + 3.0) * rho / (4.0 * e_int)
    return out


def primitive_to_conserved(w, gamma: float = DEFAULT_GAMMA):
    w = np.asarray(w, dtype=float)
    rho = w[..., 0]
    out = np.empty_like(w)
    out[..., 0] = rho
    out[..., 1:4] = rho[..., None] * w[..., 1:4]
    out[..., 4] = 0.5 * rho * np.sum(w[..., 1:4] ** 2, axis=-1) + \
        (internal_dof(gamma) + 3.0) * rho / (4.0 * w[..., 4])
    return out


def pressure(w):
    w = np.asarray(w, dtype=float)
    return w[..., 0] / (2.0 * w[..., 4])


def sound_speed(w, gamma: float = DEFAULT_GAMMA):
    w = np.asarray(w, dtype=float)
    return np.sqrt(gamma / (2.0 * w[..., 4]))
