"""Kinetic constants, state conversions, exception types and the Maxwellian
moment tables.

Mirrors gks3d/kinetic.py: the host helpers of :17-87 used for setup
(initial fields, patch references), and the MomentTable / build_moments
API (:90-162), whose tables are computed on the device (gks_moment_table,
the recurrences of csrc/gks_flux.cu k_moment_table).  psi_moments queries a
table like the reference (:191-220).  The per-point moment engine of the
flux itself only exists on the device (csrc/gks_kinetic.cuh).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

DEFAULT_GAMMA = 1.4
MAX_UORDER = 6   # kinetic.py:22
MAX_XIORDER = 2  # kinetic.py:23


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


def check_primitive(w):
    """Raise UnphysicalStateError on rho <= 0, lam <= 0 or non-finite entries (kinetic.py:80-87)."""
    w = np.asarray(w, dtype=float)
    bad = (w[..., 0] <= 0.0) | (w[..., 4] <= 0.0) | ~np.all(np.isfinite(w), axis=-1)
    if np.any(bad):
        raise UnphysicalStateError(f"invalid primitive state at {np.argwhere(bad)[:8].tolist()}")


@dataclass
class MomentTable:
    """Density-normalised Maxwellian moments of a state batch (kinetic.py:90-110):
    order-first arrays u_full[p] = <u^p>, u_pos / u_neg the u > 0 / u < 0
    half ranges, v_full, w_full the tangential moments, xi[s] = <xi^2s>."""

    u_full: np.ndarray
    u_pos: np.ndarray
    u_neg: np.ndarray
    v_full: np.ndarray
    w_full: np.ndarray
    xi: np.ndarray
    rho: np.ndarray


def build_moments(w, gamma: float = DEFAULT_GAMMA, max_order: int = MAX_UORDER) -> MomentTable:
    """Moment tables of a primitive-state batch, computed on the device."""
    from . import _native as N

    w = np.asarray(w, dtype=float)
    check_primitive(w)
    shape = w.shape[:-1]
    flat = N.f64(w.reshape(-1, 5))
    n = flat.shape[0]
    tabs = [np.empty((max_order + 1, n)) for _ in range(5)]
    xi = np.empty((MAX_XIORDER + 1, n))
    rc = N.load().gks_moment_table(n, N.dptr(flat), float(gamma), int(max_order), *(N.dptr(t) for t in tabs),
                                   N.dptr(xi))
    N.check(rc)
    for t in tabs + [xi]:
        if not np.all(np.isfinite(t)):
            raise UnphysicalStateError("moment table overflow: state out of range")
    tabs = [t.reshape((-1,) + shape) for t in tabs]
    return MomentTable(*tabs, xi.reshape((-1,) + shape), w[..., 0].copy())


def _moment(tab: MomentTable, umode, p, q, r, s):
    u = {"full": tab.u_full, "pos": tab.u_pos, "neg": tab.u_neg}[umode]
    if p >= len(u) or q >= len(tab.v_full) or r >= len(tab.w_full) or s >= len(tab.xi):
        raise ValueError(f"moment order ({p},{q},{r},{s}) exceeds tabulated range")
    return u[p] * tab.v_full[q] * tab.w_full[r] * tab.xi[s]


def psi_moments(tab: MomentTable, p: int, q: int, r: int, s: int = 0, umode: str = "full"):
    """<u^p v^q w^r xi^2s psi> per state, psi = (1, u, v, w, |c|^2 / 2): shape (..., 5)."""
    m = lambda a, b, c, d: _moment(tab, umode, a, b, c, d)  # noqa: E731
    e = 0.5 * (m(p + 2, q, r, s) + m(p, q + 2, r, s) + m(p, q, r + 2, s) + m(p, q, r, s + 1))
    return np.stack([m(p, q, r, s), m(p + 1, q, r, s), m(p, q + 1, r, s), m(p, q, r + 1, s), e], axis=-1)


def conserved_from_moments(tab: MomentTable):
    """Conserved 5-vector rho <psi> of a table (kinetic.py:315-317)."""
    return tab.rho[..., None] * psi_moments(tab, 0, 0, 0)


def _slopes(w, rhs, time_slope, gamma):
    from . import _native as N

    w = np.asarray(w, dtype=float)
    shape = w.shape
    wf = N.f64(w.reshape(-1, 5))
    r = N.f64(np.asarray(rhs, dtype=float).reshape(wf.shape[0], -1))
    out = np.empty((wf.shape[0], 5))
    lib = N.load()
    rc = lib.gks_slopes(wf.shape[0], N.dptr(wf), N.dptr(r), int(time_slope), float(gamma), N.dptr(out))
    if rc == N.GKS_ERR_UNPHYSICAL:
        raise UnphysicalStateError(lib.gks_last_error().decode())
    N.check(rc)
    return out.reshape(shape)


def solve_micro_slope(w, dq, gamma: float = DEFAULT_GAMMA):
    """a with <a psi g> = dq / rho (kinetic.py:271-302), the closed-form solve on the device."""
    return _slopes(w, dq, False, gamma)


def solve_time_slope(w, a1, a2, a3, gamma: float = DEFAULT_GAMMA, tab=None):
    """Time slope A from <(a1 u + a2 v + a3 w + A) psi> = 0 (kinetic.py:305-312), on the device."""
    a = np.stack([np.asarray(a1, dtype=float), np.asarray(a2, dtype=float), np.asarray(a3, dtype=float)], axis=-2)
    return _slopes(w, a, True, gamma)


def slope_psi_moments(tab: MomentTable, slope, p: int, q: int, r: int, umode: str = "full"):
    """<a(c) u^p v^q w^r psi> for a(c) = a1 + a2 u + a3 v + a4 w + a5 |c|^2 / 2
    (kinetic.py:222-255): a combination of the table's psi-moments."""
    a = np.asarray(slope, dtype=float)
    pm = lambda *o: psi_moments(tab, *o, umode=umode)  # noqa: E731
    out = a[..., 0, None] * pm(p, q, r, 0) + a[..., 1, None] * pm(p + 1, q, r, 0) + \
        a[..., 2, None] * pm(p, q + 1, r, 0) + a[..., 3, None] * pm(p, q, r + 1, 0)
    return out + (0.5 * a[..., 4, None]) * (pm(p + 2, q, r, 0) + pm(p, q + 2, r, 0) + pm(p, q, r + 2, 0) +
                                            pm(p, q, r, 1))


def directional_slope_psi_moments(tab: MomentTable, a1, a2, a3, p: int, q: int, r: int, umode: str = "full"):
    """<(a1 u + a2 v + a3 w) u^p v^q w^r psi> (kinetic.py:258-268)."""
    return slope_psi_moments(tab, a1, p + 1, q, r, umode) + slope_psi_moments(tab, a2, p, q + 1, r, umode) + \
        slope_psi_moments(tab, a3, p, q, r + 1, umode)
