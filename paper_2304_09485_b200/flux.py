"""Gas-kinetic interface flux API (device-backed).

Mirrors gks3d/flux.py: build_interface (:69-107), evolve_flux (:162-179),
point_value (:182-188), kfvs_flux (:200-208), collision_time (:211-227),
rotate_to_local / rotate_to_global (:230-243).  The interface distribution
is evaluated by the fused sm_100a kernel behind gks_flux_batch; the batch
object only carries the local states and slopes.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as N
from .kinetic import DEFAULT_GAMMA, UnphysicalStateError


@dataclass
class InterfaceBatch:
    wl: np.ndarray
    wr: np.ndarray
    sl: np.ndarray
    sr: np.ndarray
    gamma: float = DEFAULT_GAMMA

    @property
    def n(self):
        return self.wl.shape[0]


def _check_prim(w):
    bad = (w[:, 0] <= 0.0) | (w[:, 4] <= 0.0) | ~np.all(np.isfinite(w), axis=1)
    if np.any(bad):
        raise UnphysicalStateError(f"invalid primitive state at {np.argwhere(bad)[:8].tolist()}")


def build_interface(wl, wr, slopes_l=None, slopes_r=None, gamma: float = DEFAULT_GAMMA) -> InterfaceBatch:
    wl = N.f64(np.atleast_2d(wl))
    wr = N.f64(np.atleast_2d(wr))
    _check_prim(wl)
    _check_prim(wr)
    n = wl.shape[0]
    sl = np.zeros((n, 3, 5)) if slopes_l is None else N.f64(slopes_l, (n, 3, 5))
    sr = np.zeros((n, 3, 5)) if slopes_r is None else N.f64(slopes_r, (n, 3, 5))
    return InterfaceBatch(wl, wr, sl, sr, gamma)


def _run(ib: InterfaceBatch, tau, dt, tp):
    n = ib.n
    tau = N.f64(np.broadcast_to(np.asarray(tau, dtype=float), (n,)))
    dt = N.f64(np.broadcast_to(np.asarray(dt, dtype=float), (n,)))
    flux = np.empty((n, 5))
    point = np.empty((n, 5)) if tp is not None else None
    if tp is not None:
        tp = N.f64(np.broadcast_to(np.asarray(tp, dtype=float), (n,)))
    lib = N.load()
    rc = lib.gks_flux_batch(n, N.dptr(ib.wl), N.dptr(ib.wr), N.dptr(ib.sl), N.dptr(ib.sr),
                            N.dptr(tau), N.dptr(dt), N.dptr(tp), ib.gamma, N.dptr(flux),
                            N.dptr(point))
    if rc == N.GKS_ERR_UNPHYSICAL:
        raise UnphysicalStateError(lib.gks_last_error().decode())
    N.check(rc)
    return flux, point


def evolve_flux(ib: InterfaceBatch, tau, dt):
    """Time-averaged local-frame flux (1/dt) int_0^dt int u psi f."""
    return _run(ib, tau, dt, None)[0]


def point_value(ib: InterfaceBatch, tau, t):
    """Interface conserved state int psi f at time t, local frame."""
    return _run(ib, tau, np.ones(ib.n), t)[1]


def kfvs_flux(wl, wr, gamma: float = DEFAULT_GAMMA):
    """Collisionless split flux: the tau >> dt limit of the same kernel."""
    ib = build_interface(wl, wr, gamma=gamma)
    return evolve_flux(ib, np.inf, 1.0)


def collision_time(model, dt, p_l, p_r, mu=0.0, p_eq=None):
    p_l = np.asarray(p_l, dtype=float)
    p_r = np.asarray(p_r, dtype=float)
    jump = np.abs(p_l - p_r) / (p_l + p_r) * dt
    if model == "inviscid":
        return 0.1 * dt + jump
    if model == "viscous":
        if p_eq is None:
            raise ValueError("viscous collision time needs the equilibrium pressure")
        return mu / np.asarray(p_eq, dtype=float) + jump
    raise ValueError(f"unknown collision model {model!r}")


def rotate_to_local(q, frame):
    q = np.asarray(q, dtype=float)
    out = q.copy()
    out[..., 1:4] = np.einsum("...ij,...j->...i", frame, q[..., 1:4])
    return out


def rotate_to_global(q, frame):
    q = np.asarray(q, dtype=float)
    out = q.copy()
    out[..., 1:4] = np.einsum("...ji,...j->...i", frame, q[..., 1:4])
    return out


def random_interface_inputs(rng, n, slope_scale=0.3):
    """Random physically valid interface states and slopes (flux.py:271-286)."""
    def states(k):
        w = np.empty((k, 5))
        w[:, 0] = rng.uniform(0.4, 1.6, k)
        w[:, 1] = rng.uniform(-1.0, 1.0, k)
        w[:, 2] = rng.uniform(-0.6, 0.6, k)
        w[:, 3] = rng.uniform(-0.6, 0.6, k)
        w[:, 4] = rng.uniform(0.5, 2.5, k)
        return w

    wl = states(n)
    wr = states(n)
    sl = slope_scale * rng.normal(size=(n, 3, 5))
    sr = slope_scale * rng.normal(size=(n, 3, 5))
    return wl, wr, sl, sr
