"""Gas-kinetic interface flux API (device-backed).

Mirrors gks3d/flux.py: build_interface (:69-107), evolve_flux (:162-179),
point_value (:182-188), instantaneous_flux (:191-197), kfvs_flux (:200-208), collision_time (:211-227),
rotate_to_local / rotate_to_global (:230-243), euler_flux_local
(:246-260), compatibility_residual (:263-268).  The interface distribution
is evaluated by the fused sm_100a kernel behind gks_flux_batch; the
InterfaceBatch also carries the reference's intermediates (micro-slopes,
time slopes, compatibility state and its slopes, from gks_interface_data)
and the three moment tables (build_moments, gks_moment_table).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as N
from .kinetic import DEFAULT_GAMMA, MomentTable, UnphysicalStateError, build_moments, psi_moments


@dataclass
class InterfaceBatch:
    """States, micro-slopes and compatibility data of a point batch
    (flux.py:34-66); sl / sr keep the conserved slopes the device flux
    kernel starts from."""

    wl: np.ndarray
    wr: np.ndarray
    sl: np.ndarray
    sr: np.ndarray
    gamma: float = DEFAULT_GAMMA
    al: np.ndarray = None   # (n, 3, 5) left micro-slopes along the local axes
    ar: np.ndarray = None
    atl: np.ndarray = None  # (n, 5) left time slope
    atr: np.ndarray = None
    w0: np.ndarray = None   # (n, 5) compatibility (equilibrium) state
    abar: np.ndarray = None
    atbar: np.ndarray = None
    tab_l: MomentTable = None
    tab_r: MomentTable = None
    tab_0: MomentTable = None

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
    out = {k: np.empty((n, 3, 5) if k in ("al", "ar", "abar") else (n, 5))
           for k in ("al", "ar", "atl", "atr", "w0", "abar", "atbar")}
    lib = N.load()
    rc = lib.gks_interface_data(n, N.dptr(wl), N.dptr(wr), N.dptr(sl), N.dptr(sr), float(gamma),
                                *(N.dptr(out[k]) for k in ("al", "ar", "atl", "atr", "w0", "abar", "atbar")))
    if rc == N.GKS_ERR_UNPHYSICAL:
        raise UnphysicalStateError(lib.gks_last_error().decode())
    N.check(rc)
    return InterfaceBatch(wl, wr, sl, sr, gamma, tab_l=build_moments(wl, gamma), tab_r=build_moments(wr, gamma),
                          tab_0=build_moments(out["w0"], gamma), **out)


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


def instantaneous_flux(ib: InterfaceBatch, tau, t):
    """Local-frame moment flux int u psi f at the instant t (flux.py:191-197)."""
    n = ib.n
    tau = N.f64(np.broadcast_to(np.asarray(tau, dtype=float), (n,)))
    t = N.f64(np.broadcast_to(np.asarray(t, dtype=float), (n,)))
    flux = np.empty((n, 5))
    lib = N.load()
    rc = lib.gks_instant_flux_batch(n, N.dptr(ib.wl), N.dptr(ib.wr), N.dptr(ib.sl), N.dptr(ib.sr), N.dptr(tau),
                                    N.dptr(t), ib.gamma, N.dptr(flux))
    if rc == N.GKS_ERR_UNPHYSICAL:
        raise UnphysicalStateError(lib.gks_last_error().decode())
    N.check(rc)
    return flux


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


def euler_flux_local(w, gamma: float = DEFAULT_GAMMA):
    """Analytic Euler flux of a local-frame primitive state along the normal (flux.py:246-260)."""
    from .kinetic import primitive_to_conserved

    w = np.atleast_2d(np.asarray(w, dtype=float))
    q = primitive_to_conserved(w, gamma)
    p = w[:, 0] / (2.0 * w[:, 4])
    u = w[:, 1]
    out = q * u[:, None]
    out[:, 1] += p
    out[:, 4] += p * u
    return out


def compatibility_residual(ib: InterfaceBatch):
    """max |rho0 <psi>_0 - (rho_l <psi>_{l,u>0} + rho_r <psi>_{r,u<0})| (flux.py:263-268)."""
    lhs = ib.w0[:, 0, None] * psi_moments(ib.tab_0, 0, 0, 0)
    rhs = ib.wl[:, 0, None] * psi_moments(ib.tab_l, 0, 0, 0, umode="pos") + \
        ib.wr[:, 0, None] * psi_moments(ib.tab_r, 0, 0, 0, umode="neg")
    return float(np.max(np.abs(lhs - rhs)))


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
