"""ORACLE (test infrastructure only): gas-kinetic interface flux.

Restates /root/reference/pkg/src/gks3d/flux.py: interface construction
(:69-107), the six-family moment assembly (:110-159), the time-integrated
flux (:162-179), the interface point value (:182-188), collision time
(:211-227) and the frame rotations (:230-243).
"""

from __future__ import annotations

import numpy as np

from .kinetic import GAMMA, Moments, cons_to_prim, micro_slope, pressure, prim_to_cons, time_slope


class Interface:
    """States, micro-slopes and the compatibility equilibrium per point."""

    def __init__(self, wl, wr, sl=None, sr=None, gamma=GAMMA):
        wl = np.atleast_2d(np.asarray(wl, dtype=float))
        wr = np.atleast_2d(np.asarray(wr, dtype=float))
        n = wl.shape[0]
        sl = np.zeros((n, 3, 5)) if sl is None else np.asarray(sl, dtype=float).reshape(n, 3, 5)
        sr = np.zeros((n, 3, 5)) if sr is None else np.asarray(sr, dtype=float).reshape(n, 3, 5)
        self.gamma = gamma
        self.wl, self.wr = wl, wr
        self.ml = Moments(wl, gamma)
        self.mr = Moments(wr, gamma)
        self.ml_pos = Moments(wl, gamma, "pos")
        self.mr_neg = Moments(wr, gamma, "neg")
        self.al = np.stack([micro_slope(wl, sl[:, k], gamma) for k in range(3)], axis=1)
        self.ar = np.stack([micro_slope(wr, sr[:, k], gamma) for k in range(3)], axis=1)
        self.Al = time_slope(wl, self.al[:, 0], self.al[:, 1], self.al[:, 2], self.ml, gamma)
        self.Ar = time_slope(wr, self.ar[:, 0], self.ar[:, 1], self.ar[:, 2], self.mr, gamma)
        # compatibility: the equilibrium carries the colliding half fluxes
        rl, rr = wl[:, 0, None], wr[:, 0, None]
        q0 = rl * self.ml_pos.psi(0, 0, 0) + rr * self.mr_neg.psi(0, 0, 0)
        self.w0 = cons_to_prim(q0, gamma)
        self.m0 = Moments(self.w0, gamma)
        self.abar = np.empty((n, 3, 5))
        for k in range(3):
            dq = rl * self.ml_pos.slope(self.al[:, k], 0, 0, 0) + rr * self.mr_neg.slope(self.ar[:, k], 0, 0, 0)
            self.abar[:, k] = micro_slope(self.w0, dq, gamma)
        self.Abar = time_slope(self.w0, self.abar[:, 0], self.abar[:, 1], self.abar[:, 2], self.m0, gamma)

    @property
    def n(self):
        return self.wl.shape[0]

    def families(self, p):
        """The six moment families of flux.py:110-159 against u^p psi."""
        rho0, rl, rr = self.w0[:, 0, None], self.wl[:, 0, None], self.wr[:, 0, None]
        a0, al, ar = self.abar, self.al, self.ar
        g_base = rho0 * self.m0.psi(p, 0, 0)
        g_slope = rho0 * self.m0.directional(a0[:, 0], a0[:, 1], a0[:, 2], p, 0, 0)
        g_time = rho0 * self.m0.slope(self.Abar, p, 0, 0)
        f_base = rl * self.ml_pos.psi(p, 0, 0) + rr * self.mr_neg.psi(p, 0, 0)
        f_slope = self.ml_pos.directional(rl * al[:, 0], rl * al[:, 1], rl * al[:, 2], p, 0, 0) + \
            self.mr_neg.directional(rr * ar[:, 0], rr * ar[:, 1], rr * ar[:, 2], p, 0, 0)
        f_time = self.ml_pos.slope(rl * self.Al, p, 0, 0) + self.mr_neg.slope(rr * self.Ar, p, 0, 0)
        return g_base, g_slope, g_time, f_base, f_slope, f_time

    def combine(self, coefs, p):
        fam = self.families(p)
        out = np.zeros((self.n, 5))
        for c, f in zip(coefs, fam):
            out += np.broadcast_to(np.asarray(c, dtype=float), (self.n,))[:, None] * f
        return out


def flux_coefficients(tau, dt):
    """Analytic time integrals of the five coefficient families (flux.py:162-179)."""
    x = dt / tau
    em1 = -np.expm1(-x)
    e = np.exp(-x)
    c1 = dt - tau * em1
    c2 = 2.0 * tau * tau * em1 - tau * dt * e - tau * dt
    c3 = 0.5 * dt * dt - tau * dt + tau * tau * em1
    c4 = tau * em1
    c5 = tau * tau * em1 - tau * dt * e
    return [c / dt for c in (c1, c2, c3, c4, -(tau * c4 + c5), -tau * c4)]


def evolve_flux(ib: Interface, tau, dt):
    """(1/dt) int_0^dt int u psi f, local frame  (flux.py:162-179)."""
    tau = np.broadcast_to(np.asarray(tau, dtype=float), (ib.n,))
    dt = np.broadcast_to(np.asarray(dt, dtype=float), (ib.n,))
    return ib.combine(flux_coefficients(tau, dt), 1)


def point_value(ib: Interface, tau, t):
    """int psi f at time t  (flux.py:182-188)."""
    tau = np.broadcast_to(np.asarray(tau, dtype=float), (ib.n,))
    t = np.broadcast_to(np.asarray(t, dtype=float), (ib.n,))
    e = np.exp(-t / tau)
    coefs = (1.0 - e, (t + tau) * e - tau, t - tau + tau * e, e, -(tau + t) * e, -tau * e)
    return ib.combine(coefs, 0)


def kfvs_flux(wl, wr, gamma=GAMMA):
    """Collisionless split flux (flux.py:200-208)."""
    wl = np.atleast_2d(wl)
    wr = np.atleast_2d(wr)
    return wl[:, 0, None] * Moments(wl, gamma, "pos").psi(1, 0, 0) + \
        wr[:, 0, None] * Moments(wr, gamma, "neg").psi(1, 0, 0)


def collision_time(model, dt, p_l, p_r, mu=0.0, p_eq=None):
    """flux.py:211-227."""
    jump = np.abs(p_l - p_r) / (p_l + p_r) * dt
    if model == "inviscid":
        return 0.1 * dt + jump
    if model == "viscous":
        return mu / p_eq + jump
    raise ValueError(model)


def to_local(q, frame):
    """flux.py:230-235: velocity block into the face frame (rows n, t1, t2)."""
    out = np.array(q, dtype=float, copy=True)
    v = q[..., 1:4]
    out[..., 1:4] = np.einsum("...ij,...j->...i", frame, v)
    return out


def to_global(q, frame):
    """flux.py:238-243."""
    out = np.array(q, dtype=float, copy=True)
    out[..., 1:4] = np.einsum("...ji,...j->...i", frame, q[..., 1:4])
    return out


def euler_flux_local(w, gamma=GAMMA):
    w = np.atleast_2d(w)
    q = prim_to_cons(w, gamma)
    p = pressure(w)
    u = w[:, 1]
    return np.stack([q[:, 0] * u, q[:, 1] * u + p, q[:, 2] * u, q[:, 3] * u, (q[:, 4] + p) * u], axis=1)


def random_interfaces(rng, n, slope_scale=0.3):
    """Same distribution as flux.py:271-286 (used for seeded parity batches)."""
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
