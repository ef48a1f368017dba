"""ORACLE (test infrastructure only): Maxwellian moment engine.

Restates /root/reference/pkg/src/gks3d/kinetic.py.  Arrays are batch-first
((n, 5) states); moment tables are stored order-first ((order+1, n)).
"""

from __future__ import annotations

import numpy as np
from scipy.special import erfc

GAMMA = 1.4
U_ORDER = 6      # kinetic.py:20  MAX_UORDER
XI_ORDER = 2     # kinetic.py:21  MAX_XIORDER


class OracleUnphysical(ValueError):
    """Non-positive density / internal energy (kinetic.py:26)."""


def n_internal(gamma):
    """Internal degrees of freedom (kinetic.py:30-32)."""
    return (5.0 - 3.0 * gamma) / (gamma - 1.0)


def cons_to_prim(q, gamma=GAMMA):
    """(rho, rhoU, rhoV, rhoW, rhoE) -> (rho, U, V, W, lam)  (kinetic.py:35-51)."""
    q = np.asarray(q, dtype=float)
    rho = q[..., 0]
    if np.any(~(rho > 0.0)) or not np.all(np.isfinite(rho)):
        raise OracleUnphysical("non-positive density")
    u = q[..., 1:4] / rho[..., None]
    eint = q[..., 4] - 0.5 * (q[..., 1] * u[..., 0] + q[..., 2] * u[..., 1] + q[..., 3] * u[..., 2])
    if np.any(~(eint > 0.0)) or not np.all(np.isfinite(eint)):
        raise OracleUnphysical("non-positive internal energy")
    w = np.empty_like(q)
    w[..., 0] = rho
    w[..., 1:4] = u
    w[..., 4] = (n_internal(gamma) + 3.0) * rho / (4.0 * eint)
    return w


def prim_to_cons(w, gamma=GAMMA):
    """Inverse of cons_to_prim (kinetic.py:54-65)."""
    w = np.asarray(w, dtype=float)
    q = np.empty_like(w)
    rho = w[..., 0]
    q[..., 0] = rho
    q[..., 1:4] = rho[..., None] * w[..., 1:4]
    q[..., 4] = 0.5 * rho * (w[..., 1] ** 2 + w[..., 2] ** 2 + w[..., 3] ** 2) + \
        (n_internal(gamma) + 3.0) * rho / (4.0 * w[..., 4])
    return q


def pressure(w):
    return w[..., 0] / (2.0 * w[..., 4])


def sound_speed(w, gamma=GAMMA):
    return np.sqrt(gamma / (2.0 * w[..., 4]))


def _recur(m, mean, lam, top):
    """<c^k> = U <c^(k-1)> + (k-1)/(2 lam) <c^(k-2)>  (kinetic.py:113-120)."""
    h = 0.5 / lam
    for k in range(2, top + 1):
        m[k] = mean * m[k - 1] + (k - 1) * h * m[k - 2]
    return m


class Moments:
    """Normalized Maxwellian moments of one primitive batch (kinetic.py:90-162).

    half: None (full range in u), "pos" (u > 0) or "neg" (u < 0).
    """

    def __init__(self, w, gamma=GAMMA, half=None):
        w = np.asarray(w, dtype=float)
        bad = (w[:, 0] <= 0.0) | (w[:, 4] <= 0.0) | ~np.all(np.isfinite(w), axis=1)
        if np.any(bad):
            raise OracleUnphysical("invalid primitive state")
        n = w.shape[0]
        lam = w[:, 4]
        self.rho = w[:, 0]
        self.u = np.empty((U_ORDER + 1, n))
        if half is None:
            self.u[0] = 1.0
            self.u[1] = w[:, 1]
        else:
            # erfc seeds of the half-range integrals (kinetic.py:123-137)
            rl = np.sqrt(lam)
            g = 0.5 * np.exp(-lam * w[:, 1] ** 2) / np.sqrt(np.pi * lam)
            if half == "pos":
                self.u[0] = 0.5 * erfc(-rl * w[:, 1])
                self.u[1] = w[:, 1] * self.u[0] + g
            else:
                self.u[0] = 0.5 * erfc(rl * w[:, 1])
                self.u[1] = w[:, 1] * self.u[0] - g
        _recur(self.u, w[:, 1], lam, U_ORDER)
        self.v = np.empty((U_ORDER + 1, n))
        self.v[0], self.v[1] = 1.0, w[:, 2]
        _recur(self.v, w[:, 2], lam, U_ORDER)
        self.w = np.empty((U_ORDER + 1, n))
        self.w[0], self.w[1] = 1.0, w[:, 3]
        _recur(self.w, w[:, 3], lam, U_ORDER)
        nd = n_internal(gamma)
        self.xi = np.empty((XI_ORDER + 1, n))
        self.xi[0] = 1.0
        self.xi[1] = nd / (2.0 * lam)
        self.xi[2] = nd * (nd + 2.0) / (4.0 * lam * lam)
        self._psi = {}  # psi(a, b, c, s) memo: directional / slope revisit the same orders

    def m(self, a, b, c, s):
        """<u^a v^b w^c xi^(2s)> (kinetic.py:173-188)."""
        out = self.u[a]
        if b:
            out = out * self.v[b]
        if c:
            out = out * self.w[c]
        if s:
            out = out * self.xi[s]
        return out

    def psi(self, a, b, c, s=0):
        """<u^a v^b w^c xi^2s psi>, shape (n, 5)  (kinetic.py:191-213)."""
        key = (a, b, c, s)
        hit = self._psi.get(key)
        if hit is not None:
            return hit
        m = self.m
        out = np.empty((self.rho.shape[0], 5))
        out[:, 0] = m(a, b, c, s)
        out[:, 1] = m(a + 1, b, c, s)
        out[:, 2] = m(a, b + 1, c, s)
        out[:, 3] = m(a, b, c + 1, s)
        out[:, 4] = 0.5 * (m(a + 2, b, c, s) + m(a, b + 2, c, s) + m(a, b, c + 2, s) + m(a, b, c, s + 1))
        out.flags.writeable = False
        self._psi[key] = out
        return out

    def slope(self, coef, a, b, c):
        """<(c0 + c1 u + c2 v + c3 w + c4 |c|^2/2) u^a v^b w^c psi>  (kinetic.py:222-250)."""
        coef = np.asarray(coef, dtype=float)
        out = coef[:, 0, None] * self.psi(a, b, c)
        out += coef[:, 1, None] * self.psi(a + 1, b, c)
        out += coef[:, 2, None] * self.psi(a, b + 1, c)
        out += coef[:, 3, None] * self.psi(a, b, c + 1)
        quad = self.psi(a + 2, b, c) + self.psi(a, b + 2, c) + self.psi(a, b, c + 2) + self.psi(a, b, c, 1)
        out += (0.5 * coef[:, 4])[:, None] * quad
        return out

    def directional(self, ax, ay, az, a, b, c):
        """<(ax u + ay v + az w)-weighted slope moments>  (kinetic.py:259-263)."""
        return self.slope(ax, a + 1, b, c) + self.slope(ay, a, b + 1, c) + self.slope(az, a, b, c + 1)


def micro_slope(w, dq, gamma=GAMMA):
    """Closed-form solve of <a psi> = dq / rho  (kinetic.py:271-302)."""
    w = np.asarray(w, dtype=float)
    rho, U, V, W, lam = (w[:, k] for k in range(5))
    n3 = n_internal(gamma) + 3.0
    b = np.asarray(dq, dtype=float) / rho[:, None]
    k2 = U * U + V * V + W * W + 0.5 * n3 / lam
    r1 = b[:, 1] - U * b[:, 0]
    r2 = b[:, 2] - V * b[:, 0]
    r3 = b[:, 3] - W * b[:, 0]
    r4 = 2.0 * b[:, 4] - k2 * b[:, 0]
    a = np.empty_like(b)
    a[:, 4] = 4.0 * lam * lam * (r4 - 2.0 * (U * r1 + V * r2 + W * r3)) / n3
    a[:, 1] = 2.0 * lam * r1 - U * a[:, 4]
    a[:, 2] = 2.0 * lam * r2 - V * a[:, 4]
    a[:, 3] = 2.0 * lam * r3 - W * a[:, 4]
    a[:, 0] = b[:, 0] - U * a[:, 1] - V * a[:, 2] - W * a[:, 3] - 0.5 * a[:, 4] * k2
    return a


def time_slope(w, ax, ay, az, mom, gamma=GAMMA):
    """A with <(ax u + ay v + az w + A) psi> = 0  (kinetic.py:305-312)."""
    rhs = -w[:, 0, None] * mom.directional(ax, ay, az, 0, 0, 0)
    return micro_slope(w, rhs, gamma)
