"""ORACLE (test infrastructure only): residual, Roe Jacobian, GMRES, advance.

Restates gks3d/boundary.py:51-171 (ghost states), gks3d/stepping.py:135-296
(local time step, residual, implicit step), gks3d/jacobian.py:37-196 (Roe
blocks) and gks3d/krylov.py:24-140 (block Jacobi, GMRES).  Vectorised numpy,
single process; also the CPU baseline of bench.py (`cpu_baseline`,
`--impl reference`).
"""

from __future__ import annotations

import numpy as np
from scipy.special import erfc

from . import flux as F
from .kinetic import GAMMA, cons_to_prim, prim_to_cons, pressure
from .recon import Recon, stencils, update_gradients

WALLS = ("wall_noslip_isothermal", "wall_noslip_adiabatic", "wall_slip_adiabatic")


class OracleStepError(RuntimeError):
    pass


class OracleSolverError(RuntimeError):
    pass


# -- boundary ghosts (boundary.py:51-171) ------------------------------------

def _ref_prim(spec):
    r = np.asarray(spec.reference, dtype=float)
    return np.array([r[0], r[1], r[2], r[3], r[0] / (2.0 * r[4])])


def _half_flux(un, lam, sign):
    g = 0.5 * np.exp(-lam * un * un) / np.sqrt(np.pi * lam)
    if sign > 0:
        return un * 0.5 * erfc(-np.sqrt(lam) * un) + g
    return -(un * 0.5 * erfc(np.sqrt(lam) * un) - g)


def ghost(q, spec, n, gamma=GAMMA):
    w = cons_to_prim(np.atleast_2d(q), gamma)
    n = np.atleast_2d(n)
    o = w.copy()
    vel = w[:, 1:4]
    un = np.sum(vel * n, axis=1)
    k = spec.kind
    if k == "wall_slip_adiabatic":
        o[:, 1:4] = vel - 2.0 * un[:, None] * n
    elif k in ("wall_noslip_adiabatic", "wall_noslip_isothermal"):
        o[:, 1:4] = 2.0 * np.asarray(spec.velocity) - vel
        if k == "wall_noslip_isothermal":
            o[:, 4] = spec.lambda_wall
            ung = np.sum(o[:, 1:4] * n, axis=1)
            o[:, 0] = w[:, 0] * _half_flux(un, w[:, 4], 1.0) / _half_flux(ung, spec.lambda_wall, -1.0)
    elif k == "supersonic_inlet":
        o[:] = _ref_prim(spec)
    elif k == "farfield_riemann":
        o = _farfield(w, n, _ref_prim(spec), gamma)
    return prim_to_cons(o, gamma)


def _farfield(w, n, ref, g):
    rho, vel, lam = w[:, 0], w[:, 1:4], w[:, 4]
    p = rho / (2.0 * lam)
    a = np.sqrt(g * p / rho)
    un = np.sum(vel * n, axis=1)
    pi = ref[0] / (2.0 * ref[4])
    ai = np.sqrt(g * pi / ref[0])
    uni = n @ ref[1:4]
    g1 = g - 1.0
    rp, rm = un + 2.0 * a / g1, uni - 2.0 * ai / g1
    ub, ab = 0.5 * (rp + rm), 0.25 * g1 * (rp - rm)
    out_ = ub > 0.0
    s = np.where(out_, p / rho ** g, pi / ref[0] ** g)
    ut = np.where(out_[:, None], vel - un[:, None] * n, ref[1:4] - uni[:, None] * n)
    rb = (ab * ab / (g * s)) ** (1.0 / g1)
    pb = rb * ab * ab / g
    mach = un / a
    so, si = mach >= 1.0, mach <= -1.0
    o = np.empty_like(w)
    o[:, 0] = np.where(so, rho, np.where(si, ref[0], rb))
    o[:, 1:4] = np.where(so[:, None], vel, np.where(si[:, None], ref[1:4], ut + ub[:, None] * n))
    o[:, 4] = np.where(so, lam, np.where(si, ref[4], rb / (2.0 * pb)))
    return o


def ghost_grad(g, spec, n):
    if spec.kind not in WALLS:
        return g.copy()
    gn = np.einsum("fxk,fx->fk", g, n)
    mir = g - 2.0 * n[:, :, None] * gn[:, None, :]
    out = mir.copy()
    mom = mir[:, :, 1:4]
    if spec.kind == "wall_slip_adiabatic":
        mn = np.einsum("fxc,fc->fx", mom, n)
        out[:, :, 1:4] = mom - 2.0 * mn[:, :, None] * n[:, None, :]
    else:
        out[:, :, 1:4] = -mom
        v = np.asarray(spec.velocity)
        if np.any(v != 0.0):
            out[:, :, 1:4] += 2.0 * mir[:, :, 0:1] * v
    return out


# -- Roe Jacobian (jacobian.py:37-196) ------------------------------------------

def euler_jac(q, n, g=GAMMA):
    g1 = g - 1.0
    rho = q[:, 0]
    v = q[:, 1:4] / rho[:, None]
    un = np.sum(v * n, axis=1)
    ke = 0.5 * np.sum(v * v, axis=1)
    h = (q[:, 4] + g1 * (q[:, 4] - rho * ke)) / rho
    J = np.zeros((len(q), 5, 5))
    J[:, 0, 1:4] = n
    J[:, 1:4, 0] = g1 * ke[:, None] * n - v * un[:, None]
    J[:, 1:4, 1:4] = v[:, :, None] * n[:, None, :] - g1 * n[:, :, None] * v[:, None, :] + \
        un[:, None, None] * np.eye(3)
    J[:, 1:4, 4] = g1 * n
    J[:, 4, 0] = (g1 * ke - h) * un
    J[:, 4, 1:4] = h[:, None] * n - g1 * v * un[:, None]
    J[:, 4, 4] = g * un
    return J


def spec_radius(q, n, g=GAMMA):
    rho = q[:, 0]
    v = q[:, 1:4] / rho[:, None]
    p = (g - 1.0) * (q[:, 4] - 0.5 * rho * np.sum(v * v, axis=1))
    return np.abs(np.sum(v * n, axis=1)) + np.sqrt(g * p / rho)


class Blocks:
    """diag (nc,5,5) + CSR off-diagonal blocks sorted by (row, col)."""

    def __init__(self, diag, off, row, col, nc):
        order = np.lexsort((col, row))
        self.diag, self.off, self.row, self.col = diag, off[order], row[order], col[order]
        self.nc = nc

    def offmv(self, x):
        # scipy BSR product, as the reference does (jacobian.py:101-113)
        if not len(self.off):
            return np.zeros((self.nc, 5))
        if getattr(self, "_bsr", None) is None:
            from scipy.sparse import bsr_matrix

            rowptr = np.concatenate([[0], np.cumsum(np.bincount(self.row, minlength=self.nc))])
            self._bsr = bsr_matrix((self.off, self.col, rowptr), shape=(5 * self.nc, 5 * self.nc))
        return (self._bsr @ x.reshape(-1)).reshape(self.nc, 5)

    def mv(self, x):
        return np.einsum("cij,cj->ci", self.diag, x) + self.offmv(x)


def roe_jacobian(mesh, q, dt, ghosts=None, g=GAMMA):
    nc = mesh.ncells
    D = np.zeros((nc, 5, 5))
    D[:, np.arange(5), np.arange(5)] = (mesh.cell_volume / dt)[:, None]
    fi = np.flatnonzero(mesh.face_neighbor >= 0)
    o, nb = mesh.face_owner[fi], mesh.face_neighbor[fi]
    n, hs = mesh.face_normal[fi], 0.5 * mesh.face_area[fi]
    lam = spec_radius(0.5 * (q[o] + q[nb]), n, g)[:, None, None] * np.eye(5)
    jo, jn = euler_jac(q[o], n, g), euler_jac(q[nb], n, g)
    np.add.at(D, o, hs[:, None, None] * (jo + lam))
    np.add.at(D, nb, hs[:, None, None] * (-jn + lam))
    off = np.concatenate([hs[:, None, None] * (jn - lam), hs[:, None, None] * (-jo - lam)])
    row = np.concatenate([o, nb])
    col = np.concatenate([nb, o])
    bf = np.flatnonzero(mesh.face_neighbor < 0)
    if len(bf):
        bo = mesh.face_owner[bf]
        qb = q[bo] if ghosts is None else 0.5 * (q[bo] + ghosts)
        lb = spec_radius(qb, mesh.face_normal[bf], g)
        np.add.at(D, bo, (0.5 * mesh.face_area[bf])[:, None, None] *
                  (euler_jac(q[bo], mesh.face_normal[bf], g) + lb[:, None, None] * np.eye(5)))
    # interleave (own, nbr) per face like the reference before its lexsort
    inter = np.empty_like(off)
    inter[0::2], inter[1::2] = off[: len(fi)], off[len(fi):]
    r2, c2 = np.empty_like(row), np.empty_like(col)
    r2[0::2], r2[1::2], c2[0::2], c2[1::2] = o, nb, nb, o
    return Blocks(D, inter, r2, c2, nc)


# -- Krylov (krylov.py:24-140) ---------------------------------------------------

def jacobi(A, b, kmax, dinv):
    z = np.einsum("cij,cj->ci", dinv, b)
    for _ in range(kmax):
        z = np.einsum("cij,cj->ci", dinv, b - A.offmv(z))
    return z


def gmres(A, b, m=10, restarts=3, kmax=2, rtol=0.0, atol=0.0, matvec=None):
    """Returns (x, cycle_norms, matvecs)."""
    mv = matvec or A.mv
    dinv = np.linalg.inv(A.diag)
    if not np.all(np.isfinite(dinv)):
        raise OracleSolverError("singular diagonal block")
    shape = b.shape
    x = np.zeros(shape)
    cycles, nmv, target = [], 0, None
    for _ in range(restarts):
        rh = jacobi(A, b - mv(x), kmax, dinv).ravel()
        nmv += 1
        beta = np.linalg.norm(rh)
        if target is None:
            target = rtol * beta + atol
        if beta == 0.0 or beta <= target:
            cycles.append([beta])
            break
        V = np.zeros((m + 1, rh.size))
        V[0] = rh / beta
        H = np.zeros((m + 1, m))
        cs, sn, gv = np.zeros(m), np.zeros(m), np.zeros(m + 1)
        gv[0] = beta
        norms, used, brk = [beta], 0, False
        for j in range(m):
            w = jacobi(A, mv(V[j].reshape(shape)), kmax, dinv).ravel()
            nmv += 1
            ws = np.linalg.norm(w)
            for i in range(j + 1):
                H[i, j] = w @ V[i]
                w -= H[i, j] * V[i]
            H[j + 1, j] = np.linalg.norm(w)
            if H[j + 1, j] < 0.5 * ws:
                for i in range(j + 1):
                    c = w @ V[i]
                    H[i, j] += c
                    w -= c * V[i]
                H[j + 1, j] = np.linalg.norm(w)
            if not np.isfinite(H[j + 1, j]):
                raise OracleSolverError("non-finite Arnoldi vector")
            for i in range(j):
                t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
                H[i, j] = t
            d = np.hypot(H[j, j], H[j + 1, j])
            cs[j], sn[j] = H[j, j] / d, H[j + 1, j] / d
            H[j, j] = d
            gv[j + 1] = -sn[j] * gv[j]
            gv[j] = cs[j] * gv[j]
            norms.append(abs(gv[j + 1]))
            used = j + 1
            if H[j + 1, j] <= 1e-13 * ws:
                brk = True
                break
            if norms[-1] <= max(1e-15 * norms[0], target):
                break
            V[j + 1] = w / H[j + 1, j]
        y = np.zeros(used)
        for i in range(used - 1, -1, -1):
            y[i] = (gv[i] - H[i, i + 1: used] @ y[i + 1: used]) / H[i, i]
        x = x + (y @ V[:used]).reshape(shape)
        cycles.append(norms)
        if brk or norms[-1] <= target:
            break
    return x, cycles, nmv


# -- the solver -----------------------------------------------------------------------

class OracleSolver:
    """CPU restatement of gks3d.stepping.Solver on a given mesh."""

    def __init__(self, mesh, scheme="weno_gmres", model="inviscid", mu=0.0, gamma=GAMMA, cfl=2.0,
                 krylov_dim=10, restarts=3, jacobi_sweeps=2, gmres_rtol=0.0, weights="nonlinear",
                 time_step="local", patches=None, jacobian="roe", first_order=False):
        self.mesh = mesh
        # first order (the B200 build's low-order start option):
        # piecewise-constant face states and the collisionless split flux
        # kfvs_flux (flux.py:200-208); point values = the half-range blend at t=0
        self.first_order = first_order
        self.compact = scheme.startswith("hweno")
        self.model, self.mu, self.gamma, self.cfl = model, mu, gamma, cfl
        self.m, self.restarts, self.kmax, self.rtol = krylov_dim, restarts, jacobi_sweeps, gmres_rtol
        self.global_dt = time_step == "global"
        self.patches = patches or {}
        self.jacobian = jacobian
        self.st = stencils(mesh)
        self.recon = Recon(mesh, self.st, self.compact, weights)
        f = mesh.fq_face
        self.frame = mesh.face_frame[f]
        self.ws = mesh.fq_weight * mesh.face_area[f]
        self.own, self.nbr = mesh.face_owner[f], mesh.face_neighbor[f]
        self.inner = self.nbr >= 0
        fp = mesh.face_patch[f]
        self.patch_fq = {n: np.flatnonzero(fp == i) for i, n in enumerate(mesh.patch_names) if np.any(fp == i)}
        self.wall = np.zeros(len(f), bool)
        for n, sel in self.patch_fq.items():
            if self.patches[n].kind in WALLS:
                self.wall[sel] = True
        self.bf = np.flatnonzero(mesh.face_neighbor < 0)

    def local_dt(self, q):
        m = self.mesh
        w = cons_to_prim(q, self.gamma)
        a = np.sqrt(self.gamma / (2.0 * w[:, 4]))
        speed = np.zeros(m.ncells)
        for cells in (m.face_owner, m.face_neighbor):
            f = np.flatnonzero(cells >= 0)
            c = cells[f]
            sig = (np.abs(np.sum(w[c, 1:4] * m.face_normal[f], axis=1)) + a[c]) * m.face_area[f]
            if self.model == "viscous" and self.mu > 0.0:
                sig += self.mu / w[c, 0] * m.face_area[f] ** 2 / m.cell_volume[c]
            np.add.at(speed, c, sig)
        dt = self.cfl * m.cell_volume / speed
        return np.full_like(dt, dt.min()) if self.global_dt else dt

    def residual(self, q, grad, dt, with_gradients=None):
        if with_gradients is None:
            with_gradients = self.compact
        coef = self.recon.coefficients(q, grad)
        if self.first_order:
            coef = np.zeros_like(coef)
        vo, go, vn, gn = self.recon.face_states(q, coef)
        for name, sel in self.patch_fq.items():
            spec = self.patches[name]
            n = self.mesh.face_normal[self.mesh.fq_face[sel]]
            vn[sel] = ghost(vo[sel], spec, n, self.gamma)
            gn[sel] = ghost_grad(go[sel], spec, n)
        fr = self.frame
        wl = cons_to_prim(F.to_local(vo, fr), self.gamma)
        wr = cons_to_prim(F.to_local(vn, fr), self.gamma)

        def slopes(g):
            s = np.einsum("fkd,fdm->fkm", fr, g)
            s[..., 1:4] = np.einsum("fij,fkj->fki", fr, s[..., 1:4])
            return s

        ib = F.Interface(wl, wr, slopes(go), slopes(gn), self.gamma)
        dtf = np.where(self.inner, np.minimum(dt[self.own], dt[np.where(self.inner, self.nbr, 0)]), dt[self.own])
        tau = F.collision_time(self.model, dtf, pressure(wl), pressure(wr), self.mu, pressure(ib.w0))
        fl = F.kfvs_flux(wl, wr, self.gamma) if self.first_order else F.evolve_flux(ib, tau, dtf)
        fl[self.wall, 0] = 0.0
        con = self.ws[:, None] * F.to_global(fl, fr)
        res = np.zeros_like(q)
        np.add.at(res, self.own, -con)
        np.add.at(res, self.nbr[self.inner], con[self.inner])
        gnew = None
        if with_gradients:
            if self.first_order:
                qp = F.to_global(prim_to_cons(ib.w0, self.gamma), fr)
            else:
                qp = F.to_global(F.point_value(ib, tau, np.zeros_like(dtf)), fr)
            gnew = update_gradients(self.mesh, qp)
        return res, gnew

    def ghosts(self, q):
        if not len(self.bf):
            return None
        out = np.empty((len(self.bf), 5))
        m = self.mesh
        for k, f in enumerate(self.bf):
            spec = self.patches[m.patch_names[m.face_patch[f]]]
            out[k] = ghost(q[m.face_owner[f]], spec, m.face_normal[f], self.gamma)[0]
        return out

    def frechet(self, q, grad, v, dt, sigma=None, base=None):
        """stepping.py:298-313; `base` = L(Q) when the caller has it (the
        matrix-free GMRES of a step evaluates L(Q) once per step)."""
        if sigma is None:
            vn = np.linalg.norm(v)
            if vn == 0.0:
                return np.zeros_like(v)
            sigma = np.sqrt(np.finfo(float).eps) * (1.0 + np.linalg.norm(q)) / vn
        if base is None:
            base, _ = self.residual(q, grad, dt, False)
        return (self.residual(q + sigma * v, grad, dt, False)[0] - base) / sigma

    def advance(self, q, grad=None):
        """One backward-Euler step (stepping.py:270-296); returns (q, grad, info dict)."""
        dt = self.local_dt(q)
        retried = False
        for attempt in range(2):
            res, gnew = self.residual(q, grad, dt)
            A = roe_jacobian(self.mesh, q, dt, self.ghosts(q), self.gamma)
            mv = None
            if self.jacobian == "frechet":
                vol = self.mesh.cell_volume
                mv = lambda v: (vol / dt)[:, None] * v - self.frechet(q, grad, v, dt, base=res)  # noqa: E731
            dq, cyc, nmv = gmres(A, res, self.m, self.restarts, self.kmax, self.rtol, 0.0, mv)
            qn = q + dq
            rho = qn[:, 0]
            bad = (rho <= 0) | (qn[:, 4] - 0.5 * np.sum(qn[:, 1:4] ** 2, axis=1) / rho <= 0) | \
                ~np.all(np.isfinite(qn), axis=1)
            if not bad.any():
                info = dict(res_rho_l1=float(np.sum(np.abs(res[:, 0])) / len(q)),
                            res_l2=float(np.sqrt(np.mean(res ** 2))), dt_min=float(dt.min()),
                            solver_cycles=len(cyc), retried=retried, matvecs=nmv)
                return qn, (gnew if self.compact else None), info
            if attempt == 0:
                dt = np.where(bad, 0.5 * dt, dt)
                retried = True
        raise OracleStepError(f"unphysical update persists at cells {np.flatnonzero(bad)[:8].tolist()}")
