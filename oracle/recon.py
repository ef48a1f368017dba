"""ORACLE (test infrastructure only): stencils and reconstruction.

Restates gks3d/mesh/stencils.py:72-192 (stencil selection),
gks3d/recon.py:41-195, 216-314 (basis, pseudo-inverse operators, WENO
combination, face evaluation) and gks3d/hweno.py:45-194 (Hermite operators,
Gauss gradient update).  Loops are per cell -- fine at the oracle's sizes.
Input is a mesh object with the reference Mesh attributes (the host mesh of
paper_2304_09485_b200.mesh is bit-identical to the reference's, pinned by
tests/test_setup.py).
"""

from __future__ import annotations

import numpy as np

NC = 9
RANK_TOL = 1e-10
EPS = 1e-6
LW = 0.025

_TET_SUBS = (((0, 1, 2), 0), ((0, 1, 3), 1), ((1, 2, 3), 2), ((2, 0, 3), 3))
_HEX_SUBS = ((0, 1, 2), (0, 2, 3), (0, 3, 4), (0, 4, 1), (5, 1, 2), (5, 2, 3), (5, 3, 4), (5, 4, 1))

B2 = np.diag([0, 0, 0, 4.0, 1.0, 1.0, 4.0, 1.0, 4.0])  # recon.py:28-36


def mono(x):
    """(x,y,z, x^2,xy,xz, y^2,yz,z^2) at scaled points (recon.py:41-45)."""
    x = np.asarray(x, dtype=float)
    a, b, c = x[..., 0], x[..., 1], x[..., 2]
    return np.stack([a, b, c, a * a, a * b, a * c, b * b, b * c, c * c], axis=-1)


def dmono(x):
    """d mono / d(x,y,z) -> (..., 3, 9)  (recon.py:48-57)."""
    x = np.asarray(x, dtype=float)
    a, b, c = x[..., 0], x[..., 1], x[..., 2]
    z, o = np.zeros_like(a), np.ones_like(a)
    return np.stack([np.stack([o, z, z, 2 * a, b, c, z, z, z], -1),
                     np.stack([z, o, z, z, a, z, 2 * b, c, z], -1),
                     np.stack([z, z, o, z, z, a, z, b, 2 * c], -1)], axis=-2)


def pinv(a, need):
    """SVD pseudo-inverse with the relative rank test (recon.py:60-69); None if rank < need."""
    u, s, vt = np.linalg.svd(a, full_matrices=False)
    if len(s) == 0 or s[0] == 0.0:
        return None
    keep = s >= RANK_TOL * s[0]
    if keep.sum() < need:
        return None
    return (vt[keep].T / s[keep]) @ u[:, keep].T


# -- stencils ----------------------------------------------------------------

def _key(i, s):
    return (int(i), round(s[0], 9), round(s[1], 9), round(s[2], 9))


def _unique(members):
    seen, out = set(), []
    for i, s in members:
        k = _key(i, s)
        if k not in seen:
            seen.add(k)
            out.append((int(i), np.asarray(s, dtype=float)))
    return out


def _faces_of(mesh, c):
    """Face ids of cell c in its own order (mesh.cell_faces[c], geometry.py:152-181)."""
    s = mesh.cell_face_start
    return mesh.cell_face_list[s[c]: s[c + 1]]


def _across(mesh, c):
    """(neighbour, shift) across each interior face of c, in cell face order."""
    res = []
    for f in _faces_of(mesh, c):
        if mesh.face_neighbor[f] < 0:
            continue
        if mesh.face_owner[f] == c:
            res.append((int(mesh.face_neighbor[f]), mesh.face_shift[f].copy()))
        else:
            res.append((int(mesh.face_owner[f]), -mesh.face_shift[f]))
    return res


def face_neighbours(mesh, c):
    """Labelled face neighbours (-1 on boundary); hexes reordered pole/equator/pole."""
    faces = _faces_of(mesh, c)
    ids = np.full(len(faces), -1, dtype=np.int64)
    sh = np.zeros((len(faces), 3))
    nrm = np.empty((len(faces), 3))
    for k, f in enumerate(faces):
        sgn = 1.0 if mesh.face_owner[f] == c else -1.0
        nrm[k] = sgn * mesh.face_normal[f]
        if mesh.face_neighbor[f] < 0:
            continue
        if mesh.face_owner[f] == c:
            ids[k], sh[k] = mesh.face_neighbor[f], mesh.face_shift[f]
        else:
            ids[k], sh[k] = mesh.face_owner[f], -mesh.face_shift[f]
    if mesh.cell_kind[c] != 1:
        return ids, sh
    pb = 1 + int(np.argmin(nrm[1:] @ nrm[0]))
    rest = [k for k in range(6) if k not in (0, pb)]
    ax = nrm[0]
    e1 = nrm[rest[0]] - (nrm[rest[0]] @ ax) * ax
    e1 /= np.linalg.norm(e1)
    e2 = np.cross(ax, e1)
    ang = [np.arctan2(nrm[k] @ e2, nrm[k] @ e1) for k in rest]
    order = [0] + [rest[k] for k in np.argsort(ang)] + [pb]
    return ids[order], sh[order]


def stencils(mesh):
    """Per cell: dict(nbr, nbr_s, big, subs, weno_fb, hweno_fb)  (stencils.py:119-192)."""
    across = [_across(mesh, c) for c in range(mesh.ncells)]
    out = []
    for c in range(mesh.ncells):
        ids, sh = face_neighbours(mesh, c)
        pres = ids >= 0
        big = [(c, np.zeros(3))] + [(i, s) for i, s in zip(ids[pres], sh[pres])]
        for i, s in zip(ids[pres], sh[pres]):
            big += [(j, s + t) for j, t in across[i]]
        big = _unique(big)
        subs = []
        if mesh.cell_kind[c] == 1:
            for pat in _HEX_SUBS:
                if np.any(ids[list(pat)] < 0):
                    continue
                mem = _unique([(c, np.zeros(3))] + [(ids[k], sh[k]) for k in pat])
                if len(mem) == 4:
                    subs.append(mem)
        else:
            for kept, grow in _TET_SUBS:
                if np.any(ids[list(kept)] < 0):
                    continue
                mem = [(c, np.zeros(3))] + [(ids[k], sh[k]) for k in kept]
                host, hs = ids[grow], sh[grow]
                extra = [(j, hs + t) for j, t in across[host]
                         if not (j == c and np.max(np.abs(hs + t)) < 1e-12)]
                extra.sort(key=lambda e: (e[0], tuple(np.round(e[1], 9))))
                mem = _unique(mem + extra[:3])
                if len(mem) == 7:
                    subs.append(mem)
        wfb = len(subs) < 2
        if wfb:
            subs = []
        out.append(dict(nbr=ids, nbr_s=sh, big=big, subs=subs, weno_fb=wfb, hweno_fb=int(pres.sum()) < 2))
    return out


# -- reconstruction geometry and operators ------------------------------------

class Recon:
    """Operators of the WENO (compact=False) or HWENO (compact=True) scheme."""

    def __init__(self, mesh, st, compact, weights="nonlinear", eps=EPS, lw=LW):
        self.mesh, self.st, self.compact = mesh, st, compact
        self.linear = weights == "linear"
        self.eps, self.lw = eps, lw
        nc = mesh.ncells
        self.avg0 = np.empty((nc, NC))
        self.beta = np.empty((nc, NC, NC))
        for c in range(nc):
            p, w = self._cq(c)
            x = (p - mesh.cell_centroid[c]) / mesh.cell_h[c]
            self.avg0[c] = w @ mono(x)
            g = dmono(x)
            self.beta[c] = np.einsum("q,qxd,qxe->de", w, g, g) + B2
        self.ops = [self._weno_ops(c) if not compact else self._hweno_ops(c) for c in range(nc)]
        self._pack()

    def _pack(self):
        """Per-cell operators padded into arrays (the reference's own layout,
        recon.py:216-274 / hweno.py:62-137): padded gather slots point at the
        cell itself and carry zero columns, padded sub-stencils are inactive."""
        nc = self.mesh.ncells
        own = np.arange(nc)
        if not self.compact:
            K = max(len(o["gids"]) for o in self.ops)
            M = max((len(o["subs"]) for o in self.ops), default=0)
            S = max((len(ids) for o in self.ops for _, ids in o["subs"]), default=1)
            self.P_big = np.zeros((nc, NC, K))
            self.P_gid = np.repeat(own[:, None], K, axis=1)
            self.P_sub = np.zeros((nc, max(M, 1), 3, S))
            self.P_sid = np.repeat(own[:, None, None], max(M, 1) * S, axis=1).reshape(nc, max(M, 1), S)
            self.P_act = np.zeros((nc, max(M, 1)), dtype=bool)
            for c, o in enumerate(self.ops):
                k = len(o["gids"])
                self.P_big[c, :, :k] = o["big"]
                self.P_gid[c, :k] = o["gids"]
                for m, (op, ids) in enumerate(o["subs"]):
                    self.P_sub[c, m, :, :len(ids)] = op
                    self.P_sid[c, m, :len(ids)] = ids
                    self.P_act[c, m] = True
        else:
            A = max(len(o["avg_ids"]) for o in self.ops)
            G = max(len(o["grad_ids"]) for o in self.ops)
            M = max((len(o["subs"]) for o in self.ops), default=0)
            self.P_bigA = np.zeros((nc, NC, max(A, 1)))
            self.P_bigG = np.zeros((nc, NC, G, 3))
            self.P_aid = np.repeat(own[:, None], max(A, 1), axis=1)
            self.P_gid = np.repeat(own[:, None], G, axis=1)
            self.P_sub = np.zeros((nc, max(M, 1), 3, 7))
            self.P_sj = np.repeat(own[:, None], max(M, 1), axis=1)
            self.P_act = np.zeros((nc, max(M, 1)), dtype=bool)
            for c, o in enumerate(self.ops):
                a, g = len(o["avg_ids"]), len(o["grad_ids"])
                self.P_bigA[c, :, :a] = o["big"][:, :a]
                self.P_bigG[c, :, :g] = o["big"][:, a:].reshape(NC, g, 3)
                self.P_aid[c, :a] = o["avg_ids"]
                self.P_gid[c, :g] = o["grad_ids"]
                for m, (op, j) in enumerate(o["subs"]):
                    self.P_sub[c, m] = op
                    self.P_sj[c, m] = j
                    self.P_act[c, m] = True

    def _cq(self, c, shift=None):
        m = self.mesh
        sl = slice(m.cell_cq_start[c], m.cell_cq_start[c + 1])
        p = m.cq_point[sl] if shift is None else m.cq_point[sl] + shift
        return p, m.cq_weight[sl]

    def avg_row(self, c, j, s):
        p, w = self._cq(j, s)
        return w @ mono((p - self.mesh.cell_centroid[c]) / self.mesh.cell_h[c]) - self.avg0[c]

    def grad_rows(self, c, j, s):
        p, w = self._cq(j, s)
        h0 = self.mesh.cell_h[c]
        return self.mesh.cell_h[j] * (np.einsum("q,qxd->xd", w, dmono((p - self.mesh.cell_centroid[c]) / h0)) / h0)

    def _weno_ops(self, c):
        st = self.st[c]
        subs = []
        for mem in st["subs"]:
            rows = np.array([self.avg_row(c, j, s)[:3] for j, s in mem[1:]])
            op = pinv(rows, 3)
            if op is not None:
                subs.append((op, np.array([j for j, _ in mem[1:]])))
        if len(subs) < 2:
            subs = []
        gids = np.array([j for j, _ in st["big"][1:]], dtype=np.int64)
        rows = np.array([self.avg_row(c, j, s) for j, s in st["big"][1:]]).reshape(-1, NC)
        op = pinv(rows, NC) if subs and len(rows) >= NC else None
        if op is None:
            op = np.zeros((NC, len(rows)))
            lin = pinv(rows[:, :3], 3) if len(rows) >= 3 else None
            if lin is not None:
                op[:3] = lin
        return dict(big=op, gids=gids, subs=subs)

    def _hweno_ops(self, c):
        st = self.st[c]
        ids, sh = st["nbr"], st["nbr_s"]
        mem = [(c, np.zeros(3))] + [(j, s) for j, s in zip(ids[ids >= 0], sh[ids >= 0])]
        avg = [self.avg_row(c, j, s) for j, s in mem[1:]]
        grd = [self.grad_rows(c, j, s) for j, s in mem]
        rows = np.vstack(avg + grd) if avg else np.vstack(grd)
        op = pinv(rows, NC) if not st["hweno_fb"] and len(rows) >= NC else None
        if op is None:
            op = np.zeros((NC, len(rows)))
            lin = pinv(rows[:, :3], 3)
            if lin is not None:
                op[:3] = lin
        subs = []
        if not st["hweno_fb"]:
            g0 = self.grad_rows(c, c, np.zeros(3))[:, :3]
            for j, s in mem[1:]:
                r = np.vstack([self.avg_row(c, j, s)[:3][None], g0, self.grad_rows(c, j, s)[:, :3]])
                sop = pinv(r, 3)
                if sop is not None:
                    subs.append((sop, j))
            if len(subs) < 2:
                subs = []
        return dict(big=op, avg_ids=np.array([j for j, _ in mem[1:]], dtype=np.int64),
                    grad_ids=np.array([j for j, _ in mem], dtype=np.int64), subs=subs)

    # -- per-step reconstruction (recon.py:167-195, 276-294; hweno.py:139-169)

    def coefficients(self, q, grad=None):
        """Combined polynomial coefficients (nc, 9, 5), vectorised over cells
        like the reference (recon.py:276-294 / hweno.py:139-169)."""
        qc = q[:, None, :]
        if self.compact:
            h = self.mesh.cell_h
            cb = np.matmul(self.P_bigA, q[self.P_aid] - qc)
            gg = h[self.P_gid][:, :, None, None] * grad[self.P_gid]  # (nc, g, 3, m)
            cb += np.matmul(self.P_bigG.reshape(gg.shape[0], -1, gg.shape[1] * 3), gg.reshape(gg.shape[0], -1, gg.shape[-1]))
            if self.linear:
                return cb
            j = self.P_sj
            hg = h[:, None, None] * grad  # (nc, 3, 5)
            rhs = np.concatenate([(q[j] - qc)[:, :, None, :], np.broadcast_to(hg[:, None], j.shape + hg.shape[1:]),
                                  hg[j]], axis=2)  # (nc, M, 7, 5)
            bs = np.matmul(self.P_sub, rhs)
        else:
            cb = np.matmul(self.P_big, q[self.P_gid] - qc)
            if self.linear:
                return cb
            bs = np.matmul(self.P_sub, q[self.P_sid] - q[:, None, None, :])
        return self._combine_all(cb, bs, self.P_act)

    def _combine_all(self, cb, bs, act):
        """combine_candidates (recon.py:167-195), all cells at once: weights
        per cell and component; cells without active sub-stencils keep cb."""
        m = act.sum(axis=1).astype(float)  # (nc,)
        has = m > 0
        ms = np.where(has, m, 1.0)
        b0 = np.sum(cb * np.matmul(self.beta, cb), axis=1)
        bm = np.sum(bs * bs, axis=2)  # (nc, M, 5)
        g0 = (1.0 - self.lw * m)[:, None]
        tau = np.sum(np.where(act[:, :, None], np.abs(b0[:, None, :] - bm), 0.0), axis=1) / ms[:, None]
        w0 = g0 * (1.0 + tau / (b0 + self.eps))
        wm = np.where(act[:, :, None], self.lw * (1.0 + tau[:, None, :] / (bm + self.eps)), 0.0)
        tot = w0 + np.sum(wm, axis=1)
        g0s = np.where(has[:, None], g0, 1.0)
        out = (w0 / tot / g0s)[:, None, :] * cb
        f = np.where(act[:, :, None], wm / tot[:, None, :] - (w0 / tot * self.lw / g0s)[:, None, :], 0.0)
        out[:, :3] += np.sum(f[:, :, None, :] * bs, axis=1)
        return np.where(has[:, None, None], out, cb)

    def face_states(self, q, coef):
        """Point values / gradients on both sides of every fq point (recon.py:297-314)."""
        m = self.mesh
        own = m.face_owner[m.fq_face]
        nbr = m.face_neighbor[m.fq_face]
        inner = nbr >= 0
        nb = np.where(inner, nbr, own)
        sides = []
        for cells, pts in ((own, m.fq_point), (nb, m.fq_point - m.face_shift[m.fq_face])):
            h = m.cell_h[cells]
            x = (pts - m.cell_centroid[cells]) / h[:, None]
            phi = mono(x) - self.avg0[cells]
            dphi = dmono(x) / h[:, None, None]
            cf = coef[cells]
            sides.append((q[cells] + np.matmul(phi[:, None, :], cf)[:, 0], np.matmul(dphi, cf)))
        (vo, go), (vn, gn) = sides
        return vo, go, np.where(inner[:, None], vn, vo), np.where(inner[:, None, None], gn, go)


def update_gradients(mesh, qpt):
    """Gauss theorem gradient from interface values (hweno.py:172-194)."""
    f = mesh.fq_face
    con = (mesh.fq_weight * mesh.face_area[f])[:, None, None] * mesh.face_normal[f][:, :, None] * qpt[:, None, :]
    out = np.zeros((mesh.ncells, 3, qpt.shape[1]))
    np.add.at(out, mesh.face_owner[f], con)
    inner = mesh.face_neighbor[f] >= 0
    np.add.at(out, mesh.face_neighbor[f][inner], -con[inner])
    return out / mesh.cell_volume[:, None, None]
