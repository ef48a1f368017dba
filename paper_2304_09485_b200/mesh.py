"""Unstructured tet/hex mesh: faces, geometry, quadrature, periodic merge.

Host-side setup mirroring gks3d/mesh/geometry.py (:1-451), boxgen.py
(:16-115) and fileio.py (:42-124), vectorised with numpy so meshes of
10^6-10^7 cells build in seconds instead of the reference's per-cell Python
loops.  Conventions are the reference's, and connectivity is
bit-identical to it:

  * face ids in order of first encounter while walking cells in input order
    and each cell's face patterns in order; the first cell is the owner and
    the owner's winding is kept (geometry.py:214-233);
  * normals point owner -> neighbour, flipped defensively (:307-309);
  * periodic patches are merged into shifted interior faces (:323-375).
"""

from __future__ import annotations

import numpy as np

TET = 0
HEX = 1

_TET_FACES = np.array(((0, 2, 1), (0, 1, 3), (1, 2, 3), (0, 3, 2)))
_HEX_FACES = np.array(((0, 3, 2, 1), (4, 5, 6, 7), (0, 1, 5, 4), (1, 2, 6, 5), (2, 3, 7, 6), (3, 0, 4, 7)))
_GAUSS1 = 1.0 / np.sqrt(3.0)
_TRI_BARY = np.array([[4, 1, 1], [1, 4, 1], [1, 1, 4]]) / 6.0
_TET_ALPHA = (5.0 + 3.0 * np.sqrt(5.0)) / 20.0
_TET_BETA = (5.0 - np.sqrt(5.0)) / 20.0
_QUAD_PTS = ((-_GAUSS1, -_GAUSS1), (_GAUSS1, -_GAUSS1), (_GAUSS1, _GAUSS1), (-_GAUSS1, _GAUSS1))
_HEX_SIGNS = np.array([(-1, -1, -1), (1, -1, -1), (1, 1, -1), (-1, 1, -1), (-1, -1, 1), (1, -1, 1),
                       (1, 1, 1), (-1, 1, 1)], dtype=float)


class MeshError(ValueError):
    """Malformed, non-conforming, or inverted mesh input."""


# -- pointwise geometry (single-entity API kept for parity with the reference) --


def local_frame(normal):
    """Orthonormal (n, t1, t2): t1 = normalised rejection of the least-aligned axis."""
    return _frames(np.asarray(normal, dtype=float)[None])[0]


def _norm3(x):
    """Row norms computed exactly as numpy's 1-D norm (sqrt of x.dot(x))."""
    return np.sqrt(np.matmul(x[:, None, :], x[:, :, None])[:, 0, 0])


def _frames(n):
    axis = np.argmin(np.abs(n), axis=1)
    e = np.zeros_like(n)
    e[np.arange(len(n)), axis] = 1.0
    dot = n[np.arange(len(n)), axis]
    t1 = e - dot[:, None] * n
    t1 /= _norm3(t1)[:, None]
    t2 = np.cross(n, t1)
    return np.stack([n, t1, t2], axis=1)


def _tri_geometry(p):
    """p (k,3,3) -> qp (k,3,3), area (k), unit normal (k,3)."""
    cr = np.cross(p[:, 1] - p[:, 0], p[:, 2] - p[:, 0])
    area = 0.5 * _norm3(cr)
    if np.any(area <= 0.0):
        raise MeshError("degenerate face (zero area)")
    normal = cr / (2.0 * area)[:, None]
    qp = np.matmul(_TRI_BARY, p)
    return qp, np.full((len(p), 3), 1.0 / 3.0), area, normal


def _quad_geometry(p):
    """2x2 tensor Gauss on the bilinear map of planar quads, p (k,4,3)."""
    k = len(p)
    qp = np.empty((k, 4, 3))
    jac = np.empty((k, 4))
    nacc = np.zeros((k, 3))
    for i, (xi, eta) in enumerate(_QUAD_PTS):
        shape = 0.25 * np.array([(1 - xi) * (1 - eta), (1 + xi) * (1 - eta), (1 + xi) * (1 + eta), (1 - xi) * (1 + eta)])
        dxi = 0.25 * np.array([-(1 - eta), (1 - eta), (1 + eta), -(1 + eta)])
        deta = 0.25 * np.array([-(1 - xi), -(1 + xi), (1 + xi), (1 - xi)])
        qp[:, i] = np.matmul(shape, p)
        cr = np.cross(np.matmul(dxi, p), np.matmul(deta, p))
        jac[:, i] = _norm3(cr)
        nacc += cr
    area = jac.sum(axis=1)
    if np.any(area <= 0.0):
        raise MeshError("degenerate face (zero area)")
    normal = nacc / _norm3(nacc)[:, None]
    span = np.max(np.linalg.norm(p - p.mean(axis=1, keepdims=True), axis=2), axis=1)
    off = np.max(np.abs(np.einsum("kjd,kd->kj", p - qp[:, :1], normal)), axis=1)
    if np.any(off > 1e-8 * np.maximum(span, 1.0)):
        raise MeshError("non-planar quadrilateral face")
    return qp, jac / area[:, None], area, normal


def face_quadrature(pts):
    pts = np.asarray(pts, dtype=float)
    if len(pts) == 3:
        qp, w, a, n = _tri_geometry(pts[None])
    elif len(pts) == 4:
        qp, w, a, n = _quad_geometry(pts[None])
    else:
        raise MeshError(f"faces must have 3 or 4 nodes, got {len(pts)}")
    return qp[0], w[0], float(a[0]), n[0]


def _tet_geometry(p):
    vol = np.linalg.det(p[:, 1:] - p[:, :1]) / 6.0
    if np.any(vol <= 0.0):
        raise MeshError(f"cell {int(np.flatnonzero(vol <= 0.0)[0])}: inverted cell (negative volume)")
    bary = np.full((4, 4), _TET_BETA)
    np.fill_diagonal(bary, _TET_ALPHA)
    qp = np.matmul(bary, p)
    return qp, np.full((len(p), 4), 0.25), vol, p.mean(axis=1)


def _hex_geometry(p):
    k = len(p)
    g = _GAUSS1
    qp = np.empty((k, 8, 3))
    jac = np.empty((k, 8))
    i = 0
    for zi in (-g, g):
        for yi in (-g, g):
            for xi in (-g, g):
                ref = np.array([xi, yi, zi])
                shape = 0.125 * np.prod(1.0 + _HEX_SIGNS * ref, axis=1)
                grad = np.empty((8, 3))
                for d in range(3):
                    others = [j for j in range(3) if j != d]
                    grad[:, d] = 0.125 * _HEX_SIGNS[:, d] * np.prod(1.0 + _HEX_SIGNS[:, others] * ref[others], axis=1)
                qp[:, i] = np.matmul(shape, p)
                jac[:, i] = np.linalg.det(np.matmul(grad.T, p))
                i += 1
    if np.any(jac <= 0.0):
        raise MeshError(f"cell {int(np.flatnonzero(np.any(jac <= 0, axis=1))[0])}: inverted cell (negative volume)")
    vol = jac.sum(axis=1)
    cen = np.matmul(jac[:, None, :], qp)[:, 0] / vol[:, None]
    return qp, jac / vol[:, None], vol, cen


def tet_volume_quadrature(pts):
    qp, w, v, c = _tet_geometry(np.asarray(pts, dtype=float)[None])
    return qp[0], w[0], float(v[0]), c[0]


def hex_volume_quadrature(pts):
    qp, w, v, c = _hex_geometry(np.asarray(pts, dtype=float)[None])
    return qp[0], w[0], float(v[0]), c[0]


def _row_keys(a):
    """View rows of an int64 array as opaque fixed-size keys (for sort/match)."""
    a = np.ascontiguousarray(a, dtype=np.int64)
    return a.view(np.dtype((np.void, a.dtype.itemsize * a.shape[1]))).ravel()


class Mesh:
    """Validated unstructured mesh with all solver-facing geometry (geometry.py:152-451)."""

    def __init__(self):
        self.nodes = None
        self.cell_kind = None
        self.cell_nodes = None
        self.cell_volume = None
        self.cell_centroid = None
        self.cell_h = None
        self.cell_face_start = None
        self.cell_face_list = None
        self.face_nodes = None
        self.face_owner = None
        self.face_neighbor = None
        self.face_patch = None
        self.face_area = None
        self.face_normal = None
        self.face_frame = None
        self.face_shift = None
        self.fq_point = None
        self.fq_weight = None
        self.fq_face = None
        self.face_fq_start = None
        self.cq_point = None
        self.cq_weight = None
        self.cell_cq_start = None
        self.patch_names = []
        self._source = None

    # -- construction -----------------------------------------------------

    @classmethod
    def build(cls, nodes, tets=(), hexes=(), patch_faces=None, periodic_pairs=()):
        mesh = cls()
        nodes = np.asarray(nodes, dtype=float)
        if nodes.ndim != 2 or nodes.shape[1] != 3 or not np.all(np.isfinite(nodes)):
            raise MeshError("nodes must be a finite (N, 3) array")
        tets = np.asarray(tets, dtype=np.int64).reshape(-1, 4)
        hexes = np.asarray(hexes, dtype=np.int64).reshape(-1, 8)
        nt, nh = len(tets), len(hexes)
        ncell = nt + nh
        if ncell == 0:
            raise MeshError("mesh has no cells")
        cell_kind = np.concatenate([np.full(nt, TET, np.int8), np.full(nh, HEX, np.int8)])
        cell_nodes = np.full((ncell, 8), -1, dtype=np.int64)
        cell_nodes[:nt, :4] = tets
        cell_nodes[nt:, :8] = hexes
        if np.any(cell_nodes >= len(nodes)) or np.any(cell_nodes[:nt, :4] < 0) or np.any(hexes < 0):
            raise MeshError("cell references a node out of range")

        # all (cell, local face) entries in walk order: tets first, then hexes
        fn_t = tets[:, _TET_FACES].reshape(-1, 3)
        fn_h = hexes[:, _HEX_FACES].reshape(-1, 4)
        ent_nodes = np.full((len(fn_t) + len(fn_h), 4), -1, dtype=np.int64)
        ent_nodes[: len(fn_t), :3] = fn_t
        ent_nodes[len(fn_t):] = fn_h
        ent_cell = np.concatenate([np.repeat(np.arange(nt), 4), nt + np.repeat(np.arange(nh), 6)])
        keys = np.full_like(ent_nodes, -1)
        keys[: len(fn_t), :3] = np.sort(fn_t, axis=1)
        keys[len(fn_t):] = np.sort(fn_h, axis=1)
        kv = _row_keys(keys)
        order = np.argsort(kv, kind="stable")
        ks = kv[order]
        new = np.ones(len(ks), dtype=bool)
        new[1:] = ks[1:] != ks[:-1]
        grp = np.cumsum(new) - 1  # group id in sorted order
        starts = np.flatnonzero(new)
        counts = np.diff(np.append(starts, len(ks)))
        if np.any(counts > 2):
            bad = keys[order[starts[np.flatnonzero(counts > 2)[0]]]]
            raise MeshError(f"non-conforming mesh: face {tuple(int(x) for x in bad if x >= 0)} shared by >2 cells")
        first = order[starts]  # walk index of the owner entry (stable sort)
        # face ids by first encounter
        fid_of_group = np.empty(len(starts), dtype=np.int64)
        fid_of_group[np.argsort(first, kind="stable")] = np.arange(len(starts))
        ent_face = np.empty(len(ks), dtype=np.int64)
        ent_face[order] = fid_of_group[grp]
        nface = len(starts)
        face_owner = np.empty(nface, dtype=np.int64)
        face_owner[fid_of_group] = ent_cell[first]
        face_neighbor = np.full(nface, -1, dtype=np.int64)
        two = np.flatnonzero(counts == 2)
        face_neighbor[fid_of_group[two]] = ent_cell[order[starts[two] + 1]]
        face_nodes = np.full((nface, 4), -1, dtype=np.int64)
        face_nodes[fid_of_group] = ent_nodes[first]
        face_key_sorted = ks[starts]  # sorted keys -> group
        # cell -> faces (CSR, in each cell's pattern order)
        nfpc = np.where(cell_kind == TET, 4, 6)
        cell_face_start = np.concatenate([[0], np.cumsum(nfpc)]).astype(np.int64)
        cell_face_list = ent_face.copy()

        # boundary patches
        face_patch = np.full(nface, -1, dtype=np.int64)
        patch_names = []
        patch_faces = patch_faces or {}
        for name, flist in patch_faces.items():
            pid = len(patch_names)
            patch_names.append(name)
            if len(flist) == 0:
                continue
            pk = np.full((len(flist), 4), -1, dtype=np.int64)
            if isinstance(flist, np.ndarray) and flist.ndim == 2:
                pk[:, : flist.shape[1]] = np.sort(flist.astype(np.int64), axis=1)
            else:
                for wdt in {len(f) for f in flist}:
                    sel = [i for i, f in enumerate(flist) if len(f) == wdt]
                    pk[sel, :wdt] = np.sort(np.asarray([flist[i] for i in sel], dtype=np.int64), axis=1)
            pv = _row_keys(pk)
            pos = np.searchsorted(face_key_sorted, pv)
            pos = np.minimum(pos, len(face_key_sorted) - 1)
            found = face_key_sorted[pos] == pv
            if not np.all(found):
                i = int(np.flatnonzero(~found)[0])
                raise MeshError(f"patch {name!r} face {tuple(int(x) for x in pk[i] if x >= 0)} matches no mesh face")
            fids = fid_of_group[pos]
            if np.any(face_neighbor[fids] != -1):
                i = int(np.flatnonzero(face_neighbor[fids] != -1)[0])
                raise MeshError(f"patch {name!r} face {tuple(int(x) for x in pk[i] if x >= 0)} is interior")
            face_patch[fids] = pid

        mesh.nodes = nodes
        mesh.cell_kind = cell_kind
        mesh.cell_nodes = cell_nodes
        mesh.patch_names = patch_names
        mesh._source = (tets, hexes, dict(patch_faces))
        mesh._finalize_cells()
        mesh.face_nodes = face_nodes
        mesh.face_owner = face_owner
        mesh.face_neighbor = face_neighbor
        mesh.face_patch = face_patch
        mesh.cell_face_start = cell_face_start
        mesh.cell_face_list = cell_face_list
        mesh._finalize_faces()
        for pa, pb in periodic_pairs:
            mesh._merge_periodic(pa, pb)
        mesh._freeze()
        return mesh

    def _finalize_cells(self):
        nc = len(self.cell_kind)
        tet = np.flatnonzero(self.cell_kind == TET)
        hx = np.flatnonzero(self.cell_kind == HEX)
        self.cell_volume = np.empty(nc)
        self.cell_centroid = np.empty((nc, 3))
        nq = np.where(self.cell_kind == TET, 4, 8)
        self.cell_cq_start = np.concatenate([[0], np.cumsum(nq)]).astype(np.int64)
        self.cq_point = np.empty((int(self.cell_cq_start[-1]), 3))
        self.cq_weight = np.empty(int(self.cell_cq_start[-1]))
        for sel, fn, k, width in ((tet, _tet_geometry, 4, 4), (hx, _hex_geometry, 8, 8)):
            if not len(sel):
                continue
            qp, w, vol, cen = fn(self.nodes[self.cell_nodes[sel, :width]])
            self.cell_volume[sel] = vol
            self.cell_centroid[sel] = cen
            idx = self.cell_cq_start[sel][:, None] + np.arange(k)
            self.cq_point[idx] = qp
            self.cq_weight[idx] = w
        self.cell_h = self.cell_volume ** (1.0 / 3.0)

    def _finalize_faces(self):
        nf = len(self.face_owner)
        tri = np.flatnonzero(self.face_nodes[:, 3] < 0)
        quad = np.flatnonzero(self.face_nodes[:, 3] >= 0)
        nq = np.where(self.face_nodes[:, 3] < 0, 3, 4)
        self.face_fq_start = np.concatenate([[0], np.cumsum(nq)]).astype(np.int64)
        nfq = int(self.face_fq_start[-1])
        self.fq_point = np.empty((nfq, 3))
        self.fq_weight = np.empty(nfq)
        self.face_area = np.empty(nf)
        self.face_normal = np.empty((nf, 3))
        for sel, fn, k in ((tri, _tri_geometry, 3), (quad, _quad_geometry, 4)):
            if not len(sel):
                continue
            try:
                qp, w, area, normal = fn(self.nodes[self.face_nodes[sel, :k]])
            except MeshError as exc:
                raise MeshError(f"face: {exc}") from exc
            flip = np.einsum("kd,kd->k", normal, qp.mean(axis=1) - self.cell_centroid[self.face_owner[sel]]) < 0.0
            normal[flip] = -normal[flip]
            idx = self.face_fq_start[sel][:, None] + np.arange(k)
            self.fq_point[idx] = qp
            self.fq_weight[idx] = w
            self.face_area[sel] = area
            self.face_normal[sel] = normal
        self.face_frame = _frames(self.face_normal)
        self.face_shift = np.zeros((nf, 3))
        self.fq_face = np.repeat(np.arange(nf, dtype=np.int64), nq)

    def _merge_periodic(self, patch_a, patch_b):
        try:
            pa = self.patch_names.index(patch_a)
            pb = self.patch_names.index(patch_b)
        except ValueError as exc:
            raise MeshError(f"unknown periodic patch in pair ({patch_a}, {patch_b})") from exc
        fa = np.flatnonzero(self.face_patch == pa)
        fb = np.flatnonzero(self.face_patch == pb)
        if len(fa) != len(fb) or len(fa) == 0:
            raise MeshError(f"periodic patches {patch_a}/{patch_b} have mismatched face counts")
        nq = np.diff(self.face_fq_start)
        cen = np.empty((len(nq), 3))
        for width in (3, 4):
            sel = np.flatnonzero(nq == width)
            if len(sel):
                cen[sel] = self.fq_point[self.face_fq_start[sel][:, None] + np.arange(width)].mean(axis=1)
        shift = cen[fb].mean(axis=0) - cen[fa].mean(axis=0)
        target = cen[fa] + shift
        from scipy.spatial import cKDTree

        dist, idx = cKDTree(cen[fb]).query(target)
        tol = 1e-8 * max(1.0, float(np.max(np.abs(self.nodes))))
        if np.max(dist) > tol or len(np.unique(idx)) != len(fb):
            raise MeshError(f"periodic patches {patch_a}/{patch_b} do not tile under translation")
        g = fb[idx]
        owner_g = self.face_owner[g].copy()
        self.face_neighbor[fa] = owner_g
        self.face_shift[fa] = -shift
        self.face_patch[fa] = -1
        keep = np.ones(len(self.face_owner), dtype=bool)
        keep[g] = False
        # the owner of g now reaches the merged face instead
        repl = np.full(len(self.face_owner), -1, dtype=np.int64)
        repl[g] = fa
        hit = repl[self.cell_face_list] >= 0
        self.cell_face_list = np.where(hit, repl[self.cell_face_list], self.cell_face_list)
        self._compress_faces(keep)

    def _compress_faces(self, keep):
        remap = -np.ones(len(keep), dtype=np.int64)
        remap[keep] = np.arange(int(keep.sum()))
        for name in ("face_nodes", "face_owner", "face_neighbor", "face_patch", "face_area", "face_normal",
                     "face_frame", "face_shift"):
            setattr(self, name, getattr(self, name)[keep])
        fq_keep = keep[self.fq_face]
        self.fq_point = self.fq_point[fq_keep]
        self.fq_weight = self.fq_weight[fq_keep]
        self.fq_face = remap[self.fq_face[fq_keep]]
        counts = np.bincount(self.fq_face, minlength=int(keep.sum()))
        self.face_fq_start = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
        self.cell_face_list = remap[self.cell_face_list]
        if np.any(self.cell_face_list < 0):
            raise MeshError("internal error: cell references a removed face")

    def _freeze(self):
        for val in vars(self).values():
            if isinstance(val, np.ndarray):
                val.setflags(write=False)

    # -- queries ------------------------------------------------------------

    @property
    def ncells(self):
        return len(self.cell_kind)

    @property
    def nfaces(self):
        return len(self.face_owner)

    @property
    def nfq(self):
        return len(self.fq_face)

    @property
    def cell_faces(self):
        """Per-cell face id arrays (reference list-of-arrays view)."""
        s = self.cell_face_start
        return [self.cell_face_list[s[c]: s[c + 1]] for c in range(self.ncells)]

    def face_points(self, f):
        ids = self.face_nodes[f]
        return self.nodes[ids[ids >= 0]]

    def face_quadrature_of(self, f):
        sl = slice(self.face_fq_start[f], self.face_fq_start[f + 1])
        return self.fq_point[sl], self.fq_weight[sl]

    def cell_quadrature_of(self, c, shift=None):
        sl = slice(self.cell_cq_start[c], self.cell_cq_start[c + 1])
        pts = self.cq_point[sl]
        if shift is not None:
            pts = pts + shift
        return pts, self.cq_weight[sl]

    def cell_outward_sign(self, c, f):
        return 1.0 if self.face_owner[f] == c else -1.0

    def neighbors_of(self, c):
        out = []
        s = self.cell_face_start
        for f in self.cell_face_list[s[c]: s[c + 1]]:
            if self.face_neighbor[f] < 0:
                continue
            if self.face_owner[f] == c:
                out.append((int(self.face_neighbor[f]), self.face_shift[f].copy()))
            else:
                out.append((int(self.face_owner[f]), -self.face_shift[f]))
        return out

    # -- validation (geometry.py:425-451) ------------------------------------

    def validate(self):
        scale = max(1.0, float(np.max(np.abs(self.nodes))))
        if np.any(self.cell_volume <= 0.0):
            raise MeshError("non-positive cell volume")
        if not np.allclose(self.cell_h ** 3, self.cell_volume, rtol=1e-12):
            raise MeshError("cell h is not volume^(1/3)")
        cells = np.repeat(np.arange(self.ncells), np.diff(self.cell_face_start))
        f = self.cell_face_list
        sign = np.where(self.face_owner[f] == cells, 1.0, -1.0)
        vec = (sign * self.face_area[f])[:, None] * self.face_normal[f]
        acc = np.zeros((self.ncells, 3))
        np.add.at(acc, cells, vec)
        bad = np.max(np.abs(acc), axis=1) > 1e-12 * scale ** 2 * max(1.0, float(np.max(self.face_area)))
        if np.any(bad):
            c = int(np.flatnonzero(bad)[0])
            raise MeshError(f"cell {c} face-area vectors do not close: {acc[c]}")
        eye = np.einsum("fij,fkj->fik", self.face_frame, self.face_frame)
        if np.max(np.abs(eye - np.eye(3))) > 1e-12:
            raise MeshError("non-orthonormal face frame")
        wsum = np.bincount(self.fq_face, weights=self.fq_weight, minlength=self.nfaces)
        if np.any(np.abs(wsum - 1.0) > 1e-13):
            raise MeshError(f"face {int(np.flatnonzero(np.abs(wsum - 1.0) > 1e-13)[0])} weights do not sum to 1")
        first = self.fq_point[self.face_fq_start[self.fq_face]]
        d = np.einsum("qd,qd->q", self.fq_point - first, self.face_normal[self.fq_face])
        if np.max(np.abs(d)) > 1e-10 * scale:
            raise MeshError("face quadrature points leave the face plane")
        return True


# -- box generator (boxgen.py:16-115) ----------------------------------------

_KUHN_TETS = np.array(((0, 1, 2, 6), (0, 2, 3, 6), (0, 3, 7, 6), (0, 7, 4, 6), (0, 4, 5, 6), (0, 5, 1, 6)))
_SIDES = ("xmin", "xmax", "ymin", "ymax", "zmin", "zmax")


def generate_box_mesh(extent, divisions, split="hex", perturb=0.0, seed=None, periodic=()):
    extent = np.asarray(extent, dtype=float)
    divisions = np.asarray(divisions, dtype=int)
    if np.any(extent <= 0.0):
        raise MeshError("box extent must be positive")
    if np.any(divisions < 1):
        raise MeshError("divisions must be >= 1 per axis")
    if perturb and split != "tet":
        raise MeshError("node perturbation requires the tet split (hex faces must stay planar)")
    if perturb < 0.0 or perturb > 0.3:
        if perturb:
            raise MeshError("perturb fraction must lie in [0, 0.3]")
    nx, ny, nz = (int(d) for d in divisions)
    spacing = extent / divisions
    xs = [np.linspace(0.0, extent[d], divisions[d] + 1) for d in range(3)]
    grid = np.stack(np.meshgrid(xs[0], xs[1], xs[2], indexing="ij"), axis=-1)
    if perturb:
        rng = np.random.default_rng(seed)
        jig = rng.uniform(-perturb, perturb, grid.shape) * spacing
        jig[0, :, :, 0] = jig[-1, :, :, 0] = 0.0
        jig[:, 0, :, 1] = jig[:, -1, :, 1] = 0.0
        jig[:, :, 0, 2] = jig[:, :, -1, 2] = 0.0
        mask = np.zeros(grid.shape[:3], dtype=bool)
        mask[1:-1, 1:-1, 1:-1] = True
        grid = grid + jig * mask[..., None]
    nodes = grid.reshape(-1, 3)

    def nid(i, j, k):
        return (i * (ny + 1) + j) * (nz + 1) + k

    i, j, k = np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij")
    i, j, k = i.ravel(), j.ravel(), k.ravel()
    hexes = np.stack([nid(i, j, k), nid(i + 1, j, k), nid(i + 1, j + 1, k), nid(i, j + 1, k),
                      nid(i, j, k + 1), nid(i + 1, j, k + 1), nid(i + 1, j + 1, k + 1), nid(i, j + 1, k + 1)], axis=1)
    if split == "hex":
        tets, hx = np.zeros((0, 4), np.int64), hexes
    elif split == "tet":
        tets, hx = hexes[:, _KUHN_TETS].reshape(-1, 4), np.zeros((0, 8), np.int64)
    else:
        raise MeshError(f"unknown split {split!r}")

    def quads(a, b, fn):
        a, b = np.meshgrid(np.arange(a), np.arange(b), indexing="ij")
        return fn(a.ravel(), b.ravel())

    side = {
        "xmin": quads(ny, nz, lambda j, k: np.stack([nid(0, j, k), nid(0, j + 1, k), nid(0, j + 1, k + 1), nid(0, j, k + 1)], 1)),
        "xmax": quads(ny, nz, lambda j, k: np.stack([nid(nx, j, k), nid(nx, j + 1, k), nid(nx, j + 1, k + 1), nid(nx, j, k + 1)], 1)),
        "ymin": quads(nx, nz, lambda i, k: np.stack([nid(i, 0, k), nid(i + 1, 0, k), nid(i + 1, 0, k + 1), nid(i, 0, k + 1)], 1)),
        "ymax": quads(nx, nz, lambda i, k: np.stack([nid(i, ny, k), nid(i + 1, ny, k), nid(i + 1, ny, k + 1), nid(i, ny, k + 1)], 1)),
        "zmin": quads(nx, ny, lambda i, j: np.stack([nid(i, j, 0), nid(i + 1, j, 0), nid(i + 1, j + 1, 0), nid(i, j + 1, 0)], 1)),
        "zmax": quads(nx, ny, lambda i, j: np.stack([nid(i, j, nz), nid(i + 1, j, nz), nid(i + 1, j + 1, nz), nid(i, j + 1, nz)], 1)),
    }
    if split == "tet":
        # split along the first-to-third diagonal the Kuhn subdivision cuts (boxgen.py:105-115)
        side = {n: np.stack([q[:, [0, 1, 2]], q[:, [0, 2, 3]]], axis=1).reshape(-1, 3) for n, q in side.items()}
    patch_faces = {n: side[n] for n in _SIDES}
    pairs = []
    for axis in periodic:
        idx = "xyz".index(axis)
        pairs.append((_SIDES[2 * idx], _SIDES[2 * idx + 1]))
    return Mesh.build(nodes, tets, hx, patch_faces, periodic_pairs=pairs)


# -- ugks-mesh file I/O (fileio.py:1-124) ------------------------------------

MAGIC = "ugks-mesh"
VERSION = 1


def _load_native(path):
    """Fast path: the C++ reader in libgks.so (gks_meshio.cpp).  Returns the
    construction data, or None when the native reader rejects the file (the
    reference-shaped parser below then runs and raises its exact error)."""
    import ctypes as C

    from . import _native as N

    lib = N.load()
    h = C.c_void_p()
    if lib.gks_ugks_read(str(path).encode(), C.byref(h)) != 0:
        return None
    try:
        sz = [C.c_int64() for _ in range(4)]
        N.check(lib.gks_ugks_sizes(h, *[C.byref(x) for x in sz]))
        nn, nt, nh, npatch = (int(x.value) for x in sz)
        names, counts = [], []
        buf = C.create_string_buffer(4096)
        for k in range(npatch):
            nf = C.c_int64()
            N.check(lib.gks_ugks_patch(h, k, buf, len(buf), C.byref(nf)))
            names.append(buf.value.decode("ascii"))
            counts.append(int(nf.value))
        total = sum(counts)
        nodes = np.empty((nn, 3))
        tets = np.empty((nt, 4), dtype=np.int64)
        hexes = np.empty((nh, 8), dtype=np.int64)
        faces = np.empty((max(total, 1), 4), dtype=np.int64)
        widths = np.empty(max(total, 1), dtype=np.int8)
        N.check(lib.gks_ugks_copy(h, N.dptr(nodes), N.iptr(tets), N.iptr(hexes), N.iptr(faces),
                                  widths.ctypes.data_as(C.c_void_p)))
    finally:
        lib.gks_ugks_free(h)
    patch_faces = {}
    pos = 0
    for name, nf in zip(names, counts):
        f, w = faces[pos: pos + nf], widths[pos: pos + nf]
        pos += nf
        if nf and np.all(w == w[0]):
            patch_faces[name] = np.ascontiguousarray(f[:, : int(w[0])])
        else:
            patch_faces[name] = [tuple(int(x) for x in r[: int(k)]) for r, k in zip(f, w)]
    return nodes, tets, hexes, patch_faces


def load_mesh(path, periodic_pairs=()):
    """Parse, build and validate a ugks-mesh ASCII file (fileio.py:42-103).

    The file is read by the native parser (gks_ugks_read); anything it
    rejects is re-parsed here, line by line, to raise the reference's error."""
    fast = _load_native(path)
    if fast is not None:
        nodes, tets, hexes, patch_faces = fast
        mesh = Mesh.build(nodes, tets, hexes, patch_faces, periodic_pairs=periodic_pairs)
        mesh.validate()
        return mesh
    with open(path, "r", encoding="ascii") as fh:
        raw = [ln.split("#", 1)[0].strip() for ln in fh.read().splitlines()]
    lines = [ln for ln in raw if ln]
    pos = 0

    def nxt():
        nonlocal pos
        if pos >= len(lines):
            raise MeshError("unexpected end of mesh file")
        pos += 1
        return lines[pos - 1]

    head = nxt().split()
    if len(head) != 2 or head[0] != MAGIC or head[1] != str(VERSION):
        raise MeshError(f"bad header {head!r}; expected '{MAGIC} {VERSION}'")

    def counted(tag):
        tok = nxt().split()
        if len(tok) != 2 or tok[0] != tag:
            raise MeshError(f"expected '{tag} <count>', got {tok!r}")
        try:
            n = int(tok[1])
        except ValueError as exc:
            raise MeshError(f"bad count for {tag}: {tok[1]!r}") from exc
        if n < 0:
            raise MeshError(f"negative count for {tag}")
        return n

    def block(count, width, conv, what):
        nonlocal pos
        if pos + count > len(lines):
            raise MeshError("unexpected end of mesh file")
        rows = [ln.split() for ln in lines[pos: pos + count]]
        for i, r in enumerate(rows):
            if len(r) != width:
                raise MeshError(f"{what} {i}: expected {width} {'coordinates' if what == 'node' else 'node ids'}")
        pos += count
        return np.array(rows, dtype=conv).reshape(count, width)

    nodes = block(counted("nodes"), 3, float, "node")
    tets = block(counted("tets"), 4, np.int64, "tets")
    hexes = block(counted("hexes"), 8, np.int64, "hexes")
    npatch = counted("patches")
    patch_faces = {}
    for _ in range(npatch):
        tok = nxt().split()
        if len(tok) != 2:
            raise MeshError(f"expected '<patch-name> <faces>', got {tok!r}")
        name, nf = tok[0], int(tok[1])
        if name in patch_faces:
            raise MeshError(f"duplicate patch name {name!r}")
        faces = []
        for i in range(nf):
            ids = [int(p) for p in nxt().split()]
            if len(ids) not in (3, 4):
                raise MeshError(f"patch {name!r} face {i}: need 3 or 4 node ids")
            faces.append(tuple(ids))
        patch_faces[name] = faces
    mesh = Mesh.build(nodes, tets, hexes, patch_faces, periodic_pairs=periodic_pairs)
    mesh.validate()
    return mesh


def save_mesh(mesh: Mesh, path):
    """Write the construction data back out; floats use repr (bit-exact round trip)."""
    tets, hexes, patch_faces = mesh._source
    with open(path, "w", encoding="ascii") as fh:
        fh.write(f"{MAGIC} {VERSION}\n")
        fh.write(f"nodes {len(mesh.nodes)}\n")
        fh.writelines(f"{float(x)!r} {float(y)!r} {float(z)!r}\n" for x, y, z in mesh.nodes)
        fh.write(f"tets {len(tets)}\n")
        fh.writelines(" ".join(str(i) for i in c) + "\n" for c in tets)
        fh.write(f"hexes {len(hexes)}\n")
        fh.writelines(" ".join(str(i) for i in c) + "\n" for c in hexes)
        fh.write(f"patches {len(patch_faces)}\n")
        for name, faces in patch_faces.items():
            fh.write(f"{name} {len(faces)}\n")
            fh.writelines(" ".join(str(i) for i in f) + "\n" for f in faces)
