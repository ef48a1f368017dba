"""Locality reordering of the device mesh (north star "mesh layout").

Meshes read from files arrive in whatever order their generator wrote them;
a shuffled copy of the C2 sphere runs its step 21 % slower on the B200
(tools/reorder_probe.py: face kernel 2.88 -> 3.33 ms, reconstruction 0.84 ->
1.05 ms, Jacobi sweep 0.16 -> 0.35 ms), because every neighbour and stencil
gather misses.  `SolverOptions(reorder="rcm" | "morton")` renumbers the
cells (reverse Cuthill-McKee on the face graph, or the Morton curve of the
centroids) and sorts the faces by their new owner, so consecutive threads
gather consecutive cells.

The renumbering lives entirely inside the solver handle:
  * stencil selection and the reconstruction operators are computed on the
    reference's numbering (bit-exact selection) and then
    restricted/permuted with gks_setup_subset;
  * every per-cell summation keeps the reference's order: the mesh
    descriptor carries each face's and face point's original index
    (`face_rank`, `fq_rank`), and the handle builds its assembly, local-dt
    and Jacobian-diagonal lists in that order;
  * the Python Solver permutes arrays on the way in and out, so callers see
    the reference's numbering everywhere.
"""

from __future__ import annotations

import numpy as np

METHODS = ("none", "rcm", "morton")


def _csr_gather(start, perm):
    """Index array that gathers the CSR blocks `perm` (new -> old) in order."""
    start = np.asarray(start, dtype=np.int64)
    lens = np.diff(start)[perm]
    new_start = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    idx = np.repeat(start[perm] - new_start[:-1], lens) + np.arange(new_start[-1], dtype=np.int64)
    return idx, new_start


def cell_order(mesh, method: str) -> np.ndarray:
    """New -> old cell permutation."""
    nc = mesh.ncells
    if method == "none":
        return np.arange(nc, dtype=np.int64)
    if method == "morton":
        c = mesh.cell_centroid
        lo, hi = c.min(axis=0), c.max(axis=0)
        q = ((c - lo) / np.maximum(hi - lo, 1e-300) * ((1 << 21) - 1)).astype(np.uint64)
        code = np.zeros(nc, dtype=np.uint64)
        for b in range(21):
            for ax in range(3):
                code |= ((q[:, ax] >> np.uint64(b)) & np.uint64(1)) << np.uint64(3 * b + ax)
        return np.argsort(code, kind="stable").astype(np.int64)
    if method == "rcm":
        from scipy.sparse import coo_matrix
        from scipy.sparse.csgraph import reverse_cuthill_mckee

        own, nb = mesh.face_owner, mesh.face_neighbor
        sel = nb >= 0
        r = np.concatenate([own[sel], nb[sel]])
        c = np.concatenate([nb[sel], own[sel]])
        g = coo_matrix((np.ones(len(r), dtype=np.int8), (r, c)), shape=(nc, nc)).tocsr()
        return np.asarray(reverse_cuthill_mckee(g, symmetric_mode=True), dtype=np.int64)
    raise ValueError(f"reorder must be one of {METHODS}, got {method!r}")


class PermutedMesh:
    """Mesh-like view of `mesh` with cells renumbered by `perm` (new -> old)
    and faces sorted by their new owner; exposes the GksMeshDesc fields plus
    the original face / face-point indices (face_rank, fq_rank)."""

    def __init__(self, mesh, perm):
        perm = np.asarray(perm, dtype=np.int64)
        nc = mesh.ncells
        inv = np.empty(nc, dtype=np.int64)
        inv[perm] = np.arange(nc, dtype=np.int64)
        self.perm, self.inv = perm, inv
        self.cell_rank = perm  # reference id of each device cell (Jacobian column order)
        self.ncells, self.nfaces = nc, mesh.nfaces
        self.patch_names = list(mesh.patch_names)
        for name in ("cell_kind", "cell_volume", "cell_h", "cell_centroid"):
            setattr(self, name, getattr(mesh, name)[perm])
        qidx, self.cell_cq_start = _csr_gather(mesh.cell_cq_start, perm)
        self.cq_point = mesh.cq_point[qidx]
        self.cq_weight = mesh.cq_weight[qidx]
        # faces: by new owner, original order inside an owner (stable)
        fperm = np.argsort(inv[mesh.face_owner], kind="stable").astype(np.int64)
        finv = np.empty(mesh.nfaces, dtype=np.int64)
        finv[fperm] = np.arange(mesh.nfaces, dtype=np.int64)
        self.face_rank = fperm
        self.face_owner = inv[mesh.face_owner[fperm]]
        nb = mesh.face_neighbor[fperm]
        self.face_neighbor = np.where(nb >= 0, inv[np.maximum(nb, 0)], -1)
        for name in ("face_patch", "face_area", "face_normal", "face_frame", "face_shift"):
            setattr(self, name, getattr(mesh, name)[fperm])
        fqidx, self.face_fq_start = _csr_gather(mesh.face_fq_start, fperm)
        self.fq_rank = fqidx
        self.fq_point = mesh.fq_point[fqidx]
        self.fq_weight = mesh.fq_weight[fqidx]
        self.fq_face = finv[mesh.fq_face[fqidx]]
        # cell -> faces in each cell's own pattern order, face ids renumbered
        cidx, self.cell_face_start = _csr_gather(mesh.cell_face_start, perm)
        self.cell_face_list = finv[mesh.cell_face_list[cidx]]
