"""Domain decomposition for the multi-GPU path.

* partition_cells: recursive coordinate bisection of the cell centroids into
  nparts equal-count parts (deterministic; cut quality is adequate for the
  box / sphere meshes and needs no METIS).
* LocalDomain: one rank's view.  Local cells are ordered
      [owned (global order) | ghost layer 1 | layer 2 | ...]
  Owned cells and layer-1 ghosts are reconstructed locally (redundant
  reconstruction instead of a coefficient exchange), so the Q halo is
  `layers` deep: 3 for WENO (two-level stencils of layer-1 ghosts), 2 for
  HWENO (Q and gradients).  Local faces are every global face touching an
  owned cell, kept in global order, so each owned cell assembles its face
  contributions in exactly the single-GPU / reference order.
* Exchange maps: for every peer, the local ids this rank sends (owned cells
  the peer needs, in the peer's ghost order) and the local ids it receives
  into.  "x" maps cover layer 1 only (Krylov vectors before each
  off-diagonal product); "q" maps cover all ghost layers.

The ghost maps are checked for self-consistency against the global stencil
tables (tests/test_partition.py): every stencil member of a
locally reconstructed cell is local.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


def partition_cells(mesh, nparts: int) -> np.ndarray:
    """Part id per cell by recursive coordinate bisection (equal counts)."""
    part = np.zeros(mesh.ncells, dtype=np.int64)
    if nparts <= 1:
        return part
    cen = mesh.cell_centroid

    def split(ids, lo, n):
        if n == 1:
            part[ids] = lo
            return
        n0 = n // 2
        ext = cen[ids].max(axis=0) - cen[ids].min(axis=0)
        ax = int(np.argmax(ext))
        order = ids[np.lexsort((ids, cen[ids, ax]))]
        k = (len(ids) * n0) // n
        split(order[:k], lo, n0)
        split(order[k:], lo + n0, n - n0)

    split(np.arange(mesh.ncells), 0, nparts)
    return part


def cell_adjacency(mesh):
    """CSR of face neighbours per cell (interior faces, both directions)."""
    inner = mesh.face_neighbor >= 0
    a = np.concatenate([mesh.face_owner[inner], mesh.face_neighbor[inner]])
    b = np.concatenate([mesh.face_neighbor[inner], mesh.face_owner[inner]])
    order = np.argsort(a, kind="stable")
    start = np.concatenate([[0], np.cumsum(np.bincount(a, minlength=mesh.ncells))])
    return start, b[order]


@dataclass
class LocalDomain:
    rank: int
    nranks: int
    cells: np.ndarray            # local -> global cell id
    n_owned: int
    layer_start: list            # local index where ghost layer k (1-based) starts; last entry = n_local
    faces: np.ndarray            # local -> global face id (global order)
    owner_rank: np.ndarray       # per local cell
    q_send: dict = field(default_factory=dict)   # peer -> local ids to send (all layers)
    q_recv: dict = field(default_factory=dict)   # peer -> local ids to receive into
    x_send: dict = field(default_factory=dict)   # layer 1 only
    x_recv: dict = field(default_factory=dict)

    @property
    def n_local(self):
        return len(self.cells)

    @property
    def n_recon(self):
        """Owned + layer-1 ghosts: the cells reconstructed on this rank."""
        return self.layer_start[1] if len(self.layer_start) > 1 else self.n_owned


def build_domains(mesh, part, layers: int):
    """LocalDomain for every rank (host-side; each rank can build only its own)."""
    nparts = int(part.max()) + 1
    start, adj = cell_adjacency(mesh)
    doms = []
    g2l_all = []
    for r in range(nparts):
        owned = np.flatnonzero(part == r)
        mark = np.zeros(mesh.ncells, dtype=bool)
        mark[owned] = True
        frontier = owned
        ghost_layers = []
        for _ in range(layers):
            nb = np.unique(np.concatenate([adj[start[c]: start[c + 1]] for c in frontier])) if len(frontier) else \
                np.zeros(0, np.int64)
            nb = nb[~mark[nb]]
            mark[nb] = True
            ghost_layers.append(nb)
            frontier = nb
        cells = np.concatenate([owned] + ghost_layers)
        ls = [len(owned)]
        for gl in ghost_layers:
            ls.append(ls[-1] + len(gl))
        owned_mark = part == r
        touch = owned_mark[mesh.face_owner] | (mesh.face_neighbor >= 0) & owned_mark[np.maximum(mesh.face_neighbor, 0)]
        faces = np.flatnonzero(touch)
        doms.append(LocalDomain(r, nparts, cells, len(owned), ls, faces, part[cells]))
        g2l = np.full(mesh.ncells, -1, dtype=np.int64)
        g2l[cells] = np.arange(len(cells))
        g2l_all.append(g2l)
    # exchange maps: receiver order = local ghost order, grouped by source
    for r, d in enumerate(doms):
        for kind, last in (("q", d.n_local), ("x", d.n_recon)):
            ghosts = np.arange(d.n_owned, last)
            src = d.owner_rank[ghosts]
            for s in np.unique(src):
                ids = ghosts[src == s]
                getattr(d, f"{kind}_recv")[int(s)] = ids
                getattr(doms[s], f"{kind}_send")[r] = g2l_all[s][d.cells[ids]]
    return doms, g2l_all


class LocalMesh:
    """Mesh-like view of one rank's cells/faces with local numbering.

    Cell arrays cover every local cell; face arrays cover the local faces
    (global order).  Faces whose far cell is not local keep -1 only if it is a
    true boundary face; by construction every face touching an owned cell has
    both cells local.
    """

    def __init__(self, mesh, dom: LocalDomain, g2l):
        c = dom.cells
        f = dom.faces
        self.ncells = len(c)
        self.nfaces = len(f)
        self.cell_kind = mesh.cell_kind[c]
        self.cell_volume = mesh.cell_volume[c]
        self.cell_h = mesh.cell_h[c]
        self.cell_centroid = mesh.cell_centroid[c]
        nq = np.diff(mesh.cell_cq_start)[c]
        self.cell_cq_start = np.concatenate([[0], np.cumsum(nq)]).astype(np.int64)
        qidx = np.concatenate([np.arange(mesh.cell_cq_start[g], mesh.cell_cq_start[g + 1]) for g in c])
        self.cq_point = mesh.cq_point[qidx]
        self.cq_weight = mesh.cq_weight[qidx]
        self.face_owner = g2l[mesh.face_owner[f]]
        nb = mesh.face_neighbor[f]
        self.face_neighbor = np.where(nb >= 0, g2l[np.maximum(nb, 0)], -1)
        if np.any(self.face_owner < 0) or np.any((nb >= 0) & (self.face_neighbor < 0)):
            raise ValueError("local face references a non-local cell")
        self.face_patch = mesh.face_patch[f]
        self.face_area = mesh.face_area[f]
        self.face_normal = mesh.face_normal[f]
        self.face_frame = mesh.face_frame[f]
        self.face_shift = mesh.face_shift[f]
        fnq = np.diff(mesh.face_fq_start)[f]
        self.face_fq_start = np.concatenate([[0], np.cumsum(fnq)]).astype(np.int64)
        fq = np.concatenate([np.arange(mesh.face_fq_start[g], mesh.face_fq_start[g + 1]) for g in f])
        self.fq_global = fq
        self.fq_point = mesh.fq_point[fq]
        self.fq_weight = mesh.fq_weight[fq]
        self.fq_face = np.repeat(np.arange(len(f), dtype=np.int64), fnq)
        # cell -> local faces (only faces present locally), in each cell's face order
        f2l = np.full(mesh.nfaces, -1, dtype=np.int64)
        f2l[f] = np.arange(len(f))
        lists = []
        for g in c:
            lf = f2l[mesh.cell_face_list[mesh.cell_face_start[g]: mesh.cell_face_start[g + 1]]]
            lists.append(lf[lf >= 0])
        self.cell_face_start = np.concatenate([[0], np.cumsum([len(x) for x in lists])]).astype(np.int64)
        self.cell_face_list = np.concatenate(lists).astype(np.int64) if lists else np.zeros(0, np.int64)
        self.patch_names = list(mesh.patch_names)


def stencil_closure_ok(stencils, dom: LocalDomain, g2l) -> bool:
    """Every big/sub stencil member of a locally reconstructed cell is local (D4 self-consistency)."""
    for lc in range(dom.n_recon):
        st = stencils[int(dom.cells[lc])]
        members = [st.big_ids] + list(st.sub_ids) + [st.hbig_ids]
        for m in members:
            if np.any(g2l[np.asarray(m, dtype=np.int64)] < 0):
                return False
    return True
