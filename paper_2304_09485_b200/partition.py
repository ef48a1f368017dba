"""Domain decomposition for the multi-GPU path.

* Canonical order: the cells are ordered once per mesh, independent of the
  number of ranks, by recursive coordinate bisection (RCB) of the centroids
  (`CANON_DEPTH` levels, every cut on a multiple of the reduction granule,
  reference order kept inside each leaf).
* Partition: rank r owns the contiguous canonical range [bounds[r],
  bounds[r+1]).  For 2^k ranks (k <= CANON_DEPTH) these ranges are exactly
  the RCB parts of level k; otherwise equal ranges of the RCB curve.  Every
  boundary is a multiple of gks_reduction_granularity(nc) cells, so each
  rank owns whole reduction groups and every GMRES dot / norm is
  partition-invariant (csrc/gks_reduce.cuh): N-rank runs reproduce the
  1-rank canonical run bit for bit.
* LocalDomain: one rank's view.  Local cells are ordered
      [owned (canonical order) | ghost layer 1 | layer 2 | ...]
  (each layer in canonical order).  Owned cells and layer-1 ghosts are
  reconstructed locally (redundant reconstruction instead of a coefficient
  exchange), so the Q halo is `layers` deep: 3 for WENO (two-level stencils
  of layer-1 ghosts), 2 for HWENO (Q and gradients).
* Exchange maps: for every peer, the local ids this rank sends (owned cells
  the peer needs, in the peer's ghost order) and the local ids it receives
  into.  "x" maps cover layer 1 only (Krylov vectors before each
  off-diagonal product); "q" maps cover all ghost layers.  A rank derives
  its send lists by computing its peers' ghost layers from the cut faces
  (no exchange of index lists, no global domain list).
* LocalMesh: the rank's faces (every face touching an owned cell) sorted by
  local owner, with each face's / face point's rank in the reference order
  (face_rank, fq_rank) and each cell's reference id (cell_rank), so the
  device sums every per-cell list in the reference's order.
* SetupMesh: the rank's cells in reference-id order with ALL their faces
  (faces leaving the set become boundary faces), the input of a per-rank
  native setup: stencils and operators of every reconstructed cell are
  bit-identical to the global build (tests/test_partition.py) without
  building the global operator tables on every rank.

Everything is vectorised numpy (no per-cell Python loops).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .reorder import _csr_gather

CANON_DEPTH = 6  # RCB levels of the canonical order (exact RCB parts up to 64 ranks)


def reduction_granule(nc_global: int) -> int:
    """Cells per reduction group (csrc/gks_reduce.cuh red_group_cells)."""
    seg = 768
    nseg = -(-nc_global // seg)
    g = 1
    while -(-nseg // g) > 1024:
        g *= 2
    return seg * g


def cell_adjacency(mesh):
    """CSR of face neighbours per cell (interior faces, both directions)."""
    inner = mesh.face_neighbor >= 0
    a = np.concatenate([mesh.face_owner[inner], mesh.face_neighbor[inner]])
    b = np.concatenate([mesh.face_neighbor[inner], mesh.face_owner[inner]])
    order = np.argsort(a, kind="stable")
    start = np.concatenate([[0], np.cumsum(np.bincount(a, minlength=mesh.ncells))]).astype(np.int64)
    return start, b[order].astype(np.int64)


def _rows(start, adj, rows):
    idx, _ = _csr_gather(start, rows)
    return adj[idx]


@dataclass
class Canonical:
    perm: np.ndarray      # canonical position -> reference cell id
    pos: np.ndarray       # reference cell id -> canonical position
    levels: list          # levels[d]: boundaries of the 2^d RCB parts (len 2^d + 1, may be shorter)
    granule: int


def canonical_order(mesh, granule=None, depth=CANON_DEPTH) -> Canonical:
    nc = mesh.ncells
    granule = reduction_granule(nc) if granule is None else int(granule)
    cen = mesh.cell_centroid
    order = np.arange(nc, dtype=np.int64)
    bounds = [0, nc]
    levels = [list(bounds)]
    for _ in range(depth):
        nb = [0]
        split_all = True
        for lo, hi in zip(bounds[:-1], bounds[1:]):
            n = hi - lo
            k = int(round(n / 2 / granule)) * granule
            if k <= 0 or k >= n:
                split_all = False
                nb.append(hi)
                continue
            ids = order[lo:hi].copy()
            c = cen[ids]
            ax = int(np.argmax(c.max(axis=0) - c.min(axis=0)))
            srt = np.lexsort((ids, c[:, ax]))
            # keep the reference order inside each half (locality of the input numbering)
            order[lo:lo + k] = np.sort(ids[srt[:k]])
            order[lo + k:hi] = np.sort(ids[srt[k:]])
            nb += [lo + k, hi]
        bounds = nb
        levels.append(list(bounds) if split_all else [])
        if not split_all:
            break
    pos = np.empty(nc, dtype=np.int64)
    pos[order] = np.arange(nc, dtype=np.int64)
    return Canonical(order, pos, levels, granule)


def partition_bounds(canon: Canonical, nranks: int) -> np.ndarray:
    """Canonical position of each rank's first owned cell (len nranks + 1)."""
    nc = len(canon.perm)
    if nranks < 1:
        raise ValueError("nranks must be >= 1")
    d = nranks.bit_length() - 1
    if (1 << d) == nranks and d < len(canon.levels) and len(canon.levels[d]) == nranks + 1:
        return np.asarray(canon.levels[d], dtype=np.int64)
    g = canon.granule
    b = [min(nc, int(round(r * nc / nranks / g)) * g) for r in range(nranks)] + [nc]
    b = np.asarray(b, dtype=np.int64)
    if np.any(np.diff(b) <= 0):
        raise ValueError(f"{nc} cells cannot be split into {nranks} ranks of whole {g}-cell reduction groups")
    return b


@dataclass
class Decomposition:
    """Partition of a mesh into nranks contiguous canonical ranges."""
    canon: Canonical
    bounds: np.ndarray
    part: np.ndarray      # rank per reference cell
    nranks: int
    adj: tuple = None     # cell adjacency CSR (start, list)
    cut: np.ndarray = None  # interior faces whose two cells live on different ranks

    @classmethod
    def build(cls, mesh, nranks: int, canon: Canonical = None):
        canon = canonical_order(mesh) if canon is None else canon
        bounds = partition_bounds(canon, nranks)
        part = np.empty(mesh.ncells, dtype=np.int64)
        part[canon.perm] = np.repeat(np.arange(nranks, dtype=np.int64), np.diff(bounds))
        inner = np.flatnonzero(mesh.face_neighbor >= 0)
        cut = inner[part[mesh.face_owner[inner]] != part[mesh.face_neighbor[inner]]]
        return cls(canon, bounds, part, nranks, cell_adjacency(mesh), cut)

    def owned(self, rank: int) -> np.ndarray:
        return self.canon.perm[self.bounds[rank]:self.bounds[rank + 1]]

    def ghost_layers(self, mesh, rank: int, layers: int) -> list:
        """Reference ids of ghost layers 1..layers of `rank`, each in canonical order."""
        start, adj = self.adj
        fo, fn = mesh.face_owner[self.cut], mesh.face_neighbor[self.cut]
        po, pn = self.part[fo], self.part[fn]
        l1 = np.concatenate([fn[po == rank], fo[pn == rank]])
        mark = self.part == rank
        out = []
        frontier = None
        for k in range(layers):
            nb = l1 if k == 0 else _rows(start, adj, frontier)
            nb = np.unique(nb)
            nb = nb[~mark[nb]]
            nb = nb[np.argsort(self.canon.pos[nb], kind="stable")]
            mark[nb] = True
            out.append(nb)
            frontier = nb
        return out


@dataclass
class LocalDomain:
    rank: int
    nranks: int
    cells: np.ndarray            # local -> reference cell id
    n_owned: int
    layer_start: list            # local index where ghost layer k (1-based) starts; last entry = n_local
    owner_rank: np.ndarray       # per local cell
    owned_offset: int = 0        # canonical position of the first owned cell
    nc_global: int = 0
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

    def g2l(self, nc_global):
        m = np.full(nc_global, -1, dtype=np.int64)
        m[self.cells] = np.arange(len(self.cells), dtype=np.int64)
        return m


def build_domain(mesh, dec: Decomposition, rank: int, layers: int) -> LocalDomain:
    """One rank's LocalDomain with its exchange maps (computed locally)."""
    owned = dec.owned(rank)
    gl = dec.ghost_layers(mesh, rank, layers)
    cells = np.concatenate([owned] + gl).astype(np.int64)
    ls = [len(owned)]
    for g in gl:
        ls.append(ls[-1] + len(g))
    d = LocalDomain(rank, dec.nranks, cells, len(owned), ls, dec.part[cells], int(dec.bounds[rank]), mesh.ncells)
    # receive: my ghosts grouped by owner, in my ghost order
    ghosts = np.arange(d.n_owned, d.n_local)
    src = d.owner_rank[ghosts]
    for kind, last in (("q", d.n_local), ("x", d.n_recon)):
        g, sg = ghosts[:last - d.n_owned], src[:last - d.n_owned]
        for p in np.unique(sg):
            getattr(d, f"{kind}_recv")[int(p)] = g[sg == p]
    # send: the peers' ghosts I own, in the peer's ghost order (peers = owners
    # of my ghosts; the ghost relation is symmetric)
    for p in np.unique(src):
        p = int(p)
        pg = dec.ghost_layers(mesh, p, layers)
        for kind, nl in (("q", layers), ("x", 1)):
            theirs = np.concatenate(pg[:nl]) if nl else np.zeros(0, np.int64)
            mine = theirs[dec.part[theirs] == rank]
            getattr(d, f"{kind}_send")[p] = dec.canon.pos[mine] - dec.bounds[rank]
    return d


def build_domains(mesh, dec: Decomposition, layers: int) -> list:
    return [build_domain(mesh, dec, r, layers) for r in range(dec.nranks)]


class LocalMesh:
    """Mesh-like view of one rank's cells and faces, local numbering.

    Cell arrays cover every local cell; faces are the reference faces that
    touch an owned cell (both their cells are local by construction), sorted
    by local owner.  face_rank / fq_rank give each face's / face point's
    position in the reference order among the local ones, cell_rank the
    reference id of each local cell.
    """

    def __init__(self, mesh, dom: LocalDomain, g2l=None):
        c = dom.cells
        g2l = dom.g2l(mesh.ncells) if g2l is None else g2l
        self.ncells = len(c)
        self.cell_rank = c
        self.cell_kind = mesh.cell_kind[c]
        self.cell_volume = mesh.cell_volume[c]
        self.cell_h = mesh.cell_h[c]
        self.cell_centroid = mesh.cell_centroid[c]
        qidx, self.cell_cq_start = _csr_gather(mesh.cell_cq_start, c)
        self.cq_point = mesh.cq_point[qidx]
        self.cq_weight = mesh.cq_weight[qidx]
        own_mark = np.zeros(mesh.ncells, dtype=bool)
        own_mark[c[:dom.n_owned]] = True
        nbr = mesh.face_neighbor
        touch = own_mark[mesh.face_owner] | ((nbr >= 0) & own_mark[np.maximum(nbr, 0)])
        faces = np.flatnonzero(touch)  # reference order
        lown = g2l[mesh.face_owner[faces]]
        fnb = nbr[faces]
        lnb = np.where(fnb >= 0, g2l[np.maximum(fnb, 0)], -1)
        if np.any(lown < 0) or np.any((fnb >= 0) & (lnb < 0)):
            raise ValueError("local face references a non-local cell")
        fperm = np.lexsort((np.arange(len(faces)), lown))  # by local owner, reference order inside
        self.faces = faces[fperm]  # local face -> reference face id
        self.nfaces = len(faces)
        self.face_rank = fperm.astype(np.int64)
        self.face_owner = lown[fperm]
        self.face_neighbor = lnb[fperm]
        for name in ("face_patch", "face_area", "face_normal", "face_frame", "face_shift"):
            setattr(self, name, getattr(mesh, name)[self.faces])
        fqidx, self.face_fq_start = _csr_gather(mesh.face_fq_start, self.faces)
        fq_sorted, _ = _csr_gather(mesh.face_fq_start, faces)
        self.fq_global = fqidx
        self.fq_rank = np.searchsorted(fq_sorted, fqidx).astype(np.int64)
        self.fq_point = mesh.fq_point[fqidx]
        self.fq_weight = mesh.fq_weight[fqidx]
        self.fq_face = np.repeat(np.arange(self.nfaces, dtype=np.int64), np.diff(self.face_fq_start))
        # cell -> local faces (only faces present locally), in each cell's face order
        f2l = np.full(mesh.nfaces, -1, dtype=np.int64)
        f2l[self.faces] = np.arange(self.nfaces, dtype=np.int64)
        cidx, cstart = _csr_gather(mesh.cell_face_start, c)
        lf = f2l[mesh.cell_face_list[cidx]]
        keep = lf >= 0
        row = np.repeat(np.arange(len(c), dtype=np.int64), np.diff(cstart))
        counts = np.bincount(row[keep], minlength=len(c))
        self.cell_face_start = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
        self.cell_face_list = lf[keep]
        self.patch_names = list(mesh.patch_names)


class SetupMesh:
    """The native-setup view of a rank's cells: local cells in ascending
    reference id (so id-ordered stencil choices match the global build) and
    every face of every such cell; a face whose other cell is not local
    becomes a boundary face of the inside cell (only cells of the outermost
    ghost layer have such faces, and their own stencils are never used).

    local_to_sub / sub_to_local map between the rank-local cell order and
    this one (gks_setup_subset)."""

    def __init__(self, mesh, dom: LocalDomain):
        cells = np.sort(dom.cells)
        n = len(cells)
        self.ncells = n
        self.local_to_sub = np.searchsorted(cells, dom.cells).astype(np.int64)
        self.sub_to_local = np.empty(n, dtype=np.int64)
        self.sub_to_local[self.local_to_sub] = np.arange(n, dtype=np.int64)
        for name in ("cell_kind", "cell_volume", "cell_h", "cell_centroid"):
            setattr(self, name, getattr(mesh, name)[cells])
        qidx, self.cell_cq_start = _csr_gather(mesh.cell_cq_start, cells)
        self.cq_point = mesh.cq_point[qidx]
        self.cq_weight = mesh.cq_weight[qidx]
        cidx, self.cell_face_start = _csr_gather(mesh.cell_face_start, cells)
        cf = mesh.cell_face_list[cidx]
        faces = np.unique(cf)
        self.nfaces = len(faces)
        g2s = np.full(mesh.ncells, -1, dtype=np.int64)
        g2s[cells] = np.arange(n, dtype=np.int64)
        so = g2s[mesh.face_owner[faces]]
        fn = mesh.face_neighbor[faces]
        sn = np.where(fn >= 0, g2s[np.maximum(fn, 0)], -1)
        flip = so < 0  # owner outside: the inside neighbour owns the (now boundary) face
        sgn = np.where(flip, -1.0, 1.0)[:, None]
        self.face_owner = np.where(flip, sn, so)
        self.face_neighbor = np.where(flip, -1, sn)
        self.face_normal = mesh.face_normal[faces] * sgn
        self.face_shift = mesh.face_shift[faces] * sgn
        self.face_frame = mesh.face_frame[faces]
        self.face_area = mesh.face_area[faces]
        self.face_patch = np.where(self.face_neighbor < 0, np.maximum(mesh.face_patch[faces], 0), -1)
        self.cell_face_list = np.searchsorted(faces, cf).astype(np.int64)
        # the setup never reads face points
        self.face_fq_start = np.zeros(self.nfaces + 1, dtype=np.int64)
        self.fq_face = np.zeros(0, dtype=np.int64)
        self.fq_point = np.zeros((0, 3))
        self.fq_weight = np.zeros(0)
        self.patch_names = list(mesh.patch_names)


def stencil_closure_ok(stencils, dom: LocalDomain, g2l) -> bool:
    """Every big/sub stencil member of a locally reconstructed cell is local (D4 self-consistency)."""
    ids = []
    for lc in range(dom.n_recon):
        st = stencils[int(dom.cells[lc])]
        ids.append(np.asarray(st.big_ids, dtype=np.int64))
        ids.extend(np.asarray(m, dtype=np.int64) for m in st.sub_ids)
        ids.append(np.asarray(st.hbig_ids, dtype=np.int64))
    ids = np.concatenate(ids) if ids else np.zeros(0, np.int64)
    return bool(np.all(g2l[ids] >= 0))
