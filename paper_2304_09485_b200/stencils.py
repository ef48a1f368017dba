"""Stencil selection (native): mirrors gks3d/mesh/stencils.py.

The per-cell selection runs in C++ (csrc/gks_setup.cpp, OpenMP); this module
exposes it through the reference's StencilTable / CellStencil view
(stencils.py:42-69) for tests and the case API.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _native as N


@dataclass
class CellStencil:
    cell: int
    neighbor_ids: np.ndarray
    neighbor_shifts: np.ndarray
    big_ids: np.ndarray
    big_shifts: np.ndarray
    sub_ids: list = field(default_factory=list)
    sub_shifts: list = field(default_factory=list)
    hbig_ids: np.ndarray | None = None
    hbig_shifts: np.ndarray | None = None
    hsub_ids: list = field(default_factory=list)
    hsub_shifts: list = field(default_factory=list)
    weno_fallback: bool = False
    hweno_fallback: bool = False


class StencilTable:
    """Lazy per-cell view over the flat native stencil arrays."""

    def __init__(self, setup: N.NativeSetup, mesh):
        self.setup = setup
        self.mesh = mesh
        a = setup.array
        self.nbr_ids = a("nbr_ids")
        self.nbr_shift = a("nbr_shift")
        self.big_start = a("big_start")
        self.big_ids = a("big_ids")
        self.big_shift = a("big_shift")
        self.sub_cell_start = a("sub_cell_start")
        self.sub_member_start = a("sub_member_start")
        self.sub_ids = a("sub_ids")
        self.sub_shift = a("sub_shift")
        self.weno_fallback = a("weno_fallback").astype(bool)
        self.hweno_fallback = a("hweno_fallback").astype(bool)
        self.cells = _Cells(self)

    def __len__(self):
        return self.mesh.ncells

    def __getitem__(self, c) -> CellStencil:
        c = int(c)
        nf = int(self.mesh.cell_face_start[c + 1] - self.mesh.cell_face_start[c])
        ids = self.nbr_ids[c, :nf].copy()
        sh = self.nbr_shift[c, :nf].copy()
        b0, b1 = self.big_start[c], self.big_start[c + 1]
        st = CellStencil(c, ids, sh, self.big_ids[b0:b1].copy(), self.big_shift[b0:b1].copy())
        for s in range(self.sub_cell_start[c], self.sub_cell_start[c + 1]):
            m0, m1 = self.sub_member_start[s], self.sub_member_start[s + 1]
            st.sub_ids.append(self.sub_ids[m0:m1].copy())
            st.sub_shifts.append(self.sub_shift[m0:m1].copy())
        st.weno_fallback = bool(self.weno_fallback[c])
        st.hweno_fallback = bool(self.hweno_fallback[c])
        present = ids >= 0
        st.hbig_ids = np.concatenate([[c], ids[present]]).astype(np.int64)
        st.hbig_shifts = np.vstack([np.zeros(3), sh[present]]) if present.any() else np.zeros((1, 3))
        if not st.hweno_fallback:
            for i, s in zip(ids[present], sh[present]):
                st.hsub_ids.append(np.array([c, i], dtype=np.int64))
                st.hsub_shifts.append(np.vstack([np.zeros(3), s]))
        return st


class _Cells:
    def __init__(self, table):
        self.t = table

    def __len__(self):
        return len(self.t)

    def __getitem__(self, c):
        return self.t[c]

    def __iter__(self):
        return (self.t[c] for c in range(len(self.t)))


def build_stencils(mesh, nthreads=0) -> StencilTable:
    """Select big and sub-candidate stencils for every cell (stencils.py:119-192)."""
    return StencilTable(N.NativeSetup(mesh, schemes=0, nthreads=nthreads), mesh)  # schemes 0: stencils only
