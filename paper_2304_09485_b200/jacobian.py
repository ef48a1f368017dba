"""Roe-split block Jacobian (device-resident), mirrors gks3d/jacobian.py.

BlockJacobian wraps a GksBlockSystem on the GPU: spmv / offdiag_mv /
diag_inverses run as sm_100a kernels (csrc/gks_implicit.cu); the block
arrays are downloaded lazily only when a caller inspects them.
assemble_jacobian builds the matrix of jacobian.py:133-196 on the device.

euler_flux / euler_flux_jacobian / spectral_radius are small pointwise host
utilities kept for API parity (tests, FD probes); the solver never calls
them -- the device kernels carry their own copies.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N
from .kinetic import DEFAULT_GAMMA


def euler_flux(q, n, gamma: float = DEFAULT_GAMMA):
    q = np.atleast_2d(np.asarray(q, dtype=float))
    n = np.atleast_2d(np.asarray(n, dtype=float))
    rho = q[:, 0]
    vel = q[:, 1:4] / rho[:, None]
    un = np.sum(vel * n, axis=1)
    p = (gamma - 1.0) * (q[:, 4] - 0.5 * rho * np.sum(vel * vel, axis=1))
    out = np.empty_like(q)
    out[:, 0] = rho * un
    out[:, 1:4] = q[:, 1:4] * un[:, None] + p[:, None] * n
    out[:, 4] = (q[:, 4] + p) * un
    return out


def euler_flux_jacobian(q, n, gamma: float = DEFAULT_GAMMA):
    q = np.atleast_2d(np.asarray(q, dtype=float))
    n = np.atleast_2d(np.asarray(n, dtype=float))
    g1 = gamma - 1.0
    rho = q[:, 0]
    vel = q[:, 1:4] / rho[:, None]
    un = np.sum(vel * n, axis=1)
    ke = 0.5 * np.sum(vel * vel, axis=1)
    p = g1 * (q[:, 4] - rho * ke)
    h = (q[:, 4] + p) / rho
    jac = np.zeros((len(q), 5, 5))
    jac[:, 0, 1:4] = n
    jac[:, 1:4, 0] = g1 * ke[:, None] * n - vel * un[:, None]
    jac[:, 1:4, 1:4] = vel[:, :, None] * n[:, None, :] - g1 * n[:, :, None] * vel[:, None, :]
    jac[:, [1, 2, 3], [1, 2, 3]] += un[:, None]
    jac[:, 1:4, 4] = g1 * n
    jac[:, 4, 0] = (g1 * ke - h) * un
    jac[:, 4, 1:4] = h[:, None] * n - g1 * vel * un[:, None]
    jac[:, 4, 4] = gamma * un
    return jac


def spectral_radius(q, n, gamma: float = DEFAULT_GAMMA):
    q = np.atleast_2d(np.asarray(q, dtype=float))
    n = np.atleast_2d(np.asarray(n, dtype=float))
    rho = q[:, 0]
    vel = q[:, 1:4] / rho[:, None]
    p = (gamma - 1.0) * (q[:, 4] - 0.5 * rho * np.sum(vel * vel, axis=1))
    return np.abs(np.sum(vel * n, axis=1)) + np.sqrt(gamma * p / rho)


class BlockJacobian:
    """Block-row matrix on the device: diagonal blocks + CSR off-diagonal blocks."""

    def __init__(self, diag=None, off=None, off_col=None, off_row=None, rowptr=None, *, _handle=None,
                 _owner=None, device=0):
        self._owner = _owner  # keeps a solver alive for handle-owned views
        self._cache = {}
        lib = N.load()
        if _handle is not None:
            self._ptr = _handle
            self._owned = False
        else:
            diag = N.f64(diag)
            nc = diag.shape[0]
            off = N.f64(off).reshape(-1, 5, 5)
            off_col = np.ascontiguousarray(off_col, dtype=np.int64)
            rowptr = np.ascontiguousarray(rowptr, dtype=np.int64)
            p = C.c_void_p()
            N.check(lib.gks_blocksys_create(nc, len(off), N.dptr(diag), N.dptr(off), N.iptr(off_col),
                                            N.iptr(rowptr), device, C.byref(p)))
            self._ptr = p
            self._owned = True

    def __del__(self):
        if getattr(self, "_owned", False) and N._lib is not None and self._ptr:
            N._lib.gks_blocksys_destroy(self._ptr)
            self._ptr = None

    @property
    def ncells(self):
        return int(N.load().gks_blocksys_ncells(self._ptr))

    def _export(self):
        if "diag" not in self._cache:
            lib = N.load()
            nc = self.ncells
            nnz = int(lib.gks_blocksys_nnz(self._ptr))
            diag = np.empty((nc, 5, 5))
            off = np.empty((nnz, 5, 5))
            col = np.empty(nnz, dtype=np.int64)
            row = np.empty(nnz, dtype=np.int64)
            rowptr = np.empty(nc + 1, dtype=np.int64)
            N.check(lib.gks_blocksys_export(self._ptr, N.dptr(diag), N.dptr(off), N.iptr(col), N.iptr(row),
                                            N.iptr(rowptr)))
            self._cache.update(diag=diag, off=off, off_col=col, off_row=row, rowptr=rowptr)
        return self._cache

    def invalidate(self):
        self._cache.clear()

    diag = property(lambda self: self._export()["diag"])
    off = property(lambda self: self._export()["off"])
    off_col = property(lambda self: self._export()["off_col"])
    off_row = property(lambda self: self._export()["off_row"])
    rowptr = property(lambda self: self._export()["rowptr"])

    def spmv(self, x):
        x = N.f64(x, (self.ncells, 5))
        y = np.empty_like(x)
        N.check(N.load().gks_blocksys_spmv(self._ptr, N.dptr(x), N.dptr(y)))
        return y

    def offdiag_mv(self, x):
        x = N.f64(x, (self.ncells, 5))
        y = np.empty_like(x)
        N.check(N.load().gks_blocksys_offdiag_mv(self._ptr, N.dptr(x), N.dptr(y)))
        return y

    def diag_inverses(self):
        out = np.empty((self.ncells, 5, 5))
        N.check(N.load().gks_blocksys_diag_inverses(self._ptr, N.dptr(out)))
        return out

    def to_dense(self):
        nc = self.ncells
        dense = np.zeros((5 * nc, 5 * nc))
        for c in range(nc):
            dense[5 * c: 5 * c + 5, 5 * c: 5 * c + 5] = self.diag[c]
        for k in range(len(self.off)):
            r, c = self.off_row[k], self.off_col[k]
            dense[5 * r: 5 * r + 5, 5 * c: 5 * c + 5] = self.off[k]
        return dense


def spmv(a: BlockJacobian, x):
    return a.spmv(x)


def assemble_jacobian(mesh, q, dt_cells, gamma: float = DEFAULT_GAMMA, boundary_ghosts=None, solver=None):
    """Roe-split approximate Jacobian (jacobian.py:133-196), assembled on the GPU.

    With solver=None a throwaway device handle is built for the mesh (patch
    kinds do not enter the matrix: ghosts are frozen inputs).
    """
    from .stepping import _jacobian_handle

    if solver is not None:
        return solver.assemble_jacobian(q, dt_cells, boundary_ghosts)
    h = _jacobian_handle(mesh, gamma)
    nc = mesh.ncells
    q = N.f64(q, (nc, 5))
    dt = N.f64(np.broadcast_to(np.asarray(dt_cells, dtype=float), (nc,)))
    ghosts = None if boundary_ghosts is None else N.f64(boundary_ghosts, (-1, 5))
    lib = N.load()
    N.check(lib.gks_assemble_jacobian(h._handle, N.dptr(q), N.dptr(dt), N.dptr(ghosts)))
    # snapshot: the handle's matrix is overwritten by the next assembly
    view = BlockJacobian(_handle=lib.gks_jacobian(h._handle), _owner=h)
    ex = view._export()
    return BlockJacobian(ex["diag"], ex["off"], ex["off_col"], ex["off_row"], ex["rowptr"], device=h.device) \
        if solver is None else view


def random_block_system(rng, ncell, extra_dominance=2.0):
    """Random diagonally dominant block system on a ring+chords adjacency (jacobian.py:199-226)."""
    pairs = set()
    for c in range(ncell):
        pairs.add((c, (c + 1) % ncell))
    for _ in range(ncell):
        a, b = rng.integers(0, ncell, 2)
        if a != b:
            pairs.add((min(a, b), max(a, b)))
    entries = []
    for a, b in sorted(pairs):
        entries.append((a, b, rng.normal(size=(5, 5)) * 0.3))
        entries.append((b, a, rng.normal(size=(5, 5)) * 0.3))
    diag = np.zeros((ncell, 5, 5))
    row_abs = np.zeros(ncell)
    for r, _, blk in entries:
        row_abs[r] += np.abs(blk).sum()
    for c in range(ncell):
        diag[c] = rng.normal(size=(5, 5))
        diag[c] += np.eye(5) * (row_abs[c] + extra_dominance + np.abs(diag[c]).sum())
    off_row = np.array([e[0] for e in entries], dtype=np.int64)
    off_col = np.array([e[1] for e in entries], dtype=np.int64)
    off = np.array([e[2] for e in entries])
    order = np.lexsort((off_col, off_row))
    rowptr = np.concatenate([[0], np.cumsum(np.bincount(off_row[order], minlength=ncell))]).astype(np.int64)
    a = BlockJacobian(diag, off[order], off_col[order], off_row[order], rowptr)
    b = rng.normal(size=(ncell, 5))
    return a, b
