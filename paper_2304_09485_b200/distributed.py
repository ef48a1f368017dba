"""Multi-GPU solver: one process per GPU, cell-partitioned mesh.

Each rank owns a LocalDomain (partition.py) and a device handle created with
gks_create_local: owned cells + ghost layers, the global reconstruction
operators restricted to its cells (gks_setup_subset), halo maps, and an NCCL
communicator (gks_comm_init; the unique id travels over torch.distributed).
Inside gks_advance_resident the step then performs, on the handle's stream
and without host round trips:
  * grouped ncclSend/ncclRecv halo exchange of Q (+ gradients) at step start,
    of dt after the local time step, of the perturbed state in Frechet JVPs,
    and of every Krylov vector before each off-diagonal block product;
  * ncclAllReduce for every GMRES dot product / norm, the step norms, the
    bad-cell count, the global time step and the error word.
Control flow stays on the device: the allreduced Hessenberg scalars are
bitwise identical on all ranks, so every rank takes the same branch.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N
from .partition import LocalMesh, build_domains, partition_cells
from .stepping import Solver, SolverOptions, SolutionField, _info, _options_struct


def _halo_desc(send: dict, recv: dict, keep):
    peers = sorted(set(send) | set(recv))
    so = np.zeros(len(peers) + 1, dtype=np.int64)
    ro = np.zeros(len(peers) + 1, dtype=np.int64)
    sids, rids = [], []
    for k, p in enumerate(peers):
        s = np.asarray(send.get(p, np.zeros(0, np.int64)), dtype=np.int64)
        r = np.asarray(recv.get(p, np.zeros(0, np.int64)), dtype=np.int64)
        so[k + 1] = so[k] + len(s)
        ro[k + 1] = ro[k] + len(r)
        sids.append(s)
        rids.append(r)
    arrs = [np.asarray(peers, dtype=np.int32), so, np.concatenate(sids) if sids else np.zeros(0, np.int64), ro,
            np.concatenate(rids) if rids else np.zeros(0, np.int64)]
    arrs = [np.ascontiguousarray(a) for a in arrs]
    keep.extend(arrs)
    d = N.GksHaloDesc()
    d.npeers = len(peers)
    d.peers, d.send_offsets, d.send_ids, d.recv_offsets, d.recv_ids = (a.ctypes.data for a in arrs)
    return d


class DistributedSolver:
    """Rank-local solver over a partitioned global mesh."""

    def __init__(self, mesh, options: SolverOptions, rank=0, nranks=1, comm_id=None, part=None,
                 global_setup=None):
        self.mesh = mesh
        self.opt = options
        self.rank, self.nranks = rank, nranks
        self.compact = options.scheme.startswith("hweno")
        layers = 2 if self.compact else 3
        self.part = partition_cells(mesh, nranks) if part is None else np.asarray(part)
        doms, g2l = build_domains(mesh, self.part, layers)
        self.dom = doms[rank]
        self.g2l = g2l[rank]
        self.local_mesh = LocalMesh(mesh, self.dom, self.g2l)
        gs = global_setup or N.NativeSetup(mesh, schemes=2 if self.compact else 1)
        lib = N.load()
        cells = np.ascontiguousarray(self.dom.cells, dtype=np.int64)
        g2l_arr = np.ascontiguousarray(self.g2l, dtype=np.int64)
        sub = C.c_void_p()
        N.check(lib.gks_setup_subset(gs.handle, N.iptr(cells), len(cells), N.iptr(g2l_arr), mesh.ncells,
                                     C.byref(sub)))
        self._sub = sub
        self._keep = []
        dd = N.GksDomainDesc()
        dd.n_owned = self.dom.n_owned
        dd.n_recon = self.dom.n_recon
        dd.nc_global = mesh.ncells
        dd.q = _halo_desc(self.dom.q_send, self.dom.q_recv, self._keep)
        dd.x = _halo_desc(self.dom.x_send, self.dom.x_recv, self._keep)
        self._dd = dd
        self._desc, self._dkeep = N.mesh_desc(self.local_mesh)
        self._opts, self._parr = _options_struct(options, mesh)
        if nranks > 1 and comm_id is None:
            raise ValueError("multi-rank solver needs the NCCL unique id (DistributedSolver.unique_id())")
        h = C.c_void_p()
        N.check(lib.gks_create_local(C.byref(self._desc), sub, C.byref(self._opts), C.byref(dd), int(options.device),
                                     C.byref(h)))
        self._handle = h
        if comm_id is not None:
            buf = (C.c_char * 128).from_buffer_copy(bytes(comm_id))
            N.check(lib.gks_comm_init(h, buf, nranks, rank))

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_char * 128)()
        N.check(N.load().gks_comm_unique_id(buf, 128))
        return bytes(buf)

    def __del__(self):
        lib = N._lib
        if lib is None:
            return
        if getattr(self, "_handle", None) is not None and self._handle.value:
            lib.gks_destroy(self._handle)
            self._handle = None
        if getattr(self, "_sub", None) is not None and self._sub.value:
            lib.gks_setup_free(self._sub)
            self._sub = None

    # state transfer (global arrays in, owned rows out)
    def upload(self, fld: SolutionField):
        q = np.ascontiguousarray(fld.q[self.dom.cells], dtype=np.float64)
        g = None if fld.grad is None else np.ascontiguousarray(fld.grad[self.dom.cells], dtype=np.float64)
        N.check(N.load().gks_state_upload(self._handle, N.dptr(q), N.dptr(g)))

    def download_owned(self):
        nl = self.dom.n_local
        q = np.empty((nl, 5))
        g = np.empty((nl, 3, 5)) if self.compact else None
        N.check(N.load().gks_state_download(self._handle, N.dptr(q), N.dptr(g)))
        n = self.dom.n_owned
        return self.dom.cells[:n], q[:n], (None if g is None else g[:n])

    def advance_resident(self):
        info = N.GksStepInfo()
        rc = N.load().gks_advance_resident(self._handle, C.byref(info))
        if rc:
            Solver._raise(self, rc, "advance")
        return _info(info)

    def residual_local(self, q_local, grad_local, dt_local, with_gradients=False):
        """Residual of owned cells from a full local state (ghosts included)."""
        n = self.dom.n_local
        res = np.empty((n, 5))
        gout = np.empty((n, 3, 5)) if with_gradients else None
        rc = N.load().gks_residual(self._handle, N.dptr(N.f64(q_local)), N.dptr(None if grad_local is None else
                                                                                 N.f64(grad_local)),
                                   N.dptr(N.f64(dt_local)), int(with_gradients), N.dptr(res), N.dptr(gout))
        if rc:
            Solver._raise(self, rc, "residual")
        k = self.dom.n_owned
        return res[:k], (None if gout is None else gout[:k])
