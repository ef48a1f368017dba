"""Multi-GPU solver: cell-partitioned mesh, one rank-local handle per rank
(SURVEY 8e).

Each rank owns a contiguous range of the mesh's canonical order
(partition.py) and a device handle created with gks_create_local: owned
cells + ghost layers, its own native setup (stencils + operators built from
a SetupMesh of its local cells only -- no global operator tables), halo maps
and a communicator.  Inside gks_advance_resident the step then performs, on
the handle's stream and without host round trips:
  * halo exchange of Q (+ gradients) at step start, of dt after the local
    time step, of the perturbed state in Frechet JVPs, and of every Krylov
    vector before each off-diagonal block product;
  * for every GMRES dot product / norm and the step norms, an exchange of
    the per-rank group partials and the same final fold on every rank
    (csrc/gks_reduce.cuh): reductions are partition-invariant, so an N-rank
    run is bitwise the 1-rank canonical run, whatever the transport;
  * max / min allreduces of the error words, the bad-cell count and, for
    time_step="global", the minimum dt.
Control flow stays on the device: the reduced Hessenberg scalars are
bitwise identical on all ranks, so every rank takes the same branch.

Transports (csrc/gks_comm.cu): NCCL (one process per GPU; the unique id
travels over torch.distributed) or the in-process loopback group
(LoopbackGroup: several ranks driven by host threads of one process, e.g. on
one GPU, through the same pack/exchange/unpack and reduction code).
"""

from __future__ import annotations

import ctypes as C
import threading

import numpy as np

from . import _native as N
from .partition import Decomposition, LocalMesh, SetupMesh, build_domain
from .stepping import Solver, SolverOptions, SolutionField, _info, _options_struct


def _bind_torch_nccl():
    """libgks dlopens libnccl.so.2 with RTLD_NOLOAD first: importing torch
    before the first NCCL call makes that the NCCL build torch ships (and
    keeps torch importable afterwards -- the reverse order leaves the older
    system NCCL bound in front of torch's)."""
    try:
        import torch  # noqa: F401
    except Exception:
        pass


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


class LoopbackGroup:
    """In-process transport for nranks rank-local handles (gks_loopback_*).

    Register each DistributedSolver with loopback=(group, rank); then
    advance_all() steps every rank concurrently, one host thread per rank
    (ctypes releases the GIL), which the collectives need: each one is a
    barrier between the rank threads.
    """

    def __init__(self, nranks: int):
        h = C.c_void_p()
        N.check(N.load().gks_loopback_create(int(nranks), C.byref(h)))
        self.handle = h
        self.nranks = nranks
        self.members = []

    def advance_all(self, solvers, step=None):
        """One step on every rank; step(k, solver) -> StepInfo replaces the
        default advance_resident (e.g. the host-array advance_inplace)."""
        out = [None] * len(solvers)
        err = [None] * len(solvers)

        def run(k, s):
            try:
                out[k] = step(k, s) if step else s.advance_resident()
            except BaseException as e:  # re-raised on the caller's thread
                err[k] = e

        ts = [threading.Thread(target=run, args=(k, s)) for k, s in enumerate(solvers)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        for e in err:
            if e is not None:
                raise e
        return out

    def close(self):
        if self.handle is not None and self.handle.value and N._lib is not None:
            for s in self.members:
                s.close()
            N._lib.gks_loopback_destroy(self.handle)
        self.handle = None

    def __del__(self):
        self.close()


class DistributedSolver:
    """Rank-local solver over a partitioned global mesh.

    comm_id: NCCL unique id (one process per GPU); loopback: (LoopbackGroup,
    rank is taken from `rank`); neither: no communicator (nranks == 1 gives
    the canonical single-rank run; with nranks > 1 the ghosts come from
    uploaded global state, used by the rank-local parity tests).
    """

    def __init__(self, mesh, options: SolverOptions, rank=0, nranks=1, comm_id=None, dec=None, loopback=None):
        self.mesh = mesh
        self.opt = options
        self.rank, self.nranks = rank, nranks
        self.compact = options.scheme.startswith("hweno")
        layers = 2 if self.compact else 3
        self.dec = Decomposition.build(mesh, nranks) if dec is None else dec
        if self.dec.nranks != nranks:
            raise ValueError(f"decomposition has {self.dec.nranks} ranks, solver asked for {nranks}")
        self.dom = build_domain(mesh, self.dec, rank, layers)
        self.local_mesh = LocalMesh(mesh, self.dom)
        lib = N.load()
        # per-rank setup on the local cells only (SetupMesh: local cells in
        # reference order with all their faces): built on the device and
        # placed in the rank-local order by gks_create_local (setup="device"),
        # or by the host native setup, restricted and reordered here
        self._setup_mesh = SetupMesh(mesh, self.dom)
        self._setup = None
        sub = C.c_void_p()
        if options.setup == "host":
            self._setup = N.NativeSetup(self._setup_mesh, schemes=2 if self.compact else 1)
            N.check(lib.gks_setup_subset(self._setup.handle, N.iptr(self._setup_mesh.local_to_sub),
                                         self.dom.n_local, N.iptr(self._setup_mesh.sub_to_local),
                                         self._setup_mesh.ncells, C.byref(sub)))
        self._sub = sub
        self._keep = []
        dd = N.GksDomainDesc()
        dd.n_owned = self.dom.n_owned
        dd.n_recon = self.dom.n_recon
        dd.nc_global = mesh.ncells
        dd.owned_offset = self.dom.owned_offset
        dd.q = _halo_desc(self.dom.q_send, self.dom.q_recv, self._keep)
        dd.x = _halo_desc(self.dom.x_send, self.dom.x_recv, self._keep)
        if options.setup != "host":
            sdesc, skeep = N.mesh_desc(self._setup_mesh)
            l2s = np.ascontiguousarray(self._setup_mesh.local_to_sub, dtype=np.int64)
            s2l = np.ascontiguousarray(self._setup_mesh.sub_to_local, dtype=np.int64)
            self._keep += [sdesc, skeep, l2s, s2l]
            dd.setup_mesh = C.cast(C.pointer(sdesc), C.c_void_p)
            dd.local_to_setup = l2s.ctypes.data
            dd.setup_to_local = s2l.ctypes.data
        self._dd = dd
        self._desc, self._dkeep = N.mesh_desc(self.local_mesh)
        self._opts, self._parr = _options_struct(options, mesh)
        h = C.c_void_p()
        N.check(lib.gks_create_local(C.byref(self._desc), sub, C.byref(self._opts), C.byref(dd), int(options.device),
                                     C.byref(h)))
        self._handle = h
        # the setup tables are no longer needed once the operators are on the device
        if sub.value:
            lib.gks_setup_free(sub)
        self._sub = None
        self._setup = None
        if comm_id is not None:
            _bind_torch_nccl()
            buf = (C.c_char * 128).from_buffer_copy(bytes(comm_id))
            N.check(lib.gks_comm_init(h, buf, nranks, rank))
        elif loopback is not None:
            if loopback.nranks != nranks:
                raise ValueError("loopback group size differs from nranks")
            N.check(lib.gks_comm_init_loopback(h, loopback.handle, rank))
            loopback.members.append(self)

    @staticmethod
    def unique_id() -> bytes:
        _bind_torch_nccl()
        buf = (C.c_char * 128)()
        N.check(N.load().gks_comm_unique_id(buf, 128))
        return bytes(buf)

    def close(self):
        lib = N._lib
        if lib is None:
            return
        if getattr(self, "_handle", None) is not None and self._handle.value:
            lib.gks_destroy(self._handle)
            self._handle = None
        if getattr(self, "_sub", None) is not None and self._sub.value:
            lib.gks_setup_free(self._sub)
            self._sub = None

    def __del__(self):
        self.close()

    # state transfer (global arrays in, owned rows out)
    def upload(self, fld: SolutionField):
        q = np.ascontiguousarray(fld.q[self.dom.cells], dtype=np.float64)
        g = None if fld.grad is None else np.ascontiguousarray(fld.grad[self.dom.cells], dtype=np.float64)
        N.check(N.load().gks_state_upload(self._handle, N.dptr(q), N.dptr(g)))

    def download_owned(self):
        """(reference ids, q, grad) of the owned cells."""
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

    def advance_inplace(self, q_local, grad_local=None):
        """One step from the rank's HOST field (all local cells, local order:
        q_local = q[dom.cells]), written back in place -- the gks_advance path
        behind Solver.advance_inplace, halos exchanged on the device."""
        if q_local.dtype != np.float64 or not q_local.flags.c_contiguous or q_local.shape != (self.dom.n_local, 5):
            raise ValueError("advance_inplace needs a C-contiguous float64 (n_local, 5) field")
        if self.compact and (grad_local is None or not grad_local.flags.c_contiguous):
            raise ValueError("compact scheme needs a C-contiguous gradient field")
        info = N.GksStepInfo()
        rc = N.load().gks_advance(self._handle, N.dptr(q_local), N.dptr(grad_local) if self.compact else None,
                                  C.byref(info))
        if rc:
            Solver._raise(self, rc, "advance")
        return _info(info)

    # Solver._raise helpers: name bad cells by their reference ids
    def _bad_cells(self):
        mask = np.zeros(self.dom.n_owned, dtype=np.int8)
        if N.load().gks_bad_mask(self._handle, mask.ctypes.data):
            return None
        return np.sort(self.dom.cells[np.flatnonzero(mask)])

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


def gather_owned(parts, ncells, compact=False):
    """Assemble global (q, grad) from every rank's download_owned()."""
    q = np.full((ncells, 5), np.nan)
    g = np.full((ncells, 3, 5), np.nan) if compact else None
    for cells, qo, go in parts:
        q[cells] = qo
        if compact:
            g[cells] = go
    return q, g
