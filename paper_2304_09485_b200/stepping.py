"""Per-step orchestration: the drop-in Solver API (mirrors gks3d/stepping.py).

`Solver(mesh, SolverOptions)` keeps the reference's public surface
(stepping.py:87-313): local_time_step, residual, _boundary_ghosts, _solve,
advance, frechet_matvec.  Underneath, every call goes through the C ABI
(include/gks.h) into a device-resident handle: mesh arrays, reconstruction
operators, Jacobian and Krylov space live in HBM; host numpy arrays are
copied in/out per call.  advance() runs the whole backward-Euler step on
the GPU (one host synchronisation per attempt) unless a caller has replaced
`_solve` or `residual`, in which case it falls back to the reference's
step-by-step composition of the same device calls.

jacobian="frechet" (north-star option) swaps the GMRES operator
for the matrix-free Frechet JVP that re-invokes the residual pipeline; the
Roe blocks stay as the block-Jacobi preconditioner.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field as dc_field

import numpy as np

from . import _native as N
from .boundary import KIND_ID, WALL_KINDS
from .jacobian import BlockJacobian
from .kinetic import DEFAULT_GAMMA, UnphysicalStateError, primitive_to_conserved
from .krylov import SolverError, gmres_solve, lusgs_sweep
from .mesh import Mesh
from .stencils import StencilTable

SCHEMES = ("weno_gmres", "hweno_gmres", "weno_lusgs")
JACOBIANS = ("roe", "frechet")


class SteppingError(RuntimeError):
    pass


@dataclass
class SolutionField:
    q: np.ndarray
    grad: np.ndarray | None = None

    def copy(self):
        return SolutionField(self.q.copy(), None if self.grad is None else self.grad.copy())


@dataclass
class StepInfo:
    res_rho_l1: float
    res_l2: float
    dt_min: float
    solver_cycles: int = 0
    retried: bool = False
    matvecs: int = 0  # B200 build: GMRES operator applications (Frechet mode: residual evals)


@dataclass
class SolverOptions:
    scheme: str = "weno_gmres"
    model: str = "inviscid"
    mu: float = 0.0
    gamma: float = DEFAULT_GAMMA
    cfl: float = 2.0
    krylov_dim: int = 10
    restarts: int = 3
    jacobi_sweeps: int = 2
    gmres_rtol: float = 0.0
    weno_eps: float = 1e-6
    linear_weight: float = 0.025
    weights: str = "nonlinear"
    time_step: str = "local"
    patches: dict = dc_field(default_factory=dict)
    # B200 build additions (reference-equal defaults)
    jacobian: str = "roe"
    device: int = 0
    reorder: str = "none"  # device-side locality renumbering: "none" | "rcm" | "morton" (reorder.py)
    first_order: bool = False  # KFVS on piecewise-constant states (the paper's low-order start)
    ortho: str = "mgs"  # GMRES orthogonalisation: "mgs" (reference, krylov.py:89-106) | "cgs2" (fused multi-dots)
    setup: str = "device"  # stencils + operators built on the GPU ("device", gks_setup_dev.cu) or host C++ ("host")

    def __post_init__(self):
        if self.scheme not in SCHEMES:
            raise ValueError(f"unknown scheme {self.scheme!r}; choose from {SCHEMES}")
        if self.model not in ("inviscid", "viscous"):
            raise ValueError(f"unknown physics model {self.model!r}")
        if self.time_step not in ("local", "global"):
            raise ValueError("time_step must be 'local' or 'global'")
        if self.weights not in ("nonlinear", "linear"):
            raise ValueError(f"weights must be 'nonlinear' or 'linear', got {self.weights!r}")
        if self.jacobian not in JACOBIANS:
            raise ValueError(f"jacobian must be one of {JACOBIANS}")
        if self.ortho not in ("mgs", "cgs2"):
            raise ValueError("ortho must be 'mgs' or 'cgs2'")
        if self.setup not in ("device", "host"):
            raise ValueError("setup must be 'device' or 'host'")
        from .reorder import METHODS

        if self.reorder not in METHODS:
            raise ValueError(f"reorder must be one of {METHODS}, got {self.reorder!r}")


def _options_struct(opt: SolverOptions, mesh: Mesh):
    n = len(mesh.patch_names)
    arr = (N.GksPatchDesc * max(n, 1))()
    for pid, name in enumerate(mesh.patch_names):
        spec = opt.patches.get(name)
        d = arr[pid]
        if spec is None or spec.kind == "periodic":
            d.kind = -1
            continue
        d.kind = KIND_ID[spec.kind]
        if spec.reference is not None:
            for k in range(5):
                d.reference[k] = float(spec.reference[k])
        else:
            d.reference[0], d.reference[4] = 1.0, 1.0
        d.lambda_wall = float(spec.lambda_wall) if spec.lambda_wall is not None else 0.0
        for k in range(3):
            d.velocity[k] = float(spec.velocity[k])
    o = N.GksOptions()
    o.scheme = SCHEMES.index(opt.scheme)
    o.model = 0 if opt.model == "inviscid" else 1
    o.mu, o.gamma, o.cfl = float(opt.mu), float(opt.gamma), float(opt.cfl)
    o.krylov_dim, o.restarts, o.jacobi_sweeps = int(opt.krylov_dim), int(opt.restarts), int(opt.jacobi_sweeps)
    o.gmres_rtol = float(opt.gmres_rtol)
    o.weno_eps, o.linear_weight = float(opt.weno_eps), float(opt.linear_weight)
    o.linear_weights = int(opt.weights == "linear")
    o.global_time_step = int(opt.time_step == "global")
    o.jacobian_mode = JACOBIANS.index(opt.jacobian)
    o.npatch = n
    o.patches = arr
    o.first_order = int(bool(opt.first_order))
    o.ortho = ("mgs", "cgs2").index(opt.ortho)
    return o, arr


class Solver:
    def __init__(self, mesh: Mesh, options: SolverOptions):
        self.mesh = mesh
        self.opt = options
        self.compact = options.scheme.startswith("hweno")
        self.device = options.device
        fq_face = mesh.fq_face
        self.fq_interior = mesh.face_neighbor[fq_face] >= 0
        self.patch_fq = {}
        fq_patch = mesh.face_patch[fq_face]
        for pid, name in enumerate(mesh.patch_names):
            sel = np.flatnonzero(fq_patch == pid)
            if len(sel):
                self.patch_fq[name] = sel
        self.wall_fq = np.zeros(len(fq_face), dtype=bool)
        uncovered = np.flatnonzero(~self.fq_interior & (fq_patch < 0))
        if len(uncovered):
            raise SteppingError(f"{len(uncovered)} boundary quadrature points have no patch")
        for name in self.patch_fq:
            if name not in options.patches:
                raise SteppingError(f"no patch spec for boundary patch {name!r}")
            if options.patches[name].kind in WALL_KINDS:
                self.wall_fq[self.patch_fq[name]] = True
        self.bfaces = np.flatnonzero(mesh.face_neighbor < 0)
        self.bface_patch = [mesh.patch_names[p] for p in mesh.face_patch[self.bfaces]]

        # stencils + operators: built on the device by gks_create (setup
        # NULL, the default) or by the host native setup on the reference's
        # numbering; the device handle is optionally renumbered (reorder.py)
        self._opts, self._patch_arr = _options_struct(options, mesh)
        lib = N.load()
        self._perm = self._sub = None
        self._setup = None
        setup = None
        if options.setup == "host":
            self._setup = N.NativeSetup(mesh, schemes=2 if self.compact else 1)
            setup = self._setup.handle
        dev_mesh = mesh
        if options.reorder != "none":
            from .reorder import PermutedMesh, cell_order

            dev_mesh = PermutedMesh(mesh, cell_order(mesh, options.reorder))
            self._perm = dev_mesh.perm
            if setup is not None:
                sub = C.c_void_p()
                N.check(lib.gks_setup_subset(setup, N.iptr(dev_mesh.perm), mesh.ncells, N.iptr(dev_mesh.inv),
                                             mesh.ncells, C.byref(sub)))
                self._sub = setup = sub
        self._desc, self._keep = N.mesh_desc(dev_mesh)
        h = C.c_void_p()
        rc = lib.gks_create(C.byref(self._desc), setup, C.byref(self._opts), int(self.device), C.byref(h))
        if rc:
            msg = lib.gks_last_error().decode(errors="replace")
            if "patch" in msg:
                raise SteppingError(msg)
            N.check(rc)
        self._handle = h
        self._stencils = None

    def __del__(self):
        h = getattr(self, "_handle", None)
        if h is not None and h.value and N._lib is not None:
            N._lib.gks_destroy(h)
            self._handle = None
        sub = getattr(self, "_sub", None)
        if sub is not None and sub.value and N._lib is not None:
            N._lib.gks_setup_free(sub)
            self._sub = None

    # reference numbering <-> device numbering (identity unless reordered)
    def _dev(self, a):
        if a is None or self._perm is None:
            return a
        return np.ascontiguousarray(a[self._perm])

    def _host(self, a):
        if a is None or self._perm is None:
            return a
        out = np.empty_like(a)
        out[self._perm] = a
        return out

    @property
    def stencils(self):
        if self._stencils is None:
            # the operator setup does not keep the stencil tables: build them on demand
            self._stencils = StencilTable(N.NativeSetup(self.mesh, schemes=0), self.mesh)
        return self._stencils

    # -- helpers ----------------------------------------------------------------

    def _q(self, fld):
        return self._dev(N.f64(fld.q, (self.mesh.ncells, 5)))

    def _grad(self, fld):
        if fld.grad is None:
            return None
        return self._dev(N.f64(fld.grad, (self.mesh.ncells, 3, 5)))

    def _raise(self, rc, where):
        lib = N.load()
        msg = lib.gks_last_error().decode(errors="replace")
        if rc == N.GKS_ERR_UNPHYSICAL:
            if where == "dt":
                raise UnphysicalStateError(msg)
            if "patch" in msg:
                raise SteppingError(msg)
            raise SteppingError(f"unphysical reconstructed interface state: {msg}")
        if rc in (N.GKS_ERR_SINGULAR, N.GKS_ERR_NONFINITE):
            raise SolverError(msg)
        if rc == N.GKS_ERR_INVALID_UPDATE:
            bad = self._bad_cells()
            if bad is not None:
                msg = f"unphysical update persists after dt halving at cells {bad[:8].tolist()}"
            raise SteppingError(msg)
        N.check(rc)

    def _bad_cells(self):
        """Reference ids of the rejected update's bad cells, ascending (stepping.py:294-296)."""
        nc = int(N.load().gks_handle_info(self._handle, 9))
        mask = np.zeros(nc, dtype=np.int8)
        if N.load().gks_bad_mask(self._handle, mask.ctypes.data):
            return None
        ids = np.flatnonzero(mask)
        return np.sort(self._ref_ids(ids))

    def _ref_ids(self, dev_ids):
        """Device (handle) cell index -> reference cell id."""
        return dev_ids if self._perm is None else self._perm[dev_ids]

    # -- time step ----------------------------------------------------------------

    def local_time_step(self, fld: SolutionField):
        q = self._q(fld)
        dt = np.empty(self.mesh.ncells)
        rc = N.load().gks_local_dt(self._handle, N.dptr(q), N.dptr(dt))
        if rc:
            self._raise(rc, "dt")
        return self._host(dt)

    # -- residual -------------------------------------------------------------------

    def residual(self, fld: SolutionField, dt_cells, with_gradients=None):
        """Cell residual L(Q) and (compact) the Gauss-theorem gradient update."""
        if with_gradients is None:
            with_gradients = self.compact
        if self.compact and fld.grad is None:
            raise SteppingError("compact scheme needs a gradient field")
        nc = self.mesh.ncells
        q = self._q(fld)
        grad = self._grad(fld)
        dt = self._dev(N.f64(np.broadcast_to(np.asarray(dt_cells, dtype=float), (nc,))))
        res = np.empty((nc, 5))
        gout = np.empty((nc, 3, 5)) if with_gradients else None
        rc = N.load().gks_residual(self._handle, N.dptr(q), N.dptr(grad), N.dptr(dt), int(bool(with_gradients)),
                                   N.dptr(res), N.dptr(gout))
        if rc:
            self._raise(rc, "residual")
        return self._host(res), self._host(gout)

    # -- implicit step ----------------------------------------------------------------

    def _boundary_ghosts(self, fld: SolutionField):
        if not len(self.bfaces):
            return None
        out = np.empty((len(self.bfaces), 5))
        rc = N.load().gks_boundary_ghosts(self._handle, N.dptr(self._q(fld)), N.dptr(out))
        if rc:
            self._raise(rc, "dt")
        return out

    def _solve(self, a, res):
        if self.opt.scheme == "weno_lusgs":
            return lusgs_sweep(a, res), 0
        dq, info = gmres_solve(a, res, m=self.opt.krylov_dim, restarts=self.opt.restarts,
                               k_max=self.opt.jacobi_sweeps, rtol=self.opt.gmres_rtol)
        return dq, len(info.cycle_residuals)

    def assemble_jacobian(self, q, dt, ghosts=None) -> BlockJacobian:
        """Roe Jacobian on this solver's device handle (a view; next assembly overwrites it)."""
        lib = N.load()
        q = self._dev(N.f64(q, (self.mesh.ncells, 5)))
        dt = self._dev(N.f64(np.broadcast_to(np.asarray(dt, dtype=float), (self.mesh.ncells,))))
        g = None if ghosts is None else N.f64(ghosts, (-1, 5))  # boundary faces: reference order on the device too
        rc = lib.gks_assemble_jacobian(self._handle, N.dptr(q), N.dptr(dt), N.dptr(g))
        if rc:
            self._raise(rc, "jac")
        view = BlockJacobian(_handle=lib.gks_jacobian(self._handle), _owner=self)
        if self._perm is None:
            return view
        # renumbered handle: hand back the matrix in the reference's numbering
        # and CSR order (rows, then columns ascending; jacobian.py:181-196)
        ex = view._export()
        rows = self._perm[ex["off_row"]]
        cols = self._perm[ex["off_col"]]
        order = np.lexsort((cols, rows))
        nc = self.mesh.ncells
        rowptr = np.concatenate([[0], np.cumsum(np.bincount(rows, minlength=nc))]).astype(np.int64)
        return BlockJacobian(self._host(ex["diag"]), ex["off"][order], cols[order], rows[order], rowptr,
                             device=self.device)

    @staticmethod
    def _invalid_cells(q, gamma):
        rho = q[:, 0]
        e_int = q[:, 4] - 0.5 * np.sum(q[:, 1:4] ** 2, axis=1) / rho
        return (rho <= 0.0) | (e_int <= 0.0) | ~np.all(np.isfinite(q), axis=1)

    def _fast_path(self):
        d = self.__dict__
        return "_solve" not in d and "residual" not in d and type(self)._solve is Solver._solve \
            and type(self).residual is Solver.residual and self.opt.scheme != "weno_lusgs"

    def advance(self, fld: SolutionField):
        """One backward-Euler step; rejected updates retry once at halved dt."""
        if self._fast_path():
            if self.compact and fld.grad is None:
                raise SteppingError("compact scheme needs a gradient field")
            q = np.array(self._q(fld), copy=True)
            grad = np.array(self._grad(fld), copy=True) if self.compact else None
            info = N.GksStepInfo()
            rc = N.load().gks_advance(self._handle, N.dptr(q), N.dptr(grad), C.byref(info))
            if rc:
                self._raise(rc, "advance")
            return SolutionField(self._host(q), self._host(grad) if self.compact else None), _info(info)
        # composed path (reference structure, stepping.py:270-296) with device calls
        dt = self.local_time_step(fld)
        retried = False
        for attempt in range(2):
            res, grad_new = self.residual(fld, dt)
            ghosts = self._boundary_ghosts(fld)
            a = self.assemble_jacobian(fld.q, dt, ghosts)
            dq, cycles = self._solve(a, res)
            q_new = fld.q + dq
            bad = self._invalid_cells(q_new, self.opt.gamma)
            if not bad.any():
                info = StepInfo(float(np.sum(np.abs(res[:, 0])) / self.mesh.ncells),
                                float(np.sqrt(np.mean(res ** 2))), float(dt.min()), cycles, retried)
                return SolutionField(q_new, grad_new if self.compact else None), info
            if attempt == 0:
                dt = np.where(bad, 0.5 * dt, dt)
                retried = True
        raise SteppingError(
            f"unphysical update persists after dt halving at cells {np.flatnonzero(bad)[:8].tolist()}")

    def advance_inplace(self, fld: SolutionField) -> StepInfo:
        """advance() writing the new state into fld.q / fld.grad (no host copies).

        Lets callers keep the field in pinned host buffers (gks_host_pin) so the
        per-step H2D/D2H copies run at full PCIe bandwidth.
        """
        nc = self.mesh.ncells
        if fld.q.dtype != np.float64 or not fld.q.flags.c_contiguous or fld.q.shape != (nc, 5):
            raise ValueError("advance_inplace needs a C-contiguous float64 (nc, 5) field")
        if self.compact and (fld.grad is None or not fld.grad.flags.c_contiguous):
            raise SteppingError("compact scheme needs a C-contiguous gradient field")
        info = N.GksStepInfo()
        if self._perm is not None:
            # renumbered handle: permuted copies in and out
            q, g = self._q(fld), self._grad(fld) if self.compact else None
            rc = N.load().gks_advance(self._handle, N.dptr(q), N.dptr(g), C.byref(info))
            if rc:
                self._raise(rc, "advance")
            fld.q[...] = self._host(q)
            if self.compact:
                fld.grad[...] = self._host(g)
            return _info(info)
        rc = N.load().gks_advance(self._handle, N.dptr(fld.q), N.dptr(fld.grad) if self.compact else None,
                                  C.byref(info))
        if rc:
            self._raise(rc, "advance")
        return _info(info)

    def frechet_matvec(self, fld: SolutionField, v, dt_cells, sigma=None):
        """Directional residual derivative (L(Q + s v) - L(Q)) / s, gradients frozen."""
        v = np.asarray(v, dtype=float).reshape(np.shape(fld.q))
        if not isinstance(self, Solver) or "residual" in self.__dict__ or type(self).residual is not Solver.residual:
            # duck-typed / overridden residual: compose through self.residual
            if sigma is None:
                vn = np.linalg.norm(v)
                if vn == 0.0:
                    return np.zeros_like(v)
                sigma = np.sqrt(np.finfo(float).eps) * (1.0 + np.linalg.norm(fld.q)) / vn
            base, _ = self.residual(fld, dt_cells, with_gradients=False)
            res, _ = self.residual(SolutionField(fld.q + sigma * v, fld.grad), dt_cells, with_gradients=False)
            return (res - base) / sigma
        nc = self.mesh.ncells
        if sigma is None and np.linalg.norm(v) == 0.0:
            return np.zeros_like(v)
        q = self._q(fld)
        grad = self._grad(fld)
        dt = self._dev(N.f64(np.broadcast_to(np.asarray(dt_cells, dtype=float), (nc,))))
        vv = self._dev(N.f64(v, (nc, 5)))
        out = np.empty((nc, 5))
        rc = N.load().gks_frechet_matvec(self._handle, N.dptr(q), N.dptr(grad), N.dptr(dt), N.dptr(vv),
                                         -1.0 if sigma is None else float(sigma), N.dptr(out))
        if rc:
            self._raise(rc, "residual")
        return self._host(out)

    # -- device-resident loop (benchmark / driver) ------------------------------------

    def upload(self, fld: SolutionField):
        N.check(N.load().gks_state_upload(self._handle, N.dptr(self._q(fld)), N.dptr(self._grad(fld))))

    def download(self) -> SolutionField:
        nc = self.mesh.ncells
        q = np.empty((nc, 5))
        g = np.empty((nc, 3, 5)) if self.compact else None
        N.check(N.load().gks_state_download(self._handle, N.dptr(q), N.dptr(g)))
        return SolutionField(self._host(q), self._host(g))

    def set_cfl(self, cfl: float):
        """Change the CFL number of this solver (options.cfl) for the next steps."""
        N.check(N.load().gks_set_cfl(self._handle, float(cfl)))
        self.opt.cfl = float(cfl)

    def advance_resident(self) -> StepInfo:
        info = N.GksStepInfo()
        rc = N.load().gks_advance_resident(self._handle, C.byref(info))
        if rc:
            self._raise(rc, "advance")
        return _info(info)


def _info(ci):
    return StepInfo(float(ci.res_rho_l1), float(ci.res_l2), float(ci.dt_min), int(ci.solver_cycles),
                    bool(ci.retried), int(ci.matvecs))


_JAC_HANDLES = {}


def _jacobian_handle(mesh, gamma):
    """A device handle for free-function assemble_jacobian calls (cached per mesh)."""
    key = (id(mesh), gamma)
    h = _JAC_HANDLES.get(key)
    if h is None or h.mesh is not mesh:
        from .boundary import PatchSpec

        patches = {n: PatchSpec(n, "supersonic_outlet") for n in mesh.patch_names}
        h = Solver(mesh, SolverOptions(gamma=gamma, patches=patches))
        _JAC_HANDLES.clear()
        _JAC_HANDLES[key] = h
    return h


def initial_field(mesh: Mesh, reference, gamma: float = DEFAULT_GAMMA, compact=False):
    """Uniform reference-state field; reference = (rho, U, V, W, p)  (stepping.py:316-324)."""
    rho, u, v, w, p = np.asarray(reference, dtype=float)
    prim = np.array([rho, u, v, w, rho / (2.0 * p)])
    q = np.tile(primitive_to_conserved(prim, gamma), (mesh.ncells, 1))
    grad = np.zeros((mesh.ncells, 3, 5)) if compact else None
    return SolutionField(q, grad)
