"""ctypes binding of libgks.so (the C ABI declared in include/gks.h).

There is no fallback: if the shared library is missing or no CUDA device is
visible, calls raise.  Build with `python -m paper_2304_09485_b200.build` or
`__graft_entry__.build()`.
"""

from __future__ import annotations

import ctypes as C
import threading
from pathlib import Path

import numpy as np

import os

# GKS_LIB overrides the library path (experiment variants built with build.py --out=)
LIB_PATH = Path(os.environ.get("GKS_LIB", Path(__file__).resolve().parent / "libgks.so"))

GKS_OK = 0
GKS_ERR_BAD_ARG = 1
GKS_ERR_CUDA = 2
GKS_ERR_UNPHYSICAL = 3
GKS_ERR_SINGULAR = 4
GKS_ERR_NONFINITE = 5
GKS_ERR_MESH = 6
GKS_ERR_NCCL = 7
GKS_ERR_NO_DEVICE = 8
GKS_ERR_INVALID_UPDATE = 9

_lock = threading.Lock()
_lib = None

c_double_p = C.POINTER(C.c_double)
c_int64_p = C.POINTER(C.c_int64)
c_int32_p = C.POINTER(C.c_int32)
c_void_p = C.c_void_p


class GksMeshDesc(C.Structure):
    _fields_ = [("ncells", C.c_int64), ("nfaces", C.c_int64), ("nfq", C.c_int64), ("ncq", C.c_int64),
                ("cell_kind", C.c_void_p), ("cell_volume", C.c_void_p), ("cell_h", C.c_void_p),
                ("cell_centroid", C.c_void_p), ("cell_cq_start", C.c_void_p), ("cq_point", C.c_void_p),
                ("cq_weight", C.c_void_p), ("cell_face_start", C.c_void_p), ("cell_face_list", C.c_void_p),
                ("face_owner", C.c_void_p), ("face_neighbor", C.c_void_p), ("face_patch", C.c_void_p),
                ("face_area", C.c_void_p), ("face_normal", C.c_void_p), ("face_frame", C.c_void_p),
                ("face_shift", C.c_void_p), ("face_fq_start", C.c_void_p), ("fq_face", C.c_void_p),
                ("fq_point", C.c_void_p), ("fq_weight", C.c_void_p), ("face_rank", C.c_void_p),
                ("fq_rank", C.c_void_p), ("cell_rank", C.c_void_p)]


_DESC_FIELDS = {
    "cell_kind": np.int8, "cell_volume": np.float64, "cell_h": np.float64, "cell_centroid": np.float64,
    "cell_cq_start": np.int64, "cq_point": np.float64, "cq_weight": np.float64,
    "cell_face_start": np.int64, "cell_face_list": np.int64, "face_owner": np.int64,
    "face_neighbor": np.int64, "face_patch": np.int64, "face_area": np.float64, "face_normal": np.float64,
    "face_frame": np.float64, "face_shift": np.float64, "face_fq_start": np.int64, "fq_face": np.int64,
    "fq_point": np.float64, "fq_weight": np.float64,
}


def mesh_desc(mesh):
    """GksMeshDesc view of a host Mesh; returns (desc, keepalive)."""
    keep = {}
    desc = GksMeshDesc()
    desc.ncells = mesh.ncells
    desc.nfaces = mesh.nfaces
    desc.nfq = len(mesh.fq_face)
    desc.ncq = len(mesh.cq_weight)
    for name, dt in _DESC_FIELDS.items():
        arr = np.ascontiguousarray(getattr(mesh, name), dtype=dt)
        keep[name] = arr
        setattr(desc, name, arr.ctypes.data)
    for name in ("face_rank", "fq_rank", "cell_rank"):  # renumbered / rank-local meshes only
        val = getattr(mesh, name, None)
        if val is not None:
            arr = np.ascontiguousarray(val, dtype=np.int64)
            keep[name] = arr
            setattr(desc, name, arr.ctypes.data)
    return desc, keep


_DTYPES = {0: np.float64, 1: np.int64, 2: np.int8}


class NativeSetup:
    """Owner of a GksSetup* (stencils + reconstruction operators)."""

    def __init__(self, mesh, schemes=3, nthreads=0):
        lib = load()
        self._desc, self._keep = mesh_desc(mesh)
        h = C.c_void_p()
        check(lib.gks_setup_build(C.byref(self._desc), int(schemes), int(nthreads), C.byref(h)))
        self.handle = h
        self.schemes = schemes
        self._cache = {}

    def array(self, name):
        if name in self._cache:
            return self._cache[name]
        lib = load()
        dt, nd = C.c_int(), C.c_int()
        shape = (C.c_int64 * 4)()
        check(lib.gks_setup_query(self.handle, name.encode(), C.byref(dt), C.byref(nd), shape))
        shp = tuple(int(shape[i]) for i in range(nd.value))
        out = np.empty(shp, dtype=_DTYPES[dt.value])
        check(lib.gks_setup_copy(self.handle, name.encode(), out.ctypes.data_as(C.c_void_p), out.nbytes))
        out.setflags(write=False)
        self._cache[name] = out
        return out

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value and _lib is not None:
            _lib.gks_setup_free(h)
            self.handle = None


class GksPatchDesc(C.Structure):
    _fields_ = [("kind", C.c_int), ("reference", C.c_double * 5), ("lambda_wall", C.c_double),
                ("velocity", C.c_double * 3)]


class GksOptions(C.Structure):
    _fields_ = [("scheme", C.c_int), ("model", C.c_int), ("mu", C.c_double), ("gamma", C.c_double),
                ("cfl", C.c_double), ("krylov_dim", C.c_int), ("restarts", C.c_int), ("jacobi_sweeps", C.c_int),
                ("gmres_rtol", C.c_double), ("weno_eps", C.c_double), ("linear_weight", C.c_double),
                ("linear_weights", C.c_int), ("global_time_step", C.c_int), ("jacobian_mode", C.c_int),
                ("npatch", C.c_int), ("patches", C.POINTER(GksPatchDesc)), ("first_order", C.c_int),
                ("ortho", C.c_int)]


class GksStepInfo(C.Structure):
    _fields_ = [("res_rho_l1", C.c_double), ("res_l2", C.c_double), ("dt_min", C.c_double),
                ("solver_cycles", C.c_int), ("retried", C.c_int), ("matvecs", C.c_int), ("nbad", C.c_int),
                ("first_bad", C.c_int64 * 8)]


class GksHaloDesc(C.Structure):
    _fields_ = [("npeers", C.c_int), ("peers", C.c_void_p), ("send_offsets", C.c_void_p),
                ("send_ids", C.c_void_p), ("recv_offsets", C.c_void_p), ("recv_ids", C.c_void_p)]


class GksDomainDesc(C.Structure):
    _fields_ = [("n_owned", C.c_int64), ("n_recon", C.c_int64), ("nc_global", C.c_int64),
                ("q", GksHaloDesc), ("x", GksHaloDesc), ("owned_offset", C.c_int64),
                ("setup_mesh", C.c_void_p), ("local_to_setup", C.c_void_p), ("setup_to_local", C.c_void_p)]


class GksError(RuntimeError):
    def __init__(self, code, message, index=-1):
        super().__init__(message)
        self.code = code
        self.index = index


# (name, restype, argtypes) of every exported symbol; kept in sync with
# include/gks.h (tests/test_native_abi.py checks both directions).
SIGNATURES = [
    ("gks_abi_version", C.c_int, []),
    ("gks_last_error", C.c_char_p, []),
    ("gks_last_error_index", C.c_int64, []),
    ("gks_kernel_launches", C.c_int64, []),
    ("gks_flux_batch", C.c_int, [C.c_int64, c_double_p, c_double_p, c_double_p, c_double_p,
                                 c_double_p, c_double_p, c_double_p, C.c_double, c_double_p,
                                 c_double_p]),
    ("gks_instant_flux_batch", C.c_int, [C.c_int64] + [C.c_void_p] * 6 + [C.c_double, C.c_void_p]),
    ("gks_flux_bench", C.c_int, [C.c_int64, C.c_int, C.c_double, c_double_p]),
    ("gks_interface_data", C.c_int, [C.c_int64, c_double_p, c_double_p, c_double_p, c_double_p, C.c_double,
                                     c_double_p, c_double_p, c_double_p, c_double_p, c_double_p, c_double_p,
                                     c_double_p]),
    ("gks_moment_table", C.c_int, [C.c_int64, c_double_p, C.c_double, C.c_int, c_double_p, c_double_p,
                                   c_double_p, c_double_p, c_double_p, c_double_p]),
    ("gks_setup_build", C.c_int, [C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_void_p)]),
    ("gks_setup_free", None, [C.c_void_p]),
    ("gks_setup_query", C.c_int, [C.c_void_p, C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                  C.POINTER(C.c_int64)]),
    ("gks_setup_copy", C.c_int, [C.c_void_p, C.c_char_p, C.c_void_p, C.c_int64]),
    ("gks_create", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.POINTER(C.c_void_p)]),
    ("gks_create_local", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int,
                                   C.POINTER(C.c_void_p)]),
    ("gks_setup_subset", C.c_int, [C.c_void_p, c_int64_p, C.c_int64, c_int64_p, C.c_int64,
                                   C.POINTER(C.c_void_p)]),
    ("gks_comm_unique_id", C.c_int, [C.c_void_p, C.c_int64]),
    ("gks_comm_init", C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_int]),
    ("gks_loopback_create", C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
    ("gks_comm_init_loopback", C.c_int, [C.c_void_p, C.c_void_p, C.c_int]),
    ("gks_loopback_destroy", None, [C.c_void_p]),
    ("gks_reduction_granularity", C.c_int64, [C.c_int64]),
    ("gks_destroy", None, [C.c_void_p]),
    ("gks_local_dt", C.c_int, [C.c_void_p, c_double_p, c_double_p]),
    ("gks_residual", C.c_int, [C.c_void_p, c_double_p, c_double_p, c_double_p, C.c_int, c_double_p,
                               c_double_p]),
    ("gks_boundary_ghosts", C.c_int, [C.c_void_p, c_double_p, c_double_p]),
    ("gks_update_gradients", C.c_int, [C.c_void_p, c_double_p, c_double_p]),
    ("gks_ghost_batch", C.c_int, [C.c_int64, C.c_void_p, c_double_p, c_double_p, c_double_p, C.c_double,
                                  c_double_p, c_double_p]),
    ("gks_slopes", C.c_int, [C.c_int64, c_double_p, c_double_p, C.c_int, C.c_double, c_double_p]),
    ("gks_num_boundary_faces", C.c_int64, [C.c_void_p]),
    ("gks_handle_array", C.c_int, [C.c_void_p, C.c_char_p, C.c_void_p, C.POINTER(C.c_int64)]),
    ("gks_recon_coeffs", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p]),
    ("gks_recon_candidates", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("gks_face_values", C.c_int, [C.c_void_p] + [C.c_void_p] * 6),
    ("gks_combine_candidates", C.c_int, [C.c_int64, C.c_int, C.c_int] + [C.c_void_p] * 4 +
     [C.c_double, C.c_double] + [C.c_void_p] * 3),
    ("gks_assemble_jacobian", C.c_int, [C.c_void_p, c_double_p, c_double_p, c_double_p]),
    ("gks_jacobian", C.c_void_p, [C.c_void_p]),
    ("gks_blocksys_create", C.c_int, [C.c_int64, C.c_int64, c_double_p, c_double_p, c_int64_p, c_int64_p,
                                      C.c_int, C.POINTER(C.c_void_p)]),
    ("gks_blocksys_destroy", None, [C.c_void_p]),
    ("gks_blocksys_ncells", C.c_int64, [C.c_void_p]),
    ("gks_blocksys_nnz", C.c_int64, [C.c_void_p]),
    ("gks_blocksys_export", C.c_int, [C.c_void_p, c_double_p, c_double_p, c_int64_p, c_int64_p, c_int64_p]),
    ("gks_blocksys_spmv", C.c_int, [C.c_void_p, c_double_p, c_double_p]),
    ("gks_blocksys_offdiag_mv", C.c_int, [C.c_void_p, c_double_p, c_double_p]),
    ("gks_blocksys_dot", C.c_int, [C.c_void_p, c_double_p, c_double_p, c_double_p]),
    ("gks_blocksys_diag_inverses", C.c_int, [C.c_void_p, c_double_p]),
    ("gks_blocksys_jacobi", C.c_int, [C.c_void_p, c_double_p, C.c_int, c_double_p]),
    ("gks_gmres", C.c_int, [C.c_void_p, c_double_p, c_double_p, C.c_int, C.c_int, C.c_int, C.c_double,
                            C.c_double, C.c_int, C.c_void_p]),
    ("gks_advance", C.c_int, [C.c_void_p, c_double_p, c_double_p, C.c_void_p]),
    ("gks_state_upload", C.c_int, [C.c_void_p, c_double_p, c_double_p]),
    ("gks_state_download", C.c_int, [C.c_void_p, c_double_p, c_double_p]),
    ("gks_advance_resident", C.c_int, [C.c_void_p, C.c_void_p]),
    ("gks_set_graph", C.c_int, [C.c_void_p, C.c_int]),
    ("gks_set_cfl", C.c_int, [C.c_void_p, C.c_double]),
    ("gks_set_ortho", C.c_int, [C.c_void_p, C.c_int]),
    ("gks_bad_mask", C.c_int, [C.c_void_p, C.c_void_p]),
    ("gks_ugks_read", C.c_int, [C.c_char_p, C.c_void_p]),
    ("gks_ugks_sizes", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("gks_ugks_patch", C.c_int, [C.c_void_p, C.c_int64, C.c_char_p, C.c_int64, C.c_void_p]),
    ("gks_ugks_copy", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("gks_ugks_free", None, [C.c_void_p]),
    ("gks_event_record", C.c_int, [C.c_void_p, C.c_int]),
    ("gks_event_elapsed", C.c_int, [C.c_void_p, C.c_int, C.c_int, c_double_p]),
    ("gks_handle_info", C.c_int64, [C.c_void_p, C.c_int]),
    ("gks_fp64_peak", C.c_int, [c_double_p]),
    ("gks_host_pin", C.c_int, [C.c_void_p, C.c_int64]),
    ("gks_host_unpin", C.c_int, [C.c_void_p]),
    ("gks_profile_enable", C.c_int, [C.c_int]),
    ("gks_profile_reset", C.c_int, []),
    ("gks_profile_read", C.c_int, [c_double_p, c_int64_p, C.c_int]),
    ("gks_profile_class_name", C.c_char_p, [C.c_int]),
    ("gks_frechet_matvec", C.c_int, [C.c_void_p, c_double_p, c_double_p, c_double_p, c_double_p, C.c_double,
                                     c_double_p]),
]


def load():
    """Load libgks.so once (raises if it has not been built)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH} is missing: build the CUDA extension first "
                "(python -m paper_2304_09485_b200.build); there is no CPU fallback")
        lib = C.CDLL(str(LIB_PATH))
        for name, res, args in SIGNATURES:
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def check(rc):
    if rc != GKS_OK:
        lib = load()
        msg = lib.gks_last_error().decode(errors="replace")
        raise GksError(rc, msg, int(lib.gks_last_error_index()))


def dptr(a):
    """Pointer to a C-contiguous float64 array (None -> NULL)."""
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags.c_contiguous, (a.dtype, a.flags)
    return a.ctypes.data_as(c_double_p)


def iptr(a):
    if a is None:
        return None
    assert a.dtype == np.int64 and a.flags.c_contiguous
    return a.ctypes.data_as(c_int64_p)


def i32ptr(a):
    if a is None:
        return None
    assert a.dtype == np.int32 and a.flags.c_contiguous
    return a.ctypes.data_as(c_int32_p)


def f64(a, shape=None):
    out = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    if shape is not None:
        out = out.reshape(shape)
    return out


def kernel_launches():
    return int(load().gks_kernel_launches())


class Profiler:
    """Per-kernel-class device time (CUDA events on the launching stream)."""

    def __init__(self):
        self.lib = load()

    def start(self):
        check(self.lib.gks_profile_reset())
        check(self.lib.gks_profile_enable(1))

    def stop(self):
        check(self.lib.gks_profile_enable(0))
        n = 32
        ms = np.zeros(n)
        cnt = np.zeros(n, dtype=np.int64)
        k = self.lib.gks_profile_read(dptr(ms), iptr(cnt), n)
        return {self.lib.gks_profile_class_name(i).decode(): (float(ms[i]), int(cnt[i])) for i in range(k)}
