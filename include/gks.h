/*
 * libgks -- C ABI of the B200-native implicit HGKS hot path.
 *
 * The reference (gks3d, a pure-Python package) has no FFI; its drop-in
 * boundary is the Python object API of gks3d.stepping / flux / jacobian /
 * krylov.  Each entry point below replaces one reference call, cited as
 * file:line under /root/reference/pkg/src/gks3d.  The Python mirror in
 * paper_2304_09485_b200/ binds these through ctypes.
 *
 * Conventions
 *   - plain C types only; arrays are C-contiguous float64 / int64 host
 *     buffers owned by the caller and copied in/out per call;
 *   - every call returns GKS_OK (0) or a GKS_ERR_* code; gks_last_error()
 *     returns the thread-local message of the last failure and
 *     gks_last_error_index() the first offending cell / point (or -1);
 *   - calls are blocking (the stream is synchronised before returning) and
 *     not re-entrant per handle.
 */
#ifndef GKS_H
#define GKS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GKS_ABI_VERSION 1

enum {
  GKS_OK = 0,
  GKS_ERR_BAD_ARG = 1,
  GKS_ERR_CUDA = 2,
  GKS_ERR_UNPHYSICAL = 3,   /* UnphysicalStateError (kinetic.py:26) / SteppingError */
  GKS_ERR_SINGULAR = 4,     /* SolverError: singular diagonal block (krylov.py:29) */
  GKS_ERR_NONFINITE = 5,    /* SolverError: non-finite Arnoldi vector (krylov.py:105) */
  GKS_ERR_MESH = 6,         /* MeshError (mesh/geometry.py:35) */
  GKS_ERR_NCCL = 7,
  GKS_ERR_NO_DEVICE = 8,
  GKS_ERR_INVALID_UPDATE = 9 /* SteppingError: unphysical update after retry (stepping.py:294) */
};

int gks_abi_version(void);
const char* gks_last_error(void);
int64_t gks_last_error_index(void);
/* number of kernels this library launched since load (evidence counter) */
int64_t gks_kernel_launches(void);

/* ------------------------------------------------------------------ */
/* Minimum slice: batched interface flux.                              */
/* Replaces flux.build_interface + evolve_flux + point_value            */
/* (flux.py:69-107, 162-179, 182-188).                                  */
/*   wl, wr  (n,5)   local-frame primitive states (rho,U,V,W,lam)       */
/*   sl, sr  (n,3,5) local-frame conserved slopes (may be NULL = zero)  */
/*   tau, dt (n)     collision time and time window                     */
/*   tp      (n)     point-value time (NULL: no point value)            */
/*   flux_out (n,5), point_out (n,5) (NULL allowed)                     */
/* ------------------------------------------------------------------ */
int gks_flux_batch(int64_t n, const double* wl, const double* wr, const double* sl,
                   const double* sr, const double* tau, const double* dt, const double* tp,
                   double gamma, double* flux_out, double* point_out);

/* ------------------------------------------------------------------ */
/* Mesh view passed to the native setup and to gks_create.  All arrays   */
/* are the host Mesh arrays of paper_2304_09485_b200.mesh (same layout   */
/* as gks3d.mesh.Mesh, geometry.py:152-181); cell_faces is CSR.          */
/* ------------------------------------------------------------------ */
typedef struct GksMeshDesc {
  int64_t ncells, nfaces, nfq, ncq;
  const int8_t* cell_kind;          /* (nc) 0 tet, 1 hex */
  const double* cell_volume;        /* (nc) */
  const double* cell_h;             /* (nc) */
  const double* cell_centroid;      /* (nc,3) */
  const int64_t* cell_cq_start;     /* (nc+1) */
  const double* cq_point;           /* (ncq,3) */
  const double* cq_weight;          /* (ncq) */
  const int64_t* cell_face_start;   /* (nc+1) */
  const int64_t* cell_face_list;    /* (cell_face_start[nc]) */
  const int64_t* face_owner;        /* (nf) */
  const int64_t* face_neighbor;     /* (nf), -1 on boundary */
  const int64_t* face_patch;        /* (nf), -1 interior */
  const double* face_area;          /* (nf) */
  const double* face_normal;        /* (nf,3) */
  const double* face_frame;         /* (nf,3,3) rows n, t1, t2 */
  const double* face_shift;         /* (nf,3) */
  const int64_t* face_fq_start;     /* (nf+1) */
  const int64_t* fq_face;           /* (nfq) */
  const double* fq_point;           /* (nfq,3) */
  const double* fq_weight;          /* (nfq) */
} GksMeshDesc;

/* ------------------------------------------------------------------ */
/* Native setup (host, no GPU needed): stencil selection and the        */
/* reconstruction operators.  Replaces mesh.build_stencils              */
/* (stencils.py:119-192), ReconGeometry (recon.py:104-164),             */
/* WenoReconstructor._build_operators (recon.py:216-274) and            */
/* HwenoReconstructor._build_operators (hweno.py:62-137).               */
/* schemes: bit 0 = WENO operators, bit 1 = HWENO operators.            */
/* Arrays are exported by name (gks_setup_query / gks_setup_copy);      */
/* dtype 0 = float64, 1 = int64, 2 = int8.                              */
/* ------------------------------------------------------------------ */
typedef struct GksSetup GksSetup;
int gks_setup_build(const GksMeshDesc* mesh, int schemes, int nthreads, GksSetup** out);
void gks_setup_free(GksSetup* setup);
int gks_setup_query(const GksSetup* setup, const char* name, int* dtype, int* ndim, int64_t* shape);
int gks_setup_copy(const GksSetup* setup, const char* name, void* dst, int64_t nbytes);

/* measurement hook: kernel-only time of the fused flux on n random
   device-resident interfaces (not a reference API) */
int gks_flux_bench(int64_t n, int reps, double gamma, double* ms_per_launch);

#ifdef __cplusplus
}
#endif
#endif /* GKS_H */
