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
/* instantaneous_flux (flux.py:191-197): the moment flux of the interface
   distribution at time t (n), the same kernel with the point-value time
   coefficients */
int gks_instant_flux_batch(int64_t n, const double* wl, const double* wr, const double* sl,
                           const double* sr, const double* tau, const double* t, double gamma,
                           double* flux_out);

/* build_interface intermediates (flux.py:69-107, InterfaceBatch fields):
   al, ar (n,3,5) micro-slopes, atl, atr (n,5) time slopes, w0 (n,5)
   compatibility state, abar (n,3,5), atbar (n,5) its slopes; sl/sr NULL =
   zero slopes */
int gks_interface_data(int64_t n, const double* wl, const double* wr, const double* sl,
                       const double* sr, double gamma, double* al, double* ar, double* atl,
                       double* atr, double* w0, double* abar, double* atbar);
/* solve_micro_slope (kinetic.py:271-302, time_slope = 0: in = dq (n,5)) or
   solve_time_slope (:305-312, time_slope = 1: in = micro-slopes (n,3,5)) of
   primitive states w (n,5) -> out (n,5) */
int gks_slopes(int64_t n, const double* w, const double* in, int time_slope, double gamma, double* out);
/* build_moments (kinetic.py:140-162): order-first (order+1, n) tables of
   <u^p> full / u>0 / u<0, <v^p>, <w^p> and (3, n) <xi^2s> */
int gks_moment_table(int64_t n, const double* w, double gamma, int order, double* u_full,
                     double* u_pos, double* u_neg, double* v_full, double* w_full, double* xi);

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
  /* optional (NULL = identity): reference index of each face / face point
     of a renumbered mesh (SolverOptions.reorder, reorder.py); the handle
     sums every per-cell list in this order so results keep the
     reference's summation order */
  const int64_t* face_rank;         /* (nf) */
  const int64_t* fq_rank;           /* (nfq) */
  /* optional (NULL = identity): reference id of each cell; the Jacobian's
     off-diagonal blocks of a row are ordered by it (jacobian.py:181-196) */
  const int64_t* cell_rank;         /* (nc) */
} GksMeshDesc;

/* ------------------------------------------------------------------ */
/* Native ugks-mesh reader (host, no GPU needed).  Replaces the per-line */
/* parse of load_mesh (mesh/fileio.py:42-103); returns GKS_ERR_BAD_ARG  */
/* on any grammar violation (the Python caller then re-parses to raise  */
/* the reference's exact MeshError).  Patch faces come back (nf, 4),    */
/* padded with -1, with their widths (3 or 4).                          */
typedef struct GksUgks GksUgks;
int gks_ugks_read(const char* path, GksUgks** out);
int gks_ugks_sizes(const GksUgks* m, int64_t* nnodes, int64_t* ntets, int64_t* nhexes, int64_t* npatches);
int gks_ugks_patch(const GksUgks* m, int64_t k, char* name, int64_t cap, int64_t* nfaces);
int gks_ugks_copy(const GksUgks* m, double* nodes, int64_t* tets, int64_t* hexes, int64_t* faces, int8_t* widths);
void gks_ugks_free(GksUgks* m);

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

/* ------------------------------------------------------------------ */
/* Solver handle: device-resident mesh, operators, state and Krylov     */
/* work space on one GPU.  Replaces gks3d.stepping.Solver               */
/* (stepping.py:87-313) underneath the Python Solver mirror.            */
/* ------------------------------------------------------------------ */
enum {  /* boundary.py:18-19 PATCH_KINDS */
  GKS_PATCH_NONE = -1,
  GKS_PATCH_WALL_NOSLIP_ISOTHERMAL = 0,
  GKS_PATCH_WALL_NOSLIP_ADIABATIC = 1,
  GKS_PATCH_WALL_SLIP_ADIABATIC = 2,
  GKS_PATCH_FARFIELD_RIEMANN = 3,
  GKS_PATCH_SUPERSONIC_INLET = 4,
  GKS_PATCH_SUPERSONIC_OUTLET = 5
};

typedef struct GksPatchDesc {  /* boundary.PatchSpec (boundary.py:26-48) */
  int kind;
  double reference[5];  /* (rho, U, V, W, p) */
  double lambda_wall;
  double velocity[3];
} GksPatchDesc;

enum { GKS_SCHEME_WENO_GMRES = 0, GKS_SCHEME_HWENO_GMRES = 1, GKS_SCHEME_WENO_LUSGS = 2 };
enum { GKS_JAC_ROE = 0, GKS_JAC_FRECHET = 1 };

typedef struct GksOptions {  /* stepping.SolverOptions (stepping.py:61-84) */
  int scheme;
  int model;             /* 0 inviscid, 1 viscous */
  double mu, gamma, cfl;
  int krylov_dim, restarts, jacobi_sweeps;
  double gmres_rtol;
  double weno_eps, linear_weight;
  int linear_weights;    /* weights="linear" */
  int global_time_step;  /* time_step="global" */
  int jacobian_mode;     /* GKS_JAC_ROE (reference) or GKS_JAC_FRECHET (matrix-free) */
  int npatch;            /* == number of mesh patches; indexed by mesh patch id */
  const GksPatchDesc* patches;
  int first_order;       /* B200 build: first-order KFVS residual (piecewise-constant states,
                            collisionless flux, flux.py:200-208) -- the paper's low-order start
                             */
  int ortho;             /* B200 build: GMRES orthogonalisation, 0 = MGS + conditional second
                            pass (krylov.py:89-106), 1 = CGS2 with fused multi-dots */
} GksOptions;

typedef struct GksHandle GksHandle;

/* Build device state.  setup == NULL: stencil selection, reconstruction
   geometry and operators are built on the GPU (gks_setup_dev.cu), bit-
   identical to the records built from gks_setup_build's arrays. */
int gks_create(const GksMeshDesc* mesh, const GksSetup* setup, const GksOptions* opt, int device,
               GksHandle** out);
void gks_destroy(GksHandle* h);
/* Reconstruction pieces of recon.py / hweno.py (the reference's
   WenoReconstructor / HwenoReconstructor / evaluate_faces API) on a
   handle's cells, 5 components, host arrays:
   gks_recon_coeffs      combined_coeffs (recon.py:285-294, hweno.py:162-169),
                         linear = 1: the big candidate alone -> coef (nc,9,5);
                         the solver's own k_recon_* kernel
   gks_recon_candidates  candidate_coeffs (recon.py:276-283, hweno.py:139-160)
                         -> c_big (nc,9,5), b_sub (nc,M,3,5), M = reference
                         sub-stencil width (gks_handle_info(h, 7))
   gks_face_values       evaluate_faces (recon.py:297-314) from coef (nc,9,5)
                         -> val_o, val_n (nfq,5), grad_o, grad_n (nfq,3,5)
   gks_combine_candidates combine_candidates (recon.py:167-195) on an
                         (n,9,k) / (n,m,3,k) batch, active (n,m), beta (n,9,9)
                         -> out (n,9,k), w0n (n,k), wmn (n,m,k); m <= 16 */
int gks_recon_coeffs(GksHandle* h, const double* q, const double* grad, int linear, double* coef);
int gks_recon_candidates(GksHandle* h, const double* q, const double* grad, double* c_big, double* b_sub);
int gks_face_values(GksHandle* h, const double* q, const double* coef, double* val_o, double* grad_o,
                    double* val_n, double* grad_n);
int gks_combine_candidates(int64_t n, int k, int m, const double* c_big, const double* b_sub,
                           const int8_t* active, const double* beta, double eps, double lin_weight,
                           double* out, double* w0n, double* wmn);
/* Diagnostic copy of a device setup array of a handle (B200 build):
   "avg0", "beta", "big_op", "big_gather", "sub_op", "sub_gather",
   "sub_active", "avg_gather", "grad_gather", "grad_scale" (the padded
   per-cell records the reconstruction kernels read).  dst == NULL: only
   *nbytes is set. */
int gks_handle_array(GksHandle* h, const char* name, void* dst, int64_t* nbytes);

/* ------------------------------------------------------------------ */
/* Domain decomposition (multi-GPU; no reference counterpart) */
/* A local handle holds cells [owned | ghost layer 1 | deeper layers];   */
/* owned + layer-1 ghosts are reconstructed, owned rows are assembled /   */
/* solved.  Halo maps list, per peer rank, the local ids to send and the  */
/* local ids to receive into (q: all ghost layers, x: layer 1).          */
/* ------------------------------------------------------------------ */
typedef struct GksHaloDesc {
  int npeers;
  const int* peers;              /* (npeers) */
  const int64_t* send_offsets;   /* (npeers+1) into send_ids */
  const int64_t* send_ids;
  const int64_t* recv_offsets;   /* (npeers+1) into recv_ids */
  const int64_t* recv_ids;
} GksHaloDesc;

typedef struct GksDomainDesc {
  int64_t n_owned, n_recon, nc_global;
  GksHaloDesc q, x;
  /* position of the first owned cell in the global canonical order: owned
     cells are consecutive there and start and end on multiples of
     gks_reduction_granularity(nc_global) cells (the last rank may end at
     nc_global), which makes every reduction partition-invariant */
  int64_t owned_offset;
  /* device-side setup of a rank-local handle (gks_create_local with setup
     == NULL; B200 build): the rank's native-setup view -- its local cells
     in ascending reference id with every face of every such cell
     (partition.py SetupMesh) -- and the maps between that order and the
     local one.  NULL when a host setup is passed. */
  const struct GksMeshDesc* setup_mesh;
  const int64_t* local_to_setup;  /* (n_local) */
  const int64_t* setup_to_local;  /* (setup_mesh->ncells) */
} GksDomainDesc;
/* cells per reduction group of a mesh of nc_global cells (partition alignment) */
int64_t gks_reduction_granularity(int64_t nc_global);

int gks_create_local(const GksMeshDesc* mesh, const GksSetup* setup, const GksOptions* opt,
                     const GksDomainDesc* domain, int device, GksHandle** out);
/* restrict a global setup to local cells (local->global ids; global->local map, -1 = absent) */
int gks_setup_subset(const GksSetup* global, const int64_t* cells, int64_t n_local, const int64_t* g2l,
                     int64_t n_global, GksSetup** out);
int gks_comm_unique_id(void* out, int64_t nbytes);           /* ncclGetUniqueId (128 bytes) */
int gks_comm_init(GksHandle* h, const void* unique_id, int nranks, int rank);
/* In-process loopback transport: nranks rank-local handles of ONE process
   (one host thread per rank, e.g. Python threads each calling
   gks_advance_resident) exchange halos and reduction partials through
   device copies ordered by CUDA events and host barriers -- no kernel waits
   on another, so the ranks may share one GPU.  Same pack / exchange / unpack
   and reduction code as NCCL; steps run uncaptured. */
typedef struct GksLoopback GksLoopback;
int gks_loopback_create(int nranks, GksLoopback** out);
int gks_comm_init_loopback(GksHandle* h, GksLoopback* group, int rank);
void gks_loopback_destroy(GksLoopback* group);  /* after every member handle is destroyed */

/* Solver.local_time_step (stepping.py:135-157): q (nc,5) -> dt (nc) */
int gks_local_dt(GksHandle* h, const double* q, double* dt_out);

/* Solver.residual (stepping.py:212-238).  grad (nc,3,5) required for the
   compact scheme; grad_out (nc,3,5) written when with_gradients != 0. */
int gks_residual(GksHandle* h, const double* q, const double* grad, const double* dt,
                 int with_gradients, double* res_out, double* grad_out);

/* Solver._boundary_ghosts (stepping.py:242-249): ghost of the cell-average
   owner state per boundary face, (nbf,5) in ascending boundary-face order */
int gks_boundary_ghosts(GksHandle* h, const double* q, double* ghosts_out);
/* boundary.ghost_state / ghost_gradients (boundary.py:66-171) for n points
   of one patch: conserved q (n,5), outward normals (n,3), optional
   gradients (n,3,5) -> q_out (n,5), grad_out (n,3,5) */
struct GksPatchDesc;
int gks_ghost_batch(int64_t n, const struct GksPatchDesc* patch, const double* q, const double* normal,
                    const double* grad, double gamma, double* q_out, double* grad_out);
/* hweno.update_gradients (hweno.py:172-194): cell-averaged gradients
   (nc,3,5) from face-point values (nfq,5) by the Gauss theorem */
int gks_update_gradients(GksHandle* h, const double* qpt, double* grad_out);
int64_t gks_num_boundary_faces(const GksHandle* h);

/* ------------------------------------------------------------------ */
/* Block systems (BlockJacobian, jacobian.py:74-126) and GMRES          */
/* ------------------------------------------------------------------ */
typedef struct GksBlockSystem GksBlockSystem;

#define GKS_GMRES_MAX_DIM 64
#define GKS_GMRES_MAX_RESTARTS 64

typedef struct GksGmresInfo {  /* krylov.GmresInfo (krylov.py:37-52) */
  int ncycles;
  int matvecs;
  int breakdown;
  double ortho_error;
  int cycle_len[GKS_GMRES_MAX_RESTARTS];
  double norms[GKS_GMRES_MAX_RESTARTS * (GKS_GMRES_MAX_DIM + 1)]; /* row c: cycle c norms */
} GksGmresInfo;

typedef struct GksStepInfo {  /* stepping.StepInfo (stepping.py:52-58) */
  double res_rho_l1, res_l2, dt_min;
  int solver_cycles;
  int retried;
  int matvecs;
  int nbad;                   /* on GKS_ERR_INVALID_UPDATE: number of bad cells */
  int64_t first_bad[8];       /* ... and the first (up to) 8 of them */
} GksStepInfo;

/* assemble_jacobian(mesh, q, dt, gamma, ghosts) (jacobian.py:133-196) into
   the handle's device Jacobian; ghosts (nbf,5) may be NULL */
int gks_assemble_jacobian(GksHandle* h, const double* q, const double* dt, const double* ghosts);
/* the handle's Jacobian as a block system (owned by the handle) */
GksBlockSystem* gks_jacobian(GksHandle* h);

/* upload an arbitrary block system (random_block_system, jacobian.py:199-226) */
int gks_blocksys_create(int64_t ncells, int64_t nnz, const double* diag, const double* off,
                        const int64_t* off_col, const int64_t* rowptr, int device, GksBlockSystem** out);
void gks_blocksys_destroy(GksBlockSystem* a);
int64_t gks_blocksys_ncells(const GksBlockSystem* a);
int64_t gks_blocksys_nnz(const GksBlockSystem* a);
/* download (any pointer may be NULL) */
int gks_blocksys_export(GksBlockSystem* a, double* diag, double* off, int64_t* off_col, int64_t* off_row,
                        int64_t* rowptr);
int gks_blocksys_spmv(GksBlockSystem* a, const double* x, double* y);          /* BlockJacobian.spmv */
int gks_blocksys_offdiag_mv(GksBlockSystem* a, const double* x, double* y);    /* .offdiag_mv */
/* x . y over the system's rows with the GMRES reduction (partition-invariant
   fold, csrc/gks_reduce.cuh) -- a measurement / specification hook */
int gks_blocksys_dot(GksBlockSystem* a, const double* x, const double* y, double* out);
int gks_blocksys_diag_inverses(GksBlockSystem* a, double* out);               /* .diag_inverses */
int gks_blocksys_jacobi(GksBlockSystem* a, const double* b, int k_max, double* z); /* krylov.py:24-34 */
/* gmres_solve (krylov.py:55-140): x_out (nc,5) */
int gks_gmres(GksBlockSystem* a, const double* b, double* x_out, int m, int restarts, int k_max, double rtol,
              double atol, int check_orthogonality, GksGmresInfo* info);

/* Solver.advance (stepping.py:270-296): one backward-Euler step in place.
   grad_inout (nc,3,5) for the compact scheme (NULL otherwise). */
int gks_advance(GksHandle* h, double* q_inout, double* grad_inout, GksStepInfo* info);
/* device-resident variant for the outer loop / benchmark */
int gks_state_upload(GksHandle* h, const double* q, const double* grad);
int gks_state_download(GksHandle* h, double* q, double* grad);
int gks_advance_resident(GksHandle* h, GksStepInfo* info);
/* after GKS_ERR_INVALID_UPDATE: the validity mask of the rejected update
   (n_owned int8, 1 = bad), so the caller can name the cells in its own
   (reference) numbering (stepping.py:294-296) */
int gks_bad_mask(GksHandle* h, int8_t* out);
/* Steps after a handle's first replay one captured CUDA graph of the whole
   step (no host synchronisation inside it).  enable = 0 runs every step
   uncaptured (default: on unless the environment sets GKS_GRAPH=0). */
int gks_set_graph(GksHandle* h, int enable);
/* change SolverOptions.cfl of a live handle (a CFL ramp; next step re-captures) */
int gks_set_cfl(GksHandle* h, double cfl);
/* GMRES orthogonalisation of a live handle: 0 MGS (reference), 1 CGS2 */
int gks_set_ortho(GksHandle* h, int ortho);
/* Solver.frechet_matvec (stepping.py:298-313); sigma <= 0 selects the
   reference's automatic step.  out = (L(q + s v) - L(q)) / s */
int gks_frechet_matvec(GksHandle* h, const double* q, const double* grad, const double* dt, const double* v,
                       double sigma, double* out);

/* ------------------------------------------------------------------ */
/* Measurement hooks (not reference APIs): CUDA events on the handle's   */
/* stream, handle sizes, and the per-kernel-class profiler (events on    */
/* the launching stream around every launch while enabled).              */
/* ------------------------------------------------------------------ */
int gks_event_record(GksHandle* h, int slot);                 /* slot 0..7 */
int gks_event_elapsed(GksHandle* h, int a, int b, double* ms);
int64_t gks_handle_info(const GksHandle* h, int what);        /* 0 nc 1 nf 2 nfq 3 nfi 4 nbf 5 nnz 6 K 7 M 8 S 9 n_owned 10 assembly entries */
int gks_fp64_peak(double* tflops);                          /* DFMA throughput probe */
int gks_host_pin(void* p, int64_t nbytes);                  /* cudaHostRegister a host buffer */
int gks_host_unpin(void* p);
int gks_profile_enable(int on);
int gks_profile_reset(void);
int gks_profile_read(double* ms_out, int64_t* count_out, int ncls);  /* returns number of classes */
const char* gks_profile_class_name(int k);

/* measurement hook: kernel-only time of the fused flux on n random
   device-resident interfaces (not a reference API) */
int gks_flux_bench(int64_t n, int reps, double gamma, double* ms_per_launch);

#ifdef __cplusplus
}
#endif
#endif /* GKS_H */
