// Block systems, Krylov work space and device-side GMRES state.
#pragma once
#include <functional>

#include "gks_reduce.cuh"
#include "gks_solver.cuh"

namespace gks {

constexpr int GM_MMAX = 64;  // max Krylov dimension
constexpr int MF_REC = 6;     // doubles per face / cell record of the matrix-free Roe products (16-B aligned)
constexpr int GM_RMAX = 64;  // max restarts

// Device-resident GMRES scalars (krylov.py:55-140 state).
struct GmresDev {
  int m, restarts;
  double rtol, atol;
  int done, notdone, active, reorth, reorth_gate;
  int j_used, breakdown, breakdown_any, err, ncycles, matvecs, ny, target_set;
  double target, beta2, beta, wscale2, wscale, hnext2, hdiv;
  double dots[GM_MMAX + 1];
  double corr[GM_MMAX + 1];
  double h[(GM_MMAX + 1) * GM_MMAX];
  double cs[GM_MMAX], sn[GM_MMAX], gv[GM_MMAX + 1], y[GM_MMAX];
  double norms[GM_RMAX * (GM_MMAX + 1)];
  int nnorms[GM_RMAX];
};

struct KrylovWS {
  int64_t n = 0;     // reduction length (5 * owned rows)
  int64_t ld = 0;    // allocation length per vector (5 * (owned + layer-1 ghosts))
  int m = 0;
  int grid = 0;
  double* V = nullptr;
  double* bufs = nullptr;
  double *w = nullptr, *r = nullptr, *t = nullptr, *z = nullptr, *b = nullptr, *x = nullptr;
  // partition-invariant reductions (gks_reduce.cuh): red.gpart points at
  // gpart[parity] for the next launch (parity alternates with the loopback
  // transport's collectives; NCCL and single-rank use gpart[0])
  RedDev red;
  double* gpart[2] = {nullptr, nullptr};
  double* gall = nullptr;  // NCCL allreduce output
  GmresDev* g = nullptr;
  double ortho_error = 0.0;  // host-side Gram check (GmresParams::check_ortho)
  int64_t gen = 0;           // allocation generation (bumped on every (re)allocation)
};

// Block-row matrix: diagonal blocks + CSR off-diagonal blocks (jacobian.py:74-126)
struct BlockSys {
  int64_t nc = 0, nnz = 0;
  int64_t n_ext = 0;                                  // rows + layer-1 ghost columns
  std::function<void(double*)> halo_x;                // fill ghost entries of x before (L+U) x
  // place of the owned rows in the global canonical order (partition-invariant
  // reductions); nc_global == 0: the system's own rows, single rank
  int64_t red_nc_global = 0, red_cell_first = 0;
  Comm* comm = nullptr;   // multi-rank: group-partial exchange for every reduction
  int canonical = 0;      // partitioned handle: keep the segment chain (no fused small-system Arnoldi)
  int *rowptr = nullptr, *col = nullptr;
  double *off = nullptr, *diag = nullptr, *dinv = nullptr;
  int* status = nullptr;
  int dinv_ok = 0;
  cudaStream_t stream = nullptr;
  KrylovWS ws;
  // matrix-free Roe off-diagonal products (handle-owned Jacobians): instead of
  // streaming the stored 5x5 blocks, recompute hs*(+-J(Q_j,n) x_j - lam x_j)
  // from per-face (n, hs, lam) and per-cell primitives (v, H, ke)
  int mf = 0;
  int* ent = nullptr;      // per CSR slot: face << 1 | side (side 0: the row is the face owner)
  double* fdat = nullptr;  // per local face: nx, ny, nz, hs = S/2, lam
  double* prim = nullptr;  // per local cell: vx, vy, vz, H, ke
  double gm1 = 0.4;
};

struct GmresParams {
  int m = 10, restarts = 3, kmax = 2;
  double rtol = 0.0, atol = 0.0;
  int check_ortho = 0;
  int ortho = 0;  // 0: MGS + conditional re-orthogonalisation (krylov.py:89-106); 1: CGS2 fused multi-dots
};

struct GmresHost {
  int ncycles = 0, matvecs = 0, breakdown = 0, err = 0;
  double ortho_error = 0.0;
  int cycle_len[GM_RMAX];
  double norms[GM_RMAX * (GM_MMAX + 1)];
};

// out = A v on the device, gated by *gate (matrix-free operators)
using MatvecFn = std::function<int(const double* v, double* out, const int* gate)>;

int blocksys_alloc(BlockSys* A, int64_t nc, int64_t nnz, cudaStream_t stream);
void blocksys_free(BlockSys* A);
void krylov_free(KrylovWS* W);
// (re)allocate the Krylov space for the system's rows (5 * nc unknowns,
// 5 * n_ext per vector) and its reduction layout; m basis vectors
int krylov_ensure(BlockSys* A, int m);
int dot2(BlockSys* A, int64_t n, const double* a, const double* b, const double* c, const double* d, double* o0,
         double* o1, const int* gate);
int step_stats(BlockSys* A, int64_t nc, const double* res, const double* dt, const int8_t* bad, DevScalars* sc);
int blocksys_invert_diag(BlockSys* A);
void bs_spmv(BlockSys* A, const double* x, double* y, const int* gate);
void bs_offdiag(BlockSys* A, const double* x, double* y, const int* gate);
void bs_jacobi(BlockSys* A, const double* b, double* z, double* tmp, int kmax, const int* gate);
int gmres_device(BlockSys* A, const double* b_dev, double* x_dev, const GmresParams& P, GmresHost* out,
                 const MatvecFn* matvec);
int jacobian_assemble(Handle* H, BlockSys* A, const double* ghosts_dev);
// launch-only halves (CUDA-graph capturable) and the host readback
int jacobian_enqueue(Handle* H, BlockSys* A, const double* ghosts_dev, bool want_blocks);
int gmres_enqueue(BlockSys* A, const double* b_dev, double* x_dev, const GmresParams& P, const MatvecFn* matvec,
                  bool check_dinv);
int gmres_result(const GmresDev* gh, GmresHost* out);
__global__ void k_status_init(int* st, int n);

}  // namespace gks
