// Implicit solve on the device: Roe-split block Jacobian (K5), block spmv and
// block-Jacobi (K6/K7), left-preconditioned restarted GMRES with modified
// Gram-Schmidt (K8) and the state update with validity check (K9).
//
// Reference: gks3d/jacobian.py:37-196 (euler_flux_jacobian, spectral_radius,
// BlockJacobian, assemble_jacobian), gks3d/krylov.py:24-140
// (jacobi_precondition, gmres_solve), gks3d/stepping.py:251-296 (_solve,
// advance).
//
// GMRES control flow lives on the device: the Hessenberg / Givens scalars
// and the cycle bookkeeping sit in a GmresDev struct in device memory; every
// vector kernel reads a gate flag and returns immediately once the reference
// algorithm would have left the loop (happy breakdown, early exit, target
// reached).  The host enqueues the fixed launch sequence without a single
// synchronisation and reads the cycle norms back once at the end.
//
// Reductions are deterministic: fixed grid, per-block tree, and the last
// block to finish sums the block partials in index order.
#include <stddef.h>
#include <string.h>

#include <algorithm>
#include <vector>

#include <cooperative_groups.h>

#include "gks_implicit.cuh"
#include "gks_reduce.cuh"
#include "gks_stage.cuh"

namespace gks {

#define TRY_GM(x)          \
  do {                     \
    int _r = (x);          \
    if (_r) return _r;     \
  } while (0)

static constexpr int RB_THREADS = 256;
static constexpr int CELLS_PER_BLOCK = 32;  // (cell,row) kernels: 160 threads

// ---------------------------------------------------------------------------
// deterministic reductions
// ---------------------------------------------------------------------------
__device__ __forceinline__ double block_sum(double v, double* sm) {
  sm[threadIdx.x] = v;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sm[threadIdx.x] += sm[threadIdx.x + s];
    __syncthreads();
  }
  return sm[0];
}

// Partition-invariant dots (gks_reduce.cuh): one block per segment of
// SEG_CELLS cells (5 * SEG_CELLS vector entries).
static constexpr int64_t SEG_VALS = 5 * (int64_t)SEG_CELLS;

// out0 = a.b, out1 = c.d   (c may be null)
__global__ void __launch_bounds__(RED_T) k_dot2(int64_t n, const double* __restrict__ a,
                                                const double* __restrict__ b, const double* __restrict__ c,
                                                const double* __restrict__ d, RedDev R, RedOut out, const int* gate) {
  __shared__ double sm[9];
  if (gate && !*gate) return;
  const int64_t base = (int64_t)blockIdx.x * SEG_VALS;
  const int64_t len = min(SEG_VALS, n - base);
  a += base; b += base;
  double v[2];
  if (c) {
    c += base; d += base;
    red_lanes<2, 0>(len, [&](int64_t i, double* o) { o[0] = __dmul_rn(a[i], b[i]); o[1] = __dmul_rn(c[i], d[i]); }, v);
    red_finish<2, 0>(R, v, out, sm);
  } else {
    red_lanes<1, 0>(len, [&](int64_t i, double* o) { o[0] = __dmul_rn(a[i], b[i]); }, v);
    red_finish<1, 0>(R, v, out, sm);
  }
}

// w -= (*coef) * v ; out = w . nxt  (nxt == nullptr: out = w . w)
__global__ void __launch_bounds__(RED_T) k_axpy_dot(int64_t n, double* __restrict__ w,
                                                    const double* __restrict__ v, const double* coef,
                                                    const double* __restrict__ nxt, RedDev R, RedOut out,
                                                    const int* gate) {
  __shared__ double sm[9];
  if (gate && !*gate) return;
  const double h = *coef;
  const int64_t base = (int64_t)blockIdx.x * SEG_VALS;
  const int64_t len = min(SEG_VALS, n - base);
  w += base; v += base;
  double r[1];
  if (nxt) {
    nxt += base;
    red_lanes<1, 0>(len, [&](int64_t i, double* o) {
      const double w0 = w[i] - h * v[i];
      w[i] = w0;
      o[0] = __dmul_rn(w0, nxt[i]);
    }, r);
  } else {
    red_lanes<1, 0>(len, [&](int64_t i, double* o) {
      const double w0 = w[i] - h * v[i];
      w[i] = w0;
      o[0] = __dmul_rn(w0, w0);
    }, r);
  }
  red_finish<1, 0>(R, r, out, sm);
}

// Multi-rank final fold over the exchanged group partials (gks_reduce.cuh):
// entry g of component c is the rank-order sum (min) over the sources --
// exact, only its owner's entry is not +0 (+inf).
template <int NS, int NM>
__global__ void __launch_bounds__(RED_T) k_red_final(RedSrc src, int64_t ngrp_g, RedOut out, const int* gate) {
  __shared__ double sm[9];
  if (gate && !*gate) return;
#pragma unroll
  for (int c = 0; c < NS + NM; ++c) {
    double v;
    if (c < NS) {
      red_lanes<1, 0>(ngrp_g, [&](int64_t g, double* o) {
        double x = __ldcg(src.p[0] + c * ngrp_g + g);
        for (int r = 1; r < src.n; ++r) x += __ldcg(src.p[r] + c * ngrp_g + g);
        o[0] = x;
      }, &v);
      v = red_tree<0>(v, sm);
    } else {
      const int64_t off = (int64_t)(RED_MIN_SLOT + c - NS) * ngrp_g;
      red_lanes<0, 1>(ngrp_g, [&](int64_t g, double* o) {
        double x = __ldcg(src.p[0] + off + g);
        for (int r = 1; r < src.n; ++r) x = fmin(x, __ldcg(src.p[r] + off + g));
        o[0] = x;
      }, &v);
      v = red_tree<1>(v, sm);
    }
    if (threadIdx.x == 0 && out.o[c]) *out.o[c] = v;
  }
}

// the same with a runtime number of sum components (CGS2 multi-dots)
__global__ void __launch_bounds__(RED_T) k_red_final_n(RedSrc src, int64_t ngrp_g, int nc, RedOutN out,
                                                       const int* gate) {
  __shared__ double sm[9];
  if (gate && !*gate) return;
  for (int c = 0; c < nc; ++c) {
    double v;
    red_lanes<1, 0>(ngrp_g, [&](int64_t g, double* o) {
      double x = __ldcg(src.p[0] + c * ngrp_g + g);
      for (int r = 1; r < src.n; ++r) x += __ldcg(src.p[r] + c * ngrp_g + g);
      o[0] = x;
    }, &v);
    v = red_tree<0>(v, sm);
    if (threadIdx.x == 0) {
      double* o = c < nc - 1 ? out.base + c : out.last;
      if (o) *o = v;
    }
  }
}

// CGS2 passes over the Arnoldi basis v_0 .. v_{NV-1} (one block per segment):
//   MODE 1: c_k = v_k . w, c_NV = w . w
//   MODE 2: w -= sum_k h_k v_k, then c_k = v_k . w, c_NV = w . w
//   MODE 3: w -= sum_k h_k v_k, then c_0 = w . w
// One read of each basis vector and of w per pass (all dots fused).
template <int NV, int MODE>
__global__ void __launch_bounds__(RED_T) k_cgs(int64_t n, int64_t ld, const double* __restrict__ V,
                                               double* __restrict__ w, const double* h, RedDev R, RedOutN out,
                                               const int* gate) {
  __shared__ double sm[9];
  if (gate && !*gate) return;
  constexpr int NC = MODE == 3 ? 1 : NV + 1;
  const int64_t base = (int64_t)blockIdx.x * SEG_VALS;
  const int64_t len = min(SEG_VALS, n - base);
  double hk[NV];
  if (MODE >= 2) {
#pragma unroll
    for (int k = 0; k < NV; ++k) hk[k] = h[k];
  }
  double acc[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) acc[c] = 0.0;
  for (int64_t i = threadIdx.x; i < len; i += RED_T) {
    const int64_t e = base + i;
    double vk[NV];
#pragma unroll
    for (int k = 0; k < NV; ++k) vk[k] = V[k * ld + e];
    double wi = w[e];
    if (MODE >= 2) {
#pragma unroll
      for (int k = 0; k < NV; ++k) wi -= hk[k] * vk[k];
      w[e] = wi;
    }
    if (MODE <= 2) {
#pragma unroll
      for (int k = 0; k < NV; ++k) acc[k] += __dmul_rn(vk[k], wi);
    }
    acc[NC - 1] += __dmul_rn(wi, wi);
  }
  red_finish_n<NC>(R, acc, out, sm);
}

template <int NV>
static void launch_cgs(int mode, int grid, cudaStream_t s, int64_t n, int64_t ld, const double* V, double* w,
                       const double* h, const RedDev& R, const RedOutN& out, const int* gate) {
  if (mode == 1) GKS_LAUNCH(KC_REDUCE, (k_cgs<NV, 1>), grid, RED_T, 0, s, n, ld, V, w, h, R, out, gate);
  else if (mode == 2) GKS_LAUNCH(KC_REDUCE, (k_cgs<NV, 2>), grid, RED_T, 0, s, n, ld, V, w, h, R, out, gate);
  else GKS_LAUNCH(KC_REDUCE, (k_cgs<NV, 3>), grid, RED_T, 0, s, n, ld, V, w, h, R, out, gate);
}

constexpr int CGS_MAXV = RED_MAXC_MD - 1;  // basis vectors per pass (krylov_dim <= 15)

template <int NV>
static void cgs_dispatch(int nv, int mode, int grid, cudaStream_t s, int64_t n, int64_t ld, const double* V,
                         double* w, const double* h, const RedDev& R, const RedOutN& out, const int* gate) {
  if (nv == NV) launch_cgs<NV>(mode, grid, s, n, ld, V, w, h, R, out, gate);
  else if constexpr (NV < CGS_MAXV) cgs_dispatch<NV + 1>(nv, mode, grid, s, n, ld, V, w, h, R, out, gate);
}

// one CGS2 pass with its reduction (and, multi-rank, the partial exchange)
static int cgs_pass(BlockSys* A, int mode, int nv, int64_t n, int64_t ld, double* w, const double* h,
                    const RedOutN& out, const int* gate) {
  KrylovWS* W = &A->ws;
  W->red.gpart = A->comm ? comm_red_buffer(A->comm, W) : W->gpart[0];
  cgs_dispatch<1>(nv, mode, (int)W->red.nseg, A->stream, n, ld, W->V, w, h, W->red, out, gate);
  if (A->comm) return comm_red_final_n(A->comm, W, mode == 3 ? 1 : nv + 1, out, gate, A->stream);
  return GKS_OK;
}

template __global__ void k_red_final<1, 0>(RedSrc, int64_t, RedOut, const int*);
template __global__ void k_red_final<2, 0>(RedSrc, int64_t, RedOut, const int*);
template __global__ void k_red_final<3, 1>(RedSrc, int64_t, RedOut, const int*);

// out = in / *den
__global__ void k_div(int64_t n, double* __restrict__ out, const double* __restrict__ in, const double* den,
                      const int* gate) {
  if (gate && !*gate) return;
  const double d = *den;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = in[i] / d;
}

__global__ void k_copy(int64_t n, double* __restrict__ out, const double* __restrict__ in) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = in[i];
}

// ---------------------------------------------------------------------------
// K5: Roe-split Jacobian assembly (jacobian.py:133-196)
// ---------------------------------------------------------------------------
__global__ void k_jac_faces(int64_t nfi, const int* __restrict__ ifaces, const int* __restrict__ f_own,
                            const int* __restrict__ f_nbr, const double* __restrict__ f_normal,
                            const double* __restrict__ f_area, const double* __restrict__ q,
                            const int* __restrict__ fslot, double gam, double* __restrict__ off,
                            double* __restrict__ fdat) {
  const int64_t fi = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (fi >= nfi) return;
  const int f = ifaces[fi];
  const int64_t o = f_own[f], nb = f_nbr[f];
  double qo[5], qn[5], qm[5];
  for (int k = 0; k < 5; ++k) {
    qo[k] = q[o * 5 + k];
    qn[k] = q[nb * 5 + k];
    qm[k] = 0.5 * (qo[k] + qn[k]);
  }
  const double n[3] = {f_normal[3 * f], f_normal[3 * f + 1], f_normal[3 * f + 2]};
  const double lam = spectral_radius(qm, n, gam);
  const double hs = 0.5 * f_area[f];
  if (fdat) {
    double* fd = fdat + (int64_t)f * MF_REC;
    fd[0] = n[0]; fd[1] = n[1]; fd[2] = n[2]; fd[3] = hs; fd[4] = lam; fd[5] = 0.0;
  }
  if (!off) return;  // matrix-free step: the stored blocks are not needed
  double J[5][5];
  // rows of ghost cells (cut faces on a partitioned mesh) have no slot
  if (fslot[2 * f] >= 0) {
    euler_jacobian(qn, n, gam, J);
    double* B = off + (int64_t)fslot[2 * f] * 25;  // row own, col nbr
    for (int i = 0; i < 5; ++i)
      for (int j = 0; j < 5; ++j) B[i * 5 + j] = hs * (J[i][j] - (i == j ? lam : 0.0));
  }
  if (fslot[2 * f + 1] >= 0) {
    euler_jacobian(qo, n, gam, J);
    double* B = off + (int64_t)fslot[2 * f + 1] * 25;  // row nbr, col own
    for (int i = 0; i < 5; ++i)
      for (int j = 0; j < 5; ++j) B[i * 5 + j] = hs * (-J[i][j] - (i == j ? lam : 0.0));
  }
}

// 5x5 inverse by LU with partial pivoting (numpy.linalg.inv: LAPACK gesv on I)
__device__ __forceinline__ bool inv5(const double A[25], double X[25]) {
  double a[25];
  int piv[5];
  for (int i = 0; i < 25; ++i) a[i] = A[i];
  for (int k = 0; k < 5; ++k) {
    int p = k;
    double mx = fabs(a[k * 5 + k]);
    for (int i = k + 1; i < 5; ++i)
      if (fabs(a[i * 5 + k]) > mx) { mx = fabs(a[i * 5 + k]); p = i; }
    piv[k] = p;
    if (a[p * 5 + k] == 0.0) return false;
    if (p != k)
      for (int j = 0; j < 5; ++j) { const double t = a[k * 5 + j]; a[k * 5 + j] = a[p * 5 + j]; a[p * 5 + j] = t; }
    const double r = 1.0 / a[k * 5 + k];
    for (int i = k + 1; i < 5; ++i) {
      const double l = a[i * 5 + k] * r;
      a[i * 5 + k] = l;
      for (int j = k + 1; j < 5; ++j) a[i * 5 + j] -= l * a[k * 5 + j];
    }
  }
  for (int col = 0; col < 5; ++col) {
    double b[5] = {0, 0, 0, 0, 0};
    b[col] = 1.0;
    for (int k = 0; k < 5; ++k)
      if (piv[k] != k) { const double t = b[k]; b[k] = b[piv[k]]; b[piv[k]] = t; }
    for (int i = 1; i < 5; ++i)
      for (int j = 0; j < i; ++j) b[i] -= a[i * 5 + j] * b[j];
    for (int i = 4; i >= 0; --i) {
      for (int j = i + 1; j < 5; ++j) b[i] -= a[i * 5 + j] * b[j];
      b[i] /= a[i * 5 + i];
    }
    for (int i = 0; i < 5; ++i) X[i * 5 + col] = b[i];
  }
  for (int i = 0; i < 25; ++i)
    if (!isfinite(X[i])) return false;
  return true;
}

// diagonal blocks: V/dt I + interior(own) + interior(nbr) + boundary(own), then D^-1
// (jacobian.py:567-610, np.add.at order: interior faces as owner, interior
// faces as neighbour, boundary faces; ascending face id within each group)
__global__ void k_jac_diag(int64_t nc, const int* __restrict__ cjd_start, const int* __restrict__ cjd,
                           const int* __restrict__ f_own, const int* __restrict__ f_nbr,
                           const double* __restrict__ f_normal, const double* __restrict__ f_area,
                           const int* __restrict__ bidx_of_face, const double* __restrict__ ghosts,
                           const double* __restrict__ q, const double* __restrict__ vol,
                           const double* __restrict__ dt, double gam, double* __restrict__ diag,
                           double* __restrict__ dinv, int* status) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= nc) return;
  double D[25];
  for (int i = 0; i < 25; ++i) D[i] = 0.0;
  const double vd = vol[c] / dt[c];
  for (int i = 0; i < 5; ++i) D[i * 6] = vd;
  double qc[5];
  for (int k = 0; k < 5; ++k) qc[k] = q[c * 5 + k];
  for (int e = cjd_start[c]; e < cjd_start[c + 1]; ++e) {
    const int f = cjd[e] >> 1;
    const int side = cjd[e] & 1;
    const double n[3] = {f_normal[3 * f], f_normal[3 * f + 1], f_normal[3 * f + 2]};
    const double hs = 0.5 * f_area[f];
    const int64_t nb = f_nbr[f];
    double qm[5];
    if (nb >= 0) {
      const int64_t o = f_own[f];
      for (int k = 0; k < 5; ++k) qm[k] = 0.5 * (q[o * 5 + k] + q[nb * 5 + k]);
    } else if (ghosts) {
      // boundary face, frozen ghost sharpens |lambda| (jacobian.py:597-610)
      const int64_t b = bidx_of_face[f];
      for (int k = 0; k < 5; ++k) qm[k] = 0.5 * (qc[k] + ghosts[b * 5 + k]);
    } else {
      for (int k = 0; k < 5; ++k) qm[k] = qc[k];
    }
    const double lam = spectral_radius(qm, n, gam);
    double J[5][5];
    euler_jacobian(qc, n, gam, J);
    const double sg = side ? -1.0 : 1.0;  // neighbour side: -J(Q_j, n)
    for (int i = 0; i < 5; ++i)
      for (int j = 0; j < 5; ++j) D[i * 5 + j] += hs * ((side ? -J[i][j] : J[i][j]) + (i == j ? lam : 0.0));
    (void)sg;
  }
  for (int i = 0; i < 25; ++i) diag[(size_t)i * nc + c] = D[i];
  double X[25];
  if (!inv5(D, X)) {
    raise_dev(status, GKS_ERR_SINGULAR, (int)c);
    for (int i = 0; i < 25; ++i) X[i] = NAN;
  }
  for (int i = 0; i < 25; ++i) dinv[(size_t)i * nc + c] = X[i];
}

__global__ void k_dinv_only(int64_t nc, const double* __restrict__ diag, double* __restrict__ dinv, int* status) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= nc) return;
  double D[25], X[25];
  for (int i = 0; i < 25; ++i) D[i] = diag[(size_t)i * nc + c];
  if (!inv5(D, X)) {
    raise_dev(status, GKS_ERR_SINGULAR, (int)c);
    for (int i = 0; i < 25; ++i) X[i] = NAN;
  }
  for (int i = 0; i < 25; ++i) dinv[(size_t)i * nc + c] = X[i];
}

// ---------------------------------------------------------------------------
// K6/K7: block products, one thread per (cell,row), 32 cells per block
// ---------------------------------------------------------------------------
// mode bits: 1 = include diagonal (spmv), 2 = subtract from rhs b (t = b - ...),
//            4 = apply D^-1 to the result (cell-local via shared memory)
template <int MODE>
__global__ void __launch_bounds__(CELLS_PER_BLOCK * 5) k_block(int64_t nc, const int* __restrict__ rowptr,
                                                               const int* __restrict__ col,
                                                               const double* __restrict__ off,
                                                               const double* __restrict__ diag,
                                                               const double* __restrict__ dinv,
                                                               const double* __restrict__ x,
                                                               const double* __restrict__ b,
                                                               double* __restrict__ out,
                                                               double* __restrict__ out_pre, const int* gate) {
  __shared__ double sm[CELLS_PER_BLOCK * 5];
  if (gate && !*gate) return;
  const int lc = threadIdx.x / 5;
  const int row = threadIdx.x - lc * 5;
  const int64_t c = (int64_t)blockIdx.x * CELLS_PER_BLOCK + lc;
  double acc = 0.0;
  if (c < nc) {
    double o = 0.0;
    for (int e = rowptr[c]; e < rowptr[c + 1]; ++e) {
      const double* B = off + (int64_t)e * 25 + row * 5;
      const double* xc = x + (int64_t)col[e] * 5;
      o += B[0] * xc[0] + B[1] * xc[1] + B[2] * xc[2] + B[3] * xc[3] + B[4] * xc[4];
    }
    if (MODE & 1) {
      const double* Dr = diag + (size_t)row * 5 * nc + c;  // block-SoA: entry k at k * nc
      const double* xc = x + c * 5;
      const double d = Dr[0] * xc[0] + Dr[nc] * xc[1] + Dr[2 * nc] * xc[2] + Dr[3 * nc] * xc[3] + Dr[4 * nc] * xc[4];
      acc = d + o;
    } else {
      acc = o;
    }
    if (MODE & 2) acc = b[c * 5 + row] - acc;
    if (out_pre) out_pre[c * 5 + row] = acc;
  }
  if (MODE & 4) {
    sm[threadIdx.x] = acc;
    __syncthreads();
    if (c < nc) {
      const double* Xr = dinv + (size_t)row * 5 * nc + c;
      const double* t = sm + lc * 5;
      out[c * 5 + row] = Xr[0] * t[0] + Xr[nc] * t[1] + Xr[2 * nc] * t[2] + Xr[3 * nc] * t[3] + Xr[4 * nc] * t[4];
    }
  } else if (c < nc) {
    out[c * 5 + row] = acc;
  }
}

// z = D^-1 b
__global__ void k_dinv_apply(int64_t nc, const double* __restrict__ dinv, const double* __restrict__ b,
                             double* __restrict__ z, const int* gate) {
  if (gate && !*gate) return;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nc * 5) return;
  const int64_t c = t / 5;
  const int row = (int)(t - c * 5);
  const double* Xr = dinv + (size_t)row * 5 * nc + c;
  const double* bc = b + c * 5;
  z[t] = Xr[0] * bc[0] + Xr[nc] * bc[1] + Xr[2 * nc] * bc[2] + Xr[3 * nc] * bc[3] + Xr[4 * nc] * bc[4];
}

// ---------------------------------------------------------------------------
// GMRES scalar kernels (single thread): krylov.py:70-131
// ---------------------------------------------------------------------------
#define GH(i, jj) g->h[(i) * GM_MMAX + (jj)]

// header of the device GMRES state (only the scalars before `dots` need it)
__global__ void k_gm_init(GmresDev* g, int m, int restarts, double rtol, double atol) {
  char* p = (char*)g;
  for (size_t i = 0; i < offsetof(GmresDev, dots); ++i) p[i] = 0;
  g->m = m;
  g->restarts = restarts;
  g->rtol = rtol;
  g->atol = atol;
}

__global__ void k_status_init(int* st, int n) {
  for (int i = 0; i < n; ++i) st[4 * i] = 0, st[4 * i + 1] = 0x7fffffff, st[4 * i + 2] = 0, st[4 * i + 3] = 0;
}

__global__ void k_gm_cycle_begin(GmresDev* g) { g->notdone = !g->done; }

// cycle start: thread 0 decides (krylov.py:71-80), then the block clears the
// Hessenberg matrix and the rotated right-hand side (one thread doing 4k
// dependent stores was 11 us per cycle)
__global__ void k_gm_cycle_start(GmresDev* g, int cyc) {
  __shared__ int go;
  if (threadIdx.x == 0) {
    go = 0;
    if (!g->notdone) {
      g->active = 0;
    } else {
      g->matvecs += 1;
      const double beta = sqrt(g->beta2);
      g->beta = beta;
      if (!g->target_set) {
        g->target = g->rtol * beta + g->atol;
        g->target_set = 1;
      }
      g->j_used = 0;
      g->breakdown = 0;
      g->norms[cyc * (GM_MMAX + 1)] = beta;
      g->nnorms[cyc] = 1;
      if (beta == 0.0 || beta <= g->target) {
        g->done = 1;
        g->active = 0;
      } else if (!isfinite(beta)) {
        g->err = GKS_ERR_NONFINITE;
        g->done = 1;
        g->active = 0;
      } else {
        g->active = 1;
        go = 1;
      }
    }
  }
  __syncthreads();
  if (!go) return;
  for (int i = threadIdx.x; i < (GM_MMAX + 1) * GM_MMAX; i += blockDim.x) g->h[i] = 0.0;
  for (int i = threadIdx.x; i <= GM_MMAX; i += blockDim.x) g->gv[i] = 0.0;
  __syncthreads();
  if (threadIdx.x == 0) g->gv[0] = g->beta;
}

// after the first MGS pass of column j: Hessenberg column, re-orthogonalisation test
__device__ __forceinline__ void gm_reorth_check(GmresDev* g, int j) {
  if (!g->active) { g->reorth_gate = 0; return; }
  g->matvecs += 1;
  for (int i = 0; i <= j; ++i) GH(i, j) = g->dots[i];
  g->wscale = sqrt(g->wscale2);
  GH(j + 1, j) = sqrt(g->hnext2);
  g->reorth = GH(j + 1, j) < 0.5 * g->wscale ? 1 : 0;
  g->reorth_gate = g->reorth;
}

__global__ void k_gm_reorth_check(GmresDev* g, int j) { gm_reorth_check(g, j); }

// CGS2 column j: Hessenberg column = first + second projection; the norm is
// that of the twice-orthogonalised w (no conditional pass)
__global__ void k_gm_cgs_check(GmresDev* g, int j) {
  if (!g->active) {
    g->reorth_gate = 0;
    return;
  }
  g->matvecs += 1;
  for (int i = 0; i <= j; ++i) GH(i, j) = g->dots[i] + g->corr[i];
  g->wscale = sqrt(g->wscale2);
  GH(j + 1, j) = sqrt(g->hnext2);
  g->reorth = 0;
  g->reorth_gate = 0;
}

// Givens update of column j (krylov.py:107-124).  The column, the stored
// rotations and the right-hand side entries are read into registers before
// anything is written back: through one GmresDev* every load would otherwise
// wait for the previous store (a dependent L2 round trip per entry).
// scratch: 3 (GM_MMAX + 1) doubles of shared memory (one thread uses it)
__device__ __forceinline__ void gm_givens(GmresDev* g, int j, int cyc, double* scratch) {
  if (!g->active) return;
  double* hc = scratch;
  double* cs = scratch + GM_MMAX + 1;
  double* sn = scratch + 2 * (GM_MMAX + 1);
  for (int i = 0; i <= j + 1; ++i) hc[i] = GH(i, j);
  for (int i = 0; i < j; ++i) {
    cs[i] = g->cs[i];
    sn[i] = g->sn[i];
  }
  const double gj = g->gv[j];
  if (g->reorth) {
    for (int i = 0; i <= j; ++i) hc[i] += g->corr[i];
    hc[j + 1] = sqrt(g->hnext2);
  }
  if (!isfinite(hc[j + 1])) {
    if (g->reorth) GH(j + 1, j) = hc[j + 1];
    g->err = GKS_ERR_NONFINITE;
    g->done = 1;
    g->active = 0;
    g->j_used = 0;
    return;
  }
  for (int i = 0; i < j; ++i) {
    const double t = cs[i] * hc[i] + sn[i] * hc[i + 1];
    hc[i + 1] = -sn[i] * hc[i] + cs[i] * hc[i + 1];
    hc[i] = t;
  }
  const double denom = hypot(hc[j], hc[j + 1]);
  const double c = hc[j] / denom;
  const double sj = hc[j + 1] / denom;
  hc[j] = denom;
  for (int i = 0; i <= j + 1; ++i) GH(i, j) = hc[i];
  g->cs[j] = c;
  g->sn[j] = sj;
  g->gv[j + 1] = -sj * gj;
  g->gv[j] = c * gj;
  double* norms = g->norms + cyc * (GM_MMAX + 1);
  const double last = fabs(-sj * gj);
  const int nn = g->nnorms[cyc];
  norms[nn] = last;
  g->nnorms[cyc] = nn + 1;
  g->j_used = j + 1;
  if (hc[j + 1] <= 1e-13 * g->wscale) {
    g->breakdown = 1;
    g->breakdown_any = 1;
    g->active = 0;
  } else if (last <= fmax(1e-15 * norms[0], g->target)) {
    g->active = 0;
  } else {
    g->hdiv = hc[j + 1];
  }
}

__global__ void k_gm_givens(GmresDev* g, int j, int cyc) {
  __shared__ double scratch[3 * (GM_MMAX + 1)];
  gm_givens(g, j, cyc, scratch);
}

// Deterministic block sum (fixed shuffle tree per warp, then warp 0 over the
// warp partials); every thread gets the result.
__device__ __forceinline__ double block_sum_w(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  if (wid == 0) {
    v = lane < (int)(blockDim.x >> 5) ? red[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (lane == 0) red[32] = v;
  }
  __syncthreads();
  return red[32];
}

// Whole Arnoldi column j for small and medium systems in ONE kernel: the MGS
// pass (krylov.py:93-96), the conditional re-orthogonalisation (:97-104),
// the Givens update (:107-124) and v_{j+1} = w / h (:127).  Replaces
// 2 (j + 1) + 6 dependent launches per column (dot2, the axpy_dot chain,
// check, the gated second pass, givens, div): below ~400k unknowns the step
// is bound by that chain.  CL CTAs form one thread-block cluster; each keeps
// its slice of w in shared memory, block partials meet through distributed
// shared memory and are summed by every CTA in rank order (identical,
// deterministic totals everywhere); the scalar recurrences run on CTA 0 and
// reach the others through global memory across cluster barriers.  Same
// arithmetic per element as the multi-block kernels; the summation tree
// differs (deterministic for a given n).
// Partials alternate between two slots, so one cluster barrier per sum is
// enough: a CTA can only overwrite a slot after the next barrier, which every
// CTA reaches only once it has read that slot.
template <int CL>
__device__ __forceinline__ double cluster_sum(double v, double* red, double* part, int& slot) {
  const double b = block_sum_w(v, red);
  if (CL == 1) return b;
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  double* p = part + slot;
  slot ^= 1;
  if (threadIdx.x == 0) *p = b;
  cl.sync();
  double s = 0.0;
#pragma unroll
  for (int r = 0; r < CL; ++r) s += *cl.map_shared_rank(p, r);
  return s;
}

template <int CL>
__device__ __forceinline__ void cluster_barrier() {
  if (CL == 1) {
    __syncthreads();
  } else {
    cooperative_groups::this_cluster().sync();
  }
}

// w stays in registers: each of the 1024 threads owns up to AW elements of
// its CTA's slice (element t + u * 1024), so every pass issues all of a
// thread's loads at once (a strided loop left one L2 round trip in flight
// per iteration: 15 us per pass, measured).
static constexpr int AW = 16;

template <int CL>
__global__ void __launch_bounds__(1024, 1) k_gm_arnoldi(int n, int64_t ld, double* __restrict__ V,
                                                     const double* __restrict__ wg, GmresDev* g, int j, int cyc) {
  __shared__ double red[33];
  __shared__ double part[2];
  __shared__ double scratch[3 * (GM_MMAX + 1)];
  int slot = 0;
  if (!__ldcg(&g->active)) return;
  const int rank = CL == 1 ? 0 : (int)cooperative_groups::this_cluster().block_rank();
  const int chunk = (n + CL - 1) / CL;
  const int lo = rank * chunk, hi = min(n, lo + chunk), m = max(0, hi - lo);
  const bool lead = rank == 0 && threadIdx.x == 0;
  const int t = threadIdx.x;
  const double* V0 = V + lo;
  double w[AW];
  double s0 = 0.0, s1 = 0.0;
#pragma unroll
  for (int u = 0; u < AW; ++u) {
    const int i = t + u * 1024;
    w[u] = i < m ? wg[lo + i] : 0.0;
    const double v = i < m ? V0[i] : 0.0;
    s0 += w[u] * w[u];
    s1 += w[u] * v;
  }
  const double ww = cluster_sum<CL>(s0, red, part, slot);
  const double d0 = cluster_sum<CL>(s1, red, part, slot);
  if (lead) {
    g->wscale2 = ww;
    g->dots[0] = d0;
  }
  // pass 0: w -= h_i v_i, fused with the next dot (w . v_{i+1}, or w . w);
  // pass 1 (only on heavy cancellation): the same with the corrections.
  // Every thread carries h in a register (the reduction result), the lead
  // thread records it in the device GMRES state.
  for (int pass = 0; pass < 2; ++pass) {
    double* hv = pass == 0 ? g->dots : g->corr;
    double h = d0;
    if (pass == 1) {
      double s = 0.0;
#pragma unroll
      for (int u = 0; u < AW; ++u) {
        const int i = t + u * 1024;
        s += w[u] * (i < m ? V0[i] : 0.0);
      }
      h = cluster_sum<CL>(s, red, part, slot);
      if (lead) hv[0] = h;
    }
    for (int k = 0; k <= j; ++k) {
      const double* v = V + (int64_t)k * ld + lo;
      const double* nx = k < j ? V + (int64_t)(k + 1) * ld + lo : nullptr;
      double s = 0.0;
      if (nx) {
#pragma unroll
        for (int u = 0; u < AW; ++u) {
          const int i = t + u * 1024;
          const double vi = i < m ? __ldcg(v + i) : 0.0;
          const double xi = i < m ? __ldcg(nx + i) : 0.0;
          w[u] = w[u] - h * vi;
          s += w[u] * xi;
        }
      } else {
#pragma unroll
        for (int u = 0; u < AW; ++u) {
          const int i = t + u * 1024;
          const double vi = i < m ? __ldcg(v + i) : 0.0;
          w[u] = w[u] - h * vi;
          s += w[u] * w[u];
        }
      }
      const double r = cluster_sum<CL>(s, red, part, slot);
      if (lead) {
        if (k < j) hv[k + 1] = r;
        else g->hnext2 = r;
      }
      h = r;
    }
    if (pass == 0) {
      if (lead) gm_reorth_check(g, j);
      cluster_barrier<CL>();
      if (!__ldcg(&g->reorth)) break;
    }
  }
  if (lead) gm_givens(g, j, cyc, scratch);
  cluster_barrier<CL>();
  if (!__ldcg(&g->active)) return;
  const double d = __ldcg(&g->hdiv);
  double* vn = V + (int64_t)(j + 1) * ld + lo;
#pragma unroll
  for (int u = 0; u < AW; ++u) {
    const int i = t + u * 1024;
    if (i < m) vn[i] = w[u] / d;
  }
}

// back substitution (krylov.py:128-131) and cycle bookkeeping
// back substitution (krylov.py:128-131): the block copies the triangle and
// the rotated right-hand side into shared memory in parallel, one thread
// solves (a single thread walking the triangle in global memory waited on one
// L2 round trip per row: 10 us per cycle)
__global__ void k_gm_cycle_end(GmresDev* g, int cyc) {
  extern __shared__ double sh[];  // (m^2 + 2 m) doubles, m = g->m
  __shared__ int ju_s;
  const int mm = g->m;
  double* tri = sh;
  double* gv = sh + mm * mm;
  double* y = gv + mm;
  if (threadIdx.x == 0) {
    g->ny = 0;
    ju_s = (!g->notdone || g->err) ? 0 : g->j_used;
  }
  __syncthreads();
  if (!g->notdone) return;
  const int ju = ju_s;
  for (int t = threadIdx.x; t < ju * ju; t += blockDim.x) tri[t] = GH(t / ju, t % ju);
  for (int t = threadIdx.x; t < ju; t += blockDim.x) gv[t] = g->gv[t];
  __syncthreads();
  if (threadIdx.x != 0) return;
  for (int i = ju - 1; i >= 0; --i) {
    double dot = 0.0;
    for (int k = i + 1; k < ju; ++k) dot += tri[i * ju + k] * y[k];
    y[i] = (gv[i] - dot) / tri[i * ju + i];
  }
  for (int i = 0; i < ju; ++i) g->y[i] = y[i];
  g->ny = ju;
  g->ncycles = cyc + 1;
  const double last = g->norms[cyc * (GM_MMAX + 1) + g->nnorms[cyc] - 1];
  if (g->breakdown || last <= g->target) g->done = 1;
}
#undef GH

// x += y @ V[:ny]  (the combination is formed first, then added)
__global__ void k_gm_update_x(int64_t n, int64_t ld, double* __restrict__ x, const double* __restrict__ V,
                              const GmresDev* g) {
  const int ny = g->ny;
  if (ny == 0) return;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int k = 0; k < ny; ++k) s += g->y[k] * V[k * ld + i];
    x[i] = x[i] + s;
  }
}

// r = b - t
__global__ void k_sub(int64_t n, double* __restrict__ r, const double* __restrict__ b, const double* __restrict__ t,
                      const int* gate) {
  if (gate && !*gate) return;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    r[i] = b[i] - t[i];
}

// per-cell primitives for the matrix-free Roe products (jacobian.py:37-61 inputs)
__global__ void k_roe_prim(int64_t n, const double* __restrict__ q, double gm1, double* __restrict__ prim) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  const double rho = q[c * 5];
  const double vx = q[c * 5 + 1] / rho, vy = q[c * 5 + 2] / rho, vz = q[c * 5 + 3] / rho;
  const double ke = 0.5 * (vx * vx + vy * vy + vz * vz);
  const double p = gm1 * (q[c * 5 + 4] - rho * ke);
  double* P = prim + c * MF_REC;
  P[0] = vx; P[1] = vy; P[2] = vz; P[3] = (q[c * 5 + 4] + p) / rho; P[4] = ke; P[5] = 0.0;
}

// Same MODE bits as k_block, one thread per cell: the off-diagonal sum is
// recomputed entry by entry (in the CSR order of the stored path)
//   J(Q,n) x = (mx, v a + un x_m + n b, H a + un (b + x4)),
//   a = mx - un x0,  b = (gamma-1)(ke x0 - v.x_m + x4),  mx = n.x_m
// The face (n, S/2, lambda) and cell primitive records are padded to 6
// doubles and read as 16-byte vectors.  (Staging the block's D / D^-1
// records into shared memory by bulk copies, as the reconstruction does, was
// measured 2x slower here: each CTA then waits for its whole tile.)
static constexpr int MF_CELLS = 128;
#ifndef GKS_ROE_BATCH
#define GKS_ROE_BATCH 1
#endif

template <int MODE>
__global__ void __launch_bounds__(MF_CELLS) k_roe_mf(int64_t nc, const int* __restrict__ rowptr,
                                                     const int* __restrict__ col, const int* __restrict__ ent,
                                                     const double* __restrict__ fdat, const double* __restrict__ prim,
                                                     double gm1, const double* __restrict__ diag,
                                                     const double* __restrict__ dinv, const double* __restrict__ x,
                                                     const double* __restrict__ b, double* __restrict__ out,
                                                     double* __restrict__ out_pre, const int* gate) {
  if (gate && !*gate) return;
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= nc) return;
  double o[5] = {0, 0, 0, 0, 0};
  auto term = [&](int64_t j, int en, double2 f01, double2 f23, double2 f45, double2 p01, double2 p23, double2 p45,
                  const double* xj) {
    const double sg = (en & 1) ? -1.0 : 1.0;
    const double nx = f01.x, ny = f01.y, nz = f23.x, hs = f23.y, lam = f45.x;
    const double vx = p01.x, vy = p01.y, vz = p23.x, H = p23.y, ke = p45.x;
    const double x0 = xj[0], x1 = xj[1], x2 = xj[2], x3 = xj[3], x4 = xj[4];
    const double mx = nx * x1 + ny * x2 + nz * x3;
    const double un = nx * vx + ny * vy + nz * vz;
    const double a = mx - un * x0;
    const double bb = gm1 * (ke * x0 - (vx * x1 + vy * x2 + vz * x3) + x4);
    const double sh = sg * hs, lh = lam * hs;
    o[0] += sh * mx - lh * x0;
    o[1] += sh * (vx * a + un * x1 + nx * bb) - lh * x1;
    o[2] += sh * (vy * a + un * x2 + ny * bb) - lh * x2;
    o[3] += sh * (vz * a + un * x3 + nz * bb) - lh * x3;
    o[4] += sh * (H * a + un * (bb + x4)) - lh * x4;
  };
  const int e0 = rowptr[c], e1 = rowptr[c + 1];
  int e = e0;
#if GKS_ROE_BATCH
  // pairs of entries: both index loads, then both entries' face / cell /
  // x records in flight, then the terms in CSR order
  for (; e + 2 <= e1; e += 2) {
    const int64_t ja = col[e], jb = col[e + 1];
    const int ea = __ldg(ent + e), eb = __ldg(ent + e + 1);
    const double2* fa = (const double2*)(fdat + (int64_t)(ea >> 1) * MF_REC);
    const double2* fb = (const double2*)(fdat + (int64_t)(eb >> 1) * MF_REC);
    const double2* pa = (const double2*)(prim + ja * MF_REC);
    const double2* pb = (const double2*)(prim + jb * MF_REC);
    const double2 fa0 = __ldg(fa), fa1 = __ldg(fa + 1), fa2 = __ldg(fa + 2);
    const double2 fb0 = __ldg(fb), fb1 = __ldg(fb + 1), fb2 = __ldg(fb + 2);
    const double2 pa0 = __ldg(pa), pa1 = __ldg(pa + 1), pa2 = __ldg(pa + 2);
    const double2 pb0 = __ldg(pb), pb1 = __ldg(pb + 1), pb2 = __ldg(pb + 2);
    double xa[5], xb[5];
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      xa[k] = x[ja * 5 + k];
      xb[k] = x[jb * 5 + k];
    }
    term(ja, ea, fa0, fa1, fa2, pa0, pa1, pa2, xa);
    term(jb, eb, fb0, fb1, fb2, pb0, pb1, pb2, xb);
  }
#endif
  for (; e < e1; ++e) {
    const int64_t j = col[e];
    const int en = __ldg(ent + e);
    const double2* fd = (const double2*)(fdat + (int64_t)(en >> 1) * MF_REC);
    const double2* P = (const double2*)(prim + j * MF_REC);
    term(j, en, __ldg(fd), __ldg(fd + 1), __ldg(fd + 2), __ldg(P), __ldg(P + 1), __ldg(P + 2), x + j * 5);
  }
  double r[5];
#pragma unroll
  for (int i = 0; i < 5; ++i) {
    double acc = o[i];
    if (MODE & 1) {
      const double* Dr = diag + (size_t)i * 5 * nc + c;  // block-SoA: entry k at k * nc
      const double* xc = x + c * 5;
      acc = (Dr[0] * xc[0] + Dr[nc] * xc[1] + Dr[2 * nc] * xc[2] + Dr[3 * nc] * xc[3] + Dr[4 * nc] * xc[4]) + acc;
    }
    if (MODE & 2) acc = b[c * 5 + i] - acc;
    r[i] = acc;
    if (out_pre) out_pre[c * 5 + i] = acc;
  }
  if (MODE & 4) {
#pragma unroll
    for (int i = 0; i < 5; ++i) {
      const double* Xr = dinv + (size_t)i * 5 * nc + c;
      out[c * 5 + i] = Xr[0] * r[0] + Xr[nc] * r[1] + Xr[2 * nc] * r[2] + Xr[3 * nc] * r[3] + Xr[4 * nc] * r[4];
    }
  } else {
#pragma unroll
    for (int i = 0; i < 5; ++i) out[c * 5 + i] = r[i];
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
static int red_grid(int64_t n) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t want = (n + RB_THREADS - 1) / RB_THREADS;
  return (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)sms * 8));
}

int blocksys_alloc(BlockSys* A, int64_t nc, int64_t nnz, cudaStream_t stream) {
  A->nc = nc;
  A->nnz = nnz;
  A->stream = stream;
  GKS_CUDA(cudaMalloc(&A->rowptr, (nc + 1) * sizeof(int)));
  GKS_CUDA(cudaMalloc(&A->col, std::max<int64_t>(nnz, 1) * sizeof(int)));
  GKS_CUDA(cudaMalloc(&A->off, std::max<int64_t>(nnz, 1) * 25 * sizeof(double)));
  // (+64 B: the staged tile copies of k_roe_mf round the last chunk up to 16 B)
  GKS_CUDA(cudaMalloc(&A->diag, nc * 25 * sizeof(double) + 64));
  GKS_CUDA(cudaMalloc(&A->dinv, nc * 25 * sizeof(double) + 64));
  GKS_CUDA(cudaMalloc(&A->status, 4 * sizeof(int)));
  return GKS_OK;
}

void blocksys_free(BlockSys* A) {
  cudaFree(A->rowptr); cudaFree(A->col); cudaFree(A->off); cudaFree(A->diag); cudaFree(A->dinv);
  cudaFree(A->status);
  krylov_free(&A->ws);
}

static int64_t g_krylov_gen = 0;

void krylov_free(KrylovWS* W) {
  if (W->V) cudaFree(W->V);
  if (W->bufs) cudaFree(W->bufs);
  if (W->red.spart) cudaFree(W->red.spart);
  if (W->gpart[0]) cudaFree(W->gpart[0]);
  if (W->gpart[1]) cudaFree(W->gpart[1]);
  if (W->gall) cudaFree(W->gall);
  if (W->red.cnt) cudaFree(W->red.cnt);
  if (W->g) cudaFree(W->g);
  *W = KrylovWS{};
}

__global__ void k_red_init(int64_t ngrp_g, double* a, double* b) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < RED_SLOTS * ngrp_g;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double v = i < RED_MIN_SLOT * ngrp_g ? 0.0 : INFINITY;  // sums | the min slot
    a[i] = v;
    b[i] = v;
  }
}

// Reduction layout of a block system's rows in the global canonical order
// (gks_reduce.cuh); fails unless the rows are whole groups of that order.
static int red_setup(BlockSys* A, KrylovWS* W) {
  const int64_t nc = A->nc;
  const int64_t ncg = A->red_nc_global > 0 ? A->red_nc_global : nc;
  const int64_t first = A->red_nc_global > 0 ? A->red_cell_first : 0;
  const int G = red_group(ncg);
  const int64_t gcells = (int64_t)SEG_CELLS * G;
  if (first % gcells != 0 || (nc % gcells != 0 && first + nc != ncg) || first + nc > ncg) {
    set_error("owned cells [%lld, %lld) of %lld are not aligned to the %lld-cell reduction groups",
              (long long)first, (long long)(first + nc), (long long)ncg, (long long)gcells);
    return GKS_ERR_BAD_ARG;
  }
  RedDev& R = W->red;
  R.nseg = (nc + SEG_CELLS - 1) / SEG_CELLS;
  R.G = G;
  R.ngrp = (R.nseg + G - 1) / G;
  const int64_t nseg_g = (ncg + SEG_CELLS - 1) / SEG_CELLS;
  R.ngrp_g = (nseg_g + G - 1) / G;
  R.grp_first = first / gcells;
  R.finalize = A->comm ? 0 : 1;
  // (room for the CGS2 multi-dots: up to RED_MAXC_MD components)
  GKS_CUDA(cudaMalloc(&R.spart, (size_t)RED_SLOTS * R.nseg * sizeof(double)));
  for (int k = 0; k < 2; ++k) GKS_CUDA(cudaMalloc(&W->gpart[k], (size_t)RED_SLOTS * R.ngrp_g * sizeof(double)));
  GKS_CUDA(cudaMalloc(&W->gall, (size_t)RED_SLOTS * R.ngrp_g * sizeof(double)));
  GKS_CUDA(cudaMalloc(&R.cnt, (size_t)(R.ngrp + 1) * sizeof(unsigned)));
  GKS_CUDA(cudaMemset(R.cnt, 0, (size_t)(R.ngrp + 1) * sizeof(unsigned)));
  k_red_init<<<blocks_for(RED_SLOTS * R.ngrp_g, 256), 256>>>(R.ngrp_g, W->gpart[0], W->gpart[1]);
  GKS_CUDA(cudaGetLastError());
  GKS_CUDA(cudaDeviceSynchronize());
  R.gpart = W->gpart[0];
  return GKS_OK;
}

int krylov_ensure(BlockSys* A, int m) {
  KrylovWS* W = &A->ws;
  const int64_t n = A->nc * 5;
  int64_t ld = 5 * std::max<int64_t>(A->n_ext, A->nc);
  if (ld < n) ld = n;
  if (W->V && W->n == n && W->ld == ld && W->m >= m) return GKS_OK;
  m = std::max(m, W->m);
  krylov_free(W);
  W->n = n;
  W->ld = ld;
  W->m = m;
  W->gen = ++g_krylov_gen;  // captured step graphs holding the old buffers are stale
  GKS_CUDA(cudaMalloc(&W->V, (size_t)(m + 1) * ld * sizeof(double)));
  GKS_CUDA(cudaMemset(W->V, 0, (size_t)(m + 1) * ld * sizeof(double)));
  GKS_CUDA(cudaMalloc(&W->bufs, (size_t)6 * ld * sizeof(double)));
  GKS_CUDA(cudaMemset(W->bufs, 0, (size_t)6 * ld * sizeof(double)));
  W->w = W->bufs;
  W->r = W->bufs + ld;
  W->t = W->bufs + 2 * ld;
  W->z = W->bufs + 3 * ld;
  W->b = W->bufs + 4 * ld;
  W->x = W->bufs + 5 * ld;
  W->grid = red_grid(n);
  GKS_CUDA(cudaMalloc(&W->g, sizeof(GmresDev)));
  return red_setup(A, W);
}

static inline int cblocks(int64_t nc) { return (int)((nc + CELLS_PER_BLOCK - 1) / CELLS_PER_BLOCK); }

static inline void halo(BlockSys* A, const double* x) {
  if (A->halo_x) A->halo_x(const_cast<double*>(x));
}

// one block product of kind MODE: stored blocks (cell x row threads) or the
// matrix-free Roe form (one thread per cell)
template <int MODE>
static void block_product(BlockSys* A, const double* x, const double* b, double* out, double* pre, const int* gate) {
  const int kc = (MODE == 6) ? KC_JACOBI : KC_SPMV;
  if (A->mf) {
    GKS_LAUNCH(kc, k_roe_mf<MODE>, blocks_for(A->nc, MF_CELLS), MF_CELLS, 0, A->stream, A->nc, A->rowptr, A->col,
               A->ent, A->fdat, A->prim, A->gm1, A->diag, A->dinv, x, b, out, pre, gate);
  } else {
    GKS_LAUNCH(kc, k_block<MODE>, cblocks(A->nc), CELLS_PER_BLOCK * 5, 0, A->stream, A->nc, A->rowptr, A->col, A->off,
               A->diag, A->dinv, x, b, out, pre, gate);
  }
}

// y = A x  (diag + off)
void bs_spmv(BlockSys* A, const double* x, double* y, const int* gate) {
  halo(A, x);
  block_product<1>(A, x, nullptr, y, nullptr, gate);
}

// y = (L+U) x
void bs_offdiag(BlockSys* A, const double* x, double* y, const int* gate) {
  halo(A, x);
  block_product<0>(A, x, nullptr, y, nullptr, gate);
}

// z = P^-1 b : z0 = D^-1 b, then kmax sweeps z <- D^-1 (b - (L+U) z)  (krylov.py:24-34)
// uses tmp as the ping-pong buffer; result in z
void bs_jacobi(BlockSys* A, const double* b, double* z, double* tmp, int kmax, const int* gate) {
  const int64_t n5 = A->nc * 5;
  GKS_LAUNCH(KC_VEC, k_dinv_apply, blocks_for(n5, 256), 256, 0, A->stream, A->nc, A->dinv, b, z, gate);
  double* cur = z;
  double* nxt = tmp;
  for (int k = 0; k < kmax; ++k) {
    halo(A, cur);
    block_product<6>(A, cur, b, nxt, nullptr, gate);
    std::swap(cur, nxt);
  }
  if (cur != z) {
    GKS_LAUNCH(KC_VEC, k_copy, red_grid(n5), RB_THREADS, 0, A->stream, n5, z, cur);
  }
}

// w = P^-1 A v : fused spmv + first D^-1, then sweeps
void bs_prec_matvec(BlockSys* A, const double* v, double* w, double* t, double* tmp, int kmax, const int* gate) {
  halo(A, v);
  block_product<5>(A, v, nullptr, w, t, gate);
  double* cur = w;
  double* nxt = tmp;
  for (int k = 0; k < kmax; ++k) {
    halo(A, cur);
    block_product<6>(A, cur, t, nxt, nullptr, gate);
    std::swap(cur, nxt);
  }
  if (cur != w) {
    const int64_t n5 = A->nc * 5;
    GKS_LAUNCH(KC_VEC, k_copy, red_grid(n5), RB_THREADS, 0, A->stream, n5, w, cur);
  }
}

// Reductions over the owned rows (n = 5 * A->nc entries), partition-invariant
// (gks_reduce.cuh).  Multi-rank: each launch leaves this rank's group
// partials, the communicator exchanges them and folds the total.
int dot2(BlockSys* A, int64_t n, const double* a, const double* b, const double* c, const double* d, double* o0,
         double* o1, const int* gate) {
  KrylovWS* W = &A->ws;
  W->red.gpart = A->comm ? comm_red_buffer(A->comm, W) : W->gpart[0];
  RedOut out;
  out.o[0] = o0;
  out.o[1] = o1;
  GKS_LAUNCH(KC_REDUCE, k_dot2, (int)W->red.nseg, RED_T, 0, A->stream, n, a, b, c, d, W->red, out, gate);
  if (A->comm) return comm_red_final(A->comm, W, c ? 2 : 1, 0, out, gate, A->stream);
  return GKS_OK;
}

int axpy_dot(BlockSys* A, int64_t n, double* w, const double* v, const double* coef, const double* nxt, double* o,
             const int* gate) {
  KrylovWS* W = &A->ws;
  W->red.gpart = A->comm ? comm_red_buffer(A->comm, W) : W->gpart[0];
  RedOut out;
  out.o[0] = o;
  GKS_LAUNCH(KC_REDUCE, k_axpy_dot, (int)W->red.nseg, RED_T, 0, A->stream, n, w, v, coef, nxt, W->red, out, gate);
  if (A->comm) return comm_red_final(A->comm, W, 1, 0, out, gate, A->stream);
  return GKS_OK;
}

// step norms (stepping.py:288-290): sum |res_rho|, sum res^2, #bad, min dt
__global__ void __launch_bounds__(RED_T) k_stats(int64_t nc, const double* __restrict__ res,
                                                 const double* __restrict__ dt, const int8_t* __restrict__ bad,
                                                 RedDev R, RedOut out) {
  __shared__ double sm[9];
  const int64_t base = (int64_t)blockIdx.x * SEG_CELLS;
  const int64_t len = min((int64_t)SEG_CELLS, nc - base);
  double v[4];
  red_lanes<3, 1>(len, [&](int64_t i, double* o) {
    const double* r = res + (base + i) * 5;
    o[0] = fabs(r[0]);
    double s2 = __dmul_rn(r[0], r[0]);
#pragma unroll
    for (int k = 1; k < 5; ++k) s2 = __dadd_rn(s2, __dmul_rn(r[k], r[k]));
    o[1] = s2;
    o[2] = bad[base + i] ? 1.0 : 0.0;
    o[3] = dt[base + i];
  }, v);
  red_finish<3, 1>(R, v, out, sm);
}

int step_stats(BlockSys* A, int64_t nc, const double* res, const double* dt, const int8_t* bad, DevScalars* sc) {
  KrylovWS* W = &A->ws;
  W->red.gpart = A->comm ? comm_red_buffer(A->comm, W) : W->gpart[0];
  RedOut out;
  for (int k = 0; k < 4; ++k) out.o[k] = &sc->stat[k];
  GKS_LAUNCH(KC_UPDATE, k_stats, (int)W->red.nseg, RED_T, 0, A->stream, nc, res, dt, bad, W->red, out);
  if (A->comm) return comm_red_final(A->comm, W, 3, 1, out, nullptr, A->stream);
  return GKS_OK;
}

// Cluster size of the fused Arnoldi-column kernel for n unknowns: slices of
// <= 16k doubles (16 registers x 1024 threads) per CTA, clusters of up to 16
// CTAs (non-portable size, checked against the device once); 0 = use the
// multi-block chain.
static constexpr int kArnoldiSlice = AW * 1024;

template <int CL>
static int arnoldi_attr(size_t smem) {
  static bool ok = [smem] {
    if (CL > 8 && cudaFuncSetAttribute(k_gm_arnoldi<CL>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) !=
                      cudaSuccess)
      return false;
    if (CL == 1) return true;
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(CL);
    cfg.blockDim = dim3(1024);
    cfg.dynamicSmemBytes = 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int nclusters = 0;
    return cudaOccupancyMaxActiveClusters(&nclusters, k_gm_arnoldi<CL>, &cfg) == cudaSuccess && nclusters > 0;
  }();
  (void)smem;
  cudaGetLastError();
  return ok ? CL : 0;
}

// Preferred slice per CTA (GKS_ARNOLDI_SLICE).  More CTAs spread the vector
// passes over more SMs, at one cluster barrier per sum; measured, the
// fewest CTAs win (3k-cell cavity: 1 CTA 1.62 ms/step, 4 CTAs 1.89).
static int64_t arnoldi_target_slice() {
  static const int64_t v = [] {
    const char* e = getenv("GKS_ARNOLDI_SLICE");
    const int64_t x = e ? atoll(e) : kArnoldiSlice;
    return std::min<int64_t>(std::max<int64_t>(x, 1024), kArnoldiSlice);
  }();
  return v;
}

static int arnoldi_cluster(int64_t n) {
  if (n > 16 * (int64_t)kArnoldiSlice) return 0;
  const int64_t slice = arnoldi_target_slice();
  const int64_t need = std::max<int64_t>(std::min<int64_t>((n + slice - 1) / slice, 16),
                                         (n + kArnoldiSlice - 1) / kArnoldiSlice);
  if (need <= 1) return arnoldi_attr<1>(0);
  if (need <= 2) return arnoldi_attr<2>(0);
  if (need <= 4) return arnoldi_attr<4>(0);
  if (need <= 8) return arnoldi_attr<8>(0);
  if (need <= 16) return arnoldi_attr<16>(0);
  return 0;
}

template <int CL>
static int launch_arnoldi_cl(cudaStream_t s, int n, int64_t ld, double* V, const double* w, GmresDev* g, int j,
                             int cyc) {
  const size_t smem = 0;
  if (CL == 1) {
    GKS_LAUNCH(KC_REDUCE, k_gm_arnoldi<1>, 1, 1024, smem, s, n, ld, V, w, g, j, cyc);
    return GKS_OK;
  }
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(CL);
  cfg.blockDim = dim3(1024);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaEvent_t pa = g_prof_on ? prof_begin(s) : nullptr;
  GKS_CUDA(cudaLaunchKernelEx(&cfg, k_gm_arnoldi<CL>, n, ld, V, w, g, j, cyc));
  count_launch(1);
  if (pa) prof_end(KC_REDUCE, s, pa);
  return GKS_OK;
}

static int launch_arnoldi(int cl, cudaStream_t s, int n, int64_t ld, double* V, const double* w, GmresDev* g, int j,
                          int cyc) {
  switch (cl) {
    case 1: return launch_arnoldi_cl<1>(s, n, ld, V, w, g, j, cyc);
    case 2: return launch_arnoldi_cl<2>(s, n, ld, V, w, g, j, cyc);
    case 4: return launch_arnoldi_cl<4>(s, n, ld, V, w, g, j, cyc);
    case 8: return launch_arnoldi_cl<8>(s, n, ld, V, w, g, j, cyc);
    default: return launch_arnoldi_cl<16>(s, n, ld, V, w, g, j, cyc);
  }
}

// Restarted left-preconditioned GMRES (krylov.py:55-140) on device vectors;
// x_dev receives the solution.  matvec == nullptr: A v is the block spmv.
// gmres_enqueue only launches (no host synchronisation, so a whole implicit
// step can be captured in a CUDA graph); gmres_collect reads the device
// state back.  check_dinv: refuse a singular Jacobi preconditioner on the
// host (needs a synchronised Jacobian assembly; the graph path checks the
// Jacobian's status word after the step instead).
int gmres_enqueue(BlockSys* A, const double* b_dev, double* x_dev, const GmresParams& P, const MatvecFn* matvec,
                  bool check_dinv) {
  const int64_t n = A->nc * 5;
  const int m = P.m;
  if (m < 1 || m > GM_MMAX || P.restarts < 1 || P.restarts > GM_RMAX || P.kmax < 0) {
    set_error("gmres: krylov_dim must be in [1, %d], restarts in [1, %d]", GM_MMAX, GM_RMAX);
    return GKS_ERR_BAD_ARG;
  }
  if (check_dinv && !A->dinv_ok) {
    set_error("singular diagonal block in Jacobi preconditioner");
    return GKS_ERR_SINGULAR;
  }
  KrylovWS* W = &A->ws;
  int rc = krylov_ensure(A, m);
  if (rc) return rc;
  const int64_t ld = W->ld;
  cudaStream_t s = A->stream;
  GmresDev* g = W->g;
  GKS_LAUNCH(KC_SCALAR, k_gm_init, 1, 1, 0, s, g, m, P.restarts, P.rtol, P.atol);
  {
    // Keep the MGS working vector w resident in L2 (persisting access window
    // on the stream, captured into the step graph) when it fits the
    // persisting carve-out: the axpy/dot chain then streams only the basis
    // vectors from HBM (1.57M cells: 48 -> 38 us per pass, C1 Roe step -9 %).
    // A partial window over a larger w thrashed L2 (9.7M cells: +38 %), so
    // larger systems keep the default policy.  GKS_L2_PERSIST=0 disables.
    static const bool persist = [] {
      const char* e = getenv("GKS_L2_PERSIST");
      return !(e && e[0] == '0');
    }();
    // (an earlier launch failure must surface here, not be cleared below)
    GKS_CUDA(cudaPeekAtLastError());
    int dev = 0, maxp = 0, maxw = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, dev);
    cudaDeviceGetAttribute(&maxw, cudaDevAttrMaxAccessPolicyWindowSize, dev);
    const size_t bytes = (size_t)n * sizeof(double);
    cudaStreamAttrValue at = {};
    if (persist && bytes <= (size_t)maxp && bytes <= (size_t)maxw) {
      if (cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, bytes) != cudaSuccess) cudaGetLastError();
      at.accessPolicyWindow.base_ptr = W->w;
      at.accessPolicyWindow.num_bytes = bytes;
      at.accessPolicyWindow.hitRatio = 1.0f;
      at.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
      at.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    }
    // the window is a hint: a refused attribute only clears its own error
    if (cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &at) != cudaSuccess)  // (num_bytes 0: no window)
      cudaGetLastError();
  }
  GKS_CUDA(cudaMemsetAsync(x_dev, 0, ld * sizeof(double), s));
  const int* act = &g->active;
  const int* notdone = &g->notdone;
  const int* rgate = &g->reorth_gate;
  const int kmax = P.kmax;
  const int grid = red_grid(n);
  // single-rank systems below ~400k unknowns: one (cluster) kernel per
  // Arnoldi column, w in shared memory (k_gm_arnoldi)
  const char* small_env = getenv("GKS_GMRES_SMALL");
  int cl = 0;  // cluster size of the fused column kernel, 0 = multi-block chain
  if (P.ortho == 1 && m > CGS_MAXV) {
    set_error("gmres: ortho=cgs2 supports krylov_dim <= %d", CGS_MAXV);
    return GKS_ERR_BAD_ARG;
  }
  if (!A->comm && !A->canonical && P.ortho == 0 && !(small_env && small_env[0] == '0')) cl = arnoldi_cluster(n);
  auto Av = [&](const double* v, double* dst, const int* gate) -> int {
    if (matvec) return (*matvec)(v, dst, gate);
    bs_spmv(A, v, dst, gate);
    return GKS_OK;
  };
  for (int cyc = 0; cyc < P.restarts; ++cyc) {
    GKS_LAUNCH(KC_SCALAR, k_gm_cycle_begin, 1, 1, 0, s, g);
    // r = b - A x ; rh = P r ; beta = ||rh||
    TRY_GM(Av(x_dev, W->t, notdone));
    GKS_LAUNCH(KC_VEC, k_sub, grid, RB_THREADS, 0, s, n, W->r, b_dev, W->t, notdone);
    bs_jacobi(A, W->r, W->z, W->w, kmax, notdone);
    TRY_GM(dot2(A, n, W->z, W->z, nullptr, nullptr, &g->beta2, nullptr, notdone));
    GKS_LAUNCH(KC_SCALAR, k_gm_cycle_start, 1, 256, 0, s, g, cyc);
    GKS_LAUNCH(KC_VEC, k_div, grid, RB_THREADS, 0, s, n, W->V, W->z, &g->beta, act);
    for (int j = 0; j < m; ++j) {
      const double* vj = W->V + (int64_t)j * ld;
      // w = P^-1 A v_j
      if (matvec) {
        TRY_GM(Av(vj, W->t, act));
        bs_jacobi(A, W->t, W->w, W->r, kmax, act);
      } else {
        bs_prec_matvec(A, vj, W->w, W->t, W->r, kmax, act);
      }
      if (cl) {
        // the whole column in one kernel (k_gm_arnoldi)
        TRY_GM(launch_arnoldi(cl, s, (int)n, ld, W->V, W->w, g, j, cyc));
        continue;
      }
      if (P.ortho == 1) {
        // CGS2: three fused passes, three reductions per column (instead of
        // j + 2 sequential MGS dots plus the conditional second sweep)
        RedOutN o1, o2, o3;
        o1.base = g->dots;
        o1.last = &g->wscale2;
        o2.base = g->corr;
        o2.last = &g->hnext2;
        o3.last = &g->hnext2;
        TRY_GM(cgs_pass(A, 1, j + 1, n, ld, W->w, nullptr, o1, act));
        TRY_GM(cgs_pass(A, 2, j + 1, n, ld, W->w, g->dots, o2, act));
        TRY_GM(cgs_pass(A, 3, j + 1, n, ld, W->w, g->corr, o3, act));
        GKS_LAUNCH(KC_SCALAR, k_gm_cgs_check, 1, 1, 0, s, g, j);
        GKS_LAUNCH(KC_SCALAR, k_gm_givens, 1, 1, 0, s, g, j, cyc);
        GKS_LAUNCH(KC_VEC, k_div, grid, RB_THREADS, 0, s, n, W->V + (int64_t)(j + 1) * ld, W->w, &g->hdiv, act);
        continue;
      }
      // ||w||^2 and w.v_0 in one pass, then fused axpy + next dot (MGS)
      TRY_GM(dot2(A, n, W->w, W->w, W->w, W->V, &g->wscale2, &g->dots[0], act));
      for (int i = 0; i <= j; ++i) {
        const double* nxt = i < j ? W->V + (int64_t)(i + 1) * ld : nullptr;
        double* dst = i < j ? &g->dots[i + 1] : &g->hnext2;
        TRY_GM(axpy_dot(A, n, W->w, W->V + (int64_t)i * ld, &g->dots[i], nxt, dst, act));
      }
      GKS_LAUNCH(KC_SCALAR, k_gm_reorth_check, 1, 1, 0, s, g, j);
      // conditional second pass (krylov.py:97-104)
      TRY_GM(dot2(A, n, W->w, W->V, nullptr, nullptr, &g->corr[0], nullptr, rgate));
      for (int i = 0; i <= j; ++i) {
        const double* nxt = i < j ? W->V + (int64_t)(i + 1) * ld : nullptr;
        double* dst = i < j ? &g->corr[i + 1] : &g->hnext2;
        TRY_GM(axpy_dot(A, n, W->w, W->V + (int64_t)i * ld, &g->corr[i], nxt, dst, rgate));
      }
      GKS_LAUNCH(KC_SCALAR, k_gm_givens, 1, 1, 0, s, g, j, cyc);
      GKS_LAUNCH(KC_VEC, k_div, grid, RB_THREADS, 0, s, n, W->V + (int64_t)(j + 1) * ld, W->w, &g->hdiv, act);
    }
    GKS_LAUNCH(KC_SCALAR, k_gm_cycle_end, 1, 128, (size_t)(m * m + 2 * m) * sizeof(double), s, g, cyc);
    GKS_LAUNCH(KC_VEC, k_gm_update_x, grid, RB_THREADS, 0, s, n, ld, x_dev, W->V, g);
    if (P.check_ortho) {
      // Gram matrix of the cycle's basis (krylov.py:778-782), host-side check
      // (synchronises: never used inside a captured step)
      GmresDev gh;
      GKS_CUDA(cudaMemcpyAsync(&gh, g, offsetof(GmresDev, dots), cudaMemcpyDeviceToHost, s));
      GKS_CUDA(cudaStreamSynchronize(s));
      const int ju = gh.ny;
      if (ju > 1) {
        std::vector<double> hv((size_t)ju * ld);
        GKS_CUDA(cudaMemcpy(hv.data(), W->V, hv.size() * sizeof(double), cudaMemcpyDeviceToHost));
        for (int a = 0; a < ju; ++a)
          for (int b = 0; b < ju; ++b) {
            double acc = 0.0;
            for (int64_t i = 0; i < n; ++i) acc += hv[a * ld + i] * hv[b * ld + i];
            W->ortho_error = std::max(W->ortho_error, fabs(acc - (a == b ? 1.0 : 0.0)));
          }
      }
    }
  }
  GKS_CUDA(cudaGetLastError());
  return GKS_OK;
}

// Fill `out` from a host copy of the device GMRES state; returns its error.
int gmres_result(const GmresDev* gh, GmresHost* out) {
  if (out) {
    out->ncycles = gh->ncycles;
    out->breakdown = gh->breakdown_any;
    out->err = gh->err;
    out->matvecs = gh->matvecs;
    for (int c = 0; c < gh->ncycles; ++c) {
      out->cycle_len[c] = gh->nnorms[c];
      for (int k = 0; k < gh->nnorms[c]; ++k) out->norms[c * (GM_MMAX + 1) + k] = gh->norms[c * (GM_MMAX + 1) + k];
    }
  }
  if (gh->err) {
    set_error(gh->err == GKS_ERR_NONFINITE ? "GMRES diverged: non-finite Arnoldi vector" : "GMRES failed (%d)",
              gh->err);
    return gh->err;
  }
  return GKS_OK;
}

int gmres_device(BlockSys* A, const double* b_dev, double* x_dev, const GmresParams& P, GmresHost* out,
                 const MatvecFn* matvec) {
  A->ws.ortho_error = 0.0;
  TRY_GM(gmres_enqueue(A, b_dev, x_dev, P, matvec, true));
  GmresDev* gh = new GmresDev;
  cudaError_t e = cudaMemcpyAsync(gh, A->ws.g, sizeof(GmresDev), cudaMemcpyDeviceToHost, A->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(A->stream);
  if (e != cudaSuccess) {
    delete gh;
    return cuda_fail(e, "gmres collect", __FILE__, __LINE__);
  }
  if (out) out->ortho_error = A->ws.ortho_error;
  const int ret = gmres_result(gh, out);
  delete gh;
  return ret;
}

// ---------------------------------------------------------------------------
// Jacobian assembly on the handle's mesh
// ---------------------------------------------------------------------------
// want_blocks: also store the off-diagonal 5x5 blocks (the matrix-free
// products of a step need only the per-face records; the API assembly
// exports the blocks)
int jacobian_enqueue(Handle* H, BlockSys* A, const double* ghosts_dev, bool want_blocks) {
  GKS_LAUNCH(KC_SCALAR, k_status_init, 1, 1, 0, H->stream, A->status, 1);
  if (H->nfi)
    GKS_LAUNCH(KC_JAC_FACE, k_jac_faces, blocks_for(H->nfi, 128), 128, 0, H->stream, H->nfi, H->interior_faces, H->f_own, H->f_nbr,
                                                                 H->f_normal, H->f_area, H->q, H->face_slot,
                                                                 H->gamma, (want_blocks || !A->mf) ? A->off : nullptr,
                                                                 A->fdat);
  if (A->mf)
    GKS_LAUNCH(KC_JAC_FACE, k_roe_prim, blocks_for(H->n_recon, 128), 128, 0, H->stream, H->n_recon, H->q,
               H->gamma - 1.0, A->prim);
  GKS_LAUNCH(KC_JAC_DIAG, k_jac_diag, blocks_for(H->n_owned, 128), 128, 0, H->stream, H->n_owned, H->cjd_start,
             H->cjd, H->f_own, H->f_nbr, H->f_normal, H->f_area, H->bidx, ghosts_dev, H->q, H->vol, H->dt, H->gamma,
             A->diag, A->dinv, A->status);
  GKS_CUDA(cudaGetLastError());
  return GKS_OK;
}

int jacobian_assemble(Handle* H, BlockSys* A, const double* ghosts_dev) {
  TRY_GM(jacobian_enqueue(H, A, ghosts_dev, true));
  int st[4];
  GKS_CUDA(cudaMemcpyAsync(st, A->status, sizeof(st), cudaMemcpyDeviceToHost, H->stream));
  GKS_CUDA(cudaStreamSynchronize(H->stream));
  A->dinv_ok = st[0] == 0;
  return GKS_OK;
}

int blocksys_invert_diag(BlockSys* A) {
  const int st0[4] = {0, 0x7fffffff, 0, 0};
  GKS_CUDA(cudaMemcpyAsync(A->status, st0, sizeof(st0), cudaMemcpyHostToDevice, A->stream));
  GKS_LAUNCH(KC_JAC_DIAG, k_dinv_only, blocks_for(A->nc, 128), 128, 0, A->stream, A->nc, A->diag, A->dinv, A->status);
  int st[4];
  GKS_CUDA(cudaMemcpyAsync(st, A->status, sizeof(st), cudaMemcpyDeviceToHost, A->stream));
  GKS_CUDA(cudaStreamSynchronize(A->stream));
  A->dinv_ok = st[0] == 0;
  return GKS_OK;
}

// ---------------------------------------------------------------------------
// K9: state update, validity mask and step norms (stepping.py:264-290)
// ---------------------------------------------------------------------------
__global__ void k_update(int64_t nc, const double* __restrict__ q, const double* __restrict__ dq,
                         double* __restrict__ qn, int8_t* __restrict__ bad) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= nc) return;
  double v[5];
  bool fin = true;
  for (int k = 0; k < 5; ++k) {
    v[k] = q[c * 5 + k] + dq[c * 5 + k];
    qn[c * 5 + k] = v[k];
    fin = fin && isfinite(v[k]);
  }
  const double rho = v[0];
  const double e = v[4] - 0.5 * (v[1] * v[1] + v[2] * v[2] + v[3] * v[3]) / rho;
  bad[c] = (rho <= 0.0) || (e <= 0.0) || !fin;
}

__global__ void k_halve_dt(int64_t nc, const int8_t* __restrict__ bad, double* __restrict__ dt) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c < nc && bad[c]) dt[c] = 0.5 * dt[c];
}

// ---------------------------------------------------------------------------
// matrix-free operator (north-star option): A v = V/dt v - (L(Q + s v) - L(Q)) / s
// (stepping.py:298-313 for the directional derivative)
// ---------------------------------------------------------------------------
__global__ void k_sigma(const double* vv_qq, double* sigma, double* out_zero_flag) {
  const double vn = sqrt(vv_qq[0]);
  const double qn = sqrt(vv_qq[1]);
  *sigma = vn == 0.0 ? 0.0 : sqrt(2.220446049250313e-16) * (1.0 + qn) / vn;
  if (out_zero_flag) *out_zero_flag = vn == 0.0 ? 1.0 : 0.0;
}

__global__ void k_perturb(int64_t n, const double* __restrict__ q, const double* __restrict__ v,
                          const double* sigma, double* __restrict__ out, const int* gate) {
  if (gate && !*gate) return;
  const double s = *sigma;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = q[i] + s * v[i];
}

}  // namespace gks

