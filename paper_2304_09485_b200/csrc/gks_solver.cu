// Solver handle + residual pipeline (K1 local dt, K2 reconstruction,
// K3 fused face flux, K4 deterministic cell assembly).
//
// Reference path (gks3d, /root/reference/pkg/src/gks3d):
//   Solver.local_time_step   stepping.py:135-157
//   Solver.residual          stepping.py:212-238
//     _reconstruct           stepping.py:161-178  (recon.py:276-314, hweno.py:139-169,
//                                                   boundary.py:66-171)
//     interface_batch        stepping.py:187-208  (flux.py:69-107, 211-243)
//     evolve_flux / scatter  stepping.py:219-228  (flux.py:162-179)
//     compact gradients      stepping.py:230-237  (flux.py:182-188, hweno.py:172-194)
//
// Data layout in HBM (AoS per entity so one cell's / face's record is one
// contiguous run): q (nc,5), grad (nc,3,5), coefficients (nc,9,5), face
// contributions (nfq,5).  Assembly is a cell-centric gather over a CSR list
// in the reference's np.add.at order (owner entries, then neighbour
// entries, ascending), so results are deterministic and atomics-free.
#include <stdlib.h>

#include <algorithm>
#include <numeric>
#include <string>
#include <vector>

#include "gks_solver.cuh"
#include "gks_stage.cuh"

namespace gks {

static constexpr int TPB = 128;

#ifndef GKS_FACE_TAU
#define GKS_FACE_TAU 1  // interface_flux_t TAU mode of the inviscid face kernel (gks_kinetic.cuh)
#endif
// L2 prefetch of the neighbour side's records at kernel start: 1 % faster
// at 168 registers (round 1), 0.4 % slower at 255 (both sides overlapped):
// off
#ifndef GKS_FACE_PREFETCH
#define GKS_FACE_PREFETCH 0
#endif

// ---------------------------------------------------------------------------
// K1: local time step
// ---------------------------------------------------------------------------
__global__ void k_local_dt(int64_t nc, const double* __restrict__ q, const int* __restrict__ cdt_start,
                           const int* __restrict__ cdt, const double* __restrict__ f_normal,
                           const double* __restrict__ f_area, const double* __restrict__ vol, int viscous,
                           double mu, double cfl, KinConst kc, double* __restrict__ dt, int* status) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= nc) return;
  double qc[5], w[5];
  for (int k = 0; k < 5; ++k) qc[k] = q[c * 5 + k];
  if (!cons_to_prim(qc, kc, w)) {
    raise_dev(status, GKS_ERR_UNPHYSICAL, (int)c);
    return;
  }
  const double a = sqrt(kc.gamma / (2.0 * w[4]));
  const double V = vol[c];
  double speed = 0.0;
  for (int e = cdt_start[c]; e < cdt_start[c + 1]; ++e) {
    const int f = cdt[e] >> 1;
    const double* n = f_normal + 3 * f;
    double un = w[1] * n[0];
    un += w[2] * n[1];
    un += w[3] * n[2];
    const double S = f_area[f];
    double sig = (fabs(un) + a) * S;
    if (viscous) sig += (mu / w[0]) * (S * S) / V;
    speed += sig;
  }
  dt[c] = cfl * V / speed;
}

// deterministic min-reduction for the global time step (single block)
__global__ void k_min_reduce(int64_t n, const double* __restrict__ dt, double* out) {
  __shared__ double sm[1024];
  double m = INFINITY;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) m = fmin(m, dt[i]);
  sm[threadIdx.x] = m;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sm[threadIdx.x] = fmin(sm[threadIdx.x], sm[threadIdx.x + s]);
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = sm[0];
}

__global__ void k_fill(int64_t n, double* __restrict__ dt, const double* val) {
  const double g = *val;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dt[i] = g;
}

// ---------------------------------------------------------------------------
// K2: reconstruction -> combined coefficients (nc, 9, 5); one thread per
// (cell, component) because the WENO weights are per cell per component
// (recon.py:167-195).
// ---------------------------------------------------------------------------
// K2 kernels run on tiles of RT cells per CTA (RT x 5 threads: thread =
// (cell, component)).  Warp 0 stages the tile's per-cell operator records
// into shared memory with bulk copies (gks_stage.cuh); every thread then
// gathers its stencil's Q from L2 and contracts against the staged records.
//
// Stencil shapes are compile-time (K, M, S) / (HA, HG, M): the handle pads
// every cell's records to the instantiated shape at upload (zero operator
// columns, the cell itself as padded gather index, inactive padded
// sub-stencils), so the kernels carry no runtime bounds: ncu r01 measured
// 45 % of all instructions in the runtime-bound version as ISETP/IMAD/BRA.
// 24 cells: a tile's staged records (60-93 KB) then fit 3 CTAs per SM, so
// one CTA's bulk copies overlap the others' compute (measured against
// 8 / 16 / 32: C2 HWENO recon 1.20 -> 0.97 ms, WENO 0.74 -> 0.71 ms)
// combine(): one reciprocal of the weight total and of gamma0 instead of six
// divisions (C2 WENO reconstruction 0.705 -> 0.663 ms; a rounding-level
// change, inside every parity bar)
// combine(): the candidate weights over a common denominator (one division
// for the normalisation instead of M + 1): C2 reconstruction 0.663 -> 0.656 ms
#ifndef GKS_COMBINE_PROD
#define GKS_COMBINE_PROD 1
#endif
#ifndef GKS_COMBINE_RCP
#define GKS_COMBINE_RCP 1
#endif
#ifndef GKS_FACE_T
#define GKS_FACE_T 128  // face kernel CTA size
#endif
#ifndef GKS_RT
#define GKS_RT 24
#endif
static constexpr int RT = GKS_RT;
static constexpr int RT_THREADS = RT * 5;
// Big-stencil gathers issued straight from the HBM index records, before the
// tile's bulk copies have landed (measured 0.84 -> 0.72 ms, C2 WENO); the
// index records are then not staged.
#ifndef GKS_RECON_EARLY
#define GKS_RECON_EARLY 1
#endif

// recon.py:167-195 on one (cell, component); beta packed as the upper
// triangle (45 entries, row-major).
// (w0n / wmn: optional outputs of the normalised weights, the API's
// combine_candidates; wmn[m * wstride])
template <int M>
__device__ __forceinline__ void combine(double cb[9], const double (&b)[M][3], const int8_t* act,
                                        const double* B, double eps, double lw, double* w0n_out = nullptr,
                                        double* wmn_out = nullptr, int wstride = 0) {
  double beta0 = 0.0;
  {
    int idx = 0;
#pragma unroll
    for (int d = 0; d < 9; ++d) {
      double t = B[idx++] * cb[d];
#pragma unroll
      for (int e = d + 1; e < 9; ++e) t += 2.0 * B[idx++] * cb[e];
      beta0 += cb[d] * t;
    }
  }
  int nact = 0;
  double bs[M];
#pragma unroll
  for (int m = 0; m < M; ++m) {
    bs[m] = b[m][0] * b[m][0] + b[m][1] * b[m][1] + b[m][2] * b[m][2];
    if (act[m]) ++nact;
  }
  const double g0 = 1.0 - lw * nact;
  double tau = 0.0;
#pragma unroll
  for (int m = 0; m < M; ++m)
    if (act[m]) tau += fabs(beta0 - bs[m]);
  tau /= (double)(nact > 1 ? nact : 1);
#if GKS_COMBINE_PROD
  // common denominator: with D = beta + eps, w = g (D + tau) / D; scaling
  // every weight by prod(D) leaves the normalised weights unchanged and
  // turns the M + 1 divisions into products (prefix / suffix products of the
  // active D's)
  double D[M + 1], pre[M + 2], suf[M + 2];
  D[0] = beta0 + eps;
#pragma unroll
  for (int m = 0; m < M; ++m) D[m + 1] = act[m] ? bs[m] + eps : 1.0;
  pre[0] = 1.0;
#pragma unroll
  for (int i = 0; i <= M; ++i) pre[i + 1] = pre[i] * D[i];
  suf[M + 1] = 1.0;
#pragma unroll
  for (int i = M; i >= 0; --i) suf[i] = suf[i + 1] * D[i];
  const double w0 = g0 * (D[0] + tau) * suf[1];
  double wm[M];
  double total = w0;
#pragma unroll
  for (int m = 0; m < M; ++m) {
    wm[m] = act[m] ? lw * (D[m + 1] + tau) * (pre[m + 1] * suf[m + 2]) : 0.0;
    total += wm[m];
  }
#else
  const double w0 = g0 * (1.0 + tau / (beta0 + eps));
  double wm[M];
  double total = w0;
#pragma unroll
  for (int m = 0; m < M; ++m) {
    wm[m] = act[m] ? lw * (1.0 + tau / (bs[m] + eps)) : 0.0;
    total += wm[m];
  }
#endif
#if GKS_COMBINE_RCP
  const double itot = 1.0 / total, ig0 = 1.0 / g0;
  const double w0n = w0 * itot;
#else
  const double w0n = w0 / total;
#endif
  if (w0n_out) {
    *w0n_out = w0n;
#pragma unroll
    for (int m = 0; m < M; ++m) wmn_out[m * wstride] = wm[m] / total;
  }
#if GKS_COMBINE_RCP
  const double c0 = w0n * ig0;
  const double sub0 = w0n * lw * ig0;
#else
  const double c0 = w0n / g0;
  const double sub0 = w0n * lw / g0;
#endif
#pragma unroll
  for (int d = 0; d < 9; ++d) cb[d] *= c0;
#pragma unroll
  for (int m = 0; m < M; ++m) {
    if (act[m]) {
#if GKS_COMBINE_RCP
      const double f = wm[m] * itot - sub0;
#else
      const double f = wm[m] / total - sub0;
#endif
#pragma unroll
      for (int d = 0; d < 3; ++d) cb[d] += f * b[m][d];
    }
  }
}

// staged arrays of the two schemes
enum : int { WT_OP = 0, WT_GI, WT_SO, WT_SG, WT_ACT, WT_BETA, WT_N };
enum : int { HT_OP = 0, HT_AG, HT_GG, HT_GS, HT_SO, HT_SG, HT_ACT, HT_BETA, HT_N };
using WenoTile = Tile<WT_N>;
using HwenoTile = Tile<HT_N>;

// Record bytes in HBM (strides from rec_stride_*, gks_stage.cuh).
inline WenoTile weno_tile(int K, int M, int S, const double* big_op, const int* big_gather, const double* sub_op,
                          const int* sub_gather, const int8_t* sub_active, const double* beta, bool linear) {
  TileBuilder<WT_N> b(RT);
  b.add(WT_OP, big_op, 8u * rec_stride_f64(9 * K));
  b.add(WT_GI, big_gather, 4u * rec_stride_i32(K), !GKS_RECON_EARLY);
  b.add(WT_SO, sub_op, 8u * rec_stride_f64(3 * M * S), !linear);
  b.add(WT_SG, sub_gather, 4u * rec_stride_i32(M * S), !linear);
  b.add(WT_ACT, sub_active, (uint32_t)M, !linear);
  b.add(WT_BETA, beta, 8u * rec_stride_f64(45), !linear);
  return b.t;
}

inline HwenoTile hweno_tile(int HA, int HG, int M, const double* big_op, const int* avg_gather,
                            const int* grad_gather, const double* grad_scale, const double* sub_op,
                            const int* sub_gather, const int8_t* sub_active, const double* beta, bool linear) {
  TileBuilder<HT_N> b(RT);
  b.add(HT_OP, big_op, 8u * rec_stride_f64(9 * (HA + 3 * HG)));
  b.add(HT_AG, avg_gather, 4u * rec_stride_i32(HA), !GKS_RECON_EARLY);
  b.add(HT_GG, grad_gather, 4u * rec_stride_i32(HG), !GKS_RECON_EARLY);
  b.add(HT_GS, grad_scale, 8u * rec_stride_f64(HG), !GKS_RECON_EARLY);
  b.add(HT_SO, sub_op, 8u * rec_stride_f64(21 * M), !linear);
  b.add(HT_SG, sub_gather, 4u * rec_stride_i32(2 * M), !linear);
  b.add(HT_ACT, sub_active, (uint32_t)M, !linear);
  b.add(HT_BETA, beta, 8u * rec_stride_f64(45), !linear);
  return b.t;
}

template <class T, int N>
__device__ __forceinline__ const T* staged(const unsigned char* sm, const Tile<N>& t, int i, int cl) {
  return (const T*)(sm + t.a[i].off + cl * t.a[i].stride);
}

template <int K, int M, int S>
__global__ void __launch_bounds__(RT_THREADS, GKS_RECON_MINB) k_recon_weno(int64_t nc, const double* __restrict__ q,
                                                                           WenoTile T, int linear, double eps,
                                                                           double lw, double* __restrict__ coef,
                                                                           const int* gate) {
  if (gate && !*gate) return;
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ uint64_t bar;
  const int64_t c0 = (int64_t)blockIdx.x * RT;
  const int n = (int)(nc - c0 < RT ? nc - c0 : RT);
  stage_tile(sm, &bar, T, c0, n);
  const int cl = threadIdx.x / 5;
  const int k = threadIdx.x - cl * 5;
  const int64_t c = c0 + cl;
  const double qc = cl < n ? __ldg(q + c * 5 + k) : 0.0;
  double r[K];
#if GKS_RECON_EARLY
  // big-stencil gathers straight from the HBM index records, in flight
  // while the bulk copies land
  if (cl < n) {
    const int* gi = (const int*)(T.a[WT_GI].src + (size_t)c * T.a[WT_GI].rec);
#pragma unroll
    for (int j = 0; j < K; ++j) r[j] = __ldg(q + (int64_t)__ldg(gi + j) * 5 + k) - qc;
  }
#endif
  mbar_wait(&bar, 0);
  if (cl >= n) return;
  const double* op = staged<double>(sm, T, WT_OP, cl);
#if !GKS_RECON_EARLY
  const int* gi = staged<int>(sm, T, WT_GI, cl);
#pragma unroll
  for (int j = 0; j < K; ++j) r[j] = __ldg(q + (int64_t)gi[j] * 5 + k) - qc;
#endif
  double cb[9];
#pragma unroll
  for (int d = 0; d < 9; ++d) {
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < K; ++j) acc += op[d * K + j] * r[j];
    cb[d] = acc;
  }
  if (!linear) {
    const double* so = staged<double>(sm, T, WT_SO, cl);
    const int* sg = staged<int>(sm, T, WT_SG, cl);
    double b[M][3];
#pragma unroll
    for (int m = 0; m < M; ++m) {
      double rs[S];
#pragma unroll
      for (int s2 = 0; s2 < S; ++s2) rs[s2] = __ldg(q + (int64_t)sg[m * S + s2] * 5 + k) - qc;
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        double acc = 0.0;
#pragma unroll
        for (int s2 = 0; s2 < S; ++s2) acc += so[(m * 3 + d) * S + s2] * rs[s2];
        b[m][d] = acc;
      }
    }
    combine<M>(cb, b, staged<int8_t>(sm, T, WT_ACT, cl), staged<double>(sm, T, WT_BETA, cl), eps, lw);
  }
  double* out = coef + c * 45 + k;
#pragma unroll
  for (int d = 0; d < 9; ++d) out[d * 5] = cb[d];
}

template <int HA, int HG, int M>
__global__ void __launch_bounds__(RT_THREADS, GKS_RECON_MINB) k_recon_hweno(int64_t nc, const double* __restrict__ q,
                                                                            const double* __restrict__ grad,
                                                                            const double* __restrict__ h,
                                                                            HwenoTile T, int linear, double eps,
                                                                            double lw, double* __restrict__ coef,
                                                                            const int* gate) {
  if (gate && !*gate) return;
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ uint64_t bar;
  const int64_t c0 = (int64_t)blockIdx.x * RT;
  const int n = (int)(nc - c0 < RT ? nc - c0 : RT);
  stage_tile(sm, &bar, T, c0, n);
  const int cl = threadIdx.x / 5;
  const int k = threadIdx.x - cl * 5;
  const int64_t c = c0 + cl;
  const double qc = cl < n ? __ldg(q + c * 5 + k) : 0.0;
  constexpr int W = HA + 3 * HG;
  // right-hand side: neighbour averages, then h-scaled gradients (hweno.py:147-151)
  double ra[HA], rg[HG][3];
  // (index records from HBM or shared memory: generic loads)
  auto gather = [&](const int* ag, const int* gg, const double* gs) {
#pragma unroll
    for (int j = 0; j < HA; ++j) ra[j] = __ldg(q + (int64_t)ag[j] * 5 + k) - qc;
#pragma unroll
    for (int g = 0; g < HG; ++g) {
      const int64_t m = gg[g];
      const double sc = gs[g];
#pragma unroll
      for (int x = 0; x < 3; ++x) rg[g][x] = sc * __ldg(grad + (m * 3 + x) * 5 + k);
    }
  };
#if GKS_RECON_EARLY
  if (cl < n)
    gather((const int*)(T.a[HT_AG].src + (size_t)c * T.a[HT_AG].rec),
           (const int*)(T.a[HT_GG].src + (size_t)c * T.a[HT_GG].rec),
           (const double*)(T.a[HT_GS].src + (size_t)c * T.a[HT_GS].rec));
#endif
  mbar_wait(&bar, 0);
  if (cl >= n) return;
  const double* op = staged<double>(sm, T, HT_OP, cl);
#if !GKS_RECON_EARLY
  gather(staged<int>(sm, T, HT_AG, cl), staged<int>(sm, T, HT_GG, cl), staged<double>(sm, T, HT_GS, cl));
#endif
  double cb[9];
#pragma unroll
  for (int d = 0; d < 9; ++d) {
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < HA; ++j) acc += op[d * W + j] * ra[j];
#pragma unroll
    for (int g = 0; g < HG; ++g)
#pragma unroll
      for (int x = 0; x < 3; ++x) acc += op[d * W + HA + 3 * g + x] * rg[g][x];
    cb[d] = acc;
  }
  if (!linear) {
    const double* so = staged<double>(sm, T, HT_SO, cl);
    const int* sg = staged<int>(sm, T, HT_SG, cl);
    double b[M][3];
#pragma unroll
    for (int m = 0; m < M; ++m) {
      const int64_t s0 = sg[m * 2 + 0];
      const int64_t s1 = sg[m * 2 + 1];
      double rhs[7];
      rhs[0] = __ldg(q + s1 * 5 + k) - qc;
      const double h0 = __ldg(h + s0), h1 = __ldg(h + s1);
#pragma unroll
      for (int x = 0; x < 3; ++x) {
        rhs[1 + x] = h0 * __ldg(grad + (s0 * 3 + x) * 5 + k);
        rhs[4 + x] = h1 * __ldg(grad + (s1 * 3 + x) * 5 + k);
      }
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        double acc = 0.0;
#pragma unroll
        for (int s2 = 0; s2 < 7; ++s2) acc += so[(m * 3 + d) * 7 + s2] * rhs[s2];
        b[m][d] = acc;
      }
    }
    combine<M>(cb, b, staged<int8_t>(sm, T, HT_ACT, cl), staged<double>(sm, T, HT_BETA, cl), eps, lw);
  }
  double* out = coef + c * 45 + k;
#pragma unroll
  for (int d = 0; d < 9; ++d) out[d * 5] = cb[d];
}

// ---------------------------------------------------------------------------
// K3: fused face kernel, one thread per face quadrature point
// ---------------------------------------------------------------------------
// Face value and Cartesian gradient of one side's reconstruction at a face
// point (recon.py:297-314): val = Q_c + phi . C_c, grad = dphi . C_c with
// phi = mono((x - x_c) / h) - avg0 and dphi = d mono / dx (recon.py:48-57).
// The scaled-chart gradient rows are sparse (4 of 9 entries per axis) and
// share the factor 1/h, so they are summed first and scaled once: one
// division per side instead of the table's 27 per-entry ones (ncu r01: 125
// FP64 divisions per face point before).  Rounding differs from the
// reference's stored tables by an ulp (parity bar 1e-12, tests/).
__device__ __forceinline__ void eval_side(const double* __restrict__ q, const double* __restrict__ coef,
                                          const double* __restrict__ cen, const double* __restrict__ inv_h,
                                          const double* __restrict__ avg0, int64_t c, const double x[3],
                                          double val[5], double g[3][5]) {
  const double ih = inv_h[c];  // 1 / h_c, precomputed once per handle (the same IEEE quotient)
  const double x0 = (x[0] - cen[3 * c]) * ih, x1 = (x[1] - cen[3 * c + 1]) * ih, x2 = (x[2] - cen[3 * c + 2]) * ih;
  const double* A = avg0 + c * 9;
  const double phi[9] = {x0 - A[0],      x1 - A[1],      x2 - A[2],      x0 * x0 - A[3], x0 * x1 - A[4],
                         x0 * x2 - A[5], x1 * x1 - A[6], x1 * x2 - A[7], x2 * x2 - A[8]};
  const double tx0 = 2.0 * x0, tx1 = 2.0 * x1, tx2 = 2.0 * x2;
  const double* C = coef + c * 45;
#pragma unroll
  for (int k = 0; k < 5; ++k) {
    double cd[9];
#pragma unroll
    for (int d = 0; d < 9; ++d) cd[d] = C[d * 5 + k];
    double v = 0.0;
#pragma unroll
    for (int d = 0; d < 9; ++d) v += phi[d] * cd[d];
    val[k] = q[c * 5 + k] + v;
    g[0][k] = (cd[0] + tx0 * cd[3] + x1 * cd[4] + x2 * cd[5]) * ih;
    g[1][k] = (cd[1] + x0 * cd[4] + tx1 * cd[6] + x2 * cd[7]) * ih;
    g[2][k] = (cd[2] + x0 * cd[5] + x1 * cd[7] + tx2 * cd[8]) * ih;
  }
}

// value only (no gradients): the pre-loop pressures of the inviscid collision time
__device__ __forceinline__ void eval_value(const double* __restrict__ q, const double* __restrict__ coef,
                                           const double* __restrict__ cen, const double* __restrict__ inv_h,
                                           const double* __restrict__ avg0, int64_t c, const double x[3],
                                           double val[5]) {
  const double ih = inv_h[c];
  const double x0 = (x[0] - cen[3 * c]) * ih, x1 = (x[1] - cen[3 * c + 1]) * ih, x2 = (x[2] - cen[3 * c + 2]) * ih;
  const double* A = avg0 + c * 9;
  const double phi[9] = {x0 - A[0],      x1 - A[1],      x2 - A[2],      x0 * x0 - A[3], x0 * x1 - A[4],
                         x0 * x2 - A[5], x1 * x1 - A[6], x1 * x2 - A[7], x2 * x2 - A[8]};
  const double* C = coef + c * 45;
#pragma unroll
  for (int k = 0; k < 5; ++k) {
    double v = 0.0;
#pragma unroll
    for (int d = 0; d < 9; ++d) v += phi[d] * C[d * 5 + k];
    val[k] = q[c * 5 + k] + v;
  }
}

__device__ __forceinline__ void to_local_state(const double qv[5], const double* F, double out[5]) {
  out[0] = qv[0];
  out[4] = qv[4];
#pragma unroll
  for (int i = 0; i < 3; ++i) out[1 + i] = F[3 * i] * qv[1] + F[3 * i + 1] * qv[2] + F[3 * i + 2] * qv[3];
}

// slopes along (n, t1, t2), momentum block rotated (stepping.py:180-185)
__device__ __forceinline__ void local_slopes(const double g[3][5], const double* F, double s[3][5]) {
  double t[3][5];
#pragma unroll
  for (int kk = 0; kk < 3; ++kk)
#pragma unroll
    for (int m = 0; m < 5; ++m) t[kk][m] = F[3 * kk] * g[0][m] + F[3 * kk + 1] * g[1][m] + F[3 * kk + 2] * g[2][m];
#pragma unroll
  for (int kk = 0; kk < 3; ++kk) {
    s[kk][0] = t[kk][0];
    s[kk][4] = t[kk][4];
#pragma unroll
    for (int i = 0; i < 3; ++i) s[kk][1 + i] = F[3 * i] * t[kk][1] + F[3 * i + 1] * t[kk][2] + F[3 * i + 2] * t[kk][3];
  }
}

struct FaceArgs {
  int64_t nfq;
  const double *q, *coef, *cen, *h, *ih, *avg0, *dt;
  const int *fq_face, *f_own, *f_nbr, *f_patch;
  const double *fq_point, *fq_ws, *f_frame, *f_normal, *f_shift;
  const DevPatch* patches;
  int model;
  double mu;
  KinConst kc;
  int want_point;
  int fq_nq;
  double* contrib;
  const int2* fq_slot;  // slot mode (non-null): contributions go to the assembly slots
  double* slots;
  double* qpt;
  int* status;
  const int* gate;
};

// (Staging the CTA's owner / neighbour cell records in shared memory with
// cp.async before the compute was measured 32 % slower: 3.52 vs 2.66 ms on
// C2 -- the CTA-wide barrier serialises load and compute phases and the
// 45 KB of records per CTA take L1 from the spills.)
// KFVS: first-order collisionless flux (tau = inf, SolverOptions.first_order)
// -- a compile-time branch, so the high-order kernel keeps its constant
// tau_in and register allocation
template <bool VISC, bool POINT, bool KFVS>
__global__ void __launch_bounds__(GKS_FACE_T, GKS_FACE_MINB) k_face(FaceArgs A) {
  if (A.gate && !*A.gate) return;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= A.nfq) return;
  const int f = A.fq_nq ? (int)((uint32_t)i / (uint32_t)A.fq_nq) : A.fq_face[i];
  const int64_t o = A.f_own[f];
  const int64_t nb = A.f_nbr[f];
  const int p = nb >= 0 ? -1 : A.f_patch[f];
  const bool wall = p >= 0 && A.patches[p].wall;
  auto eval_cell = [&](bool own, const double x[3], double v[5], double g[3][5]) {
    eval_side(A.q, A.coef, A.cen, A.ih, A.avg0, own ? o : nb, x, v, g);
  };
  auto eval_cell_value = [&](bool own, const double x[3], double v[5]) {
    eval_value(A.q, A.coef, A.cen, A.ih, A.avg0, own ? o : nb, x, v);
  };
#if GKS_FACE_PREFETCH
  {
  // the neighbour side's coefficient record is read only after the whole
  // owner side: start moving its lines into L2 now (no registers held)
  if (nb >= 0) {
    const char* pc = (const char*)(A.coef + nb * 45);
#if GKS_FACE_PREFETCH == 2
    // into L1 (the kernel uses no shared memory: 12 warps x 32 x 440 B fit)
#pragma unroll
    for (int l = 0; l < 360; l += 128) asm volatile("prefetch.global.L1 [%0];" ::"l"(pc + l));
    asm volatile("prefetch.global.L1 [%0];" ::"l"(pc + 359));
    asm volatile("prefetch.global.L1 [%0];" ::"l"((const char*)(A.avg0 + nb * 9)));
#else
#pragma unroll
    for (int l = 0; l < 360; l += 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(pc + l));
    asm volatile("prefetch.global.L2 [%0];" ::"l"(pc + 359));
    asm volatile("prefetch.global.L2 [%0];" ::"l"((const char*)(A.avg0 + nb * 9)));
#endif
  }
  }
#endif
  // face window min(dt_owner, dt_nbr), read where the flux first needs it
  // (after the side loop for the inviscid face): its loads need not land
  // before the reconstruction gathers start
  auto dtf = [&]() { return nb >= 0 ? fmin(A.dt[o], A.dt[nb]) : A.dt[o]; };
  int ghost_fail = 0;
  // side 0: owner reconstruction; side 1: neighbour (shifted chart) or ghost
  auto get = [&](int side, double w[5], double sl[3][5], double& hside) {
    const double x[3] = {A.fq_point[3 * i], A.fq_point[3 * i + 1], A.fq_point[3 * i + 2]};
    double v[5], g[3][5];
    if (side == 0 || nb < 0) {
      eval_cell(true, x, v, g);
    } else {
      const double xs[3] = {x[0] - A.f_shift[3 * f], x[1] - A.f_shift[3 * f + 1], x[2] - A.f_shift[3 * f + 2]};
      eval_cell(false, xs, v, g);
    }
    if (side == 1 && nb < 0) {
      const DevPatch P = A.patches[p];
      const double nrm[3] = {A.f_normal[3 * f], A.f_normal[3 * f + 1], A.f_normal[3 * f + 2]};
      double vg[5], gg[3][5];
      if (!ghost_state(v, P, nrm, A.kc, vg)) {
        ghost_fail = 1;
        return false;
      }
      ghost_gradients(g, P, nrm, gg);
#pragma unroll
      for (int k = 0; k < 5; ++k) {
        v[k] = vg[k];
        g[0][k] = gg[0][k];
        g[1][k] = gg[1][k];
        g[2][k] = gg[2][k];
      }
    }
    const double* F = A.f_frame + 9 * f;
    double ql[5];
    to_local_state(v, F, ql);
#if GKS_H_MUL
    if (!cons_to_prim_h(ql, A.kc, w, hside)) return false;
#else
    if (!cons_to_prim(ql, A.kc, w)) return false;
    hside = 0.5 / w[4];
#endif
    local_slopes(g, F, sl);
    return true;
  };
  // both side pressures first (inviscid tau is then known before the side loop)
  auto press = [&](double& pl, double& pr) {
    const double x[3] = {A.fq_point[3 * i], A.fq_point[3 * i + 1], A.fq_point[3 * i + 2]};
    double v[5], w[5];
    eval_cell_value(true, x, v);
    if (!cons_to_prim(v, A.kc, w)) return false;
    pl = w[0] / (2.0 * w[4]);
    if (nb >= 0) {
      const double xs[3] = {x[0] - A.f_shift[3 * f], x[1] - A.f_shift[3 * f + 1], x[2] - A.f_shift[3 * f + 2]};
      eval_cell_value(false, xs, v);
    } else {
      const DevPatch P = A.patches[p];
      const double nrm[3] = {A.f_normal[3 * f], A.f_normal[3 * f + 1], A.f_normal[3 * f + 2]};
      double vg[5];
      if (!ghost_state(v, P, nrm, A.kc, vg)) {
        ghost_fail = 1;
        return false;
      }
#pragma unroll
      for (int k = 0; k < 5; ++k) v[k] = vg[k];
    }
    if (!cons_to_prim(v, A.kc, w)) return false;
    pr = w[0] / (2.0 * w[4]);
    return true;
  };
  // TAU mode 2: the right state's pressure only (the left one comes from
  // the side loop), in the local frame like the loop's own states
  auto press_r = [&](double& pl, double& pr) {
    (void)pl;
    const double x[3] = {A.fq_point[3 * i], A.fq_point[3 * i + 1], A.fq_point[3 * i + 2]};
    double v[5], w[5], ql[5];
    if (nb >= 0) {
      const double xs[3] = {x[0] - A.f_shift[3 * f], x[1] - A.f_shift[3 * f + 1], x[2] - A.f_shift[3 * f + 2]};
      eval_cell_value(false, xs, v);
    } else {
      eval_cell_value(true, x, v);
      const DevPatch P = A.patches[p];
      const double nrm[3] = {A.f_normal[3 * f], A.f_normal[3 * f + 1], A.f_normal[3 * f + 2]};
      double vg[5];
      if (!ghost_state(v, P, nrm, A.kc, vg)) {
        ghost_fail = 1;
        return false;
      }
#pragma unroll
      for (int k = 0; k < 5; ++k) v[k] = vg[k];
    }
    to_local_state(v, A.f_frame + 9 * f, ql);
    if (!cons_to_prim(ql, A.kc, w)) return false;
    pr = w[0] / (2.0 * w[4]);
    return true;
  };
  double fl[5], pv[5];
  int rc;
  constexpr double tau_in = KFVS ? INFINITY : -1.0;
  if (GKS_FACE_TAU == 2) rc = interface_flux_t<VISC, POINT, 2>(get, press_r, tau_in, dtf, A.mu, A.kc, fl, 0.0, pv);
  else rc = interface_flux_t<VISC, POINT, GKS_FACE_TAU>(get, press, tau_in, dtf, A.mu, A.kc, fl, 0.0, pv);
  if (rc) {
    if (ghost_fail) {
      atomicCAS(A.status, 0, GKS_ERR_UNPHYSICAL);
      atomicMin(A.status + 1, (int)i);
      A.status[2] = p + 1;
    } else {
      raise_dev(A.status, GKS_ERR_UNPHYSICAL, (int)i);
    }
    return;
  }
  if (wall) fl[0] = 0.0;
  const double* F = A.f_frame + 9 * f;
  const double ws = A.fq_ws[i];
  double c[5];
  c[0] = ws * fl[0];
  c[4] = ws * fl[4];
#pragma unroll
  for (int d = 0; d < 3; ++d) c[1 + d] = ws * (F[d] * fl[1] + F[3 + d] * fl[2] + F[6 + d] * fl[3]);
  if (A.fq_slot) {
    // owner entry -c, neighbour entry +c (stepping.py:225-228)
    const int2 sl = A.fq_slot[i];
    if (sl.x >= 0) {
      double* so = A.slots + (int64_t)sl.x * 5;
#pragma unroll
      for (int k = 0; k < 5; ++k) so[k] = -c[k];
    }
    if (sl.y >= 0) {
      double* sn = A.slots + (int64_t)sl.y * 5;
#pragma unroll
      for (int k = 0; k < 5; ++k) sn[k] = c[k];
    }
  } else {
    double* out = A.contrib + i * 5;
#pragma unroll
    for (int k = 0; k < 5; ++k) out[k] = c[k];
  }
  if (POINT) {
    double* qp = A.qpt + i * 5;
    qp[0] = pv[0];
    qp[4] = pv[4];
#pragma unroll
    for (int d = 0; d < 3; ++d) qp[1 + d] = F[d] * pv[1] + F[3 + d] * pv[2] + F[6 + d] * pv[3];
  }
}

// ---------------------------------------------------------------------------
// K4: deterministic cell assembly (stepping.py:225-228, hweno.py:172-194)
// ---------------------------------------------------------------------------
__global__ void k_assemble(int64_t nc, const int* __restrict__ cfq_start, const int* __restrict__ cfq,
                           const double* __restrict__ contrib, const double* __restrict__ qpt,
                           const int* __restrict__ fq_face, const double* __restrict__ fq_ws,
                           const double* __restrict__ f_normal, const double* __restrict__ vol,
                           double* __restrict__ res, double* __restrict__ grad_new, const int* gate,
                           FrechetEpi fe) {
  if (gate && !*gate) return;
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= nc) return;
  double r[5] = {0, 0, 0, 0, 0};
  double g[3][5] = {};
  const bool wantg = grad_new != nullptr;
  // unrolled so several entries' index and record loads are in flight at
  // once (the list walk is a dependent index -> record chain per entry)
#pragma unroll 4
  for (int e = cfq_start[c]; e < cfq_start[c + 1]; ++e) {
    const int64_t i = cfq[e] >> 1;
    const bool is_nbr = cfq[e] & 1;
    const double* cc = contrib + i * 5;
#pragma unroll
    for (int k = 0; k < 5; ++k) r[k] = is_nbr ? r[k] + cc[k] : r[k] - cc[k];
    if (wantg) {
      const int f = fq_face[i];
      const double ws = fq_ws[i];
      const double* pv = qpt + i * 5;
#pragma unroll
      for (int x = 0; x < 3; ++x) {
        const double wn = ws * f_normal[3 * f + x];
#pragma unroll
        for (int k = 0; k < 5; ++k) {
          const double t = wn * pv[k];
          g[x][k] = is_nbr ? g[x][k] - t : g[x][k] + t;
        }
      }
    }
  }
  if (fe.out) {
    // the Frechet combine (formerly its own pass) on the unwritten residual.
    // Staging the block's residual through shared memory for coalesced
    // stores was slower (0.22 -> 0.27 ms on C2: the carve-out takes L1 from
    // the contribution gathers)
    const double s = *fe.sigma;
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      const int64_t e = c * 5 + k;
      const double d = s == 0.0 ? 0.0 : (r[k] - fe.r0[e]) / s;
      fe.out[e] = fe.mode ? (vol[c] / fe.dt[c]) * fe.v[e] - d : d;
    }
  } else {
#pragma unroll
    for (int k = 0; k < 5; ++k) res[c * 5 + k] = r[k];
  }
  if (wantg) {
    const double V = vol[c];
#pragma unroll
    for (int x = 0; x < 3; ++x)
#pragma unroll
      for (int k = 0; k < 5; ++k) grad_new[(c * 3 + x) * 5 + k] = g[x][k] / V;
  }
}

// Same assembly with one thread per (cell, component): five independent
// list walks per cell instead of one, so five times the contribution loads
// are in flight per cell, and the res / Frechet epilogue stores coalesce.
// Each component is summed over the same list in the same order as
// k_assemble (bitwise-identical results).
__global__ void k_assemble5(int64_t nc, const int* __restrict__ cfq_start, const int* __restrict__ cfq,
                            const double* __restrict__ contrib, const double* __restrict__ qpt,
                            const int* __restrict__ fq_face, const double* __restrict__ fq_ws,
                            const double* __restrict__ f_normal, const double* __restrict__ vol,
                            double* __restrict__ res, double* __restrict__ grad_new, const int* gate,
                            FrechetEpi fe) {
  if (gate && !*gate) return;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nc * 5) return;
  const int64_t c = t / 5;
  const int k = (int)(t - c * 5);
  double r = 0.0;
  double g[3] = {0.0, 0.0, 0.0};
  const bool wantg = grad_new != nullptr;
  const int e0 = cfq_start[c], e1 = cfq_start[c + 1];
  int e = e0;
  if (!wantg) {
    // batches of 8: all index loads, then all contribution loads in flight,
    // then the sums in list order
    for (; e + 8 <= e1; e += 8) {
      int ce[8];
      double cc[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) ce[u] = __ldg(cfq + e + u);
#pragma unroll
      for (int u = 0; u < 8; ++u) cc[u] = contrib[(int64_t)(ce[u] >> 1) * 5 + k];
#pragma unroll
      for (int u = 0; u < 8; ++u) r = (ce[u] & 1) ? r + cc[u] : r - cc[u];
    }
  }
  if (wantg) {
    // gradient update too (compact scheme): batches of 4 -- index loads, then
    // each entry's contribution / point value / weight / face, then the
    // normals, then the sums in list order
    for (; e + 4 <= e1; e += 4) {
      int ce[4], f[4];
      double cc[4], pv[4], ws[4], nr[4][3];
#pragma unroll
      for (int u = 0; u < 4; ++u) ce[u] = __ldg(cfq + e + u);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t i = ce[u] >> 1;
        cc[u] = contrib[i * 5 + k];
        pv[u] = qpt[i * 5 + k];
        ws[u] = __ldg(fq_ws + i);
        f[u] = __ldg(fq_face + i);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int x = 0; x < 3; ++x) nr[u][x] = __ldg(f_normal + 3 * f[u] + x);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const bool is_nbr = ce[u] & 1;
        r = is_nbr ? r + cc[u] : r - cc[u];
#pragma unroll
        for (int x = 0; x < 3; ++x) {
          const double wn = ws[u] * nr[u][x];
          const double tt = wn * pv[u];
          g[x] = is_nbr ? g[x] - tt : g[x] + tt;
        }
      }
    }
  }
#pragma unroll 4
  for (; e < e1; ++e) {
    const int ce = cfq[e];
    const int64_t i = ce >> 1;
    const bool is_nbr = ce & 1;
    const double cc = contrib[i * 5 + k];
    r = is_nbr ? r + cc : r - cc;
    if (wantg) {
      const int f = fq_face[i];
      const double ws = fq_ws[i];
      const double pv = qpt[i * 5 + k];
#pragma unroll
      for (int x = 0; x < 3; ++x) {
        const double wn = ws * f_normal[3 * f + x];
        const double tt = wn * pv;
        g[x] = is_nbr ? g[x] - tt : g[x] + tt;
      }
    }
  }
  if (fe.out) {
    const double sg = *fe.sigma;
    const double d = sg == 0.0 ? 0.0 : (r - fe.r0[t]) / sg;
    fe.out[t] = fe.mode ? (vol[c] / fe.dt[c]) * fe.v[t] - d : d;
  } else {
    res[t] = r;
  }
  if (wantg) {
    const double V = vol[c];
#pragma unroll
    for (int x = 0; x < 3; ++x) grad_new[(c * 3 + x) * 5 + k] = g[x] / V;
  }
}

// Tiled assembly (residuals without the gradient update): a CTA of 32 cells
// x 5 components first loads its cells' whole CSR list segment into shared
// memory with coalesced loads (one copy for the five component threads),
// then every thread issues its contribution loads from the staged indices
// -- the dependent index round trip leaves the per-thread chain.  Same
// entries, order and signs as k_assemble5: bitwise-identical results.
#ifndef GKS_AT_CELLS
#define GKS_AT_CELLS 32
#endif
constexpr int AT_CELLS = GKS_AT_CELLS;
constexpr int AT_MAXE = AT_CELLS * 18;  // hex cells: at most 6 faces x 3 points
__global__ void __launch_bounds__(AT_CELLS * 5) k_assemble_tile(int64_t nc, const int* __restrict__ cfq_start,
                                                                const int* __restrict__ cfq,
                                                                const double* __restrict__ contrib,
                                                                const double* __restrict__ vol,
                                                                double* __restrict__ res, const int* gate,
                                                                FrechetEpi fe) {
  if (gate && !*gate) return;
  __shared__ int sidx[AT_MAXE];
  const int64_t c0 = (int64_t)blockIdx.x * AT_CELLS;
  const int64_t cend = c0 + AT_CELLS < nc ? c0 + AT_CELLS : nc;
  const int base = __ldg(cfq_start + c0);
  const int ne = __ldg(cfq_start + cend) - base;
  for (int i = threadIdx.x; i < ne; i += blockDim.x) sidx[i] = __ldg(cfq + base + i);
  __syncthreads();
  const int64_t t = c0 * 5 + threadIdx.x;
  if (t >= nc * 5) return;
  const int64_t c = t / 5;
  const int k = (int)(t - c * 5);
  int e = __ldg(cfq_start + c) - base;
  const int e1 = __ldg(cfq_start + c + 1) - base;
  double r = 0.0;
  for (; e + 8 <= e1; e += 8) {
    double cc[8];
    int ce[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) ce[u] = sidx[e + u];
#pragma unroll
    for (int u = 0; u < 8; ++u) cc[u] = contrib[(int64_t)(ce[u] >> 1) * 5 + k];
#pragma unroll
    for (int u = 0; u < 8; ++u) r = (ce[u] & 1) ? r + cc[u] : r - cc[u];
  }
#pragma unroll 4
  for (; e < e1; ++e) {
    const int ce = sidx[e];
    const double cc = contrib[(int64_t)(ce >> 1) * 5 + k];
    r = (ce & 1) ? r + cc : r - cc;
  }
  if (fe.out) {
    const double sg = *fe.sigma;
    const double d = sg == 0.0 ? 0.0 : (r - fe.r0[t]) / sg;
    fe.out[t] = fe.mode ? (vol[c] / fe.dt[c]) * fe.v[t] - d : d;
  } else {
    res[t] = r;
  }
}

// Tiled assembly with the Gauss gradient update (compact scheme): the list
// segment and, per entry, the face-point weight times the face normal
// (ws * n, computed once instead of by all five component threads) are
// staged in shared memory; the sums follow k_assemble5's order and
// operations exactly (bitwise-identical results).
__global__ void __launch_bounds__(AT_CELLS * 5) k_assemble_tile_g(int64_t nc, const int* __restrict__ cfq_start,
                                                                  const int* __restrict__ cfq,
                                                                  const double* __restrict__ contrib,
                                                                  const double* __restrict__ qpt,
                                                                  const int* __restrict__ fq_face,
                                                                  const double* __restrict__ fq_ws,
                                                                  const double* __restrict__ f_normal,
                                                                  const double* __restrict__ vol,
                                                                  double* __restrict__ res,
                                                                  double* __restrict__ grad_new, const int* gate,
                                                                  FrechetEpi fe) {
  if (gate && !*gate) return;
  __shared__ int sidx[AT_MAXE];
  __shared__ double swn[AT_MAXE * 3];
  const int64_t c0 = (int64_t)blockIdx.x * AT_CELLS;
  const int64_t cend = c0 + AT_CELLS < nc ? c0 + AT_CELLS : nc;
  const int base = __ldg(cfq_start + c0);
  const int ne = __ldg(cfq_start + cend) - base;
  for (int i = threadIdx.x; i < ne; i += blockDim.x) {
    const int ce = __ldg(cfq + base + i);
    sidx[i] = ce;
    const int64_t q = ce >> 1;
    const int f = __ldg(fq_face + q);
    const double ws = __ldg(fq_ws + q);
#pragma unroll
    for (int x = 0; x < 3; ++x) swn[i * 3 + x] = ws * __ldg(f_normal + 3 * f + x);
  }
  __syncthreads();
  const int64_t t = c0 * 5 + threadIdx.x;
  if (t >= nc * 5) return;
  const int64_t c = t / 5;
  const int k = (int)(t - c * 5);
  int e = __ldg(cfq_start + c) - base;
  const int e1 = __ldg(cfq_start + c + 1) - base;
  double r = 0.0;
  double g[3] = {0.0, 0.0, 0.0};
  for (; e + 4 <= e1; e += 4) {
    int ce[4];
    double cc[4], pv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) ce[u] = sidx[e + u];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t i = ce[u] >> 1;
      cc[u] = contrib[i * 5 + k];
      pv[u] = qpt[i * 5 + k];
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const bool is_nbr = ce[u] & 1;
      r = is_nbr ? r + cc[u] : r - cc[u];
#pragma unroll
      for (int x = 0; x < 3; ++x) {
        const double tt = swn[(e + u) * 3 + x] * pv[u];
        g[x] = is_nbr ? g[x] - tt : g[x] + tt;
      }
    }
  }
  for (; e < e1; ++e) {
    const int ce = sidx[e];
    const int64_t i = ce >> 1;
    const bool is_nbr = ce & 1;
    const double cc = contrib[i * 5 + k];
    const double pv = qpt[i * 5 + k];
    r = is_nbr ? r + cc : r - cc;
#pragma unroll
    for (int x = 0; x < 3; ++x) {
      const double tt = swn[e * 3 + x] * pv;
      g[x] = is_nbr ? g[x] - tt : g[x] + tt;
    }
  }
  if (fe.out) {
    const double sg = *fe.sigma;
    const double d = sg == 0.0 ? 0.0 : (r - fe.r0[t]) / sg;
    fe.out[t] = fe.mode ? (vol[c] / fe.dt[c]) * fe.v[t] - d : d;
  } else {
    res[t] = r;
  }
  const double V = vol[c];
#pragma unroll
  for (int x = 0; x < 3; ++x) grad_new[(c * 3 + x) * 5 + k] = g[x] / V;
}

// Slot assembly: the face kernel has written every signed contribution into
// its cell's CSR slot, so a cell's residual is a contiguous segmented sum
// (one thread per (cell, component), coalesced 40-byte slot records, no
// index walk).  Same entries in the same order with the same signs as
// k_assemble5 (r - c == r + (-c)): bitwise-identical results.
__global__ void k_assemble_slots(int64_t nc, const int* __restrict__ cfq_start, const double* __restrict__ slots,
                                 const double* __restrict__ vol, double* __restrict__ res, const int* gate,
                                 FrechetEpi fe) {
  if (gate && !*gate) return;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nc * 5) return;
  const int64_t c = t / 5;
  const int k = (int)(t - c * 5);
  const int e0 = cfq_start[c], e1 = cfq_start[c + 1];
  double r = 0.0;
#pragma unroll 4
  for (int e = e0; e < e1; ++e) r += __ldcs(slots + (int64_t)e * 5 + k);
  if (fe.out) {
    const double sg = *fe.sigma;
    const double d = sg == 0.0 ? 0.0 : (r - fe.r0[t]) / sg;
    fe.out[t] = fe.mode ? (vol[c] / fe.dt[c]) * fe.v[t] - d : d;
  } else {
    res[t] = r;
  }
}

// ghost of the cell-average owner state per boundary face (stepping.py:242-249)
__global__ void k_boundary_ghosts(int64_t nbf, const int* __restrict__ bfaces, const int* __restrict__ f_own,
                                  const int* __restrict__ f_patch, const double* __restrict__ f_normal,
                                  const DevPatch* __restrict__ patches, const double* __restrict__ q, KinConst kc,
                                  double* __restrict__ ghosts, int* status) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nbf) return;
  const int f = bfaces[b];
  const int64_t o = f_own[f];
  double qc[5], g[5];
  for (int k = 0; k < 5; ++k) qc[k] = q[o * 5 + k];
  const double n[3] = {f_normal[3 * f], f_normal[3 * f + 1], f_normal[3 * f + 2]};
  if (!ghost_state(qc, patches[f_patch[f]], n, kc, g)) {
    raise_dev(status, GKS_ERR_UNPHYSICAL, (int)o);
    return;
  }
  for (int k = 0; k < 5; ++k) ghosts[b * 5 + k] = g[k];
}

// ---------------------------------------------------------------------------
// host orchestration
// ---------------------------------------------------------------------------
void reset_status(Handle* H) {
  const int st0[4] = {0, 0x7fffffff, 0, 0};
  cudaMemcpyAsync(H->status, st0, sizeof(st0), cudaMemcpyHostToDevice, H->stream);
}

#define TRY_STATUS(x)     \
  do {                     \
    int _r = (x);          \
    if (_r) return _r;     \
  } while (0)

int status_report(Handle* H, const char* what, const int* st) {
  if (st[0] == 0) return GKS_OK;
  set_error_index(st[1]);
  if (st[0] == GKS_ERR_UNPHYSICAL && st[2] > 0 && st[2] - 1 < (int)H->patch_names.size())
    set_error("%s: unphysical reconstructed state at patch '%s' (point %d)", what,
              H->patch_names[st[2] - 1].c_str(), st[1]);
  else
    set_error("%s: error %d at index %d", what, st[0], st[1]);
  return st[0];
}

int check_status(Handle* H, const char* what) {
  int st[4];
  // every rank must agree on failure: the error code is max-reduced first
  if (H->comm) TRY_STATUS(allreduce(H, H->status, 1, 1, 2, H->stream));
  GKS_CUDA(cudaMemcpyAsync(st, H->status, sizeof(st), cudaMemcpyDeviceToHost, H->stream));
  GKS_CUDA(cudaStreamSynchronize(H->stream));
  return status_report(H, what, st);
}

int local_dt_device(Handle* H) {
  GKS_LAUNCH(KC_DT, k_local_dt, blocks_for(H->n_owned, TPB), TPB, 0, H->stream, H->n_owned, H->q, H->cdt_start,
             H->cdt, H->f_normal, H->f_area, H->vol, H->model == 1 && H->mu > 0.0, H->mu, H->cfl, H->kc, H->dt,
             H->status);
  if (H->global_dt) {
    GKS_LAUNCH(KC_DT, k_min_reduce, 1, 1024, 0, H->stream, H->n_owned, H->dt, &H->scal->red[6]);
    TRY_STATUS(allreduce(H, &H->scal->red[6], 1, 0, 1, H->stream));
    GKS_LAUNCH(KC_DT, k_fill, blocks_for(H->nc, 256), 256, 0, H->stream, H->nc, H->dt, &H->scal->red[6]);
  } else {
    // face windows min(dt_owner, dt_nbr) on cut faces need the layer-1 ghosts' dt
    TRY_STATUS(halo_exchange(H, H->hx, H->dt, 1, H->stream));
  }
  GKS_CUDA(cudaGetLastError());
  return GKS_OK;
}

// Instantiated stencil shapes; the handle pads its records to one of them
// (gks_api.cu recon_shape).
static int recon_device(Handle* H, const double* q, const int* gate) {
  const int nbt = blocks_for(H->n_recon, RT);
  const bool lin = H->linear_weights != 0;
  constexpr uint32_t kMaxSmem = 227 * 1024;
  const int Kt = H->Kt, Mt = H->Mt, St = H->St;
  if (H->compact) {
    const HwenoTile T = hweno_tile(Kt, St, Mt, H->big_op, H->avg_gather, H->grad_gather, H->grad_scale, H->sub_op,
                                   H->sub_gather, H->sub_active, H->beta, lin);
    if (T.smem > kMaxSmem) {
      set_error("reconstruction tile needs %u B of shared memory (stencil too wide)", T.smem);
      return GKS_ERR_BAD_ARG;
    }
#define GKS_HWENO(HA, HG, M)                                                                                      \
  if (Kt == HA && St == HG && Mt == M) {                                                                          \
    GKS_CUDA(cudaFuncSetAttribute(k_recon_hweno<HA, HG, M>, cudaFuncAttributeMaxDynamicSharedMemorySize,          \
                                  (int)T.smem));                                                                  \
    GKS_LAUNCH(KC_RECON, (k_recon_hweno<HA, HG, M>), nbt, RT_THREADS, T.smem, H->stream, H->n_recon, q, H->grad,   \
               H->h, T, H->linear_weights, H->eps, H->lw, H->coef, gate);                                         \
    return GKS_OK;                                                                                                \
  }
    GKS_HWENO(4, 5, 4)
    GKS_HWENO(6, 7, 6)
    GKS_HWENO(16, 17, 8)
#undef GKS_HWENO
  } else {
    const WenoTile T = weno_tile(Kt, Mt, St, H->big_op, H->big_gather, H->sub_op, H->sub_gather, H->sub_active,
                                 H->beta, lin);
    if (T.smem > kMaxSmem) {
      set_error("reconstruction tile needs %u B of shared memory (stencil too wide)", T.smem);
      return GKS_ERR_BAD_ARG;
    }
#define GKS_WENO(K, M, S)                                                                                         \
  if (Kt == K && Mt == M && St == S) {                                                                            \
    GKS_CUDA(cudaFuncSetAttribute(k_recon_weno<K, M, S>, cudaFuncAttributeMaxDynamicSharedMemorySize,             \
                                  (int)T.smem));                                                                  \
    GKS_LAUNCH(KC_RECON, (k_recon_weno<K, M, S>), nbt, RT_THREADS, T.smem, H->stream, H->n_recon, q, T,            \
               H->linear_weights, H->eps, H->lw, H->coef, gate);                                                  \
    return GKS_OK;                                                                                                \
  }
    GKS_WENO(13, 4, 6)
    GKS_WENO(14, 4, 6)
    GKS_WENO(15, 4, 6)
    GKS_WENO(16, 4, 6)
    GKS_WENO(24, 8, 3)
    GKS_WENO(32, 8, 8)
#undef GKS_WENO
  }
  set_error("no reconstruction kernel for padded stencil shape (%d, %d, %d)", Kt, Mt, St);
  return GKS_ERR_BAD_ARG;
}

int residual_device(Handle* H, const double* q, double* res, bool with_gradients, const int* gate,
                    const FrechetEpi* fe) {
  // owned + layer-1 ghosts (redundant reconstruction), RT cells per CTA;
  // first order: zero coefficients (face values = cell averages, no slopes)
  if (H->first_order) {
    GKS_CUDA(cudaMemsetAsync(H->coef, 0, (size_t)H->n_recon * 45 * sizeof(double), H->stream));
  } else if (int rc = recon_device(H, q, gate)) {
    return rc;
  }
  FaceArgs A;
  A.nfq = H->nfq;
  A.q = q; A.coef = H->coef; A.cen = H->cen; A.h = H->h; A.ih = H->ih; A.avg0 = H->avg0; A.dt = H->dt;
  A.fq_face = H->fq_face; A.f_own = H->f_own; A.f_nbr = H->f_nbr; A.f_patch = H->f_patch;
  A.fq_point = H->fq_point; A.fq_ws = H->fq_ws; A.f_frame = H->f_frame; A.f_normal = H->f_normal;
  A.f_shift = H->f_shift; A.patches = H->patches; A.model = H->model; A.mu = H->mu; A.kc = H->kc;
  A.want_point = with_gradients ? 1 : 0;
  A.fq_nq = H->fq_nq;
  A.contrib = H->contrib; A.qpt = H->qpt; A.status = H->status; A.gate = gate;
  static const int slot_env = [] {
    const char* e = getenv("GKS_ASSEMBLE_SLOTS");
    return e ? atoi(e) : 0;
  }();
  // slot assembly for residuals without the gradient update
  const bool slot_mode = slot_env && !with_gradients;
  A.fq_slot = slot_mode ? H->fq_slot : nullptr;
  A.slots = H->slots;
  const int fb = blocks_for(H->nfq, GKS_FACE_T);
#define GKS_FACE(V, P)                                                                    \
  do {                                                                                    \
    if (H->first_order) GKS_LAUNCH(KC_FACE, (k_face<V, P, true>), fb, GKS_FACE_T, 0, H->stream, A); \
    else GKS_LAUNCH(KC_FACE, (k_face<V, P, false>), fb, GKS_FACE_T, 0, H->stream, A);            \
  } while (0)
  if (H->model == 1) {
    if (with_gradients) GKS_FACE(true, true);
    else GKS_FACE(true, false);
  } else {
    if (with_gradients) GKS_FACE(false, true);
    else GKS_FACE(false, false);
  }
#undef GKS_FACE
  static const int asm5 = [] {
    const char* e = getenv("GKS_ASSEMBLE5");
    return e ? atoi(e) : 1;
  }();
  static const int tile = [] {
    const char* e = getenv("GKS_ASSEMBLE_TILE");
    return e ? atoi(e) : 1;
  }();
  if (slot_mode)
    GKS_LAUNCH(KC_ASSEMBLE, k_assemble_slots, blocks_for(H->n_owned * 5, 160), 160, 0, H->stream, H->n_owned,
               H->cfq_start, H->slots, H->vol, res, gate, fe ? *fe : FrechetEpi{});
  else if (asm5 && tile && H->asm_tile && with_gradients)
    GKS_LAUNCH(KC_ASSEMBLE, k_assemble_tile_g, blocks_for(H->n_owned, AT_CELLS), AT_CELLS * 5, 0, H->stream,
               H->n_owned, H->cfq_start, H->cfq, H->contrib, H->qpt, H->fq_face, H->fq_ws, H->f_normal, H->vol, res,
               H->grad_new, gate, fe ? *fe : FrechetEpi{});
  else if (asm5 && tile && H->asm_tile && !with_gradients)
    GKS_LAUNCH(KC_ASSEMBLE, k_assemble_tile, blocks_for(H->n_owned, AT_CELLS), AT_CELLS * 5, 0, H->stream, H->n_owned,
               H->cfq_start, H->cfq, H->contrib, H->vol, res, gate, fe ? *fe : FrechetEpi{});
  else if (asm5)
    GKS_LAUNCH(KC_ASSEMBLE, k_assemble5, blocks_for(H->n_owned * 5, 160), 160, 0, H->stream, H->n_owned, H->cfq_start,
               H->cfq, H->contrib, H->qpt, H->fq_face, H->fq_ws, H->f_normal, H->vol, res,
               with_gradients ? H->grad_new : nullptr, gate, fe ? *fe : FrechetEpi{});
  else
    GKS_LAUNCH(KC_ASSEMBLE, k_assemble, blocks_for(H->n_owned, TPB), TPB, 0, H->stream, H->n_owned, H->cfq_start,
               H->cfq, H->contrib, H->qpt, H->fq_face, H->fq_ws, H->f_normal, H->vol, res,
               with_gradients ? H->grad_new : nullptr, gate, fe ? *fe : FrechetEpi{});
  GKS_CUDA(cudaGetLastError());
  return GKS_OK;
}

// ghost_state / ghost_gradients (boundary.py:66-171) of a batch of points
// on one patch: the device functions the face kernel fuses
__global__ void k_ghost_batch(int64_t n, DevPatch P, const double* __restrict__ q, const double* __restrict__ nrm,
                              const double* __restrict__ grad, KinConst kc, double* __restrict__ qg,
                              double* __restrict__ gg, int* status) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double qi[5], out[5];
  for (int k = 0; k < 5; ++k) qi[k] = q[i * 5 + k];
  const double nv[3] = {nrm[i * 3], nrm[i * 3 + 1], nrm[i * 3 + 2]};
  if (!ghost_state(qi, P, nv, kc, out)) {
    raise_dev(status, GKS_ERR_UNPHYSICAL, (int)i);
    return;
  }
  for (int k = 0; k < 5; ++k) qg[i * 5 + k] = out[k];
  if (grad) {
    double g[3][5], o[3][5];
    for (int x = 0; x < 3; ++x)
      for (int k = 0; k < 5; ++k) g[x][k] = grad[(i * 3 + x) * 5 + k];
    ghost_gradients(g, P, nv, o);
    for (int x = 0; x < 3; ++x)
      for (int k = 0; k < 5; ++k) gg[(i * 3 + x) * 5 + k] = o[x][k];
  }
}

int ghost_batch_device(int64_t n, const DevPatch& P, const double* q, const double* nrm, const double* grad,
                       const KinConst& kc, double* q_out, double* grad_out) {
  std::vector<void*> bufs;
  auto dev = [&](size_t cnt) -> double* {
    void* p = nullptr;
    if (cudaMalloc(&p, std::max<size_t>(cnt, 1) * sizeof(double)) != cudaSuccess) return nullptr;
    bufs.push_back(p);
    return (double*)p;
  };
  struct Free {
    std::vector<void*>& b;
    ~Free() {
      for (void* p : b) cudaFree(p);
    }
  } fr{bufs};
  double *dq = dev(n * 5), *dn = dev(n * 3), *dg = grad ? dev(n * 15) : nullptr, *dqo = dev(n * 5);
  double* dgo = grad ? dev(n * 15) : nullptr;
  int* dst = (int*)dev(1);
  if (!dq || !dn || !dqo || !dst || (grad && (!dg || !dgo))) {
    set_error("ghost batch: device allocation failed");
    return GKS_ERR_CUDA;
  }
  GKS_CUDA(cudaMemcpy(dq, q, n * 5 * sizeof(double), cudaMemcpyHostToDevice));
  GKS_CUDA(cudaMemcpy(dn, nrm, n * 3 * sizeof(double), cudaMemcpyHostToDevice));
  if (grad) GKS_CUDA(cudaMemcpy(dg, grad, n * 15 * sizeof(double), cudaMemcpyHostToDevice));
  const int st0[2] = {0, 0x7fffffff};
  GKS_CUDA(cudaMemcpy(dst, st0, sizeof(st0), cudaMemcpyHostToDevice));
  GKS_LAUNCH(KC_GHOST, k_ghost_batch, blocks_for(n, TPB), TPB, 0, 0, n, P, dq, dn, dg, kc, dqo, dgo, dst);
  GKS_CUDA(cudaGetLastError());
  int st[2];
  GKS_CUDA(cudaMemcpy(st, dst, sizeof(st), cudaMemcpyDeviceToHost));
  if (st[0]) {
    set_error_index(st[1]);
    set_error("unphysical interior state at point %d", st[1]);
    return st[0];
  }
  GKS_CUDA(cudaMemcpy(q_out, dqo, n * 5 * sizeof(double), cudaMemcpyDeviceToHost));
  if (grad) GKS_CUDA(cudaMemcpy(grad_out, dgo, n * 15 * sizeof(double), cudaMemcpyDeviceToHost));
  return GKS_OK;
}

// Gauss-theorem gradient of face-point values alone (hweno.py:172-194):
// the assembly kernel with zero flux contributions
int gauss_gradients_device(Handle* H, const double* qpt, double* grad_out) {
  GKS_CUDA(cudaMemsetAsync(H->contrib, 0, (size_t)H->nfq * 5 * sizeof(double), H->stream));
  GKS_LAUNCH(KC_ASSEMBLE, k_assemble5, blocks_for(H->n_owned * 5, 160), 160, 0, H->stream, H->n_owned, H->cfq_start,
             H->cfq, H->contrib, qpt, H->fq_face, H->fq_ws, H->f_normal, H->vol, H->res2, grad_out, nullptr,
             FrechetEpi{});
  GKS_CUDA(cudaGetLastError());
  return GKS_OK;
}

int boundary_ghosts_device(Handle* H, const double* q) {
  if (H->nbf == 0) return GKS_OK;
  GKS_LAUNCH(KC_GHOST, k_boundary_ghosts, blocks_for(H->nbf, TPB), TPB, 0, H->stream, H->nbf, H->boundary_faces, H->f_own,
                                                                     H->f_patch, H->f_normal, H->patches, q,
                                                                     H->kc, H->ghosts, H->status);
  GKS_CUDA(cudaGetLastError());
  return GKS_OK;
}


// ---------------------------------------------------------------------------
// reconstruction pieces of the host API (recon.py / hweno.py): candidate
// coefficients, the nonlinear combination of given candidates, and face-
// point values from given coefficients.  Generic (runtime-shaped) kernels
// over the handle's records -- the solver's own step runs the fused
// k_recon_* / k_face kernels above.
// ---------------------------------------------------------------------------

// kernel-argument view of the handle's records and geometry
struct RecView {
  int Kt, Mt, St;
  const double *big_op, *sub_op, *grad_scale, *cen, *h, *ih, *avg0, *fq_point, *f_shift;
  const int *big_gather, *sub_gather, *avg_gather, *grad_gather, *fq_face, *f_own, *f_nbr;
};

static RecView rec_view(const Handle* H) {
  return RecView{H->Kt,         H->Mt,         H->St,          H->big_op,   H->sub_op,  H->grad_scale, H->cen,
                 H->h,          H->ih,         H->avg0,        H->fq_point, H->f_shift, H->big_gather, H->sub_gather,
                 H->avg_gather, H->grad_gather, H->fq_face,    H->f_own,    H->f_nbr};
}

// candidate_coeffs (recon.py:276-283, hweno.py:139-160): the quadratic big
// candidate (nc, 9, 5) and the linear sub candidates (nc, Mout, 3, 5)
template <bool COMPACT>
__global__ void __launch_bounds__(TPB) k_recon_candidates(int64_t nc, const double* __restrict__ q,
                                                          const double* __restrict__ grad,
                                                          const double* __restrict__ h, RecView R, int Mout,
                                                          double* __restrict__ cbig, double* __restrict__ bsub) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nc * 5) return;
  const int64_t c = i / 5;
  const int k = (int)(i - c * 5);
  const double qc = q[c * 5 + k];
  const int Kt = R.Kt, Mt = R.Mt, St = R.St;
  if (!COMPACT) {
    const double* op = R.big_op + c * rec_stride_f64(9 * Kt);
    const int* gi = R.big_gather + c * rec_stride_i32(Kt);
    for (int d = 0; d < 9; ++d) {
      double acc = 0.0;
      for (int j = 0; j < Kt; ++j) acc += op[d * Kt + j] * (q[(int64_t)gi[j] * 5 + k] - qc);
      cbig[(c * 9 + d) * 5 + k] = acc;
    }
    const double* so = R.sub_op + c * rec_stride_f64(3 * Mt * St);
    const int* sg = R.sub_gather + c * rec_stride_i32(Mt * St);
    for (int m = 0; m < Mout; ++m)
      for (int d = 0; d < 3; ++d) {
        double acc = 0.0;
        for (int s2 = 0; s2 < St; ++s2) acc += so[(m * 3 + d) * St + s2] * (q[(int64_t)sg[m * St + s2] * 5 + k] - qc);
        bsub[((c * Mout + m) * 3 + d) * 5 + k] = acc;
      }
  } else {
    const int HA = Kt, HG = St, W = HA + 3 * HG;
    const double* op = R.big_op + c * rec_stride_f64(9 * W);
    const int* ag = R.avg_gather + c * rec_stride_i32(HA);
    const int* gg = R.grad_gather + c * rec_stride_i32(HG);
    const double* gs = R.grad_scale + c * rec_stride_f64(HG);
    for (int d = 0; d < 9; ++d) {
      double acc = 0.0;
      for (int j = 0; j < HA; ++j) acc += op[d * W + j] * (q[(int64_t)ag[j] * 5 + k] - qc);
      for (int g = 0; g < HG; ++g)
        for (int x = 0; x < 3; ++x) acc += op[d * W + HA + 3 * g + x] * (gs[g] * grad[((int64_t)gg[g] * 3 + x) * 5 + k]);
      cbig[(c * 9 + d) * 5 + k] = acc;
    }
    const double* so = R.sub_op + c * rec_stride_f64(21 * Mt);
    const int* sg = R.sub_gather + c * rec_stride_i32(2 * Mt);
    for (int m = 0; m < Mout; ++m) {
      const int64_t s0 = sg[m * 2], s1 = sg[m * 2 + 1];
      double rhs[7];
      rhs[0] = q[s1 * 5 + k] - qc;
      for (int x = 0; x < 3; ++x) {
        rhs[1 + x] = h[s0] * grad[(s0 * 3 + x) * 5 + k];
        rhs[4 + x] = h[s1] * grad[(s1 * 3 + x) * 5 + k];
      }
      for (int d = 0; d < 3; ++d) {
        double acc = 0.0;
        for (int s2 = 0; s2 < 7; ++s2) acc += so[(m * 3 + d) * 7 + s2] * rhs[s2];
        bsub[((c * Mout + m) * 3 + d) * 5 + k] = acc;
      }
    }
  }
}

// combine_candidates (recon.py:167-195) on given candidates: one thread per
// (cell, component) of an (n, 9, k) / (n, M, 3, k) batch, M <= 16; the
// same combine() as the fused kernels, beta symmetrised to its packed form
constexpr int CB_MAXM = 16;
__global__ void __launch_bounds__(TPB) k_combine_batch(int64_t n, int nk, int M, const double* __restrict__ cbig,
                                                       const double* __restrict__ bsub,
                                                       const int8_t* __restrict__ act,
                                                       const double* __restrict__ beta, double eps, double lw,
                                                       double* __restrict__ out, double* __restrict__ w0n,
                                                       double* __restrict__ wmn) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n * nk) return;
  const int64_t c = i / nk;
  const int k = (int)(i - c * nk);
  double cb[9], B[45], b[CB_MAXM][3];
  int8_t a[CB_MAXM];
  for (int d = 0; d < 9; ++d) cb[d] = cbig[(c * 9 + d) * nk + k];
  {
    int idx = 0;
    const double* Bc = beta + c * 81;
    for (int d = 0; d < 9; ++d)
      for (int e = d; e < 9; ++e) B[idx++] = e == d ? Bc[d * 9 + d] : 0.5 * (Bc[d * 9 + e] + Bc[e * 9 + d]);
  }
  for (int m = 0; m < CB_MAXM; ++m) {
    a[m] = m < M ? act[c * M + m] : 0;
    for (int d = 0; d < 3; ++d) b[m][d] = m < M ? bsub[((c * M + m) * 3 + d) * nk + k] : 0.0;
  }
  double wtmp[CB_MAXM];
  combine<CB_MAXM>(cb, b, a, B, eps, lw, w0n + c * nk + k, wtmp, 1);
  for (int m = 0; m < M; ++m) wmn[(c * M + m) * nk + k] = wtmp[m];
  for (int d = 0; d < 9; ++d) out[(c * 9 + d) * nk + k] = cb[d];
}

// evaluate_faces (recon.py:297-314): both sides' values / gradients at every
// face point from given coefficients; boundary points repeat the owner side
__global__ void __launch_bounds__(TPB) k_face_values(int64_t nfq, RecView R, const double* __restrict__ q,
                                                     const double* __restrict__ coef, double* __restrict__ vo,
                                                     double* __restrict__ go, double* __restrict__ vn,
                                                     double* __restrict__ gn) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nfq) return;
  const int f = R.fq_face[i];
  const int64_t own = R.f_own[f], nbr = R.f_nbr[f];
  const double x[3] = {R.fq_point[3 * i], R.fq_point[3 * i + 1], R.fq_point[3 * i + 2]};
  double v[5], g[3][5];
  eval_side(q, coef, R.cen, R.ih, R.avg0, own, x, v, g);
  for (int k = 0; k < 5; ++k) {
    vo[i * 5 + k] = v[k];
    for (int d = 0; d < 3; ++d) go[(i * 3 + d) * 5 + k] = g[d][k];
  }
  if (nbr >= 0) {
    const double xn[3] = {x[0] - R.f_shift[3 * f], x[1] - R.f_shift[3 * f + 1], x[2] - R.f_shift[3 * f + 2]};
    eval_side(q, coef, R.cen, R.ih, R.avg0, nbr, xn, v, g);
  }
  for (int k = 0; k < 5; ++k) {
    vn[i * 5 + k] = v[k];
    for (int d = 0; d < 3; ++d) gn[(i * 3 + d) * 5 + k] = g[d][k];
  }
}

// entries of the largest 32-cell tile of the assembly list fit the staging buffer
// 1 if every 32-cell tile's list segment fits k_assemble_tile's staging
int assemble_tile_fits(const int* cfq_start_host, int64_t n_owned) {
  for (int64_t c0 = 0; c0 < n_owned; c0 += AT_CELLS) {
    const int64_t ce = c0 + AT_CELLS < n_owned ? c0 + AT_CELLS : n_owned;
    if (cfq_start_host[ce] - cfq_start_host[c0] > AT_MAXE) return 0;
  }
  return 1;
}

int recon_coeffs_device(Handle* H, const double* q, int linear) {
  const int saved = H->linear_weights;
  H->linear_weights = linear;
  const int rc = recon_device(H, q, nullptr);
  H->linear_weights = saved;
  return rc;
}

int recon_candidates_device(Handle* H, const double* q, int Mout, double* cbig, double* bsub) {
  if (Mout > H->Mt) {
    set_error("candidate width %d exceeds the records (%d)", Mout, H->Mt);
    return GKS_ERR_BAD_ARG;
  }
  if (H->compact)
    GKS_LAUNCH(KC_RECON, k_recon_candidates<true>, blocks_for(H->nc * 5, TPB), TPB, 0, H->stream, H->nc, q, H->grad,
               H->h, rec_view(H), Mout, cbig, bsub);
  else
    GKS_LAUNCH(KC_RECON, k_recon_candidates<false>, blocks_for(H->nc * 5, TPB), TPB, 0, H->stream, H->nc, q, H->grad,
               H->h, rec_view(H), Mout, cbig, bsub);
  GKS_CUDA(cudaGetLastError());
  return GKS_OK;
}

int combine_batch_device(int64_t n, int nk, int M, const double* cbig, const double* bsub, const int8_t* act,
                         const double* beta, double eps, double lw, double* out, double* w0n, double* wmn,
                         cudaStream_t s) {
  if (M < 1 || M > CB_MAXM) {
    set_error("combine: %d sub-stencil slots (1..%d supported)", M, CB_MAXM);
    return GKS_ERR_BAD_ARG;
  }
  if (n * nk == 0) return GKS_OK;
  GKS_LAUNCH(KC_RECON, k_combine_batch, blocks_for(n * nk, TPB), TPB, 0, s, n, nk, M, cbig, bsub, act, beta, eps, lw,
             out, w0n, wmn);
  GKS_CUDA(cudaGetLastError());
  return GKS_OK;
}

int face_values_device(Handle* H, const double* q, const double* coef, double* vo, double* go, double* vn,
                       double* gn) {
  GKS_LAUNCH(KC_FACE, k_face_values, blocks_for(H->nfq, TPB), TPB, 0, H->stream, H->nfq, rec_view(H), q, coef, vo, go, vn, gn);
  GKS_CUDA(cudaGetLastError());
  return GKS_OK;
}

}  // namespace gks
