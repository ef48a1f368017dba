// Partition-invariant reductions (GMRES dots and norms, step norms).
//
// Every sum over cells is defined on the GLOBAL canonical cell order, so its
// value does not depend on how the cells are split across ranks or thread
// blocks:
//   values            -> segment partials  (SEG_CELLS consecutive cells)
//   segment partials  -> group partials    (G consecutive segments)
//   group partials    -> total             (all groups of the mesh)
// and every level is the same fixed fold (red_lanes + red_tree): position i of a level
// goes to lane i % 256 and accumulator (i / 256) % 4, the four accumulators
// are combined pairwise and the 256 lanes by a fixed shuffle tree.
//
// A rank owns whole groups (partitions are aligned to SEG_CELLS * G cells of
// the canonical order, red_group_cells), so it finishes its group partials
// alone; a multi-rank run exchanges only the group partials (<= 1024 doubles
// per sum, zeros outside the owner's range, so the exchange is exact) and
// every rank evaluates the same final fold.  N-rank reductions are therefore
// bitwise those of one rank, and independent of the collective's algorithm.
// Products are rounded before they are added (__dmul_rn: no FMA
// contraction), so the fold is exactly restated by a plain IEEE numpy
// evaluation (tests/_fold.py), which the tests use as its specification.
#pragma once
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

namespace gks {

constexpr int SEG_CELLS = 768;   // cells per segment (5 * 768 = 15 * 256 vector entries)
constexpr int RED_T = 256;       // threads per reduction block (one segment per block)
constexpr int RED_MAXC = 4;      // components per reduction (step stats: 3 sums + 1 min)
constexpr int RED_MAXGRP = 1024; // groups per mesh (bounds the exchanged partials)
constexpr int RED_MAXC_MD = 16;  // sum components of the CGS2 multi-dots (krylov_dim <= 14)
// buffer layout [component][group]: sums at 0 .. RED_MAXC_MD-1, the min
// component (step stats' dt) at RED_MIN_SLOT, +inf outside the owner's range
constexpr int RED_MIN_SLOT = RED_MAXC_MD;
constexpr int RED_SLOTS = RED_MAXC_MD + 1;
__host__ __device__ constexpr int red_slot(int c, int ns) { return c < ns ? c : RED_MIN_SLOT + (c - ns); }

// Segments per group for a mesh of nc_global cells: the smallest power of two
// that keeps the number of groups <= RED_MAXGRP.  A function of the global
// mesh only, so every partition of the mesh uses the same tree.
inline int red_group(int64_t nc_global) {
  const int64_t nseg = (nc_global + SEG_CELLS - 1) / SEG_CELLS;
  int g = 1;
  while ((nseg + g - 1) / g > RED_MAXGRP) g *= 2;
  return g;
}
inline int64_t red_group_cells(int64_t nc_global) { return (int64_t)SEG_CELLS * red_group(nc_global); }

struct Comm;  // gks_comm.cu

// Kernel-side description of one handle's reduction layout.
struct RedDev {
  int64_t nseg = 0;       // local segments
  int G = 1;              // segments per group
  int64_t ngrp = 0;       // local groups
  int64_t ngrp_g = 0;     // global groups
  int64_t grp_first = 0;  // global index of local group 0
  double* spart = nullptr;  // [RED_SLOTS][nseg] segment partials
  double* gpart = nullptr;  // [RED_SLOTS][ngrp_g] group partials (this rank's entries only)
  unsigned* cnt = nullptr;  // [ngrp + 1] arrival counters (self-resetting)
  int finalize = 1;         // single rank: the last block folds the group partials
};

struct RedOut {
  double* o[RED_MAXC] = {nullptr, nullptr, nullptr, nullptr};
};

// op 0: sum (identity +0, so no partial is ever -0), op 1: min (identity +inf)
template <int OP>
__device__ __forceinline__ double red_op(double a, double b) {
  return OP == 0 ? a + b : fmin(a, b);
}
template <int OP>
__device__ __forceinline__ double red_id() {
  return OP == 0 ? 0.0 : INFINITY;
}

// Fixed tree over the block's 256 lane values; every thread gets the result.
// sm: >= 9 doubles of shared memory (reused across calls after a barrier).
template <int OP>
__device__ __forceinline__ double red_tree(double v, double* sm) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = red_op<OP>(v, __shfl_down_sync(0xffffffffu, v, o));
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sm[wid] = v;
  __syncthreads();
  if (wid == 0) {
    v = lane < RED_T / 32 ? sm[lane] : red_id<OP>();
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) v = red_op<OP>(v, __shfl_down_sync(0xffffffffu, v, o));
    if (lane == 0) sm[8] = v;
  }
  __syncthreads();
  return sm[8];
}

// Per-lane part of the canonical fold of len positions: position i ->
// lane i % 256, accumulator (i / 256) % 4; accumulators are combined as
// (a0 . a1) . (a2 . a3).  get(i, v) writes the NS + NM component values of
// position i (components [0, NS) summed, [NS, NS + NM) min-reduced).
template <int NS, int NM, class Get>
__device__ __forceinline__ void red_lanes(int64_t len, Get get, double* out) {
  constexpr int NC = NS + NM;
  double a[4][NC];
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int c = 0; c < NC; ++c) a[u][c] = c < NS ? 0.0 : INFINITY;
  auto acc = [&](int u, const double* v) {
#pragma unroll
    for (int c = 0; c < NC; ++c) a[u][c] = c < NS ? a[u][c] + v[c] : fmin(a[u][c], v[c]);
  };
  int64_t i = threadIdx.x;
  double v[4][NC];
  for (; i + 3 * RED_T < len; i += 4 * RED_T) {
#pragma unroll
    for (int u = 0; u < 4; ++u) get(i + u * RED_T, v[u]);
#pragma unroll
    for (int u = 0; u < 4; ++u) acc(u, v[u]);
  }
#pragma unroll
  for (int u = 0; u < 3; ++u)
    if (i + u * RED_T < len) {
      get(i + u * RED_T, v[u]);
      acc(u, v[u]);
    }
#pragma unroll
  for (int c = 0; c < NC; ++c)
    out[c] = c < NS ? (a[0][c] + a[1][c]) + (a[2][c] + a[3][c])
                    : fmin(fmin(a[0][c], a[1][c]), fmin(a[2][c], a[3][c]));
}

template <int OP>
__device__ __forceinline__ double red_fold_arr(const double* p, int64_t len, double* sm) {
  double v;
  if (OP == 0) red_lanes<1, 0>(len, [p](int64_t i, double* o) { o[0] = __ldcg(p + i); }, &v);
  else red_lanes<0, 1>(len, [p](int64_t i, double* o) { o[0] = __ldcg(p + i); }, &v);
  return red_tree<OP>(v, sm);
}

// Finish one segment: v[c] are this thread's lane values of the segment's
// fold (components [0, NS) sums, [NS, NS + NM) mins).  Writes the segment
// partials; the last block of a group writes the group partial, and with
// R.finalize the last group folds all group partials into out.
template <int NS, int NM>
__device__ __forceinline__ void red_finish(const RedDev& R, const double* v, const RedOut& out, double* sm) {
  constexpr int NC = NS + NM;
  __shared__ bool last;
  const int64_t b = blockIdx.x;
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const double t = c < NS ? red_tree<0>(v[c], sm) : red_tree<1>(v[c], sm);
    if (threadIdx.x == 0) R.spart[red_slot(c, NS) * R.nseg + b] = t;
  }
  const int64_t gl = b / R.G;
  const int64_t g0 = gl * R.G;
  const int gsz = (int)min((int64_t)R.G, R.nseg - g0);
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicInc(R.cnt + gl, (unsigned)gsz - 1u) == (unsigned)gsz - 1u;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const double* sp = R.spart + red_slot(c, NS) * R.nseg + g0;
    const double t = c < NS ? red_fold_arr<0>(sp, gsz, sm) : red_fold_arr<1>(sp, gsz, sm);
    if (threadIdx.x == 0) R.gpart[red_slot(c, NS) * R.ngrp_g + R.grp_first + gl] = t;
  }
  if (!R.finalize) return;
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicInc(R.cnt + R.ngrp, (unsigned)R.ngrp - 1u) == (unsigned)R.ngrp - 1u;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const double* gp = R.gpart + red_slot(c, NS) * R.ngrp_g;
    const double t = c < NS ? red_fold_arr<0>(gp, R.ngrp_g, sm) : red_fold_arr<1>(gp, R.ngrp_g, sm);
    if (threadIdx.x == 0 && out.o[c]) *out.o[c] = t;
  }
}

// Multi-component sums (the CGS2 multi-dots): NC components written to
// base[0..NC-2] and last, folded like red_finish (one tree per component).
struct RedOutN {
  double* base = nullptr;  // components 0 .. NC-2
  double* last = nullptr;  // component NC-1
};

template <int NC>
__device__ __forceinline__ void red_finish_n(const RedDev& R, const double* v, const RedOutN& out, double* sm) {
  __shared__ bool last;
  const int64_t b = blockIdx.x;
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const double t = red_tree<0>(v[c], sm);
    if (threadIdx.x == 0) R.spart[c * R.nseg + b] = t;
  }
  const int64_t gl = b / R.G;
  const int64_t g0 = gl * R.G;
  const int gsz = (int)min((int64_t)R.G, R.nseg - g0);
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicInc(R.cnt + gl, (unsigned)gsz - 1u) == (unsigned)gsz - 1u;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const double t = red_fold_arr<0>(R.spart + c * R.nseg + g0, gsz, sm);
    if (threadIdx.x == 0) R.gpart[c * R.ngrp_g + R.grp_first + gl] = t;
  }
  if (!R.finalize) return;
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicInc(R.cnt + R.ngrp, (unsigned)R.ngrp - 1u) == (unsigned)R.ngrp - 1u;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const double t = red_fold_arr<0>(R.gpart + c * R.ngrp_g, R.ngrp_g, sm);
    if (threadIdx.x == 0) {
      double* o = c < NC - 1 ? out.base + c : out.last;
      if (o) *o = t;
    }
  }
}

// Multi-rank final fold over the exchanged group partials: nsrc source
// arrays (the NCCL-summed array, or every loopback rank's own array, summed
// in rank order -- exact, as all but one entry are +0 / +inf).
struct RedSrc {
  const double* p[16];
  int n;
};

}  // namespace gks
