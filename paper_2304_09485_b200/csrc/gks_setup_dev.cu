// Device-side setup: stencil selection, reconstruction geometry and the
// WENO / HWENO operators of every cell, built on the GPU straight into the
// handle's padded per-cell records (the layout gks_api.cu's host path
// uploads).  One thread per cell runs the shared per-cell code of
// gks_setup_cell.cuh (stencils.py:72-192, recon.py:60-274,
// hweno.py:45-137).  This translation unit is compiled with -fmad=false
// (build.py): with contraction off on both sides and IEEE sqrt / division,
// every record is the host build's bit for bit
// (tests/test_device_setup_gpu.py), without the host's per-cell operator
// tables (37 GB at 10^7 cells) or its OpenMP pass.
//
// Passes: k_setup_sizes (stencil sizes -> record shape upper bounds),
// k_setup_ops<COMPACT> (geometry + operators; gathers the reference layout
// leaves as padding are marked -1), k_setup_fix<COMPACT> (padding gathers ->
// 0 inside the reference widths, the cell's own id beyond them, as the host
// path's pad_records writes them).
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <vector>

#include "gks_setup_cell.cuh"
#include "gks_solver.cuh"
#include "gks_stage.cuh"

namespace gks {

bool weno_shape(int K, int M, int S, int* Kt, int* Mt, int* St);
bool hweno_shape(int HA, int HG, int M, int* At, int* Gt, int* Mt);

namespace {

constexpr int SETUP_T = 128;

#define TRY(x)           \
  do {                   \
    int _rc = (x);       \
    if (_rc) return _rc; \
  } while (0)
constexpr size_t kTail = 64;  // tail padding of every handle array (gks_api.cu kTailPad)

enum : int { SZ_K = 0, SZ_MUP, SZ_SUP, SZ_AMAX, SZ_M, SZ_S, SZ_HM, SZ_N };

__global__ void __launch_bounds__(SETUP_T) k_setup_sizes(GksMeshDesc m, int64_t n, int* sz) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  su::Stencil st;
  su::build_stencil(m, c, st);
  int sup = 0;
  for (int k = 0; k < st.nsub; ++k) sup = max(sup, st.sublen[k] - 1);
  atomicMax(&sz[SZ_K], st.nbig - 1);
  atomicMax(&sz[SZ_MUP], st.nsub);
  atomicMax(&sz[SZ_SUP], sup);
  atomicMax(&sz[SZ_AMAX], st.present());
}

struct Recs {
  // WENO: big_op (9, Kt), big_gather (Kt), sub_op (Mt, 3, St), sub_gather (Mt, St), sub_active (Mt)
  // HWENO: big_op (9, At + 3 Gt), avg_gather (At), grad_gather (Gt), grad_scale (Gt),
  //        sub_op (Mt, 21), sub_gather (Mt, 2), sub_active (Mt)
  double *big_op, *sub_op, *grad_scale, *avg0, *beta;
  int *big_gather, *sub_gather, *avg_gather, *grad_gather;
  int8_t* sub_active;
  int Kt, Mt, St;                  // WENO (Kt, Mt, St) / HWENO (At, Mt, Gt)
  int e_bop, e_bg, e_sop, e_sg;    // record strides (elements)
  int e_ag, e_gg, e_gs;            // HWENO
};

struct WenoSink {
  const Recs& r;
  int64_t c;
  __device__ void sub_op(int slot, int d, int k, double v) { r.sub_op[c * r.e_sop + (slot * 3 + d) * r.St + k] = v; }
  __device__ void sub_gather(int slot, int k, int64_t id) { r.sub_gather[c * r.e_sg + slot * r.St + k] = (int)id; }
  __device__ void sub_active(int slot) { r.sub_active[c * r.Mt + slot] = 1; }
  __device__ void drop_subs(int n) {
    for (int mm = 0; mm < n; ++mm) {
      r.sub_active[c * r.Mt + mm] = 0;
      for (int k = 0; k < 3 * r.St; ++k) r.sub_op[c * r.e_sop + mm * 3 * r.St + k] = 0.0;
      for (int k = 0; k < r.St; ++k) r.sub_gather[c * r.e_sg + mm * r.St + k] = -1;
    }
  }
  __device__ void big_op(int d, int k, double v) { r.big_op[c * r.e_bop + d * r.Kt + k] = v; }
  __device__ void big_gather(int k, int64_t id) { r.big_gather[c * r.e_bg + k] = (int)id; }
  __device__ void big_degree(int) {}
};

struct HwenoSink {
  const Recs& r;
  int64_t c;
  int na;
  __device__ void big_op(int d, int k, double v) {
    r.big_op[c * r.e_bop + d * (r.Kt + 3 * r.St) + (k < na ? k : r.Kt + (k - na))] = v;
  }
  __device__ void avg_gather(int k, int64_t id) { r.avg_gather[c * r.e_ag + k] = (int)id; }
  __device__ void grad_gather(int k, int64_t id, double h) {
    r.grad_gather[c * r.e_gg + k] = (int)id;
    r.grad_scale[c * r.e_gs + k] = h;
  }
  __device__ void big_ncols(int) {}
  __device__ void big_degree(int) {}
  __device__ void sub_op(int slot, int i, double v) { r.sub_op[c * r.e_sop + slot * 21 + i] = v; }
  __device__ void sub_gather(int slot, int64_t id) {
    r.sub_gather[c * r.e_sg + slot * 2 + 0] = (int)c;
    r.sub_gather[c * r.e_sg + slot * 2 + 1] = (int)id;
  }
  __device__ void sub_active(int slot) { r.sub_active[c * r.Mt + slot] = 1; }
  __device__ void drop_subs(int n) {
    for (int mm = 0; mm < n; ++mm) {
      r.sub_active[c * r.Mt + mm] = 0;
      for (int i = 0; i < 21; ++i) r.sub_op[c * r.e_sop + mm * 21 + i] = 0.0;
      r.sub_gather[c * r.e_sg + mm * 2] = -1;
      r.sub_gather[c * r.e_sg + mm * 2 + 1] = -1;
    }
  }
};

// geometry (avg0, packed upper triangle of beta) + operators of one cell;
// the arrays arrive zeroed, gathers are pre-marked -1 (padding)
template <bool COMPACT>
__global__ void __launch_bounds__(SETUP_T) k_setup_ops(GksMeshDesc m, int64_t n, Recs r, int* sz) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  double avg0c[9], B[81];
  su::cell_geometry(m, c, avg0c, B);
  for (int d = 0; d < 9; ++d) r.avg0[c * 9 + d] = avg0c[d];
  {
    int idx = 0;
    for (int d = 0; d < 9; ++d)
      for (int e = d; e < 9; ++e) r.beta[c * 45 + idx++] = B[d * 9 + e];
  }
  su::Stencil st;
  su::build_stencil(m, c, st);
  if (!COMPACT) {
    for (int k = 0; k < r.Kt; ++k) r.big_gather[c * r.e_bg + k] = -1;
    for (int k = 0; k < r.Mt * r.St; ++k) r.sub_gather[c * r.e_sg + k] = -1;
    WenoSink sink{r, c};
    const int res = su::weno_cell(m, c, st, avg0c, sink);
    atomicMax(&sz[SZ_M], res & 0xff);
    atomicMax(&sz[SZ_S], res >> 8);
  } else {
    for (int k = 0; k < r.Kt; ++k) r.avg_gather[c * r.e_ag + k] = -1;
    for (int k = 0; k < r.St; ++k) r.grad_gather[c * r.e_gg + k] = -1;
    for (int k = 0; k < 2 * r.Mt; ++k) r.sub_gather[c * r.e_sg + k] = -1;
    HwenoSink sink{r, c, st.present()};
    atomicMax(&sz[SZ_HM], su::hweno_cell(m, c, st, avg0c, sink));
  }
}

// padding gathers: the reference arrays' zero padding inside the reference
// widths (pad0: cell 0 of the reference numbering, i.e. 0 unless the mesh is
// renumbered -- gks_setup_subset renumbers that padding the same way), the
// cell itself beyond them (pad_records' self fill)
template <bool COMPACT>
__global__ void __launch_bounds__(256) k_setup_fix(int64_t n, Recs r, int w0, int w1, int w2, int pad0) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  const int self = (int)c;
  if (!COMPACT) {  // w0 = K, w1 = M, w2 = S
    for (int k = 0; k < r.Kt; ++k) {
      int* g = &r.big_gather[c * r.e_bg + k];
      if (*g < 0) *g = k < w0 ? pad0 : self;
    }
    for (int mm = 0; mm < r.Mt; ++mm)
      for (int k = 0; k < r.St; ++k) {
        int* g = &r.sub_gather[c * r.e_sg + mm * r.St + k];
        if (*g < 0) *g = (mm < w1 && k < w2) ? pad0 : self;
      }
  } else {  // w0 = HA, w1 = HG, w2 = HM
    for (int k = 0; k < r.Kt; ++k) {
      int* g = &r.avg_gather[c * r.e_ag + k];
      if (*g < 0) *g = k < w0 ? pad0 : self;
    }
    for (int k = 0; k < r.St; ++k) {
      int* g = &r.grad_gather[c * r.e_gg + k];
      if (*g < 0) *g = k < w1 ? pad0 : self;
    }
    for (int mm = 0; mm < r.Mt; ++mm)
      for (int j = 0; j < 2; ++j) {
        int* g = &r.sub_gather[c * r.e_sg + mm * 2 + j];
        if (*g < 0) *g = mm < w2 ? pad0 : self;
      }
  }
}

// temporary device copy of the mesh arrays the per-cell code reads
struct DevMeshCopy {
  GksMeshDesc d{};
  std::vector<void*> bufs;
  ~DevMeshCopy() {
    for (void* p : bufs) cudaFree(p);
  }
  template <class T>
  int put(const T*& dst, const T* src, size_t n) {
    if (!src) { dst = nullptr; return GKS_OK; }
    void* p = nullptr;
    GKS_CUDA(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)));
    bufs.push_back(p);
    GKS_CUDA(cudaMemcpy(p, src, n * sizeof(T), cudaMemcpyHostToDevice));
    dst = static_cast<const T*>(p);
    return GKS_OK;
  }
};

template <class T>
int dalloc(Handle* H, T** p, size_t n) {
  GKS_CUDA(cudaMalloc(p, std::max<size_t>(n, 1) * sizeof(T) + kTail));
  H->allocs.push_back(*p);
  GKS_CUDA(cudaMemset(*p, 0, std::max<size_t>(n, 1) * sizeof(T) + kTail));
  return GKS_OK;
}

inline unsigned grid_of(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

// rank-local records from the setup-mesh build: rows in local order,
// gathers renumbered to local ids, padding as k_setup_fix (pad0 = the local
// id of setup cell 0: gks_setup_subset renumbers the reference arrays' zero
// padding the same way)
template <bool COMPACT>
__global__ void __launch_bounds__(256) k_setup_place(int64_t nl, Recs s, Recs d, const int64_t* __restrict__ l2s,
                                                     const int64_t* __restrict__ s2l, int w0, int w1, int w2,
                                                     int pad0) {
  const int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= nl) return;
  const int64_t c = l2s[l];
  const int self = (int)l;
  auto map = [&](int v, bool inside) { return v < 0 ? (inside ? pad0 : self) : (int)s2l[v]; };
  for (int k = 0; k < 9; ++k) d.avg0[l * 9 + k] = s.avg0[c * 9 + k];
  for (int k = 0; k < 45; ++k) d.beta[l * 45 + k] = s.beta[c * 45 + k];
  for (int k = 0; k < s.e_bop; ++k) d.big_op[l * d.e_bop + k] = s.big_op[c * s.e_bop + k];
  for (int k = 0; k < s.e_sop; ++k) d.sub_op[l * d.e_sop + k] = s.sub_op[c * s.e_sop + k];
  for (int k = 0; k < s.Mt; ++k) d.sub_active[l * d.Mt + k] = s.sub_active[c * s.Mt + k];
  if (!COMPACT) {
    for (int k = 0; k < s.Kt; ++k) d.big_gather[l * d.e_bg + k] = map(s.big_gather[c * s.e_bg + k], k < w0);
    for (int mm = 0; mm < s.Mt; ++mm)
      for (int k = 0; k < s.St; ++k)
        d.sub_gather[l * d.e_sg + mm * s.St + k] = map(s.sub_gather[c * s.e_sg + mm * s.St + k], mm < w1 && k < w2);
  } else {
    for (int k = 0; k < s.Kt; ++k) d.avg_gather[l * d.e_ag + k] = map(s.avg_gather[c * s.e_ag + k], k < w0);
    for (int k = 0; k < s.St; ++k) {
      d.grad_gather[l * d.e_gg + k] = map(s.grad_gather[c * s.e_gg + k], k < w1);
      d.grad_scale[l * d.e_gs + k] = s.grad_scale[c * s.e_gs + k];
    }
    for (int mm = 0; mm < s.Mt; ++mm)
      for (int j = 0; j < 2; ++j) d.sub_gather[l * d.e_sg + mm * 2 + j] = map(s.sub_gather[c * s.e_sg + mm * 2 + j], mm < w2);
  }
}

}  // namespace

// Build avg0, beta and the reconstruction records of the handle's cells on
// the device (the host path's "cells" geometry + "operators" phases).  A
// rank-local handle (dom->setup_mesh set) builds on its setup mesh -- the
// local cells in ascending reference id with all their faces, so stencil
// choices match the global build -- and places the records in local order.
int device_setup(Handle* H, const GksMeshDesc* local, const GksDomainDesc* dom) {
  GKS_NVTX("gks_device_setup");
  const bool mapped = dom && dom->setup_mesh;
  const GksMeshDesc* m = mapped ? dom->setup_mesh : local;
  const int64_t nc = m->ncells, nl = local->ncells;
  if (mapped && (!dom->local_to_setup || !dom->setup_to_local)) {
    set_error("device setup: a setup mesh needs local_to_setup / setup_to_local");
    return GKS_ERR_BAD_ARG;
  }
  int nfpc = 0;
  for (int64_t c = 0; c < nc; ++c) {
    const int nf = (int)(m->cell_face_start[c + 1] - m->cell_face_start[c]);
    if ((m->cell_kind[c] == 1 && nf != 6) || (m->cell_kind[c] != 1 && nf != 4)) {
      set_error("device setup: cell %lld has %d faces (tet 4 / hex 6 only)", (long long)c, nf);
      return GKS_ERR_BAD_ARG;
    }
    nfpc = std::max(nfpc, nf);
  }
  int pad0 = 0;  // handle id of reference cell 0 (renumbered meshes / rank-local handles)
  if (mapped) {
    for (int64_t l = 0; l < nl; ++l)
      if (dom->local_to_setup[l] < 0 || dom->local_to_setup[l] >= nc) {
        set_error("device setup: local_to_setup[%lld] out of range", (long long)l);
        return GKS_ERR_BAD_ARG;
      }
    for (int64_t c = 0; c < nc; ++c)
      if (dom->setup_to_local[c] < 0 || dom->setup_to_local[c] >= nl) {
        set_error("device setup: setup_to_local[%lld] out of range", (long long)c);
        return GKS_ERR_BAD_ARG;
      }
    pad0 = (int)dom->setup_to_local[0];
  } else if (m->cell_rank) {
    for (int64_t c = 0; c < nc; ++c)
      if (m->cell_rank[c] == 0) { pad0 = (int)c; break; }
  }
  DevMeshCopy dm;
  GksMeshDesc& d = dm.d;
  d.ncells = nc; d.nfaces = m->nfaces; d.nfq = m->nfq; d.ncq = m->ncq;
  const int64_t nf = m->nfaces, ncq = m->ncq, nlist = m->cell_face_start[nc];
  TRY(dm.put(d.cell_kind, m->cell_kind, nc));
  TRY(dm.put(d.cell_h, m->cell_h, nc));
  TRY(dm.put(d.cell_centroid, m->cell_centroid, nc * 3));
  TRY(dm.put(d.cell_cq_start, m->cell_cq_start, nc + 1));
  TRY(dm.put(d.cq_point, m->cq_point, ncq * 3));
  TRY(dm.put(d.cq_weight, m->cq_weight, ncq));
  TRY(dm.put(d.cell_face_start, m->cell_face_start, nc + 1));
  TRY(dm.put(d.cell_face_list, m->cell_face_list, nlist));
  TRY(dm.put(d.face_owner, m->face_owner, nf));
  TRY(dm.put(d.face_neighbor, m->face_neighbor, nf));
  TRY(dm.put(d.face_normal, m->face_normal, nf * 3));
  TRY(dm.put(d.face_shift, m->face_shift, nf * 3));
  TRY(dm.put(d.cell_rank, m->cell_rank, nc));
  const int64_t* l2s = nullptr;
  const int64_t* s2l = nullptr;
  if (mapped) {
    TRY(dm.put(l2s, dom->local_to_setup, nl));
    TRY(dm.put(s2l, dom->setup_to_local, nc));
  }

  int* sz = nullptr;
  GKS_CUDA(cudaMalloc(&sz, SZ_N * sizeof(int)));
  dm.bufs.push_back(sz);
  GKS_CUDA(cudaMemset(sz, 0, SZ_N * sizeof(int)));
  k_setup_sizes<<<grid_of(nc, SETUP_T), SETUP_T, 0, H->stream>>>(d, nc, sz);
  GKS_CUDA(cudaGetLastError());
  int hs[SZ_N];
  GKS_CUDA(cudaMemcpyAsync(hs, sz, sizeof(hs), cudaMemcpyDeviceToHost, H->stream));
  GKS_CUDA(cudaStreamSynchronize(H->stream));

  // build records: the handle's own (single handle) or temporaries in
  // setup-mesh order (rank-local handle)
  auto balloc = [&](auto** p, size_t n) -> int {
    if (!mapped) return dalloc(H, p, n);
    const size_t bytes = std::max<size_t>(n, 1) * sizeof(**p) + kTail;
    GKS_CUDA(cudaMalloc(p, bytes));
    dm.bufs.push_back(*p);
    GKS_CUDA(cudaMemset(*p, 0, bytes));
    return GKS_OK;
  };
  auto alloc_recs = [&](Recs& r, int64_t rows, auto&& al) -> int {
    TRY(al(&r.avg0, rows * 9));
    TRY(al(&r.beta, rows * 45));
    if (!H->compact) {
      r.e_bop = rec_stride_f64(9 * r.Kt);
      r.e_bg = rec_stride_i32(r.Kt);
      r.e_sop = rec_stride_f64(r.Mt * 3 * r.St);
      r.e_sg = rec_stride_i32(r.Mt * r.St);
      TRY(al(&r.big_op, (size_t)rows * r.e_bop));
      TRY(al(&r.big_gather, (size_t)rows * r.e_bg));
    } else {
      r.e_bop = rec_stride_f64(9 * (r.Kt + 3 * r.St));
      r.e_ag = rec_stride_i32(r.Kt);
      r.e_gg = rec_stride_i32(r.St);
      r.e_gs = rec_stride_f64(r.St);
      r.e_sop = rec_stride_f64(r.Mt * 21);
      r.e_sg = rec_stride_i32(r.Mt * 2);
      TRY(al(&r.big_op, (size_t)rows * r.e_bop));
      TRY(al(&r.avg_gather, (size_t)rows * r.e_ag));
      TRY(al(&r.grad_gather, (size_t)rows * r.e_gg));
      TRY(al(&r.grad_scale, (size_t)rows * r.e_gs));
    }
    TRY(al(&r.sub_op, (size_t)rows * r.e_sop));
    TRY(al(&r.sub_gather, (size_t)rows * r.e_sg));
    TRY(al(&r.sub_active, (size_t)rows * r.Mt));
    return GKS_OK;
  };
  static_assert(rec_stride_f64(45) == 45, "beta records are stored unpadded");

  const bool compact = H->compact;
  const int K = std::max(hs[SZ_K], 1), mup = std::max(hs[SZ_MUP], 1), sup = std::max(hs[SZ_SUP], 1);
  const int HA = std::max(hs[SZ_AMAX], 1), HG = hs[SZ_AMAX] + 1;
  int Kt, Mt, St;
  if (!compact ? !weno_shape(K, mup, sup, &Kt, &Mt, &St) : !hweno_shape(HA, HG, std::max(nfpc, 1), &Kt, &St, &Mt)) {
    set_error("device setup: stencil shape (%d, %d, %d) exceeds the reconstruction kernels", K, mup, sup);
    return GKS_ERR_BAD_ARG;
  }
  for (int attempt = 0; attempt < 2; ++attempt) {
    Recs r{};
    r.Kt = Kt; r.Mt = Mt; r.St = St;
    TRY(alloc_recs(r, nc, balloc));
    if (!compact)
      k_setup_ops<false><<<grid_of(nc, SETUP_T), SETUP_T, 0, H->stream>>>(d, nc, r, sz);
    else
      k_setup_ops<true><<<grid_of(nc, SETUP_T), SETUP_T, 0, H->stream>>>(d, nc, r, sz);
    GKS_CUDA(cudaGetLastError());
    GKS_CUDA(cudaMemcpyAsync(hs, sz, sizeof(hs), cudaMemcpyDeviceToHost, H->stream));
    GKS_CUDA(cudaStreamSynchronize(H->stream));
    // exact reference widths -> the record shape the host path would pick
    int Kx, Mx, Sx;
    const int M = std::max(hs[SZ_M], 1), S = std::max(hs[SZ_S], 1), HM = std::max(hs[SZ_HM], 1);
    if (!compact ? !weno_shape(K, M, S, &Kx, &Mx, &Sx) : !hweno_shape(HA, HG, HM, &Kx, &Sx, &Mx)) {
      set_error("device setup: stencil shape exceeds the reconstruction kernels");
      return GKS_ERR_BAD_ARG;
    }
    if (Kx != Kt || Mx != Mt || Sx != St) {
      if (attempt) {
        set_error("device setup: record shape did not settle");
        return GKS_ERR_BAD_ARG;
      }
      // rebuild with the exact shape (an oversized single-handle build stays
      // allocated until the handle is destroyed; only mixed meshes get here)
      Kt = Kx; Mt = Mx; St = Sx;
      GKS_CUDA(cudaMemsetAsync(sz + SZ_M, 0, 3 * sizeof(int), H->stream));
      continue;
    }
    const int w0 = compact ? HA : K, w1 = compact ? HG : M, w2 = compact ? HM : S;
    Recs f = r;
    if (mapped) {
      f = Recs{};
      f.Kt = Kt; f.Mt = Mt; f.St = St;
      TRY(alloc_recs(f, nl, [&](auto** p, size_t n) { return dalloc(H, p, n); }));
      if (!compact)
        k_setup_place<false><<<grid_of(nl, 256), 256, 0, H->stream>>>(nl, r, f, l2s, s2l, w0, w1, w2, pad0);
      else
        k_setup_place<true><<<grid_of(nl, 256), 256, 0, H->stream>>>(nl, r, f, l2s, s2l, w0, w1, w2, pad0);
    } else if (!compact) {
      k_setup_fix<false><<<grid_of(nc, 256), 256, 0, H->stream>>>(nc, r, w0, w1, w2, pad0);
    } else {
      k_setup_fix<true><<<grid_of(nc, 256), 256, 0, H->stream>>>(nc, r, w0, w1, w2, pad0);
    }
    GKS_CUDA(cudaGetLastError());
    GKS_CUDA(cudaStreamSynchronize(H->stream));
    if (!compact) {
      H->K = K; H->M = M; H->S = S;
    } else {
      H->HA = HA; H->HG = HG; H->HM = HM;
    }
    H->avg0 = f.avg0;
    H->beta = f.beta;
    H->big_gather = f.big_gather;
    H->avg_gather = f.avg_gather;
    H->grad_gather = f.grad_gather;
    H->grad_scale = f.grad_scale;
    H->Kt = Kt; H->Mt = Mt; H->St = St;
    H->big_op = f.big_op;
    H->sub_op = f.sub_op;
    H->sub_gather = f.sub_gather;
    H->sub_active = f.sub_active;
    return GKS_OK;
  }
  set_error("device setup: record shape did not settle");
  return GKS_ERR_BAD_ARG;
}

}  // namespace gks
