// C ABI of the solver handle: creation (host CSR construction + upload),
// residual / Jacobian / GMRES / advance entry points.  Every entry point
// copies host arrays in, runs the device path and copies results out; the
// *_device variants keep the state resident for the benchmark loop.
#include <chrono>
#include <stddef.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <numeric>
#include <string>
#include <vector>

#include "gks_implicit.cuh"
#include "gks_stage.cuh"

extern "C" {
// native setup internals (gks_setup.cpp)
int gks_setup_query(const GksSetup* setup, const char* name, int* dtype, int* ndim, int64_t* shape);
int gks_setup_copy(const GksSetup* setup, const char* name, void* dst, int64_t nbytes);
}

struct GksBlockSystem {
  gks::BlockSys sys;
  bool owned = true;  // false for the handle's Jacobian view
};

// Phases of one implicit step with their own device error words, read back
// once after the step (so the step needs no host synchronisation inside and
// can be captured in a CUDA graph).
enum : int { PH_DT = 0, PH_RES, PH_GHOST, PH_N };

// Host mirror of everything the host needs after a step (pinned memory).
struct StepHost {
  int st[4 * PH_N];
  int jst[4];
  gks::DevScalars sc;
  gks::GmresDev g;
};

// One captured implicit step.  The graph bakes in the state buffers, and
// the step swaps q/q_new (grad/grad_new), so two executables alternate.
struct StepGraph {
  cudaGraphExec_t exec = nullptr;
  const double* q = nullptr;
  const double* grad = nullptr;
  int64_t launches = 0;  // kernel nodes (launch accounting on replay)
  int64_t ws_gen = 0;    // Krylov workspace generation the graph was captured against
};

struct GksHandle {
  gks::Handle H;
  GksBlockSystem jac;
  bool jac_valid = false;
  int* phase_status = nullptr;  // device, 4 * PH_N ints
  StepHost* sh = nullptr;       // pinned
  StepGraph graphs[2];
  int64_t steps = 0;            // steps advanced through this handle
  int graph = -1;               // CUDA-graph steps: -1 env default (GKS_GRAPH), 0 off, 1 on
  // staging buffers of the host-API entry points (residual, local dt,
  // Jacobian, Frechet matvec): they never overwrite the resident state
  double *api_q = nullptr, *api_grad = nullptr, *api_dt = nullptr, *api_qpt = nullptr;
};

// Swaps the handle's state pointers for the API staging buffers for the
// duration of one host-API call (uncaptured; the step graphs keep theirs).
struct ApiStage {
  gks::Handle* H;
  double *q, *grad, *dt;
  explicit ApiStage(GksHandle* G) : H(&G->H), q(G->H.q), grad(G->H.grad), dt(G->H.dt) {
    H->q = G->api_q;
    H->grad = G->api_grad;
    H->dt = G->api_dt;
  }
  ~ApiStage() {
    H->q = q;
    H->grad = grad;
    H->dt = dt;
  }
};

namespace gks {

static int setup_array(const GksSetup* S, const char* name, std::vector<double>* f, std::vector<int64_t>* i,
                       std::vector<int8_t>* b, std::vector<int64_t>* shape) {
  int dt, nd;
  int64_t shp[4];
  int rc = gks_setup_query(S, name, &dt, &nd, shp);
  if (rc) return rc;
  int64_t n = 1;
  shape->assign(shp, shp + nd);
  for (int k = 0; k < nd; ++k) n *= shp[k];
  if (dt == 0) { f->resize(n); return gks_setup_copy(S, name, f->data(), n * 8); }
  if (dt == 1) { i->resize(n); return gks_setup_copy(S, name, i->data(), n * 8); }
  b->resize(n);
  return gks_setup_copy(S, name, b->data(), n);
}

// Every device array carries 64 bytes of tail padding: the bulk-copy staging
// of the reconstruction kernels rounds a tile's chunk up to 16 bytes and may
// read up to 15 bytes past the last record (gks_stage.cuh).
static constexpr size_t kTailPad = 64;

template <class T>
static int upload(Handle* H, T** dst, const T* src, size_t n) {
  GKS_CUDA(cudaMalloc(dst, std::max<size_t>(n, 1) * sizeof(T) + kTailPad));
  H->allocs.push_back(*dst);
  if (n) GKS_CUDA(cudaMemcpy(*dst, src, n * sizeof(T), cudaMemcpyHostToDevice));
  return GKS_OK;
}

// GKS_POISON=1 builds fill every work allocation with 0xFF bytes (NaN
// doubles, -1 ints): a kernel reading device memory no kernel or copy wrote
// then turns results into NaN and the parity tests fail (the initcheck of a
// pool without compute-sanitizer).
#ifndef GKS_POISON
#define GKS_POISON 0
#endif
template <class T>
static int alloc(Handle* H, T** dst, size_t n) {
  GKS_CUDA(cudaMalloc(dst, std::max<size_t>(n, 1) * sizeof(T) + kTailPad));
  H->allocs.push_back(*dst);
  if (GKS_POISON) GKS_CUDA(cudaMemset(*dst, 0xFF, std::max<size_t>(n, 1) * sizeof(T) + kTailPad));
  return GKS_OK;
}

static std::vector<int> to_i32(const int64_t* p, size_t n) {
  std::vector<int> out(n);
  for (size_t k = 0; k < n; ++k) out[k] = (int)p[k];
  return out;
}

#define TRY(x)                 \
  do {                         \
    int _rc = (x);             \
    if (_rc) return _rc;       \
  } while (0)

// Structural memory check of every static index array before it reaches the
// device (compute-sanitizer is unavailable on the GPU pool): each gathered
// or scattered index, shifted right by `shift` (tagged CSR entries), must lie
// in [lo, hi).  All device gathers index through these arrays (or through
// indices derived from them), so a handle that passes cannot read or write
// out of bounds.
static int check_range(const char* what, const int* v, size_t n, int64_t lo, int64_t hi, int shift = 0) {
  for (size_t k = 0; k < n; ++k) {
    const int64_t x = (int64_t)(v[k] >> shift);
    if (x < lo || x >= hi) {
      set_error("index check: %s[%zu] = %lld outside [%lld, %lld)", what, k, (long long)x, (long long)lo,
                (long long)hi);
      return GKS_ERR_BAD_ARG;
    }
  }
  return GKS_OK;
}
template <class V>
static int check_vec(const char* what, const V& v, int64_t lo, int64_t hi, int shift = 0) {
  return check_range(what, v.data(), v.size(), lo, hi, shift);
}

static int upload_halo(Handle* H, HaloMap& X, const GksHaloDesc& d) {
  X.peers.assign(d.peers, d.peers + d.npeers);
  X.soff.assign(d.send_offsets, d.send_offsets + d.npeers + 1);
  X.roff.assign(d.recv_offsets, d.recv_offsets + d.npeers + 1);
  X.ns = X.soff.back();
  X.nr = X.roff.back();
  auto si = to_i32(d.send_ids, X.ns), ri = to_i32(d.recv_ids, X.nr);
  TRY(check_vec("halo send ids", si, 0, H->n_owned));
  TRY(check_vec("halo recv ids", ri, H->n_owned, H->nc));
  for (size_t p = 0; p + 1 < X.soff.size(); ++p)
    if (X.soff[p] > X.soff[p + 1] || X.roff[p] > X.roff[p + 1]) {
      set_error("halo offsets not ascending");
      return GKS_ERR_BAD_ARG;
    }
  TRY(upload(H, &X.sids, si.data(), si.size()));
  TRY(upload(H, &X.rids, ri.data(), ri.size()));
  return GKS_OK;
}

// Reconstruction records are padded per cell to a compile-time stencil
// shape of the K2 kernels (gks_solver.cu recon_device): extra operator
// columns are zero, extra gather slots point at the cell itself (so the
// right-hand side entry is Q_c - Q_c = 0 exactly), extra sub-stencils are
// inactive.  (rows, cols) -> (rows, cols_t) per cell.
template <class T, class Fill>
static std::vector<T> pad_records(const std::vector<T>& src, int64_t nc, int64_t rows, int64_t cols, int64_t rows_t,
                                  int64_t cols_t, Fill fill) {
  std::vector<T> out((size_t)nc * rows_t * cols_t);
  for (int64_t c = 0; c < nc; ++c)
    for (int64_t r = 0; r < rows_t; ++r)
      for (int64_t j = 0; j < cols_t; ++j)
        out[(c * rows_t + r) * cols_t + j] =
            (r < rows && j < cols) ? src[(c * rows + r) * cols + j] : fill(c);
  return out;
}

// Re-stride per-cell records of E entries to the staging stride (gks_stage.cuh
// rec_stride_*), zero-filled.
template <class T>
static std::vector<T> restride(const std::vector<T>& src, int64_t nc, int64_t E) {
  const int64_t Es = sizeof(T) == 8 ? rec_stride_f64((int)E) : (sizeof(T) == 4 ? rec_stride_i32((int)E) : E);
  if (Es == E) return src;
  std::vector<T> out((size_t)nc * Es, T(0));
  for (int64_t c = 0; c < nc; ++c)
    for (int64_t e = 0; e < E; ++e) out[c * Es + e] = src[c * E + e];
  return out;
}

template <class T>
static int upload_rec(Handle* H, T** dst, const std::vector<T>& src, int64_t nc) {
  const std::vector<T> v = restride(src, nc, nc ? (int64_t)src.size() / nc : 0);
  return upload(H, dst, v.data(), v.size());
}

int device_setup(Handle* H, const GksMeshDesc* m, const GksDomainDesc* dom);  // gks_setup_dev.cu

bool weno_shape(int K, int M, int S, int* Kt, int* Mt, int* St) {
  if (M <= 4 && S <= 6 && K <= 16) { *Kt = std::max(K, 13); *Mt = 4; *St = 6; return true; }
  if (M <= 8 && S <= 3 && K <= 24) { *Kt = 24; *Mt = 8; *St = 3; return true; }
  if (M <= 8 && S <= 8 && K <= 32) { *Kt = 32; *Mt = 8; *St = 8; return true; }
  return false;
}

bool hweno_shape(int HA, int HG, int M, int* At, int* Gt, int* Mt) {
  if (HA <= 4 && HG <= 5 && M <= 4) { *At = 4; *Gt = 5; *Mt = 4; return true; }
  if (HA <= 6 && HG <= 7 && M <= 6) { *At = 6; *Gt = 7; *Mt = 6; return true; }
  if (HA <= 16 && HG <= 17 && M <= 8) { *At = 16; *Gt = 17; *Mt = 8; return true; }
  return false;
}

// PatchSpec (boundary.py:26-48) -> device record: reference state as a
// primitive (rho, U, V, W, lam) (boundary.py:50-53), wall flags
static DevPatch dev_patch(const GksPatchDesc& d) {
  DevPatch P;
  P.kind = d.kind;
  P.wall = d.kind == PK_WALL_NOSLIP_ISOTHERMAL || d.kind == PK_WALL_NOSLIP_ADIABATIC ||
           d.kind == PK_WALL_SLIP_ADIABATIC;
  P.wall_moving = d.velocity[0] != 0.0 || d.velocity[1] != 0.0 || d.velocity[2] != 0.0;
  P.ref[0] = d.reference[0]; P.ref[1] = d.reference[1]; P.ref[2] = d.reference[2];
  P.ref[3] = d.reference[3];
  P.ref[4] = d.reference[0] / (2.0 * d.reference[4]);
  P.lambda_wall = d.lambda_wall;
  for (int k = 0; k < 3; ++k) P.vel[k] = d.velocity[k];
  return P;
}

int create_handle(GksHandle* G, const GksMeshDesc* m, const GksSetup* S, const GksOptions* o, int device,
                  const GksDomainDesc* dom) {
  Handle* H = &G->H;
  // GKS_SETUP_TIMING=1: host wall time of each construction phase on stderr
  const bool timing = getenv("GKS_SETUP_TIMING") != nullptr;
  auto t_last = std::chrono::steady_clock::now();
  auto tick = [&](const char* what) {
    if (!timing) return;
    auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "gks_create %-16s %8.3f s\n", what, std::chrono::duration<double>(now - t_last).count());
    t_last = now;
  };
  H->device = device;
  GKS_CUDA(cudaSetDevice(device));
  GKS_CUDA(cudaStreamCreateWithFlags(&H->stream, cudaStreamNonBlocking));
  const int64_t nc = m->ncells, nf = m->nfaces, nfq = m->nfq;
  if (nc > INT32_MAX / 16 || nfq > INT32_MAX / 2) {
    set_error("mesh too large for 32-bit device indices");
    return GKS_ERR_BAD_ARG;
  }
  H->nc = nc; H->nf = nf; H->nfq = nfq;
  H->n_owned = dom ? dom->n_owned : nc;
  H->n_recon = dom ? dom->n_recon : nc;
  H->nc_global = dom ? dom->nc_global : nc;
  H->cell_first = dom ? dom->owned_offset : 0;
  if (H->n_owned < 1 || H->n_owned > H->n_recon || H->n_recon > nc) {
    set_error("bad domain sizes (owned %lld, recon %lld, local %lld)", (long long)H->n_owned,
              (long long)H->n_recon, (long long)nc);
    return GKS_ERR_BAD_ARG;
  }
  H->scheme = o->scheme;
  H->compact = o->scheme == GKS_SCHEME_HWENO_GMRES;
  H->model = o->model;
  H->mu = o->mu; H->gamma = o->gamma; H->cfl = o->cfl;
  H->eps = o->weno_eps; H->lw = o->linear_weight;
  H->linear_weights = o->linear_weights;
  H->global_dt = o->global_time_step;
  H->jac_mode = o->jacobian_mode;
  H->first_order = o->first_order;
  H->ortho = o->ortho;
  H->krylov_dim = o->krylov_dim; H->restarts = o->restarts; H->jacobi_sweeps = o->jacobi_sweeps;
  H->gmres_rtol = o->gmres_rtol;
  H->kc = make_kin(o->gamma);

  tick("init");
  // patches
  int maxpatch = -1;
  for (int64_t f = 0; f < nf; ++f) maxpatch = std::max<int>(maxpatch, (int)m->face_patch[f]);
  if (o->npatch < maxpatch + 1) {
    set_error("options list %d patches, mesh uses %d", o->npatch, maxpatch + 1);
    return GKS_ERR_BAD_ARG;
  }
  H->npatch = o->npatch;
  H->patches_h.resize(std::max(o->npatch, 1));
  for (int p = 0; p < o->npatch; ++p) H->patches_h[p] = dev_patch(o->patches[p]);
  for (int64_t f = 0; f < nf; ++f) {
    if (m->face_neighbor[f] < 0) {
      const int p = (int)m->face_patch[f];
      if (p < 0 || H->patches_h[p].kind < 0) {
        set_error("boundary face %lld has no patch spec", (long long)f);
        return GKS_ERR_BAD_ARG;
      }
    }
  }
  TRY(upload(H, &H->patches, H->patches_h.data(), H->patches_h.size()));

  tick("patches");
  // cells
  std::vector<double> hf;
  std::vector<int64_t> hi, shp;
  std::vector<int8_t> hb;
  TRY(upload(H, &H->vol, m->cell_volume, nc));
  TRY(upload(H, &H->h, m->cell_h, nc));
  {
    std::vector<double> ih(nc);
    for (int64_t c = 0; c < nc; ++c) ih[c] = 1.0 / m->cell_h[c];
    TRY(upload(H, &H->ih, ih.data(), nc));
  }
  TRY(upload(H, &H->cen, m->cell_centroid, nc * 3));
  if (S) {  // host setup; otherwise device_setup builds avg0 / beta with the operators
  TRY(setup_array(S, "avg0", &hf, &hi, &hb, &shp));
  TRY(upload(H, &H->avg0, hf.data(), hf.size()));
  TRY(setup_array(S, "beta_mat", &hf, &hi, &hb, &shp));
  {
    // symmetric smoothness-indicator matrices: keep the upper triangle (45 of 81)
    std::vector<double> packed(nc * 45);
    for (int64_t c = 0; c < nc; ++c) {
      int idx = 0;
      for (int d = 0; d < 9; ++d)
        for (int e = d; e < 9; ++e) packed[c * 45 + idx++] = hf[c * 81 + d * 9 + e];
    }
    TRY(upload_rec(H, &H->beta, packed, nc));
  }
  }

  tick("cells");
  // faces
  {
    auto own = to_i32(m->face_owner, nf), nbr = to_i32(m->face_neighbor, nf), pat = to_i32(m->face_patch, nf);
    TRY(check_vec("face_owner", own, 0, nc));
    TRY(check_vec("face_neighbor", nbr, -1, nc));
    TRY(upload(H, &H->f_own, own.data(), nf));
    TRY(upload(H, &H->f_nbr, nbr.data(), nf));
    TRY(upload(H, &H->f_patch, pat.data(), nf));
  }
  TRY(upload(H, &H->f_area, m->face_area, nf));
  TRY(upload(H, &H->f_normal, m->face_normal, nf * 3));
  TRY(upload(H, &H->f_frame, m->face_frame, nf * 9));
  TRY(upload(H, &H->f_shift, m->face_shift, nf * 3));
  {
    auto fqf = to_i32(m->fq_face, nfq);
    TRY(check_vec("fq_face", fqf, 0, nf));
    TRY(upload(H, &H->fq_face, fqf.data(), nfq));
    // uniform points per face in face order: the face kernel derives the
    // face from the point index instead of loading it (one dependent load less)
    H->fq_nq = 0;
    if (nf > 0 && nfq % nf == 0 && nfq / nf <= 64) {
      const int nq = (int)(nfq / nf);
      bool uni = true;
      for (int64_t i = 0; i < nfq && uni; ++i) uni = fqf[i] == (int)(i / nq);
      if (uni) H->fq_nq = nq;
    }
    std::vector<double> ws(nfq);
    for (int64_t i = 0; i < nfq; ++i) ws[i] = m->fq_weight[i] * m->face_area[m->fq_face[i]];
    TRY(upload(H, &H->fq_ws, ws.data(), nfq));
  }
  TRY(upload(H, &H->fq_point, m->fq_point, nfq * 3));

  tick("faces");
  // visiting orders: the reference's face / face-point order (identity
  // unless the mesh was renumbered, reorder.py)
  std::vector<int64_t> forder(nf), qorder(nfq);
  if (m->face_rank) {
    for (int64_t f = 0; f < nf; ++f) forder[m->face_rank[f]] = f;
  } else {
    std::iota(forder.begin(), forder.end(), 0);
  }
  if (m->fq_rank) {
    for (int64_t i = 0; i < nfq; ++i) qorder[m->fq_rank[i]] = i;
  } else {
    std::iota(qorder.begin(), qorder.end(), 0);
  }

  tick("orders");
  // CSR lists (counting sorts keep ascending order inside each group)
  {
    // assembly: owner fq entries, then neighbour fq entries (stepping.py:225-228),
    // visited in the reference's face-point order
    std::vector<int> cnt(nc + 1, 0);
    for (int64_t i = 0; i < nfq; ++i) {
      const int64_t f = m->fq_face[i];
      cnt[m->face_owner[f] + 1]++;
      if (m->face_neighbor[f] >= 0) cnt[m->face_neighbor[f] + 1]++;
    }
    std::partial_sum(cnt.begin(), cnt.end(), cnt.begin());
    std::vector<int> pos(cnt.begin(), cnt.end() - 1), list(cnt[nc]);
    for (int64_t k = 0; k < nfq; ++k) {
      const int64_t i = qorder[k];
      list[pos[m->face_owner[m->fq_face[i]]]++] = (int)(i << 1);
    }
    for (int64_t k = 0; k < nfq; ++k) {
      const int64_t i = qorder[k];
      const int64_t nb = m->face_neighbor[m->fq_face[i]];
      if (nb >= 0) list[pos[nb]++] = (int)((i << 1) | 1);
    }
    TRY(upload(H, &H->cfq_start, cnt.data(), nc + 1));
    H->asm_tile = assemble_tile_fits(cnt.data(), H->n_owned);
    TRY(check_vec("assembly list", list, 0, nfq, 1));
    TRY(upload(H, &H->cfq, list.data(), list.size()));
    {
      std::vector<int2> slot(nfq, make_int2(-1, -1));
      const int64_t nent = cnt[H->n_owned];  // entries of owned cells (they come first)
      H->nent = nent;
      for (int64_t e = 0; e < nent; ++e) {
        const int v = list[e];
        if (v & 1) slot[v >> 1].y = (int)e;
        else slot[v >> 1].x = (int)e;
      }
      TRY(upload(H, &H->fq_slot, slot.data(), slot.size()));
      TRY(alloc(H, &H->slots, std::max<int64_t>(nent, 1) * 5));
    }
  }
  {
    // local dt: owner faces then neighbour faces (stepping.py:144-154)
    std::vector<int> cnt(nc + 1, 0);
    for (int64_t f = 0; f < nf; ++f) {
      cnt[m->face_owner[f] + 1]++;
      if (m->face_neighbor[f] >= 0) cnt[m->face_neighbor[f] + 1]++;
    }
    std::partial_sum(cnt.begin(), cnt.end(), cnt.begin());
    std::vector<int> pos(cnt.begin(), cnt.end() - 1), list(cnt[nc]);
    for (int64_t k = 0; k < nf; ++k) {
      const int64_t f = forder[k];
      list[pos[m->face_owner[f]]++] = (int)(f << 1);
    }
    for (int64_t k = 0; k < nf; ++k) {
      const int64_t f = forder[k];
      if (m->face_neighbor[f] >= 0) list[pos[m->face_neighbor[f]]++] = (int)((f << 1) | 1);
    }
    TRY(upload(H, &H->cdt_start, cnt.data(), nc + 1));
    TRY(check_vec("local-dt list", list, 0, nf, 1));
    TRY(upload(H, &H->cdt, list.data(), list.size()));
    // Jacobian diagonal: interior own, interior nbr, boundary own (jacobian.py:582-610)
    std::vector<int> pos2(cnt.begin(), cnt.end() - 1), list2(cnt[nc]);
    for (int64_t k = 0; k < nf; ++k) {
      const int64_t f = forder[k];
      if (m->face_neighbor[f] >= 0) list2[pos2[m->face_owner[f]]++] = (int)(f << 1);
    }
    for (int64_t k = 0; k < nf; ++k) {
      const int64_t f = forder[k];
      if (m->face_neighbor[f] >= 0) list2[pos2[m->face_neighbor[f]]++] = (int)((f << 1) | 1);
    }
    for (int64_t k = 0; k < nf; ++k) {
      const int64_t f = forder[k];
      if (m->face_neighbor[f] < 0) list2[pos2[m->face_owner[f]]++] = (int)(f << 1);
    }
    TRY(upload(H, &H->cjd_start, cnt.data(), nc + 1));
    TRY(check_vec("Jacobian-diagonal list", list2, 0, nf, 1));
    TRY(upload(H, &H->cjd, list2.data(), list2.size()));
  }
  {
    // interior / boundary face lists, Jacobian CSR (lexsort by (row, col), stable)
    // boundary faces in the reference's face order (ghost rows, stepping.py:242-249)
    std::vector<int> ifaces, bfaces, bidx(nf, -1);
    for (int64_t k = 0; k < nf; ++k) {
      const int64_t f = forder[k];
      if (m->face_neighbor[f] >= 0) ifaces.push_back((int)f);
      else { bidx[f] = (int)bfaces.size(); bfaces.push_back((int)f); }
    }
    H->nfi = ifaces.size();
    H->nbf = bfaces.size();
    const int64_t nnz = 2 * H->nfi;
    H->nnz = nnz;
    std::vector<int64_t> erow(nnz), ecol(nnz);
    for (int64_t k = 0; k < H->nfi; ++k) {
      const int64_t f = ifaces[k];
      erow[2 * k] = m->face_owner[f]; ecol[2 * k] = m->face_neighbor[f];
      erow[2 * k + 1] = m->face_neighbor[f]; ecol[2 * k + 1] = m->face_owner[f];
    }
    // columns ascending in the REFERENCE numbering (jacobian.py:181-196
    // lexsort), so a renumbered or rank-local handle sums every row's
    // off-diagonal products in the reference's order.  Stable counting sort
    // by row (rows of ghost cells live on their owner rank), then a stable
    // insertion sort of each row (at most one entry per cell face).
    const int64_t* cref = m->cell_rank;
    std::vector<int> rowptr(H->n_owned + 1, 0);
    for (int64_t e = 0; e < nnz; ++e)
      if (erow[e] < H->n_owned) rowptr[erow[e] + 1]++;
    std::partial_sum(rowptr.begin(), rowptr.end(), rowptr.begin());
    const int64_t nkept = rowptr[H->n_owned];
    std::vector<int64_t> order(std::max<int64_t>(nkept, 1));
    {
      std::vector<int> pos(rowptr.begin(), rowptr.end() - 1);
      for (int64_t e = 0; e < nnz; ++e)
        if (erow[e] < H->n_owned) order[pos[erow[e]]++] = e;
    }
    auto ckey = [&](int64_t e) { return cref ? cref[ecol[e]] : ecol[e]; };
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < H->n_owned; ++r)
      for (int64_t i = rowptr[r] + 1; i < rowptr[r + 1]; ++i)
        for (int64_t j = i; j > rowptr[r] && ckey(order[j]) < ckey(order[j - 1]); --j) std::swap(order[j], order[j - 1]);
    H->nnz = nkept;
    std::vector<int> col(std::max<int64_t>(nkept, 1)), fslot(2 * nf, -1), ent(std::max<int64_t>(nkept, 1));
    for (int64_t p = 0; p < nkept; ++p) {
      const int64_t e = order[p];
      col[p] = (int)ecol[e];
      ent[p] = (ifaces[e / 2] << 1) | (int)(e & 1);
      fslot[2 * ifaces[e / 2] + (e & 1)] = (int)p;
    }
    TRY(upload(H, &H->interior_faces, ifaces.data(), ifaces.size()));
    TRY(upload(H, &H->boundary_faces, bfaces.data(), bfaces.size()));
    TRY(upload(H, &H->face_slot, fslot.data(), fslot.size()));
    TRY(upload(H, &H->bidx, bidx.data(), bidx.size()));
    BlockSys* A = &G->jac.sys;
    TRY(blocksys_alloc(A, H->n_owned, nkept, H->stream));
    A->n_ext = H->n_recon;
    A->red_nc_global = H->nc_global;
    A->red_cell_first = H->cell_first;
    A->canonical = dom ? 1 : 0;
    GKS_CUDA(cudaMemcpy(A->rowptr, rowptr.data(), (H->n_owned + 1) * sizeof(int), cudaMemcpyHostToDevice));
    TRY(check_vec("Jacobian columns", col, 0, H->n_recon));
    TRY(check_range("Jacobian entries", ent.data(), (size_t)nkept, 0, nf, 1));
    if (nkept) GKS_CUDA(cudaMemcpy(A->col, col.data(), nkept * sizeof(int), cudaMemcpyHostToDevice));
    G->jac.owned = false;
    // matrix-free Roe products for the handle's Jacobian (GKS_ROE_MF=0 streams the stored blocks)
    const char* mf = getenv("GKS_ROE_MF");
    A->mf = (mf && mf[0] == '0') ? 0 : 1;
    A->gm1 = o->gamma - 1.0;
    TRY(upload(H, &A->ent, ent.data(), ent.size()));
    TRY(alloc(H, &A->fdat, (size_t)std::max<int64_t>(nf, 1) * MF_REC));
    TRY(alloc(H, &A->prim, (size_t)nc * MF_REC));
  }

  tick("csr+jacobian");
  // reconstruction operators
  // (records padded to the kernel's stencil shape, see pad_records)
  auto zero_d = [](int64_t) { return 0.0; };
  auto self_i = [](int64_t c) { return (int)c; };
  auto zero_b = [](int64_t) { return (int8_t)0; };
  if (!S) {
    // device-side setup (gks_setup_dev.cu): stencils, geometry and operators
    // built on the GPU into the same records
    TRY(device_setup(H, m, dom));
  } else if (H->compact) {
    std::vector<double> op, gs, so;
    std::vector<int> ag, gg, sg;
    std::vector<int8_t> act;
    TRY(setup_array(S, "hweno_big_op", &op, &hi, &hb, &shp));
    TRY(setup_array(S, "hweno_big_avg_gather", &hf, &hi, &hb, &shp));
    H->HA = (int)shp[1];
    ag = to_i32(hi.data(), hi.size());
    TRY(setup_array(S, "hweno_big_grad_gather", &hf, &hi, &hb, &shp));
    H->HG = (int)shp[1];
    gg = to_i32(hi.data(), hi.size());
    TRY(setup_array(S, "hweno_big_grad_scale", &gs, &hi, &hb, &shp));
    TRY(setup_array(S, "hweno_sub_op", &so, &hi, &hb, &shp));
    H->HM = (int)shp[1];
    TRY(setup_array(S, "hweno_sub_gather", &hf, &hi, &hb, &shp));
    sg = to_i32(hi.data(), hi.size());
    TRY(setup_array(S, "hweno_sub_active", &hf, &hi, &act, &shp));
    int At, Gt, Mt;
    if (!hweno_shape(H->HA, H->HG, H->HM, &At, &Gt, &Mt)) {
      set_error("HWENO stencil shape (%d, %d, %d) exceeds the reconstruction kernels", H->HA, H->HG, H->HM);
      return GKS_ERR_BAD_ARG;
    }
    H->Kt = At; H->St = Gt; H->Mt = Mt;
    // big operator columns: [averages HA | gradients 3 HG] -> [At | 3 Gt]
    {
      const int W = H->HA + 3 * H->HG, Wt = At + 3 * Gt;
      std::vector<double> opt((size_t)nc * 9 * Wt, 0.0);
      for (int64_t c = 0; c < nc; ++c)
        for (int d = 0; d < 9; ++d) {
          const double* src = &op[(c * 9 + d) * W];
          double* dst = &opt[(c * 9 + d) * Wt];
          for (int j = 0; j < H->HA; ++j) dst[j] = src[j];
          for (int j = 0; j < 3 * H->HG; ++j) dst[At + j] = src[H->HA + j];
        }
      TRY(upload_rec(H, &H->big_op, opt, nc));
    }
    {
      auto v = pad_records(ag, nc, 1, H->HA, 1, At, self_i);
      TRY(check_range("HWENO average gathers", v.data(), (size_t)H->n_recon * At, 0, nc));
      TRY(upload_rec(H, &H->avg_gather, v, nc));
    }
    {
      auto v = pad_records(gg, nc, 1, H->HG, 1, Gt, self_i);
      TRY(check_range("HWENO gradient gathers", v.data(), (size_t)H->n_recon * Gt, 0, nc));
      TRY(upload_rec(H, &H->grad_gather, v, nc));
    }
    { auto v = pad_records(gs, nc, 1, H->HG, 1, Gt, zero_d); TRY(upload_rec(H, &H->grad_scale, v, nc)); }
    { auto v = pad_records(so, nc, H->HM, 21, Mt, 21, zero_d); TRY(upload_rec(H, &H->sub_op, v, nc)); }
    {
      auto v = pad_records(sg, nc, H->HM, 2, Mt, 2, self_i);
      TRY(check_range("HWENO sub-stencil gathers", v.data(), (size_t)H->n_recon * Mt * 2, 0, nc));
      TRY(upload_rec(H, &H->sub_gather, v, nc));
    }
    { auto v = pad_records(act, nc, 1, H->HM, 1, Mt, zero_b); TRY(upload_rec(H, &H->sub_active, v, nc)); }
  } else {
    std::vector<double> op, so;
    std::vector<int> bg, sg;
    std::vector<int8_t> act;
    TRY(setup_array(S, "weno_big_op", &op, &hi, &hb, &shp));
    H->K = (int)shp[2];
    TRY(setup_array(S, "weno_big_gather", &hf, &hi, &hb, &shp));
    bg = to_i32(hi.data(), hi.size());
    TRY(setup_array(S, "weno_sub_op", &so, &hi, &hb, &shp));
    H->M = (int)shp[1];
    H->S = (int)shp[3];
    TRY(setup_array(S, "weno_sub_gather", &hf, &hi, &hb, &shp));
    sg = to_i32(hi.data(), hi.size());
    TRY(setup_array(S, "weno_sub_active", &hf, &hi, &act, &shp));
    int Kt, Mt, St;
    if (!weno_shape(H->K, H->M, H->S, &Kt, &Mt, &St)) {
      set_error("WENO stencil shape (%d, %d, %d) exceeds the reconstruction kernels", H->K, H->M, H->S);
      return GKS_ERR_BAD_ARG;
    }
    H->Kt = Kt; H->Mt = Mt; H->St = St;
    { auto v = pad_records(op, nc, 9, H->K, 9, Kt, zero_d); TRY(upload_rec(H, &H->big_op, v, nc)); }
    {
      auto v = pad_records(bg, nc, 1, H->K, 1, Kt, self_i);
      TRY(check_range("WENO big-stencil gathers", v.data(), (size_t)H->n_recon * Kt, 0, nc));
      TRY(upload_rec(H, &H->big_gather, v, nc));
    }
    {
      // sub operator (M, 3, S) -> (Mt, 3, St)
      auto v = pad_records(so, nc * H->M, 3, H->S, 3, St, zero_d);  // pad S
      auto w = pad_records(v, nc, H->M, 3 * St, Mt, 3 * St, zero_d);  // pad M
      TRY(upload_rec(H, &H->sub_op, w, nc));
    }
    {
      std::vector<int> v((size_t)nc * Mt * St);
      for (int64_t c = 0; c < nc; ++c)
        for (int mm = 0; mm < Mt; ++mm)
          for (int s2 = 0; s2 < St; ++s2)
            v[(c * Mt + mm) * St + s2] = (mm < H->M && s2 < H->S) ? sg[(c * H->M + mm) * H->S + s2] : (int)c;
      TRY(check_range("WENO sub-stencil gathers", v.data(), (size_t)H->n_recon * Mt * St, 0, nc));
      TRY(upload_rec(H, &H->sub_gather, v, nc));
    }
    { auto v = pad_records(act, nc, 1, H->M, 1, Mt, zero_b); TRY(upload_rec(H, &H->sub_active, v, nc)); }
  }

  tick("operators");
  // state and work buffers
  TRY(alloc(H, &H->q, nc * 5));
  TRY(alloc(H, &G->api_q, nc * 5));
  TRY(alloc(H, &G->api_grad, nc * 15));
  TRY(alloc(H, &G->api_dt, nc));
  GKS_CUDA(cudaMemset(G->api_grad, 0, nc * 15 * sizeof(double)));
  TRY(alloc(H, &H->grad, nc * 15));
  TRY(alloc(H, &H->dt, nc));
  TRY(alloc(H, &H->coef, nc * 45));
  TRY(alloc(H, &H->contrib, nfq * 5));
  TRY(alloc(H, &H->qpt, H->compact ? nfq * 5 : 1));
  TRY(alloc(H, &H->res, nc * 5));
  TRY(alloc(H, &H->grad_new, nc * 15));
  TRY(alloc(H, &H->ghosts, std::max<int64_t>(H->nbf, 1) * 5));
  TRY(alloc(H, &H->q_new, nc * 5));
  TRY(alloc(H, &H->dq, nc * 5));
  TRY(alloc(H, &H->qtmp, nc * 5));
  TRY(alloc(H, &H->res2, nc * 5));
  TRY(alloc(H, &H->bad, nc));
  TRY(alloc(H, &H->scal, 1));
  GKS_CUDA(cudaMemset(H->scal, 0, sizeof(DevScalars)));
  TRY(alloc(H, &H->status, 4));
  TRY(alloc(H, &G->phase_status, 4 * PH_N));
  GKS_CUDA(cudaMallocHost(&G->sh, sizeof(StepHost)));
  GKS_CUDA(cudaMemset(H->grad, 0, nc * 15 * sizeof(double)));
  if (dom) {
    TRY(upload_halo(H, H->hq, dom->q));
    TRY(upload_halo(H, H->hx, dom->x));
    const int64_t mx = std::max(std::max(H->hq.ns, H->hq.nr), std::max(H->hx.ns, H->hx.nr));
    TRY(alloc(H, &H->hsend, std::max<int64_t>(mx, 1) * 15 * 2));  // two parity halves (loopback)
    H->hsend_half = std::max<int64_t>(mx, 1) * 15;
    TRY(alloc(H, &H->hrecv, std::max<int64_t>(mx, 1) * 15));
  }
  tick("buffers");
  return GKS_OK;
}

void destroy_handle(GksHandle* G) {
  Handle* H = &G->H;
  cudaSetDevice(H->device);
  comm_destroy(H);
  if (H->stream) cudaStreamSynchronize(H->stream);
  for (StepGraph& g : G->graphs)
    if (g.exec) cudaGraphExecDestroy(g.exec);
  if (G->sh) cudaFreeHost(G->sh);
  for (void* p : H->allocs) cudaFree(p);
  blocksys_free(&G->jac.sys);
  if (H->stream) cudaStreamDestroy(H->stream);
}

int jacobian_assemble(Handle* H, BlockSys* A, const double* ghosts_dev);

}  // namespace gks

using namespace gks;

namespace {
struct DevTmp {
  std::vector<void*> p;
  ~DevTmp() {
    for (void* x : p) cudaFree(x);
  }
  template <class T>
  T* get(size_t n) {
    void* x = nullptr;
    if (cudaMalloc(&x, std::max<size_t>(n, 1) * sizeof(T)) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    p.push_back(x);
    return (T*)x;
  }
};
}  // namespace

static int no_device() {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    set_error("no CUDA device visible: the B200 path has no CPU fallback");
    return GKS_ERR_NO_DEVICE;
  }
  return GKS_OK;
}

extern "C" {

int gks_create(const GksMeshDesc* mesh, const GksSetup* setup, const GksOptions* opt, int device,
               GksHandle** out) {
  GKS_NVTX("gks_create");
  set_error_index(-1);
  if (!mesh || !opt || !out) {
    set_error("gks_create: bad arguments");
    return GKS_ERR_BAD_ARG;
  }
  if (int rc = no_device()) return rc;
  // setup == NULL: stencils and operators are built on the device
  GksHandle* G = new GksHandle();
  int rc = create_handle(G, mesh, setup, opt, device, nullptr);
  if (rc) {
    destroy_handle(G);
    delete G;
    return rc;
  }
  *out = G;
  return GKS_OK;
}

int gks_create_local(const GksMeshDesc* mesh, const GksSetup* setup, const GksOptions* opt,
                     const GksDomainDesc* domain, int device, GksHandle** out) {
  GKS_NVTX("gks_create_local");
  set_error_index(-1);
  if (!mesh || !opt || !out || !domain || (!setup && !domain->setup_mesh)) {
    set_error("gks_create_local: bad arguments");
    return GKS_ERR_BAD_ARG;
  }
  if (int rc = no_device()) return rc;
  GksHandle* G = new GksHandle();
  int rc = create_handle(G, mesh, setup, opt, device, domain);
  if (rc) {
    destroy_handle(G);
    delete G;
    return rc;
  }
  *out = G;
  return GKS_OK;
}

static int comm_attach(GksHandle* G);

int gks_comm_init(GksHandle* G, const void* unique_id, int nranks, int rank) {
  Handle* H = &G->H;
  if (H->comm) {
    set_error("handle already has a communicator");
    return GKS_ERR_BAD_ARG;
  }
  TRY(comm_init(H, unique_id, nranks, rank));
  return comm_attach(G);
}

int gks_comm_init_loopback(GksHandle* G, GksLoopback* lb, int rank) {
  Handle* H = &G->H;
  if (H->comm || !lb) {
    set_error(H->comm ? "handle already has a communicator" : "null loopback group");
    return GKS_ERR_BAD_ARG;
  }
  TRY(comm_init_loopback(H, loopback_group(lb), rank));
  G->graph = 0;  // cross-stream event waits: steps run uncaptured
  return comm_attach(G);
}

static int comm_attach(GksHandle* G) {
  Handle* H = &G->H;
  // captured steps predate the communicator: re-capture with the exchanges
  for (StepGraph& g : G->graphs) {
    if (g.exec) cudaGraphExecDestroy(g.exec);
    g = StepGraph();
  }
  BlockSys* A = &G->jac.sys;
  A->halo_x = [H](double* x) { halo_exchange(H, H->hx, x, 5, H->stream); };
  A->comm = H->comm;
  krylov_free(&A->ws);  // the reduction layout changes (group-partial exchange)
  return GKS_OK;
}

void gks_destroy(GksHandle* G) {
  if (!G) return;
  destroy_handle(G);
  delete G;
}

int64_t gks_num_boundary_faces(const GksHandle* G) { return G ? G->H.nbf : -1; }

int gks_handle_array(GksHandle* G, const char* name, void* dst, int64_t* nbytes) {
  if (!G || !name || !nbytes) return GKS_ERR_BAD_ARG;
  Handle* H = &G->H;
  const int64_t nc = H->nc;
  const std::string n(name);
  const void* src = nullptr;
  int64_t bytes = 0;
  const bool c = H->compact;
  if (n == "avg0") { src = H->avg0; bytes = nc * 9 * 8; }
  else if (n == "beta") { src = H->beta; bytes = nc * rec_stride_f64(45) * 8; }
  else if (n == "big_op") { src = H->big_op; bytes = nc * rec_stride_f64(9 * (c ? H->Kt + 3 * H->St : H->Kt)) * 8; }
  else if (n == "big_gather" && !c) { src = H->big_gather; bytes = nc * rec_stride_i32(H->Kt) * 4; }
  else if (n == "sub_op") { src = H->sub_op; bytes = nc * rec_stride_f64(c ? H->Mt * 21 : H->Mt * 3 * H->St) * 8; }
  else if (n == "sub_gather") { src = H->sub_gather; bytes = nc * rec_stride_i32(c ? H->Mt * 2 : H->Mt * H->St) * 4; }
  else if (n == "sub_active") { src = H->sub_active; bytes = nc * H->Mt; }
  else if (n == "avg_gather" && c) { src = H->avg_gather; bytes = nc * rec_stride_i32(H->Kt) * 4; }
  else if (n == "grad_gather" && c) { src = H->grad_gather; bytes = nc * rec_stride_i32(H->St) * 4; }
  else if (n == "grad_scale" && c) { src = H->grad_scale; bytes = nc * rec_stride_f64(H->St) * 8; }
  else {
    set_error("gks_handle_array: unknown array '%s' for this scheme", name);
    return GKS_ERR_BAD_ARG;
  }
  if (!dst) { *nbytes = bytes; return GKS_OK; }
  if (*nbytes != bytes) {
    set_error("gks_handle_array: '%s' needs %lld bytes", name, (long long)bytes);
    return GKS_ERR_BAD_ARG;
  }
  GKS_CUDA(cudaSetDevice(H->device));
  GKS_CUDA(cudaStreamSynchronize(H->stream));
  GKS_CUDA(cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost));
  return GKS_OK;
}

int64_t gks_reduction_granularity(int64_t nc_global) { return red_group_cells(nc_global); }

int gks_local_dt(GksHandle* G, const double* q, double* dt_out) {
  GKS_NVTX("gks_local_dt");
  Handle* H = &G->H;
  set_error_index(-1);
  GKS_CUDA(cudaSetDevice(H->device));
  ApiStage stage(G);
  GKS_CUDA(cudaMemcpyAsync(H->q, q, H->nc * 5 * sizeof(double), cudaMemcpyHostToDevice, H->stream));
  reset_status(H);
  if (int rc = local_dt_device(H)) return rc;
  if (int rc = check_status(H, "local_time_step")) return rc;
  GKS_CUDA(cudaMemcpyAsync(dt_out, H->dt, H->nc * sizeof(double), cudaMemcpyDeviceToHost, H->stream));
  GKS_CUDA(cudaStreamSynchronize(H->stream));
  return GKS_OK;
}

int gks_residual(GksHandle* G, const double* q, const double* grad, const double* dt, int with_gradients,
                 double* res_out, double* grad_out) {
  GKS_NVTX("gks_residual");
  Handle* H = &G->H;
  set_error_index(-1);
  GKS_CUDA(cudaSetDevice(H->device));
  if (H->compact && !grad) {
    set_error("compact scheme needs a gradient field");
    return GKS_ERR_BAD_ARG;
  }
  ApiStage stage(G);
  GKS_CUDA(cudaMemcpyAsync(H->q, q, H->nc * 5 * sizeof(double), cudaMemcpyHostToDevice, H->stream));
  if (grad) GKS_CUDA(cudaMemcpyAsync(H->grad, grad, H->nc * 15 * sizeof(double), cudaMemcpyHostToDevice, H->stream));
  GKS_CUDA(cudaMemcpyAsync(H->dt, dt, H->nc * sizeof(double), cudaMemcpyHostToDevice, H->stream));
  reset_status(H);
  if (int rc = residual_device(H, H->q, H->res, with_gradients != 0, nullptr)) return rc;
  if (int rc = check_status(H, "residual")) return rc;
  GKS_CUDA(cudaMemcpyAsync(res_out, H->res, H->nc * 5 * sizeof(double), cudaMemcpyDeviceToHost, H->stream));
  if (with_gradients && grad_out)
    GKS_CUDA(cudaMemcpyAsync(grad_out, H->grad_new, H->nc * 15 * sizeof(double), cudaMemcpyDeviceToHost, H->stream));
  GKS_CUDA(cudaStreamSynchronize(H->stream));
  return GKS_OK;
}

int gks_ghost_batch(int64_t n, const GksPatchDesc* patch, const double* q, const double* normal,
                    const double* grad, double gamma, double* q_out, double* grad_out) {
  set_error_index(-1);
  if (n < 0 || !patch || !q || !normal || !q_out || (grad && !grad_out)) {
    set_error("gks_ghost_batch: bad arguments");
    return GKS_ERR_BAD_ARG;
  }
  if (patch->kind < PK_WALL_NOSLIP_ISOTHERMAL || patch->kind > PK_SUPERSONIC_OUTLET) {
    set_error("patch kind %d has no ghost state", patch->kind);
    return GKS_ERR_BAD_ARG;
  }
  if (n == 0) return GKS_OK;
  if (int rc = no_device()) return rc;
  return ghost_batch_device(n, dev_patch(*patch), q, normal, grad, make_kin(gamma), q_out, grad_out);
}

// reconstruction pieces of recon.py / hweno.py on the handle's cells
int gks_recon_coeffs(GksHandle* G, const double* q, const double* grad, int linear, double* coef) {
  Handle* H = &G->H;
  set_error_index(-1);
  if (!q || !coef || (H->compact && !grad)) {
    set_error("gks_recon_coeffs: bad arguments (the compact scheme needs gradients)");
    return GKS_ERR_BAD_ARG;
  }
  if (H->n_recon != H->nc) {
    set_error("gks_recon_coeffs: rank-local handles reconstruct owned + layer-1 cells only");
    return GKS_ERR_BAD_ARG;
  }
  GKS_CUDA(cudaSetDevice(H->device));
  ApiStage stage(G);
  GKS_CUDA(cudaMemcpyAsync(H->q, q, H->nc * 5 * sizeof(double), cudaMemcpyHostToDevice, H->stream));
  if (grad) GKS_CUDA(cudaMemcpyAsync(H->grad, grad, H->nc * 15 * sizeof(double), cudaMemcpyHostToDevice, H->stream));
  if (int rc = recon_coeffs_device(H, H->q, linear ? 1 : 0)) return rc;
  GKS_CUDA(cudaMemcpyAsync(coef, H->coef, H->nc * 45 * sizeof(double), cudaMemcpyDeviceToHost, H->stream));
  GKS_CUDA(cudaStreamSynchronize(H->stream));
  return GKS_OK;
}


int gks_recon_candidates(GksHandle* G, const double* q, const double* grad, double* c_big, double* b_sub) {
  Handle* H = &G->H;
  set_error_index(-1);
  if (!q || !c_big || !b_sub || (H->compact && !grad)) {
    set_error("gks_recon_candidates: bad arguments (the compact scheme needs gradients)");
    return GKS_ERR_BAD_ARG;
  }
  GKS_CUDA(cudaSetDevice(H->device));
  const int M = H->compact ? H->HM : H->M;
  DevTmp t;
  double* cb = t.get<double>(H->nc * 45);
  double* bs = t.get<double>(H->nc * M * 15);
  if (!cb || !bs) {
    set_error("gks_recon_candidates: device allocation failed");
    return GKS_ERR_CUDA;
  }
  ApiStage stage(G);
  GKS_CUDA(cudaMemcpyAsync(H->q, q, H->nc * 5 * sizeof(double), cudaMemcpyHostToDevice, H->stream));
  if (grad) GKS_CUDA(cudaMemcpyAsync(H->grad, grad, H->nc * 15 * sizeof(double), cudaMemcpyHostToDevice, H->stream));
  if (int rc = recon_candidates_device(H, H->q, M, cb, bs)) return rc;
  GKS_CUDA(cudaMemcpyAsync(c_big, cb, H->nc * 45 * sizeof(double), cudaMemcpyDeviceToHost, H->stream));
  GKS_CUDA(cudaMemcpyAsync(b_sub, bs, H->nc * M * 15 * sizeof(double), cudaMemcpyDeviceToHost, H->stream));
  GKS_CUDA(cudaStreamSynchronize(H->stream));
  return GKS_OK;
}

int gks_face_values(GksHandle* G, const double* q, const double* coef, double* val_o, double* grad_o, double* val_n,
                    double* grad_n) {
  Handle* H = &G->H;
  set_error_index(-1);
  if (!q || !coef || !val_o || !grad_o || !val_n || !grad_n) {
    set_error("gks_face_values: bad arguments");
    return GKS_ERR_BAD_ARG;
  }
  GKS_CUDA(cudaSetDevice(H->device));
  const int64_t nfq = H->nfq;
  DevTmp t;
  double* vo = t.get<double>(nfq * 5);
  double* go = t.get<double>(nfq * 15);
  double* vn = t.get<double>(nfq * 5);
  double* gn = t.get<double>(nfq * 15);
  if (!vo || !go || !vn || !gn) {
    set_error("gks_face_values: device allocation failed");
    return GKS_ERR_CUDA;
  }
  ApiStage stage(G);
  GKS_CUDA(cudaMemcpyAsync(H->q, q, H->nc * 5 * sizeof(double), cudaMemcpyHostToDevice, H->stream));
  GKS_CUDA(cudaMemcpyAsync(H->coef, coef, H->nc * 45 * sizeof(double), cudaMemcpyHostToDevice, H->stream));
  if (int rc = face_values_device(H, H->q, H->coef, vo, go, vn, gn)) return rc;
  GKS_CUDA(cudaMemcpyAsync(val_o, vo, nfq * 5 * sizeof(double), cudaMemcpyDeviceToHost, H->stream));
  GKS_CUDA(cudaMemcpyAsync(grad_o, go, nfq * 15 * sizeof(double), cudaMemcpyDeviceToHost, H->stream));
  GKS_CUDA(cudaMemcpyAsync(val_n, vn, nfq * 5 * sizeof(double), cudaMemcpyDeviceToHost, H->stream));
  GKS_CUDA(cudaMemcpyAsync(grad_n, gn, nfq * 15 * sizeof(double), cudaMemcpyDeviceToHost, H->stream));
  GKS_CUDA(cudaStreamSynchronize(H->stream));
  return GKS_OK;
}

int gks_combine_candidates(int64_t n, int k, int m, const double* c_big, const double* b_sub, const int8_t* active,
                           const double* beta, double eps, double lin_weight, double* out, double* w0n,
                           double* wmn) {
  set_error_index(-1);
  if (n < 0 || k < 1 || m < 1 || !c_big || !b_sub || !active || !beta || !out || !w0n || !wmn) {
    set_error("gks_combine_candidates: bad arguments");
    return GKS_ERR_BAD_ARG;
  }
  if (n == 0) return GKS_OK;
  if (int rc = no_device()) return rc;
  DevTmp t;
  double* cb = t.get<double>(n * 9 * k);
  double* bs = t.get<double>(n * m * 3 * k);
  int8_t* ac = t.get<int8_t>(n * m);
  double* be = t.get<double>(n * 81);
  double* o = t.get<double>(n * 9 * k);
  double* w0 = t.get<double>(n * k);
  double* wm = t.get<double>(n * m * k);
  if (!cb || !bs || !ac || !be || !o || !w0 || !wm) {
    set_error("gks_combine_candidates: device allocation failed");
    return GKS_ERR_CUDA;
  }
  GKS_CUDA(cudaMemcpy(cb, c_big, n * 9 * k * sizeof(double), cudaMemcpyHostToDevice));
  GKS_CUDA(cudaMemcpy(bs, b_sub, n * m * 3 * k * sizeof(double), cudaMemcpyHostToDevice));
  GKS_CUDA(cudaMemcpy(ac, active, n * m, cudaMemcpyHostToDevice));
  GKS_CUDA(cudaMemcpy(be, beta, n * 81 * sizeof(double), cudaMemcpyHostToDevice));
  if (int rc = combine_batch_device(n, k, m, cb, bs, ac, be, eps, lin_weight, o, w0, wm, 0)) return rc;
  GKS_CUDA(cudaMemcpy(out, o, n * 9 * k * sizeof(double), cudaMemcpyDeviceToHost));
  GKS_CUDA(cudaMemcpy(w0n, w0, n * k * sizeof(double), cudaMemcpyDeviceToHost));
  GKS_CUDA(cudaMemcpy(wmn, wm, n * m * k * sizeof(double), cudaMemcpyDeviceToHost));
  return GKS_OK;
}

int gks_update_gradients(GksHandle* G, const double* qpt, double* grad_out) {
  Handle* H = &G->H;
  set_error_index(-1);
  GKS_CUDA(cudaSetDevice(H->device));
  if (!G->api_qpt) TRY(alloc(H, &G->api_qpt, H->nfq * 5));
  GKS_CUDA(cudaMemcpyAsync(G->api_qpt, qpt, H->nfq * 5 * sizeof(double), cudaMemcpyHostToDevice, H->stream));
  TRY(gauss_gradients_device(H, G->api_qpt, G->api_grad));
  GKS_CUDA(cudaMemcpyAsync(grad_out, G->api_grad, H->n_owned * 15 * sizeof(double), cudaMemcpyDeviceToHost,
                           H->stream));
  GKS_CUDA(cudaStreamSynchronize(H->stream));
  return GKS_OK;
}

int gks_boundary_ghosts(GksHandle* G, const double* q, double* ghosts_out) {
  Handle* H = &G->H;
  set_error_index(-1);
  GKS_CUDA(cudaSetDevice(H->device));
  if (H->nbf == 0) return GKS_OK;
  GKS_CUDA(cudaMemcpyAsync(H->qtmp, q, H->nc * 5 * sizeof(double), cudaMemcpyHostToDevice, H->stream));
  reset_status(H);
  if (int rc = boundary_ghosts_device(H, H->qtmp)) return rc;
  if (int rc = check_status(H, "boundary_ghosts")) return rc;
  GKS_CUDA(cudaMemcpyAsync(ghosts_out, H->ghosts, H->nbf * 5 * sizeof(double), cudaMemcpyDeviceToHost, H->stream));
  GKS_CUDA(cudaStreamSynchronize(H->stream));
  return GKS_OK;
}

}  // extern "C"

// ===========================================================================
// implicit-solve entry points
// ===========================================================================
namespace gks {
__global__ void k_update(int64_t nc, const double* q, const double* dq, double* qn, int8_t* bad);
__global__ void k_halve_dt(int64_t nc, const int8_t* bad, double* dt);
__global__ void k_sigma(const double* vv_qq, double* sigma, double* out_zero_flag);
__global__ void k_perturb(int64_t n, const double* q, const double* v, const double* sigma, double* out,
                          const int* gate);

// J v (mode 0: Frechet derivative; mode 1: V/dt v - derivative) with the step
// residual H->res as the base point; q_base = H->q, dt = H->dt.
// qq_cached: ||Q||^2 is already in red[1] (constant over one GMRES solve;
// the same reduction, so sigma is bit-identical to recomputing it)
static int frechet_apply(Handle* H, BlockSys* A, const double* v, double* out, int mode, const int* gate,
                         const double* fixed_sigma, bool qq_cached = false) {
  const int64_t n = H->n_owned * 5;
  double* sig = &H->scal->sigma;
  if (!fixed_sigma) {
    if (qq_cached) TRY(dot2(A, n, v, v, nullptr, nullptr, &H->scal->red[0], nullptr, gate));
    else TRY(dot2(A, n, v, v, H->q, H->q, &H->scal->red[0], &H->scal->red[1], gate));
    GKS_LAUNCH(KC_SCALAR, k_sigma, 1, 1, 0, H->stream, H->scal->red, sig, nullptr);
  } else {
    sig = const_cast<double*>(fixed_sigma);
  }
  GKS_LAUNCH(KC_VEC, k_perturb, blocks_for(n, 256), 256, 0, H->stream, n, H->q, v, sig, H->qtmp, gate);
  TRY(halo_exchange(H, H->hq, H->qtmp, 5, H->stream));
  // the combine runs as the assembly's epilogue (no r1 round trip through HBM)
  FrechetEpi fe;
  fe.r0 = H->res;
  fe.sigma = sig;
  fe.v = v;
  fe.dt = H->dt;
  fe.mode = mode;
  fe.out = out;
  return residual_device(H, H->qtmp, H->res2, false, gate, &fe);
}

// One attempt of the step on the current dt: residual -> Roe Jacobian ->
// GMRES -> update -> norms (stepping.py:270-296).  Launch-only.
static int enqueue_attempt(GksHandle* G) {
  Handle* H = &G->H;
  BlockSys* A = &G->jac.sys;
  // residual-pipeline errors (including those of the Frechet JVPs' residual
  // evaluations inside GMRES, stepping.py:298-313) land in the PH_RES word
  struct StatusScope {
    Handle* H;
    int* saved;
    ~StatusScope() { H->status = saved; }
  } scope{H, H->status};
  H->status = G->phase_status + 4 * PH_RES;
  // the Krylov workspace must exist before the first reduction of the step
  // (the Frechet ||Q||^2 below runs ahead of gmres_enqueue)
  TRY(krylov_ensure(A, H->krylov_dim));
  TRY(residual_device(H, H->q, H->res, H->compact != 0, nullptr));
  if (H->nbf) {
    H->status = G->phase_status + 4 * PH_GHOST;
    TRY(boundary_ghosts_device(H, H->q));
    H->status = G->phase_status + 4 * PH_RES;
  }
  TRY(jacobian_enqueue(H, A, H->nbf ? H->ghosts : nullptr, false));
  GmresParams P;
  P.m = H->krylov_dim;
  P.restarts = H->restarts;
  P.kmax = H->jacobi_sweeps;
  P.rtol = H->gmres_rtol;
  P.ortho = H->ortho;
  MatvecFn mf = [H, A](const double* v, double* out, const int* gate) {
    return frechet_apply(H, A, v, out, 1, gate, nullptr, true);
  };
  if (H->jac_mode == GKS_JAC_FRECHET) {
    const int64_t n = H->n_owned * 5;
    TRY(dot2(A, n, H->q, H->q, nullptr, nullptr, &H->scal->red[1], nullptr, nullptr));
  }
  TRY(gmres_enqueue(A, H->res, H->dq, P, H->jac_mode == GKS_JAC_FRECHET ? &mf : nullptr, false));
  GKS_LAUNCH(KC_UPDATE, k_update, blocks_for(H->n_owned, 256), 256, 0, H->stream, H->n_owned, H->q, H->dq, H->q_new,
             H->bad);
  TRY(step_stats(A, H->n_owned, H->res, H->dt, H->bad, H->scal));
  if (H->comm) {
    // every rank must agree on failure: error codes are max-reduced
    for (int ph = 0; ph < PH_N; ++ph) TRY(allreduce(H, G->phase_status + 4 * ph, 1, 1, 2, H->stream));
    TRY(allreduce(H, A->status, 1, 1, 2, H->stream));
  }
  return GKS_OK;
}

// The whole step up to the first attempt's norms.
static int enqueue_step(GksHandle* G) {
  Handle* H = &G->H;
  GKS_LAUNCH(KC_SCALAR, k_status_init, 1, 1, 0, H->stream, G->phase_status, PH_N);
  // ghost layers are stale after the previous update: refresh Q (+grad)
  TRY(halo_exchange(H, H->hq, H->q, 5, H->stream));
  if (H->compact) TRY(halo_exchange(H, H->hq, H->grad, 15, H->stream));
  int* const status = H->status;
  H->status = G->phase_status + 4 * PH_DT;
  const int rc = local_dt_device(H);
  H->status = status;
  TRY(rc);
  return enqueue_attempt(G);
}

// Read the step's device records back (one synchronisation) and report the
// first error in program order, as the reference raises it.
static int collect_step(GksHandle* G, GmresHost* gh) {
  Handle* H = &G->H;
  BlockSys* A = &G->jac.sys;
  StepHost* sh = G->sh;
  GKS_CUDA(cudaMemcpyAsync(sh->st, G->phase_status, sizeof(sh->st), cudaMemcpyDeviceToHost, H->stream));
  GKS_CUDA(cudaMemcpyAsync(sh->jst, A->status, sizeof(sh->jst), cudaMemcpyDeviceToHost, H->stream));
  GKS_CUDA(cudaMemcpyAsync(&sh->sc, H->scal, sizeof(DevScalars), cudaMemcpyDeviceToHost, H->stream));
  GKS_CUDA(cudaMemcpyAsync(&sh->g, A->ws.g, sizeof(GmresDev), cudaMemcpyDeviceToHost, H->stream));
  GKS_CUDA(cudaStreamSynchronize(H->stream));
  static const char* what[PH_N] = {"local_time_step", "residual", "boundary_ghosts"};
  for (int ph = 0; ph < PH_N; ++ph) TRY(status_report(H, what[ph], sh->st + 4 * ph));
  A->dinv_ok = sh->jst[0] == 0;
  if (!A->dinv_ok) {
    set_error("singular diagonal block in Jacobi preconditioner");
    return GKS_ERR_SINGULAR;
  }
  return gmres_result(&sh->g, gh);
}

// CUDA graphs for the step (GKS_GRAPH=0 disables; the per-launch profiler
// runs uncaptured).  The first step of a handle runs uncaptured so every
// lazily allocated workspace exists before capture.
static bool graph_enabled(const GksHandle* G) {
  static const bool env_on = [] {
    const char* e = getenv("GKS_GRAPH");
    return !(e && e[0] == '0');
  }();
  const bool on = G->graph < 0 ? env_on : G->graph != 0;
  return on && !g_prof_on && G->steps > 0;
}

static int run_step_graph(GksHandle* G) {
  Handle* H = &G->H;
  StepGraph* slot = nullptr;
  const int64_t gen = G->jac.sys.ws.gen;
  for (StepGraph& g : G->graphs) {
    if (g.exec && g.ws_gen != gen) {
      // the Krylov workspace was reallocated (host-API gmres with a larger m,
      // a Frechet matvec of another length): the graph points at freed memory
      cudaGraphExecDestroy(g.exec);
      g = StepGraph();
    }
    if (g.exec && g.q == H->q && g.grad == H->grad) slot = &g;
  }
  if (!slot) {
    slot = !G->graphs[0].exec ? &G->graphs[0] : &G->graphs[1];
    if (slot->exec) {
      cudaGraphExecDestroy(slot->exec);
      slot->exec = nullptr;
    }
    cudaGraph_t graph = nullptr;
    const int64_t l0 = gks_kernel_launches();
    GKS_CUDA(cudaStreamBeginCapture(H->stream, cudaStreamCaptureModeRelaxed));
    const int rc = enqueue_step(G);
    const cudaError_t e = cudaStreamEndCapture(H->stream, &graph);
    if (rc) {
      if (graph) cudaGraphDestroy(graph);
      return rc;
    }
    GKS_CUDA(e);
    const cudaError_t ei = cudaGraphInstantiate(&slot->exec, graph, 0);
    cudaGraphDestroy(graph);
    GKS_CUDA(ei);
    slot->q = H->q;
    slot->grad = H->grad;
    slot->ws_gen = G->jac.sys.ws.gen;
    slot->launches = gks_kernel_launches() - l0;
    count_launch((int)-slot->launches);  // captured, not launched
  }
  GKS_CUDA(cudaGraphLaunch(slot->exec, H->stream));
  count_launch((int)slot->launches);
  return GKS_OK;
}

static int advance_device(GksHandle* G, GksStepInfo* info) {
  Handle* H = &G->H;
  memset(info, 0, sizeof(*info));
  if (H->scheme == GKS_SCHEME_WENO_LUSGS) {
    set_error("scheme 'weno_lusgs' (sequential LUSGS sweep) is not part of the device path");
    return GKS_ERR_BAD_ARG;
  }
  bool launched = false;
  if (graph_enabled(G)) {
    if (run_step_graph(G) == GKS_OK) {
      launched = true;
    } else {
      // capture/instantiation refused (nothing of the step has run): step
      // uncaptured from now on rather than fail
      cudaGetLastError();
      G->graph = 0;
      for (StepGraph& g : G->graphs) {
        if (g.exec) cudaGraphExecDestroy(g.exec);
        g = StepGraph();
      }
    }
  }
  if (!launched) TRY(enqueue_step(G));
  int retried = 0;
  for (int attempt = 0; attempt < 2; ++attempt) {
    GmresHost gh;
    TRY(collect_step(G, &gh));
    const DevScalars& sc = G->sh->sc;
    info->matvecs += gh.matvecs;
    const int nbad = (int)sc.stat[2];
    if (nbad == 0) {
      std::swap(H->q, H->q_new);
      if (H->compact) std::swap(H->grad, H->grad_new);
      info->res_rho_l1 = sc.stat[0] / (double)H->nc_global;
      info->res_l2 = sqrt(sc.stat[1] / (double)(5 * H->nc_global));
      info->dt_min = sc.stat[3];
      info->solver_cycles = gh.ncycles;
      info->retried = retried;
      G->steps += 1;
      if (g_prof_on) prof_harvest();
      return GKS_OK;
    }
    info->nbad = nbad;
    if (attempt == 0) {
      // stepping.py:286-293: halve dt on the offending cells and redo the attempt (uncaptured)
      GKS_LAUNCH(KC_UPDATE, k_halve_dt, blocks_for(H->n_owned, 256), 256, 0, H->stream, H->n_owned, H->bad, H->dt);
      TRY(halo_exchange(H, H->hx, H->dt, 1, H->stream));
      GKS_LAUNCH(KC_SCALAR, k_status_init, 1, 1, 0, H->stream, G->phase_status, PH_N);
      TRY(enqueue_attempt(G));
      retried = 1;
    }
  }
  std::vector<int8_t> bad(H->n_owned);
  GKS_CUDA(cudaMemcpy(bad.data(), H->bad, H->n_owned, cudaMemcpyDeviceToHost));
  int k = 0;
  std::string lst;
  for (int64_t c = 0; c < H->n_owned && k < 8; ++c)
    if (bad[c]) {
      info->first_bad[k++] = c;
      lst += (lst.empty() ? "" : ", ") + std::to_string(c);
    }
  for (; k < 8; ++k) info->first_bad[k] = -1;
  set_error("unphysical update persists after dt halving at cells [%s]", lst.c_str());
  return GKS_ERR_INVALID_UPDATE;
}

}  // namespace gks

// Diagonal blocks live on the device in block-SoA order (entry k of every
// cell contiguous: [k * nc + c]) so the one-thread-per-cell products read
// them coalesced; the C ABI exchanges the reference's (nc, 5, 5) layout.
static std::vector<double> blocks_to_soa(const double* aos, int64_t nc) {
  std::vector<double> v((size_t)nc * 25);
  for (int64_t c = 0; c < nc; ++c)
    for (int k = 0; k < 25; ++k) v[(size_t)k * nc + c] = aos[c * 25 + k];
  return v;
}

static void blocks_from_soa(const std::vector<double>& soa, int64_t nc, double* aos) {
  for (int64_t c = 0; c < nc; ++c)
    for (int k = 0; k < 25; ++k) aos[c * 25 + k] = soa[(size_t)k * nc + c];
}

static int bs_check_size(GksBlockSystem* a) {
  if (!a) {
    set_error("null block system");
    return GKS_ERR_BAD_ARG;
  }
  return GKS_OK;
}

extern "C" {

int gks_assemble_jacobian(GksHandle* G, const double* q, const double* dt, const double* ghosts) {
  GKS_NVTX("gks_assemble_jacobian");
  Handle* H = &G->H;
  set_error_index(-1);
  GKS_CUDA(cudaSetDevice(H->device));
  ApiStage stage(G);
  GKS_CUDA(cudaMemcpyAsync(H->q, q, H->nc * 5 * sizeof(double), cudaMemcpyHostToDevice, H->stream));
  GKS_CUDA(cudaMemcpyAsync(H->dt, dt, H->nc * sizeof(double), cudaMemcpyHostToDevice, H->stream));
  if (ghosts && H->nbf)
    GKS_CUDA(cudaMemcpyAsync(H->ghosts, ghosts, H->nbf * 5 * sizeof(double), cudaMemcpyHostToDevice, H->stream));
  TRY(jacobian_assemble(H, &G->jac.sys, ghosts && H->nbf ? H->ghosts : nullptr));
  G->jac_valid = true;
  return GKS_OK;
}

GksBlockSystem* gks_jacobian(GksHandle* G) { return G ? &G->jac : nullptr; }

int gks_blocksys_create(int64_t nc, int64_t nnz, const double* diag, const double* off, const int64_t* off_col,
                        const int64_t* rowptr, int device, GksBlockSystem** out) {
  set_error_index(-1);
  if (nc <= 0 || nnz < 0 || !diag || !rowptr || !out || (nnz && (!off || !off_col))) {
    set_error("gks_blocksys_create: bad arguments");
    return GKS_ERR_BAD_ARG;
  }
  if (int rc = no_device()) return rc;
  GKS_CUDA(cudaSetDevice(device));
  GksBlockSystem* a = new GksBlockSystem();
  cudaStream_t s;
  GKS_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  TRY(blocksys_alloc(&a->sys, nc, nnz, s));
  std::vector<int> rp = to_i32(rowptr, nc + 1), cl = to_i32(off_col, nnz);
  GKS_CUDA(cudaMemcpy(a->sys.rowptr, rp.data(), (nc + 1) * sizeof(int), cudaMemcpyHostToDevice));
  if (nnz) {
    GKS_CUDA(cudaMemcpy(a->sys.col, cl.data(), nnz * sizeof(int), cudaMemcpyHostToDevice));
    GKS_CUDA(cudaMemcpy(a->sys.off, off, nnz * 25 * sizeof(double), cudaMemcpyHostToDevice));
  }
  {
    const std::vector<double> d = blocks_to_soa(diag, nc);
    GKS_CUDA(cudaMemcpy(a->sys.diag, d.data(), nc * 25 * sizeof(double), cudaMemcpyHostToDevice));
  }
  TRY(blocksys_invert_diag(&a->sys));
  a->owned = true;
  *out = a;
  return GKS_OK;
}

void gks_blocksys_destroy(GksBlockSystem* a) {
  if (!a || !a->owned) return;
  cudaStream_t s = a->sys.stream;
  blocksys_free(&a->sys);
  if (s) cudaStreamDestroy(s);
  delete a;
}

int64_t gks_blocksys_ncells(const GksBlockSystem* a) { return a ? a->sys.nc : -1; }
int64_t gks_blocksys_nnz(const GksBlockSystem* a) { return a ? a->sys.nnz : -1; }

int gks_blocksys_export(GksBlockSystem* a, double* diag, double* off, int64_t* off_col, int64_t* off_row,
                        int64_t* rowptr) {
  TRY(bs_check_size(a));
  BlockSys* A = &a->sys;
  GKS_CUDA(cudaStreamSynchronize(A->stream));
  if (diag) {
    std::vector<double> d((size_t)A->nc * 25);
    GKS_CUDA(cudaMemcpy(d.data(), A->diag, d.size() * sizeof(double), cudaMemcpyDeviceToHost));
    blocks_from_soa(d, A->nc, diag);
  }
  if (off && A->nnz) GKS_CUDA(cudaMemcpy(off, A->off, A->nnz * 25 * sizeof(double), cudaMemcpyDeviceToHost));
  std::vector<int> rp(A->nc + 1), cl(std::max<int64_t>(A->nnz, 1));
  GKS_CUDA(cudaMemcpy(rp.data(), A->rowptr, (A->nc + 1) * sizeof(int), cudaMemcpyDeviceToHost));
  if (A->nnz) GKS_CUDA(cudaMemcpy(cl.data(), A->col, A->nnz * sizeof(int), cudaMemcpyDeviceToHost));
  if (rowptr)
    for (int64_t c = 0; c <= A->nc; ++c) rowptr[c] = rp[c];
  if (off_col)
    for (int64_t e = 0; e < A->nnz; ++e) off_col[e] = cl[e];
  if (off_row)
    for (int64_t c = 0; c < A->nc; ++c)
      for (int e = rp[c]; e < rp[c + 1]; ++e) off_row[e] = c;
  return GKS_OK;
}

static int bs_vec_op(GksBlockSystem* a, const double* x, double* y, int which) {
  TRY(bs_check_size(a));
  BlockSys* A = &a->sys;
  const int64_t n = A->nc * 5;
  TRY(krylov_ensure(A, 1));
  GKS_CUDA(cudaMemcpyAsync(A->ws.x, x, n * sizeof(double), cudaMemcpyHostToDevice, A->stream));
  if (which == 0) bs_spmv(A, A->ws.x, A->ws.b, nullptr);
  else bs_offdiag(A, A->ws.x, A->ws.b, nullptr);
  GKS_CUDA(cudaGetLastError());
  GKS_CUDA(cudaMemcpyAsync(y, A->ws.b, n * sizeof(double), cudaMemcpyDeviceToHost, A->stream));
  GKS_CUDA(cudaStreamSynchronize(A->stream));
  return GKS_OK;
}

int gks_blocksys_spmv(GksBlockSystem* a, const double* x, double* y) { return bs_vec_op(a, x, y, 0); }

int gks_blocksys_dot(GksBlockSystem* a, const double* x, const double* y, double* out) {
  TRY(bs_check_size(a));
  BlockSys* A = &a->sys;
  const int64_t n = A->nc * 5;
  TRY(krylov_ensure(A, 1));
  GKS_CUDA(cudaMemcpyAsync(A->ws.x, x, n * sizeof(double), cudaMemcpyHostToDevice, A->stream));
  GKS_CUDA(cudaMemcpyAsync(A->ws.b, y, n * sizeof(double), cudaMemcpyHostToDevice, A->stream));
  TRY(dot2(A, n, A->ws.x, A->ws.b, nullptr, nullptr, &A->ws.g->beta2, nullptr, nullptr));
  GKS_CUDA(cudaGetLastError());
  GKS_CUDA(cudaMemcpyAsync(out, &A->ws.g->beta2, sizeof(double), cudaMemcpyDeviceToHost, A->stream));
  GKS_CUDA(cudaStreamSynchronize(A->stream));
  return GKS_OK;
}
int gks_blocksys_offdiag_mv(GksBlockSystem* a, const double* x, double* y) { return bs_vec_op(a, x, y, 1); }

int gks_blocksys_diag_inverses(GksBlockSystem* a, double* out) {
  TRY(bs_check_size(a));
  BlockSys* A = &a->sys;
  GKS_CUDA(cudaStreamSynchronize(A->stream));
  {
    std::vector<double> d((size_t)A->nc * 25);
    GKS_CUDA(cudaMemcpy(d.data(), A->dinv, d.size() * sizeof(double), cudaMemcpyDeviceToHost));
    blocks_from_soa(d, A->nc, out);
  }
  return GKS_OK;
}

int gks_blocksys_jacobi(GksBlockSystem* a, const double* b, int k_max, double* z) {
  TRY(bs_check_size(a));
  BlockSys* A = &a->sys;
  if (!A->dinv_ok) {
    set_error("singular diagonal block in Jacobi preconditioner");
    return GKS_ERR_SINGULAR;
  }
  const int64_t n = A->nc * 5;
  TRY(krylov_ensure(A, 1));
  GKS_CUDA(cudaMemcpyAsync(A->ws.b, b, n * sizeof(double), cudaMemcpyHostToDevice, A->stream));
  bs_jacobi(A, A->ws.b, A->ws.z, A->ws.w, k_max, nullptr);
  GKS_CUDA(cudaGetLastError());
  GKS_CUDA(cudaMemcpyAsync(z, A->ws.z, n * sizeof(double), cudaMemcpyDeviceToHost, A->stream));
  GKS_CUDA(cudaStreamSynchronize(A->stream));
  return GKS_OK;
}

int gks_gmres(GksBlockSystem* a, const double* b, double* x_out, int m, int restarts, int k_max, double rtol,
              double atol, int check_orthogonality, GksGmresInfo* info) {
  GKS_NVTX("gks_gmres");
  TRY(bs_check_size(a));
  set_error_index(-1);
  BlockSys* A = &a->sys;
  const int64_t n = A->nc * 5;
  TRY(krylov_ensure(A, m));
  double* db;
  double* dx;
  GKS_CUDA(cudaMalloc(&db, n * sizeof(double)));
  GKS_CUDA(cudaMalloc(&dx, n * sizeof(double)));
  GKS_CUDA(cudaMemcpyAsync(db, b, n * sizeof(double), cudaMemcpyHostToDevice, A->stream));
  GmresParams P;
  P.m = m; P.restarts = restarts; P.kmax = k_max; P.rtol = rtol; P.atol = atol;
  P.check_ortho = check_orthogonality;
  GmresHost* gh = new GmresHost();
  int rc = gmres_device(A, db, dx, P, gh, nullptr);
  if (rc == GKS_OK) {
    cudaMemcpyAsync(x_out, dx, n * sizeof(double), cudaMemcpyDeviceToHost, A->stream);
    cudaStreamSynchronize(A->stream);
  }
  if (info) {
    info->ncycles = gh->ncycles;
    info->matvecs = gh->matvecs;
    info->breakdown = gh->breakdown;
    info->ortho_error = gh->ortho_error;
    for (int c = 0; c < gh->ncycles; ++c) {
      info->cycle_len[c] = gh->cycle_len[c];
      for (int k = 0; k < gh->cycle_len[c]; ++k)
        info->norms[c * (GKS_GMRES_MAX_DIM + 1) + k] = gh->norms[c * (GM_MMAX + 1) + k];
    }
  }
  delete gh;
  cudaFree(db);
  cudaFree(dx);
  return rc;
}

int gks_event_record(GksHandle* G, int slot) {
  Handle* H = &G->H;
  if (slot < 0 || slot >= 8) return GKS_ERR_BAD_ARG;
  if (!H->ev_ready) {
    for (int k = 0; k < 8; ++k) GKS_CUDA(cudaEventCreate(&H->ev[k]));
    H->ev_ready = 1;
  }
  GKS_CUDA(cudaEventRecord(H->ev[slot], H->stream));
  return GKS_OK;
}

int gks_event_elapsed(GksHandle* G, int a, int b, double* ms) {
  Handle* H = &G->H;
  if (!H->ev_ready || a < 0 || b < 0 || a >= 8 || b >= 8) return GKS_ERR_BAD_ARG;
  GKS_CUDA(cudaEventSynchronize(H->ev[b]));
  float f = 0.f;
  GKS_CUDA(cudaEventElapsedTime(&f, H->ev[a], H->ev[b]));
  *ms = f;
  return GKS_OK;
}

int64_t gks_handle_info(const GksHandle* G, int what) {
  const Handle* H = &G->H;
  switch (what) {
    case 0: return H->nc;
    case 1: return H->nf;
    case 2: return H->nfq;
    case 3: return H->nfi;
    case 4: return H->nbf;
    case 5: return H->nnz;
    case 6: return H->compact ? H->HA + 3 * H->HG : H->K;   /* big-op width */
    case 7: return H->compact ? H->HM : H->M;               /* sub-stencil slots */
    case 8: return H->compact ? 7 : H->S;                   /* sub-stencil width */
    case 9: return H->n_owned;
    case 10: return H->nent;  /* assembly entries (slots) of the owned cells */
    default: return -1;
  }
}

int gks_state_upload(GksHandle* G, const double* q, const double* grad) {
  Handle* H = &G->H;
  GKS_CUDA(cudaSetDevice(H->device));
  GKS_CUDA(cudaMemcpyAsync(H->q, q, H->nc * 5 * sizeof(double), cudaMemcpyHostToDevice, H->stream));
  if (grad) GKS_CUDA(cudaMemcpyAsync(H->grad, grad, H->nc * 15 * sizeof(double), cudaMemcpyHostToDevice, H->stream));
  GKS_CUDA(cudaStreamSynchronize(H->stream));
  return GKS_OK;
}

int gks_state_download(GksHandle* G, double* q, double* grad) {
  Handle* H = &G->H;
  GKS_CUDA(cudaSetDevice(H->device));
  if (q) GKS_CUDA(cudaMemcpyAsync(q, H->q, H->nc * 5 * sizeof(double), cudaMemcpyDeviceToHost, H->stream));
  if (grad) GKS_CUDA(cudaMemcpyAsync(grad, H->grad, H->nc * 15 * sizeof(double), cudaMemcpyDeviceToHost, H->stream));
  GKS_CUDA(cudaStreamSynchronize(H->stream));
  return GKS_OK;
}

int gks_set_cfl(GksHandle* G, double cfl) {
  if (!G || !(cfl > 0.0)) {
    set_error("gks_set_cfl: bad arguments");
    return GKS_ERR_BAD_ARG;
  }
  G->H.cfl = cfl;
  // the captured steps carry the old CFL as a kernel argument
  for (StepGraph& g : G->graphs) {
    if (g.exec) cudaGraphExecDestroy(g.exec);
    g = StepGraph();
  }
  return GKS_OK;
}

int gks_set_ortho(GksHandle* G, int ortho) {
  if (!G || ortho < 0 || ortho > 1) {
    set_error("gks_set_ortho: bad arguments");
    return GKS_ERR_BAD_ARG;
  }
  G->H.ortho = ortho;
  for (StepGraph& g : G->graphs) {
    if (g.exec) cudaGraphExecDestroy(g.exec);
    g = StepGraph();
  }
  return GKS_OK;
}

int gks_set_graph(GksHandle* G, int enable) {
  if (!G) return GKS_ERR_BAD_ARG;
  G->graph = enable ? 1 : 0;
  return GKS_OK;
}

int gks_bad_mask(GksHandle* G, int8_t* out) {
  Handle* H = &G->H;
  GKS_CUDA(cudaSetDevice(H->device));
  GKS_CUDA(cudaStreamSynchronize(H->stream));
  GKS_CUDA(cudaMemcpy(out, H->bad, H->n_owned, cudaMemcpyDeviceToHost));
  return GKS_OK;
}

int gks_advance_resident(GksHandle* G, GksStepInfo* info) {
  GKS_NVTX("gks_advance_resident");
  set_error_index(-1);
  GKS_CUDA(cudaSetDevice(G->H.device));
  return advance_device(G, info);
}

int gks_advance(GksHandle* G, double* q_inout, double* grad_inout, GksStepInfo* info) {
  GKS_NVTX("gks_advance");
  Handle* H = &G->H;
  if (H->compact && !grad_inout) {
    set_error("compact scheme needs a gradient field");
    return GKS_ERR_BAD_ARG;
  }
  TRY(gks_state_upload(G, q_inout, H->compact ? grad_inout : nullptr));
  TRY(gks_advance_resident(G, info));
  return gks_state_download(G, q_inout, H->compact ? grad_inout : nullptr);
}

int gks_frechet_matvec(GksHandle* G, const double* q, const double* grad, const double* dt, const double* v,
                       double sigma, double* out) {
  GKS_NVTX("gks_frechet_matvec");
  Handle* H = &G->H;
  set_error_index(-1);
  GKS_CUDA(cudaSetDevice(H->device));
  if (H->compact && !grad) {
    set_error("compact scheme needs a gradient field");
    return GKS_ERR_BAD_ARG;
  }
  const int64_t n = H->nc * 5;
  BlockSys* A = &G->jac.sys;
  // the step's workspace shape (owned rows, krylov_dim): no reallocation
  TRY(krylov_ensure(A, std::max(1, H->krylov_dim)));
  const int64_t nv = std::min<int64_t>(n, A->ws.ld);  // owned rows + layer-1 ghosts are read
  ApiStage stage(G);
  GKS_CUDA(cudaMemcpyAsync(H->q, q, n * sizeof(double), cudaMemcpyHostToDevice, H->stream));
  if (grad) GKS_CUDA(cudaMemcpyAsync(H->grad, grad, H->nc * 15 * sizeof(double), cudaMemcpyHostToDevice, H->stream));
  GKS_CUDA(cudaMemcpyAsync(H->dt, dt, H->nc * sizeof(double), cudaMemcpyHostToDevice, H->stream));
  GKS_CUDA(cudaMemcpyAsync(A->ws.x, v, nv * sizeof(double), cudaMemcpyHostToDevice, H->stream));
  reset_status(H);
  TRY(residual_device(H, H->q, H->res, false, nullptr));
  const double* fixed = nullptr;
  if (sigma > 0.0) {
    GKS_CUDA(cudaMemcpyAsync(&H->scal->red[7], &sigma, sizeof(double), cudaMemcpyHostToDevice, H->stream));
    fixed = &H->scal->red[7];
  }
  TRY(frechet_apply(H, A, A->ws.x, A->ws.b, 0, nullptr, fixed));
  TRY(check_status(H, "frechet_matvec"));
  GKS_CUDA(cudaMemcpyAsync(out, A->ws.b, A->nc * 5 * sizeof(double), cudaMemcpyDeviceToHost, H->stream));
  GKS_CUDA(cudaStreamSynchronize(H->stream));
  return GKS_OK;
}

}  // extern "C"
