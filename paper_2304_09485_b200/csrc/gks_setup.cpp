// Host-side native setup: stencil selection and reconstruction operators.
//
// Runs the per-cell arithmetic of gks_setup_cell.cuh over all cells in
// parallel (OpenMP) and keeps the reference's padded operator layout
// (exported through gks_setup_query / gks_setup_copy).  The same per-cell
// code also runs on the device (gks_setup_dev.cu, the default path of
// gks_create); this build serves the host API (StencilTable, the operator
// arrays) and the per-rank setups of the distributed solver.
//   gks3d/mesh/stencils.py:72-192   _ordered_neighbors, _dedup, build_stencils
//   gks3d/recon.py:60-69            _pinv (SVD pseudo-inverse, rank tol 1e-10)
//   gks3d/recon.py:104-164          ReconGeometry (avg0, beta matrices)
//   gks3d/recon.py:216-274          WenoReconstructor._build_operators
//   gks3d/hweno.py:45-137           HwenoReconstructor._grad_rows/_build_operators
// Stencil selection is integer work and is bit-identical to the reference
// (tests/test_setup.py).  The pseudo-inverses use a one-sided Jacobi SVD
// instead of LAPACK; they agree to rounding (their bits are unpinned by the
// reference).
//
// This file must be compiled without FP contraction (-ffp-contract=off) so
// the hex-face angle ordering reproduces numpy's arithmetic exactly and the
// operators equal the device build's bit for bit.
#include <math.h>
#include <omp.h>
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <array>
#include <map>
#include <string>
#include <vector>

#include "gks.h"
#include "gks_setup_cell.cuh"

namespace gks {
void set_error(const char* fmt, ...);
}

using gks::su::NCOEF;

struct GksSetup {
  int64_t nc = 0;
  int nfpc = 0;  // max faces per cell (4 tet, 6 hex)
  // ordered face neighbours (nc, nfpc), shifts (nc, nfpc, 3)
  std::vector<int64_t> nbr_ids;
  std::vector<double> nbr_shift;
  // WENO big stencil CSR (members include the target first)
  std::vector<int64_t> big_start, big_ids;
  std::vector<double> big_shift;
  // WENO sub-stencils: per cell count, CSR over subs then members
  std::vector<int64_t> sub_cell_start, sub_member_start, sub_ids;
  std::vector<double> sub_shift;
  std::vector<int8_t> weno_fallback, hweno_fallback;
  // recon geometry
  std::vector<double> avg0, beta;
  // WENO operators (reference padded layout)
  int64_t w_kmax = 0, w_mmax = 0, w_smax = 0;
  std::vector<double> w_big_op, w_sub_op;
  std::vector<int64_t> w_big_gather, w_sub_gather;
  std::vector<int8_t> w_sub_active, w_big_degree;
  // HWENO operators
  int64_t h_amax = 0, h_gmax = 0, h_mmax = 0;
  std::vector<double> h_big_op, h_big_grad_scale, h_sub_op;
  std::vector<int64_t> h_big_avg_gather, h_big_grad_gather, h_sub_gather, h_big_ncols;
  std::vector<int8_t> h_sub_active, h_big_degree;

  struct Arr {
    const void* p;
    int dtype;  // 0 f64, 1 i64, 2 i8
    int ndim;
    int64_t shape[4];
  };
  std::map<std::string, Arr> arrays;
  std::vector<std::vector<char>> owned_storage;  // backing store of subset setups
  template <class T>
  void reg(const char* name, const std::vector<T>& v, int dtype, std::initializer_list<int64_t> shp) {
    Arr a{v.data(), dtype, (int)shp.size(), {0, 0, 0, 0}};
    int i = 0;
    for (int64_t s : shp) a.shape[i++] = s;
    arrays[name] = a;
  }
};


namespace {

using gks::su::Stencil;
using gks::su::build_stencil;

// reference-layout sinks of the per-cell operator builders
struct HostWenoSink {
  GksSetup* S;
  int64_t c, mup, sup, kmax;
  void sub_op(int slot, int d, int k, double v) { S->w_sub_op[((c * mup + slot) * 3 + d) * sup + k] = v; }
  void sub_gather(int slot, int k, int64_t id) { S->w_sub_gather[(c * mup + slot) * sup + k] = id; }
  void sub_active(int slot) { S->w_sub_active[c * mup + slot] = 1; }
  void drop_subs(int n) {
    for (int mm = 0; mm < n; ++mm) {
      S->w_sub_active[c * mup + mm] = 0;
      for (int64_t k = 0; k < 3 * sup; ++k) S->w_sub_op[(c * mup + mm) * 3 * sup + k] = 0.0;
      for (int64_t k = 0; k < sup; ++k) S->w_sub_gather[(c * mup + mm) * sup + k] = 0;
    }
  }
  void big_op(int d, int k, double v) { S->w_big_op[(c * NCOEF + d) * kmax + k] = v; }
  void big_gather(int k, int64_t id) { S->w_big_gather[c * kmax + k] = id; }
  void big_degree(int deg) { S->w_big_degree[c] = (int8_t)deg; }
};

struct HostHwenoSink {
  GksSetup* S;
  const GksMeshDesc* m;
  int64_t c, mup, amax, gmax, W;
  int na;
  void big_op(int d, int k, double v) {
    S->h_big_op[(c * NCOEF + d) * W + (k < na ? k : amax + (k - na))] = v;
  }
  void avg_gather(int k, int64_t id) { S->h_big_avg_gather[c * amax + k] = id; }
  void grad_gather(int k, int64_t id, double h) {
    S->h_big_grad_gather[c * gmax + k] = id;
    S->h_big_grad_scale[c * gmax + k] = h;
  }
  void big_ncols(int R) { S->h_big_ncols[c] = R; }
  void big_degree(int deg) { S->h_big_degree[c] = (int8_t)deg; }
  void sub_op(int slot, int i, double v) { S->h_sub_op[(c * mup + slot) * 21 + i] = v; }
  void sub_gather(int slot, int64_t id) {
    S->h_sub_gather[(c * mup + slot) * 2 + 0] = c;
    S->h_sub_gather[(c * mup + slot) * 2 + 1] = id;
  }
  void sub_active(int slot) { S->h_sub_active[c * mup + slot] = 1; }
  void drop_subs(int n) {
    for (int mm = 0; mm < n; ++mm) {
      S->h_sub_active[c * mup + mm] = 0;
      for (int i = 0; i < 21; ++i) S->h_sub_op[(c * mup + mm) * 21 + i] = 0.0;
      S->h_sub_gather[(c * mup + mm) * 2] = 0;
      S->h_sub_gather[(c * mup + mm) * 2 + 1] = 0;
    }
  }
};

}  // namespace

extern "C" {

// Memory-lean build (10^7-cell meshes): a sizing pass, then every cell
// rebuilds its stencil and writes its operators straight into the final
// padded arrays; per-cell stencil objects are never kept.  The CSR stencil
// tables are only exported when asked for (schemes == 0 or bit 2).
int gks_setup_build(const GksMeshDesc* m, int schemes, int nthreads, GksSetup** out) {
  if (!m || !out || m->ncells <= 0) {
    gks::set_error("gks_setup_build: bad arguments");
    return GKS_ERR_BAD_ARG;
  }
  if (nthreads > 0) omp_set_num_threads(nthreads);
  const int64_t nc = m->ncells;
  int nfpc = 0;
  for (int64_t c = 0; c < nc; ++c) {
    const int nf = (int)(m->cell_face_start[c + 1] - m->cell_face_start[c]);
    if (nf > gks::su::NF || (m->cell_kind[c] == 1 && nf != 6) || (m->cell_kind[c] != 1 && nf != 4)) {
      gks::set_error("gks_setup_build: cell %lld has %d faces (tet 4 / hex 6 only)", (long long)c, nf);
      return GKS_ERR_BAD_ARG;
    }
    nfpc = std::max(nfpc, nf);
  }
  GksSetup* S = new GksSetup();
  S->nc = nc;
  S->nfpc = nfpc;
  const GksMeshDesc& M = *m;
  const bool want_weno = schemes & 1, want_hweno = schemes & 2;
  const bool want_stencils = schemes == 0 || (schemes & 4);

  // ---- pass A: sizes ------------------------------------------------------
  std::vector<int32_t> big_n(nc), sub_n(nc), nbr_n(nc);
  std::vector<int8_t> wfb(nc), hfb(nc);
  int64_t sub_len_max = 0;
#pragma omp parallel for schedule(dynamic, 256) reduction(max : sub_len_max)
  for (int64_t c = 0; c < nc; ++c) {
    Stencil st;
    build_stencil(M, c, st);
    big_n[c] = st.nbig;
    sub_n[c] = st.nsub;
    nbr_n[c] = st.present();
    wfb[c] = st.weno_fallback;
    hfb[c] = st.hweno_fallback;
    for (int k = 0; k < st.nsub; ++k) sub_len_max = std::max<int64_t>(sub_len_max, st.sublen[k] - 1);
  }
  S->weno_fallback = wfb;
  S->hweno_fallback = hfb;

  // ---- optional stencil export (CSR) ---------------------------------------
  if (want_stencils) {
    S->nbr_ids.assign(nc * nfpc, -1);
    S->nbr_shift.assign(nc * nfpc * 3, 0.0);
    S->big_start.assign(nc + 1, 0);
    S->sub_cell_start.assign(nc + 1, 0);
    for (int64_t c = 0; c < nc; ++c) {
      S->big_start[c + 1] = S->big_start[c] + big_n[c];
      S->sub_cell_start[c + 1] = S->sub_cell_start[c] + sub_n[c];
    }
    S->big_ids.resize(S->big_start[nc]);
    S->big_shift.resize(S->big_start[nc] * 3);
    std::vector<int64_t> sub_len(S->sub_cell_start[nc], 0);
#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t c = 0; c < nc; ++c) {
      Stencil st;
      build_stencil(M, c, st);
      int64_t si = S->sub_cell_start[c];
      for (int k = 0; k < st.nsub; ++k) sub_len[si++] = st.sublen[k];
    }
    S->sub_member_start.assign(sub_len.size() + 1, 0);
    for (size_t k = 0; k < sub_len.size(); ++k) S->sub_member_start[k + 1] = S->sub_member_start[k] + sub_len[k];
    S->sub_ids.resize(S->sub_member_start.back());
    S->sub_shift.resize(S->sub_member_start.back() * 3);
#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t c = 0; c < nc; ++c) {
      Stencil st;
      build_stencil(M, c, st);
      for (int k = 0; k < st.nf; ++k) {
        S->nbr_ids[c * nfpc + k] = st.nbr[k];
        S->nbr_shift[(c * nfpc + k) * 3 + 0] = st.nbr_s[k].x;
        S->nbr_shift[(c * nfpc + k) * 3 + 1] = st.nbr_s[k].y;
        S->nbr_shift[(c * nfpc + k) * 3 + 2] = st.nbr_s[k].z;
      }
      int64_t b = S->big_start[c];
      for (int k = 0; k < st.nbig; ++k) {
        const auto& mb = st.big[k];
        S->big_ids[b] = mb.id;
        S->big_shift[3 * b] = mb.s.x; S->big_shift[3 * b + 1] = mb.s.y; S->big_shift[3 * b + 2] = mb.s.z;
        ++b;
      }
      int64_t si = S->sub_cell_start[c];
      for (int k = 0; k < st.nsub; ++k) {
        int64_t q = S->sub_member_start[si++];
        for (int j = 0; j < st.sublen[k]; ++j) {
          const auto& mb = st.sub[k][j];
          S->sub_ids[q] = mb.id;
          S->sub_shift[3 * q] = mb.s.x; S->sub_shift[3 * q + 1] = mb.s.y; S->sub_shift[3 * q + 2] = mb.s.z;
          ++q;
        }
      }
    }
  }

  // ---- recon geometry (recon.py:104-146) ----------------------------------
  S->avg0.assign(nc * NCOEF, 0.0);
  S->beta.assign(nc * NCOEF * NCOEF, 0.0);
#pragma omp parallel for schedule(static)
  for (int64_t c = 0; c < nc; ++c) gks::su::cell_geometry(M, c, &S->avg0[c * NCOEF], &S->beta[c * 81]);

  if (want_weno) {
    // WENO operators (recon.py:216-274) written in place with upper-bound widths
    int64_t kmax = 1, mup = 1;
    for (int64_t c = 0; c < nc; ++c) {
      kmax = std::max<int64_t>(kmax, std::max(big_n[c] - 1, 1));
      mup = std::max<int64_t>(mup, sub_n[c]);
    }
    const int64_t sup = std::max<int64_t>(sub_len_max, 1);
    S->w_big_op.assign(nc * NCOEF * kmax, 0.0);
    S->w_big_gather.assign(nc * kmax, 0);
    S->w_sub_op.assign(nc * mup * 3 * sup, 0.0);
    S->w_sub_gather.assign(nc * mup * sup, 0);
    S->w_sub_active.assign(nc * mup, 0);
    S->w_big_degree.assign(nc, 2);
    std::vector<int32_t> msurv(nc, 0), ssurv(nc, 0);
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t c = 0; c < nc; ++c) {
      Stencil st;
      build_stencil(M, c, st);
      HostWenoSink sink{S, c, mup, sup, kmax};
      const int r = gks::su::weno_cell(M, c, st, &S->avg0[c * NCOEF], sink);
      msurv[c] = r & 0xff;
      ssurv[c] = r >> 8;
    }
    // reference widths: mmax = max(surviving subs, 1), smax = max surviving sub columns (default 1)
    int64_t mmax = 0, smax = 0;
    for (int64_t c = 0; c < nc; ++c) {
      mmax = std::max<int64_t>(mmax, msurv[c]);
      smax = std::max<int64_t>(smax, ssurv[c]);
    }
    mmax = std::max<int64_t>(mmax, 1);
    smax = std::max<int64_t>(smax, 1);
    if (mmax != mup || smax != sup) {
      std::vector<double> op2(nc * mmax * 3 * smax, 0.0);
      std::vector<int64_t> g2(nc * mmax * smax, 0);
      std::vector<int8_t> a2(nc * mmax, 0);
      for (int64_t c = 0; c < nc; ++c)
        for (int64_t mm = 0; mm < mmax; ++mm) {
          a2[c * mmax + mm] = S->w_sub_active[c * mup + mm];
          for (int64_t d = 0; d < 3; ++d)
            for (int64_t k = 0; k < smax; ++k)
              op2[((c * mmax + mm) * 3 + d) * smax + k] = S->w_sub_op[((c * mup + mm) * 3 + d) * sup + k];
          for (int64_t k = 0; k < smax; ++k) g2[(c * mmax + mm) * smax + k] = S->w_sub_gather[(c * mup + mm) * sup + k];
        }
      S->w_sub_op.swap(op2);
      S->w_sub_gather.swap(g2);
      S->w_sub_active.swap(a2);
    }
    S->w_kmax = kmax;
    S->w_mmax = mmax;
    S->w_smax = smax;
  }

  if (want_hweno) {
    // HWENO operators (hweno.py:62-137)
    int64_t amax = 0, gmax = 0;
    for (int64_t c = 0; c < nc; ++c) {
      amax = std::max<int64_t>(amax, nbr_n[c]);
      gmax = std::max<int64_t>(gmax, nbr_n[c] + 1);
    }
    amax = std::max<int64_t>(amax, 1);
    const int64_t mup = std::max<int64_t>(nfpc, 1);
    const int64_t W = amax + 3 * gmax;
    S->h_big_op.assign(nc * NCOEF * W, 0.0);
    S->h_big_avg_gather.assign(nc * amax, 0);
    S->h_big_grad_gather.assign(nc * gmax, 0);
    S->h_big_grad_scale.assign(nc * gmax, 0.0);
    S->h_big_ncols.assign(nc, 0);
    S->h_big_degree.assign(nc, 2);
    S->h_sub_op.assign(nc * mup * 21, 0.0);
    S->h_sub_gather.assign(nc * mup * 2, 0);
    S->h_sub_active.assign(nc * mup, 0);
    std::vector<int32_t> msurv(nc, 0);
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t c = 0; c < nc; ++c) {
      Stencil st;
      build_stencil(M, c, st);
      HostHwenoSink sink{S, m, c, mup, amax, gmax, W, st.present()};
      msurv[c] = gks::su::hweno_cell(M, c, st, &S->avg0[c * NCOEF], sink);
    }
    int64_t mmax = 0;
    for (int64_t c = 0; c < nc; ++c) mmax = std::max<int64_t>(mmax, msurv[c]);
    mmax = std::max<int64_t>(mmax, 1);
    if (mmax != mup) {
      std::vector<double> op2(nc * mmax * 21, 0.0);
      std::vector<int64_t> g2(nc * mmax * 2, 0);
      std::vector<int8_t> a2(nc * mmax, 0);
      for (int64_t c = 0; c < nc; ++c)
        for (int64_t mm = 0; mm < mmax; ++mm) {
          a2[c * mmax + mm] = S->h_sub_active[c * mup + mm];
          for (int i = 0; i < 21; ++i) op2[(c * mmax + mm) * 21 + i] = S->h_sub_op[(c * mup + mm) * 21 + i];
          g2[(c * mmax + mm) * 2] = S->h_sub_gather[(c * mup + mm) * 2];
          g2[(c * mmax + mm) * 2 + 1] = S->h_sub_gather[(c * mup + mm) * 2 + 1];
        }
      S->h_sub_op.swap(op2);
      S->h_sub_gather.swap(g2);
      S->h_sub_active.swap(a2);
    }
    S->h_amax = amax;
    S->h_gmax = gmax;
    S->h_mmax = mmax;
  }

  // register exports
  if (want_stencils) {
    S->reg("nbr_ids", S->nbr_ids, 1, {nc, nfpc});
    S->reg("nbr_shift", S->nbr_shift, 0, {nc, nfpc, 3});
    S->reg("big_start", S->big_start, 1, {nc + 1});
    S->reg("big_ids", S->big_ids, 1, {(int64_t)S->big_ids.size()});
    S->reg("big_shift", S->big_shift, 0, {(int64_t)S->big_ids.size(), 3});
    S->reg("sub_cell_start", S->sub_cell_start, 1, {nc + 1});
    S->reg("sub_member_start", S->sub_member_start, 1, {(int64_t)S->sub_member_start.size()});
    S->reg("sub_ids", S->sub_ids, 1, {(int64_t)S->sub_ids.size()});
    S->reg("sub_shift", S->sub_shift, 0, {(int64_t)S->sub_ids.size(), 3});
  }
  S->reg("weno_fallback", S->weno_fallback, 2, {nc});
  S->reg("hweno_fallback", S->hweno_fallback, 2, {nc});
  S->reg("avg0", S->avg0, 0, {nc, NCOEF});
  S->reg("beta_mat", S->beta, 0, {nc, NCOEF, NCOEF});
  if (want_weno) {
    S->reg("weno_big_op", S->w_big_op, 0, {nc, NCOEF, S->w_kmax});
    S->reg("weno_big_gather", S->w_big_gather, 1, {nc, S->w_kmax});
    S->reg("weno_big_degree", S->w_big_degree, 2, {nc});
    S->reg("weno_sub_op", S->w_sub_op, 0, {nc, S->w_mmax, 3, S->w_smax});
    S->reg("weno_sub_gather", S->w_sub_gather, 1, {nc, S->w_mmax, S->w_smax});
    S->reg("weno_sub_active", S->w_sub_active, 2, {nc, S->w_mmax});
  }
  if (want_hweno) {
    const int64_t W = S->h_amax + 3 * S->h_gmax;
    S->reg("hweno_big_op", S->h_big_op, 0, {nc, NCOEF, W});
    S->reg("hweno_big_avg_gather", S->h_big_avg_gather, 1, {nc, S->h_amax});
    S->reg("hweno_big_grad_gather", S->h_big_grad_gather, 1, {nc, S->h_gmax});
    S->reg("hweno_big_grad_scale", S->h_big_grad_scale, 0, {nc, S->h_gmax});
    S->reg("hweno_big_ncols", S->h_big_ncols, 1, {nc});
    S->reg("hweno_big_degree", S->h_big_degree, 2, {nc});
    S->reg("hweno_sub_op", S->h_sub_op, 0, {nc, S->h_mmax, 3, 7});
    S->reg("hweno_sub_gather", S->h_sub_gather, 1, {nc, S->h_mmax, 2});
    S->reg("hweno_sub_active", S->h_sub_active, 2, {nc, S->h_mmax});
  }
  *out = S;
  return GKS_OK;
}

void gks_setup_free(GksSetup* s) { delete s; }

// Restrict a global setup to local cells: rows of every per-cell array are
// gathered in local order and cell-id gathers are renumbered to local ids
// (ids outside the local set map to 0 -- only rows of cells that are not
// reconstructed locally can contain them).
int gks_setup_subset(const GksSetup* g, const int64_t* cells, int64_t n_local, const int64_t* g2l,
                     int64_t n_global, GksSetup** out) {
  if (!g || !cells || !g2l || !out || n_local <= 0 || n_global != g->nc) {
    gks::set_error("gks_setup_subset: bad arguments");
    return GKS_ERR_BAD_ARG;
  }
  static const char* gathers[] = {"weno_big_gather", "weno_sub_gather", "hweno_big_avg_gather",
                                  "hweno_big_grad_gather", "hweno_sub_gather"};
  GksSetup* S = new GksSetup();
  S->nc = n_local;
  S->nfpc = g->nfpc;
  for (const auto& kv : g->arrays) {
    const auto& a = kv.second;
    if (a.ndim < 1 || a.shape[0] != g->nc) continue;  // CSR stencil tables are not per-cell arrays
    const int esz = a.dtype == 2 ? 1 : 8;
    int64_t row = esz;
    for (int d = 1; d < a.ndim; ++d) row *= a.shape[d];
    S->owned_storage.emplace_back((size_t)(n_local * row));
    std::vector<char>& buf = S->owned_storage.back();
    const char* src = static_cast<const char*>(a.p);
    for (int64_t c = 0; c < n_local; ++c) memcpy(buf.data() + c * row, src + cells[c] * row, row);
    bool is_gather = false;
    for (const char* nm : gathers) is_gather |= kv.first == nm;
    if (is_gather) {
      int64_t* v = reinterpret_cast<int64_t*>(buf.data());
      const int64_t n = n_local * row / 8;
      for (int64_t k = 0; k < n; ++k) {
        const int64_t l = (v[k] >= 0 && v[k] < n_global) ? g2l[v[k]] : -1;
        v[k] = l >= 0 ? l : 0;
      }
    }
    GksSetup::Arr b = a;
    b.p = buf.data();
    b.shape[0] = n_local;
    S->arrays[kv.first] = b;
  }
  *out = S;
  return GKS_OK;
}

int gks_setup_query(const GksSetup* s, const char* name, int* dtype, int* ndim, int64_t* shape) {
  if (!s || !name) return GKS_ERR_BAD_ARG;
  auto it = s->arrays.find(name);
  if (it == s->arrays.end()) {
    gks::set_error("gks_setup_query: unknown array '%s'", name);
    return GKS_ERR_BAD_ARG;
  }
  *dtype = it->second.dtype;
  *ndim = it->second.ndim;
  for (int i = 0; i < 4; ++i) shape[i] = it->second.shape[i];
  return GKS_OK;
}

int gks_setup_copy(const GksSetup* s, const char* name, void* dst, int64_t nbytes) {
  if (!s || !name || !dst) return GKS_ERR_BAD_ARG;
  auto it = s->arrays.find(name);
  if (it == s->arrays.end()) {
    gks::set_error("gks_setup_copy: unknown array '%s'", name);
    return GKS_ERR_BAD_ARG;
  }
  const auto& a = it->second;
  int64_t n = 1;
  for (int i = 0; i < a.ndim; ++i) n *= a.shape[i];
  const int64_t bytes = n * (a.dtype == 2 ? 1 : 8);
  if (bytes != nbytes) {
    gks::set_error("gks_setup_copy: '%s' needs %lld bytes, got %lld", name, (long long)bytes, (long long)nbytes);
    return GKS_ERR_BAD_ARG;
  }
  if (bytes) memcpy(dst, a.p, bytes);
  return GKS_OK;
}

}  // extern "C"
