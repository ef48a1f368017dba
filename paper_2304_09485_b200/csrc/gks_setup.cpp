// Host-side native setup: stencil selection and reconstruction operators.
//
// Restates, per cell and in parallel (OpenMP):
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
// the hex-face angle ordering reproduces numpy's arithmetic exactly.
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

namespace gks {
void set_error(const char* fmt, ...);
}

namespace {

constexpr int NCOEF = 9;
constexpr double RANK_TOL = 1e-10;

struct V3 {
  double x, y, z;
};
inline V3 add(V3 a, V3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
inline V3 neg(V3 a) { return {-a.x, -a.y, -a.z}; }

struct Member {
  int64_t id;
  V3 s;
};

inline std::array<int64_t, 3> skey(const V3& s) {
  return {llround(s.x * 1e9), llround(s.y * 1e9), llround(s.z * 1e9)};
}

// _dedup (stencils.py:106-116): keep the first occurrence of (id, rounded shift)
std::vector<Member> dedup(const std::vector<Member>& in) {
  std::vector<Member> out;
  std::vector<std::array<int64_t, 4>> seen;
  out.reserve(in.size());
  seen.reserve(in.size());
  for (const Member& m : in) {
    auto k = skey(m.s);
    std::array<int64_t, 4> key{m.id, k[0], k[1], k[2]};
    bool dup = false;
    for (auto& q : seen)
      if (q == key) { dup = true; break; }
    if (dup) continue;
    seen.push_back(key);
    out.push_back(m);
  }
  return out;
}

inline double dot3(const double* a, const double* b) {
  double acc = 0.0;
  acc += a[0] * b[0];
  acc += a[1] * b[1];
  acc += a[2] * b[2];
  return acc;
}

const int TET_KEPT[4][3] = {{0, 1, 2}, {0, 1, 3}, {1, 2, 3}, {2, 0, 3}};
const int TET_ENL[4] = {0, 1, 2, 3};
const int HEX_PAT[8][3] = {{0, 1, 2}, {0, 2, 3}, {0, 3, 4}, {0, 4, 1},
                           {5, 1, 2}, {5, 2, 3}, {5, 3, 4}, {5, 4, 1}};

// ---------------------------------------------------------------------------
// small dense linear algebra
// ---------------------------------------------------------------------------

// One-sided Jacobi SVD of A (m x n, row-major, m >= n).  Returns singular
// values s (descending), U (m x n), V (n x n), both column-orthonormal.
void svd_jacobi(int m, int n, const double* A, double* s, double* U, double* V) {
  std::vector<double> a(A, A + (size_t)m * n);
  for (int i = 0; i < n * n; ++i) V[i] = 0.0;
  for (int i = 0; i < n; ++i) V[i * n + i] = 1.0;
  for (int sweep = 0; sweep < 60; ++sweep) {
    double off = 0.0;
    for (int p = 0; p < n - 1; ++p)
      for (int q = p + 1; q < n; ++q) {
        double al = 0, be = 0, ga = 0;
        for (int i = 0; i < m; ++i) {
          const double x = a[i * n + p], y = a[i * n + q];
          al += x * x;
          be += y * y;
          ga += x * y;
        }
        if (ga == 0.0) continue;
        const double rel = fabs(ga) / sqrt(al * be);
        if (!(rel > 1e-17)) continue;
        off = std::max(off, rel);
        const double zeta = (be - al) / (2.0 * ga);
        const double t = (zeta >= 0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / sqrt(1.0 + t * t), sn = c * t;
        for (int i = 0; i < m; ++i) {
          const double x = a[i * n + p], y = a[i * n + q];
          a[i * n + p] = c * x - sn * y;
          a[i * n + q] = sn * x + c * y;
        }
        for (int i = 0; i < n; ++i) {
          const double x = V[i * n + p], y = V[i * n + q];
          V[i * n + p] = c * x - sn * y;
          V[i * n + q] = sn * x + c * y;
        }
      }
    if (off < 1e-16) break;
  }
  std::vector<double> sv(n);
  for (int j = 0; j < n; ++j) {
    double acc = 0;
    for (int i = 0; i < m; ++i) acc += a[i * n + j] * a[i * n + j];
    sv[j] = sqrt(acc);
  }
  std::vector<int> ord(n);
  for (int j = 0; j < n; ++j) ord[j] = j;
  std::stable_sort(ord.begin(), ord.end(), [&](int x, int y) { return sv[x] > sv[y]; });
  std::vector<double> Vs(V, V + n * n);
  for (int jj = 0; jj < n; ++jj) {
    const int j = ord[jj];
    s[jj] = sv[j];
    for (int i = 0; i < m; ++i) U[i * n + jj] = sv[j] > 0 ? a[i * n + j] / sv[j] : 0.0;
    for (int i = 0; i < n; ++i) V[i * n + jj] = Vs[i * n + j];
  }
}

// _pinv (recon.py:60-69): pinv of A (m x n) -> P (n x m), or false if rank <
// rank_needed.  Requires m >= n (always true at the call sites).
bool pinv(int m, int n, const double* A, int rank_needed, double* P) {
  if (m < n || n == 0) return false;
  std::vector<double> s(n), U((size_t)m * n), V((size_t)n * n);
  svd_jacobi(m, n, A, s.data(), U.data(), V.data());
  if (s[0] == 0.0) return false;
  int rank = 0;
  for (int j = 0; j < n; ++j)
    if (s[j] >= RANK_TOL * s[0]) ++rank;
  if (rank < rank_needed) return false;
  for (int i = 0; i < n; ++i)
    for (int k = 0; k < m; ++k) {
      double acc = 0;
      for (int j = 0; j < rank; ++j) acc += V[i * n + j] * (1.0 / s[j]) * U[k * n + j];
      P[i * m + k] = acc;
    }
  return true;
}

inline void mono_rows(const double* xt, double* r) {
  const double x = xt[0], y = xt[1], z = xt[2];
  r[0] = x; r[1] = y; r[2] = z;
  r[3] = x * x; r[4] = x * y; r[5] = x * z; r[6] = y * y; r[7] = y * z; r[8] = z * z;
}

inline void mono_grad_rows(const double* xt, double g[3][NCOEF]) {
  const double x = xt[0], y = xt[1], z = xt[2];
  const double gx[9] = {1, 0, 0, 2 * x, y, z, 0, 0, 0};
  const double gy[9] = {0, 1, 0, 0, x, 0, 2 * y, z, 0};
  const double gz[9] = {0, 0, 1, 0, 0, x, 0, y, 2 * z};
  for (int d = 0; d < 9; ++d) { g[0][d] = gx[d]; g[1][d] = gy[d]; g[2][d] = gz[d]; }
}

}  // namespace

// ---------------------------------------------------------------------------
// setup object
// ---------------------------------------------------------------------------

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

struct MeshView {
  const GksMeshDesc* m;
  std::vector<Member> neighbors_of(int64_t c) const {
    std::vector<Member> out;
    for (int64_t k = m->cell_face_start[c]; k < m->cell_face_start[c + 1]; ++k) {
      const int64_t f = m->cell_face_list[k];
      if (m->face_neighbor[f] < 0) continue;
      const double* s = m->face_shift + 3 * f;
      if (m->face_owner[f] == c)
        out.push_back({m->face_neighbor[f], {s[0], s[1], s[2]}});
      else
        out.push_back({m->face_owner[f], {-s[0], -s[1], -s[2]}});
    }
    return out;
  }
};

// _ordered_neighbors (stencils.py:72-103)
void ordered_neighbors(const GksMeshDesc* m, int64_t c, std::vector<int64_t>& ids,
                       std::vector<V3>& sh) {
  const int64_t f0 = m->cell_face_start[c];
  const int nf = (int)(m->cell_face_start[c + 1] - f0);
  ids.assign(nf, -1);
  sh.assign(nf, V3{0, 0, 0});
  std::vector<std::array<double, 3>> nrm(nf);
  for (int k = 0; k < nf; ++k) {
    const int64_t f = m->cell_face_list[f0 + k];
    const double sg = m->face_owner[f] == c ? 1.0 : -1.0;
    for (int d = 0; d < 3; ++d) nrm[k][d] = sg * m->face_normal[3 * f + d];
    if (m->face_neighbor[f] < 0) continue;
    const double* s = m->face_shift + 3 * f;
    if (m->face_owner[f] == c) {
      ids[k] = m->face_neighbor[f];
      sh[k] = {s[0], s[1], s[2]};
    } else {
      ids[k] = m->face_owner[f];
      sh[k] = {-s[0], -s[1], -s[2]};
    }
  }
  if (m->cell_kind[c] != 1) return;
  // hex: (pole a, equator by angle, pole b)
  int pole_b = 1;
  double best = 0;
  for (int k = 1; k < 6; ++k) {
    const double d = dot3(nrm[k].data(), nrm[0].data());
    if (k == 1 || d < best) { best = d; pole_b = k; }
  }
  std::vector<int> rest;
  for (int k = 1; k < 6; ++k)
    if (k != pole_b) rest.push_back(k);
  const double* axis = nrm[0].data();
  const double* r0 = nrm[rest[0]].data();
  const double pr = dot3(r0, axis);
  double b1[3] = {r0[0] - pr * axis[0], r0[1] - pr * axis[1], r0[2] - pr * axis[2]};
  const double nb = sqrt(dot3(b1, b1));
  for (double& x : b1) x /= nb;
  const double b2[3] = {axis[1] * b1[2] - axis[2] * b1[1], axis[2] * b1[0] - axis[0] * b1[2],
                        axis[0] * b1[1] - axis[1] * b1[0]};
  std::vector<double> ang(4);
  for (int i = 0; i < 4; ++i) ang[i] = atan2(dot3(nrm[rest[i]].data(), b2), dot3(nrm[rest[i]].data(), b1));
  std::vector<int> o = {0, 1, 2, 3};
  std::stable_sort(o.begin(), o.end(), [&](int a, int b) { return ang[a] < ang[b]; });
  std::vector<int> order = {0, rest[o[0]], rest[o[1]], rest[o[2]], rest[o[3]], pole_b};
  std::vector<int64_t> ids2(6);
  std::vector<V3> sh2(6);
  for (int k = 0; k < 6; ++k) { ids2[k] = ids[order[k]]; sh2[k] = sh[order[k]]; }
  ids = ids2;
  sh = sh2;
}

struct CellStencil {
  std::vector<int64_t> nbr;
  std::vector<V3> nbr_s;
  std::vector<Member> big;
  std::vector<std::vector<Member>> subs;
  bool weno_fallback = false, hweno_fallback = false;
};

void build_cell_stencil(const GksMeshDesc* m, const MeshView& mv, int64_t c, CellStencil& st) {
  ordered_neighbors(m, c, st.nbr, st.nbr_s);
  const int nf = (int)st.nbr.size();
  std::vector<Member> big;
  big.push_back({c, {0, 0, 0}});
  for (int k = 0; k < nf; ++k)
    if (st.nbr[k] >= 0) big.push_back({st.nbr[k], st.nbr_s[k]});
  for (int k = 0; k < nf; ++k) {
    if (st.nbr[k] < 0) continue;
    for (const Member& jt : mv.neighbors_of(st.nbr[k])) big.push_back({jt.id, add(st.nbr_s[k], jt.s)});
  }
  st.big = dedup(big);
  st.subs.clear();
  if (m->cell_kind[c] == 1) {
    for (auto& pat : HEX_PAT) {
      if (st.nbr[pat[0]] < 0 || st.nbr[pat[1]] < 0 || st.nbr[pat[2]] < 0) continue;
      std::vector<Member> mi = {{c, {0, 0, 0}}};
      for (int k : pat) mi.push_back({st.nbr[k], st.nbr_s[k]});
      auto di = dedup(mi);
      if (di.size() == 4) st.subs.push_back(di);
    }
  } else {
    for (int p = 0; p < 4; ++p) {
      const int* kept = TET_KEPT[p];
      if (st.nbr[kept[0]] < 0 || st.nbr[kept[1]] < 0 || st.nbr[kept[2]] < 0) continue;
      std::vector<Member> mi = {{c, {0, 0, 0}}};
      for (int q = 0; q < 3; ++q) mi.push_back({st.nbr[kept[q]], st.nbr_s[kept[q]]});
      const int64_t host = st.nbr[TET_ENL[p]];
      const V3 hs = st.nbr_s[TET_ENL[p]];
      std::vector<Member> added;
      for (const Member& jt : mv.neighbors_of(host)) {
        const V3 tot = add(hs, jt.s);
        const double mx = std::max(fabs(tot.x), std::max(fabs(tot.y), fabs(tot.z)));
        if (jt.id == c && mx < 1e-12) continue;
        added.push_back({jt.id, tot});
      }
      std::stable_sort(added.begin(), added.end(), [](const Member& a, const Member& b) {
        if (a.id != b.id) return a.id < b.id;
        return skey(a.s) < skey(b.s);
      });
      for (size_t q = 0; q < added.size() && q < 3; ++q) mi.push_back(added[q]);
      auto di = dedup(mi);
      if (di.size() == 7) st.subs.push_back(di);
    }
  }
  if (st.subs.size() < 2) {
    st.subs.clear();
    st.weno_fallback = true;
  }
  int present = 0;
  for (int k = 0; k < nf; ++k) present += st.nbr[k] >= 0;
  st.hweno_fallback = present < 2;
}

struct Geo {
  const GksMeshDesc* m;
  // cell-average rows of the basis over member (j, shift) in the chart of c
  void avg_row(int64_t c, int64_t j, const V3& s, double* row) const {
    const double* c0 = m->cell_centroid + 3 * c;
    const double h0 = m->cell_h[c];
    for (int d = 0; d < NCOEF; ++d) row[d] = 0.0;
    for (int64_t q = m->cell_cq_start[j]; q < m->cell_cq_start[j + 1]; ++q) {
      const double* p = m->cq_point + 3 * q;
      const double xt[3] = {((p[0] + s.x) - c0[0]) / h0, ((p[1] + s.y) - c0[1]) / h0,
                            ((p[2] + s.z) - c0[2]) / h0};
      double r[NCOEF];
      mono_rows(xt, r);
      const double w = m->cq_weight[q];
      for (int d = 0; d < NCOEF; ++d) row[d] += w * r[d];
    }
  }
  // h_j * mean gradient rows of the basis over member (j, s), chart of c (hweno.py:45-60)
  void grad_rows(int64_t c, int64_t j, const V3& s, double out[3][NCOEF]) const {
    const double* c0 = m->cell_centroid + 3 * c;
    const double h0 = m->cell_h[c];
    double acc[3][NCOEF] = {};
    for (int64_t q = m->cell_cq_start[j]; q < m->cell_cq_start[j + 1]; ++q) {
      const double* p = m->cq_point + 3 * q;
      const double xt[3] = {((p[0] + s.x) - c0[0]) / h0, ((p[1] + s.y) - c0[1]) / h0,
                            ((p[2] + s.z) - c0[2]) / h0};
      double g[3][NCOEF];
      mono_grad_rows(xt, g);
      const double w = m->cq_weight[q];
      for (int x = 0; x < 3; ++x)
        for (int d = 0; d < NCOEF; ++d) acc[x][d] += w * g[x][d];
    }
    for (int x = 0; x < 3; ++x)
      for (int d = 0; d < NCOEF; ++d) out[x][d] = m->cell_h[j] * (acc[x][d] / h0);
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
  GksSetup* S = new GksSetup();
  const int64_t nc = m->ncells;
  S->nc = nc;
  int nfpc = 0;
  for (int64_t c = 0; c < nc; ++c)
    nfpc = std::max<int>(nfpc, (int)(m->cell_face_start[c + 1] - m->cell_face_start[c]));
  S->nfpc = nfpc;
  MeshView mv{m};
  const bool want_weno = schemes & 1, want_hweno = schemes & 2;
  const bool want_stencils = schemes == 0 || (schemes & 4);

  // ---- pass A: sizes ------------------------------------------------------
  std::vector<int32_t> big_n(nc), sub_n(nc), nbr_n(nc);
  std::vector<int8_t> wfb(nc), hfb(nc);
  int64_t sub_len_max = 0;
#pragma omp parallel for schedule(dynamic, 256) reduction(max : sub_len_max)
  for (int64_t c = 0; c < nc; ++c) {
    CellStencil st;
    build_cell_stencil(m, mv, c, st);
    big_n[c] = (int32_t)st.big.size();
    sub_n[c] = (int32_t)st.subs.size();
    int present = 0;
    for (int64_t id : st.nbr) present += id >= 0;
    nbr_n[c] = present;
    wfb[c] = st.weno_fallback;
    hfb[c] = st.hweno_fallback;
    for (auto& sub : st.subs) sub_len_max = std::max<int64_t>(sub_len_max, (int64_t)sub.size() - 1);
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
    // member counts per sub need the stencils: one more pass
#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t c = 0; c < nc; ++c) {
      CellStencil st;
      build_cell_stencil(m, mv, c, st);
      int64_t si = S->sub_cell_start[c];
      for (auto& sub : st.subs) sub_len[si++] = (int64_t)sub.size();
    }
    S->sub_member_start.assign(sub_len.size() + 1, 0);
    for (size_t k = 0; k < sub_len.size(); ++k) S->sub_member_start[k + 1] = S->sub_member_start[k] + sub_len[k];
    S->sub_ids.resize(S->sub_member_start.back());
    S->sub_shift.resize(S->sub_member_start.back() * 3);
#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t c = 0; c < nc; ++c) {
      CellStencil st;
      build_cell_stencil(m, mv, c, st);
      for (size_t k = 0; k < st.nbr.size(); ++k) {
        S->nbr_ids[c * nfpc + k] = st.nbr[k];
        S->nbr_shift[(c * nfpc + k) * 3 + 0] = st.nbr_s[k].x;
        S->nbr_shift[(c * nfpc + k) * 3 + 1] = st.nbr_s[k].y;
        S->nbr_shift[(c * nfpc + k) * 3 + 2] = st.nbr_s[k].z;
      }
      int64_t b = S->big_start[c];
      for (auto& mb : st.big) {
        S->big_ids[b] = mb.id;
        S->big_shift[3 * b] = mb.s.x; S->big_shift[3 * b + 1] = mb.s.y; S->big_shift[3 * b + 2] = mb.s.z;
        ++b;
      }
      int64_t si = S->sub_cell_start[c];
      for (auto& sub : st.subs) {
        int64_t q = S->sub_member_start[si++];
        for (auto& mb : sub) {
          S->sub_ids[q] = mb.id;
          S->sub_shift[3 * q] = mb.s.x; S->sub_shift[3 * q + 1] = mb.s.y; S->sub_shift[3 * q + 2] = mb.s.z;
          ++q;
        }
      }
    }
  }

  // ---- recon geometry (recon.py:104-146) ----------------------------------
  Geo geo{m};
  S->avg0.assign(nc * NCOEF, 0.0);
  S->beta.assign(nc * NCOEF * NCOEF, 0.0);
#pragma omp parallel for schedule(static)
  for (int64_t c = 0; c < nc; ++c) {
    geo.avg_row(c, c, V3{0, 0, 0}, &S->avg0[c * NCOEF]);
    double* B = &S->beta[c * 81];
    const double* c0 = m->cell_centroid + 3 * c;
    const double h0 = m->cell_h[c];
    for (int64_t q = m->cell_cq_start[c]; q < m->cell_cq_start[c + 1]; ++q) {
      const double* p = m->cq_point + 3 * q;
      const double xt[3] = {(p[0] - c0[0]) / h0, (p[1] - c0[1]) / h0, (p[2] - c0[2]) / h0};
      double g[3][NCOEF];
      mono_grad_rows(xt, g);
      const double w = m->cq_weight[q];
      for (int d = 0; d < 9; ++d)
        for (int e = 0; e < 9; ++e) B[d * 9 + e] += w * (g[0][d] * g[0][e] + g[1][d] * g[1][e] + g[2][d] * g[2][e]);
    }
    // + B2 (second-derivative rows, recon.py:28-36)
    B[3 * 9 + 3] += 4.0; B[4 * 9 + 4] += 1.0; B[5 * 9 + 5] += 1.0;
    B[6 * 9 + 6] += 4.0; B[7 * 9 + 7] += 1.0; B[8 * 9 + 8] += 4.0;
  }
  auto member_row = [&](int64_t c, const Member& mb, double* row) {
    geo.avg_row(c, mb.id, mb.s, row);
    for (int d = 0; d < NCOEF; ++d) row[d] -= S->avg0[c * NCOEF + d];
  };

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
      CellStencil st;
      build_cell_stencil(m, mv, c, st);
      int nsurv = 0, scols = 0;
      for (auto& sub : st.subs) {
        const int S1 = (int)sub.size() - 1;
        std::vector<double> rows(S1 * 3), full(NCOEF), op(3 * S1);
        for (int k = 1; k <= S1; ++k) {
          member_row(c, sub[k], full.data());
          for (int d = 0; d < 3; ++d) rows[(k - 1) * 3 + d] = full[d];
        }
        if (!pinv(S1, 3, rows.data(), 3, op.data())) continue;
        for (int d = 0; d < 3; ++d)
          for (int k = 0; k < S1; ++k) S->w_sub_op[((c * mup + nsurv) * 3 + d) * sup + k] = op[d * S1 + k];
        for (int k = 0; k < S1; ++k) S->w_sub_gather[(c * mup + nsurv) * sup + k] = sub[k + 1].id;
        S->w_sub_active[c * mup + nsurv] = 1;
        scols = std::max(scols, S1);
        ++nsurv;
      }
      if (nsurv < 2) {  // fewer than two candidates: drop them all
        for (int mm = 0; mm < nsurv; ++mm) {
          S->w_sub_active[c * mup + mm] = 0;
          for (int64_t k = 0; k < 3 * sup; ++k) S->w_sub_op[(c * mup + mm) * 3 * sup + k] = 0.0;
          for (int64_t k = 0; k < sup; ++k) S->w_sub_gather[(c * mup + mm) * sup + k] = 0;
        }
        nsurv = 0;
        scols = 0;
      }
      msurv[c] = nsurv;
      ssurv[c] = scols;
      const int R = (int)st.big.size() - 1;
      std::vector<double> rows((size_t)std::max(R, 0) * NCOEF);
      for (int k = 1; k <= R; ++k) member_row(c, st.big[k], &rows[(k - 1) * NCOEF]);
      std::vector<double> op;
      bool ok = false;
      if (nsurv && R >= NCOEF) {
        op.assign((size_t)NCOEF * R, 0.0);
        ok = pinv(R, NCOEF, rows.data(), NCOEF, op.data());
      }
      int cols = R;
      if (!ok) {
        S->w_big_degree[c] = 1;
        cols = std::max(R, 1);
        op.assign((size_t)NCOEF * cols, 0.0);
        if (R >= 3) {
          std::vector<double> lr(R * 3), lin(3 * R);
          for (int k = 0; k < R; ++k)
            for (int d = 0; d < 3; ++d) lr[k * 3 + d] = rows[k * NCOEF + d];
          if (pinv(R, 3, lr.data(), 3, lin.data()))
            for (int d = 0; d < 3; ++d)
              for (int k = 0; k < R; ++k) op[d * cols + k] = lin[d * R + k];
        }
      }
      for (int d = 0; d < NCOEF; ++d)
        for (int k = 0; k < cols; ++k) S->w_big_op[(c * NCOEF + d) * kmax + k] = op[d * cols + k];
      for (int k = 1; k <= R; ++k) S->w_big_gather[c * kmax + k - 1] = st.big[k].id;
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
      CellStencil st;
      build_cell_stencil(m, mv, c, st);
      std::vector<Member> ids = {{c, {0, 0, 0}}};
      for (size_t k = 0; k < st.nbr.size(); ++k)
        if (st.nbr[k] >= 0) ids.push_back({st.nbr[k], st.nbr_s[k]});
      const int na = (int)ids.size() - 1;
      const int R = na + 3 * (int)ids.size();
      std::vector<double> rows((size_t)R * NCOEF);
      for (int k = 1; k <= na; ++k) member_row(c, ids[k], &rows[(k - 1) * NCOEF]);
      for (size_t k = 0; k < ids.size(); ++k) {
        double g[3][NCOEF];
        geo.grad_rows(c, ids[k].id, ids[k].s, g);
        for (int x = 0; x < 3; ++x)
          for (int d = 0; d < NCOEF; ++d) rows[(na + 3 * k + x) * NCOEF + d] = g[x][d];
      }
      std::vector<double> op((size_t)NCOEF * R, 0.0);
      bool ok = false;
      if (!st.hweno_fallback && R >= NCOEF) ok = pinv(R, NCOEF, rows.data(), NCOEF, op.data());
      if (!ok) {
        S->h_big_degree[c] = 1;
        std::fill(op.begin(), op.end(), 0.0);
        std::vector<double> lr(R * 3), lin(3 * R);
        for (int k = 0; k < R; ++k)
          for (int d = 0; d < 3; ++d) lr[k * 3 + d] = rows[k * NCOEF + d];
        if (pinv(R, 3, lr.data(), 3, lin.data()))
          for (int d = 0; d < 3; ++d)
            for (int k = 0; k < R; ++k) op[d * R + k] = lin[d * R + k];
      }
      S->h_big_ncols[c] = R;
      for (int d = 0; d < NCOEF; ++d) {
        for (int k = 0; k < na; ++k) S->h_big_op[(c * NCOEF + d) * W + k] = op[d * R + k];
        for (int k = na; k < R; ++k) S->h_big_op[(c * NCOEF + d) * W + amax + (k - na)] = op[d * R + k];
      }
      S->h_big_grad_gather[c * gmax] = c;
      S->h_big_grad_scale[c * gmax] = m->cell_h[c];
      for (int k = 1; k <= na; ++k) {
        S->h_big_avg_gather[c * amax + k - 1] = ids[k].id;
        S->h_big_grad_gather[c * gmax + k] = ids[k].id;
        S->h_big_grad_scale[c * gmax + k] = m->cell_h[ids[k].id];
      }
      int nsurv = 0;
      if (!st.hweno_fallback) {
        double g0[3][NCOEF];
        geo.grad_rows(c, c, V3{0, 0, 0}, g0);
        for (int k = 1; k <= na; ++k) {
          // rows: [avg row of the neighbour (3 cols); grad rows of target; grad rows of neighbour]
          double srows[7 * 3];
          double full[NCOEF];
          member_row(c, ids[k], full);
          for (int d = 0; d < 3; ++d) srows[d] = full[d];
          for (int x = 0; x < 3; ++x)
            for (int d = 0; d < 3; ++d) srows[(1 + x) * 3 + d] = g0[x][d];
          double g[3][NCOEF];
          geo.grad_rows(c, ids[k].id, ids[k].s, g);
          for (int x = 0; x < 3; ++x)
            for (int d = 0; d < 3; ++d) srows[(4 + x) * 3 + d] = g[x][d];
          double sop[21];
          if (!pinv(7, 3, srows, 3, sop)) continue;
          for (int i = 0; i < 21; ++i) S->h_sub_op[(c * mup + nsurv) * 21 + i] = sop[i];
          S->h_sub_gather[(c * mup + nsurv) * 2 + 0] = c;
          S->h_sub_gather[(c * mup + nsurv) * 2 + 1] = ids[k].id;
          S->h_sub_active[c * mup + nsurv] = 1;
          ++nsurv;
        }
        if (nsurv < 2) {
          for (int mm = 0; mm < nsurv; ++mm) {
            S->h_sub_active[c * mup + mm] = 0;
            for (int i = 0; i < 21; ++i) S->h_sub_op[(c * mup + mm) * 21 + i] = 0.0;
            S->h_sub_gather[(c * mup + mm) * 2] = 0;
            S->h_sub_gather[(c * mup + mm) * 2 + 1] = 0;
          }
          nsurv = 0;
        }
      }
      msurv[c] = nsurv;
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
