// Per-cell setup arithmetic shared by the host build (gks_setup.cpp, g++,
// -ffp-contract=off) and the device build (gks_setup_dev.cu, nvcc
// -fmad=false): stencil selection, the one-sided Jacobi SVD pseudo-inverse
// and the reconstruction operators of one cell.  Both translation units
// compile the same statements in the same order without contraction, with
// IEEE sqrt / division on both sides, so the device-built operators are the
// host-built ones bit for bit (tests/test_device_setup_gpu.py).
//
// Restates:
//   gks3d/mesh/stencils.py:72-116   _ordered_neighbors, _dedup
//   gks3d/mesh/stencils.py:119-192  build_stencils (big stencil, sub-stencils)
//   gks3d/recon.py:28-36, 60-69     B2, _pinv (rank tolerance 1e-10)
//   gks3d/recon.py:104-164          ReconGeometry (avg0, beta)
//   gks3d/recon.py:216-274          WenoReconstructor._build_operators
//   gks3d/hweno.py:45-137           HwenoReconstructor._grad_rows / _build_operators
// Fixed-capacity arrays replace the host vectors: at most 6 faces per cell
// (tet 4, hex 6), so a big stencil has at most 1 + 6 + 36 members before
// deduplication and at most 42 neighbour rows.
#pragma once

#include <math.h>
#include <stdint.h>

#include "gks.h"

#ifdef __CUDACC__
#define GKS_HD __host__ __device__ inline
#else
#define GKS_HD inline
#endif

namespace gks {
namespace su {

constexpr int NCOEF = 9;
constexpr double RANK_TOL = 1e-10;
constexpr int NF = 6;                   // faces per cell
constexpr int BIGCAP = 1 + NF + NF * NF;
constexpr int RMAX = BIGCAP - 1;        // rows of a pseudo-inverse
constexpr int NSUBCAP = 8;              // sub-stencils per cell (hex 8, tet 4)
constexpr int SUBCAP = 7;               // members of a sub-stencil (tet 7, hex 4)

struct V3 {
  double x, y, z;
};
GKS_HD V3 add(V3 a, V3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }

struct Member {
  int64_t id;
  V3 s;
};

GKS_HD void skey(const V3& s, int64_t k[3]) {
  k[0] = llround(s.x * 1e9);
  k[1] = llround(s.y * 1e9);
  k[2] = llround(s.z * 1e9);
}

// lexicographic order of the rounded shifts (std::array operator<)
GKS_HD bool skey_less(const V3& a, const V3& b) {
  int64_t ka[3], kb[3];
  skey(a, ka);
  skey(b, kb);
  for (int i = 0; i < 3; ++i) {
    if (ka[i] < kb[i]) return true;
    if (kb[i] < ka[i]) return false;
  }
  return false;
}

GKS_HD bool same_member(const Member& a, const Member& b) {
  if (a.id != b.id) return false;
  int64_t ka[3], kb[3];
  skey(a.s, ka);
  skey(b.s, kb);
  return ka[0] == kb[0] && ka[1] == kb[1] && ka[2] == kb[2];
}

// _dedup (stencils.py:106-116): keep the first occurrence of (id, rounded
// shift), in place; returns the new length
GKS_HD int dedup(Member* m, int n) {
  int out = 0;
  for (int i = 0; i < n; ++i) {
    bool dup = false;
    for (int j = 0; j < out; ++j)
      if (same_member(m[j], m[i])) { dup = true; break; }
    if (!dup) m[out++] = m[i];
  }
  return out;
}

GKS_HD double dot3(const double* a, const double* b) {
  double acc = 0.0;
  acc += a[0] * b[0];
  acc += a[1] * b[1];
  acc += a[2] * b[2];
  return acc;
}

// interior-face neighbours of cell c in its face order (Mesh.cell_neighbors)
GKS_HD int neighbors_of(const GksMeshDesc& m, int64_t c, Member* out) {
  int n = 0;
  for (int64_t k = m.cell_face_start[c]; k < m.cell_face_start[c + 1]; ++k) {
    const int64_t f = m.cell_face_list[k];
    if (m.face_neighbor[f] < 0) continue;
    const double* s = m.face_shift + 3 * f;
    if (m.face_owner[f] == c)
      out[n++] = {m.face_neighbor[f], {s[0], s[1], s[2]}};
    else
      out[n++] = {m.face_owner[f], {-s[0], -s[1], -s[2]}};
  }
  return n;
}

// _ordered_neighbors (stencils.py:72-103): one slot per face (-1 boundary);
// hex faces reordered as (pole a, equator by angle, pole b).  Returns the
// face count.
GKS_HD int ordered_neighbors(const GksMeshDesc& m, int64_t c, int64_t* ids, V3* sh) {
  const int64_t f0 = m.cell_face_start[c];
  const int nf = (int)(m.cell_face_start[c + 1] - f0);
  double nrm[NF][3];
  for (int k = 0; k < nf; ++k) {
    ids[k] = -1;
    sh[k] = V3{0, 0, 0};
    const int64_t f = m.cell_face_list[f0 + k];
    const double sg = m.face_owner[f] == c ? 1.0 : -1.0;
    for (int d = 0; d < 3; ++d) nrm[k][d] = sg * m.face_normal[3 * f + d];
    if (m.face_neighbor[f] < 0) continue;
    const double* s = m.face_shift + 3 * f;
    if (m.face_owner[f] == c) {
      ids[k] = m.face_neighbor[f];
      sh[k] = {s[0], s[1], s[2]};
    } else {
      ids[k] = m.face_owner[f];
      sh[k] = {-s[0], -s[1], -s[2]};
    }
  }
  if (m.cell_kind[c] != 1) return nf;
  int pole_b = 1;
  double best = 0;
  for (int k = 1; k < 6; ++k) {
    const double d = dot3(nrm[k], nrm[0]);
    if (k == 1 || d < best) { best = d; pole_b = k; }
  }
  int rest[4], nr = 0;
  for (int k = 1; k < 6; ++k)
    if (k != pole_b) rest[nr++] = k;
  const double* axis = nrm[0];
  const double* r0 = nrm[rest[0]];
  const double pr = dot3(r0, axis);
  double b1[3] = {r0[0] - pr * axis[0], r0[1] - pr * axis[1], r0[2] - pr * axis[2]};
  const double nb = sqrt(dot3(b1, b1));
  for (int d = 0; d < 3; ++d) b1[d] /= nb;
  const double b2[3] = {axis[1] * b1[2] - axis[2] * b1[1], axis[2] * b1[0] - axis[0] * b1[2],
                        axis[0] * b1[1] - axis[1] * b1[0]};
  double ang[4];
  for (int i = 0; i < 4; ++i) ang[i] = atan2(dot3(nrm[rest[i]], b2), dot3(nrm[rest[i]], b1));
  int o[4] = {0, 1, 2, 3};
  for (int i = 1; i < 4; ++i)  // stable insertion sort by angle
    for (int j = i; j > 0 && ang[o[j]] < ang[o[j - 1]]; --j) {
      const int t = o[j]; o[j] = o[j - 1]; o[j - 1] = t;
    }
  const int order[6] = {0, rest[o[0]], rest[o[1]], rest[o[2]], rest[o[3]], pole_b};
  int64_t ids2[6];
  V3 sh2[6];
  for (int k = 0; k < 6; ++k) { ids2[k] = ids[order[k]]; sh2[k] = sh[order[k]]; }
  for (int k = 0; k < 6; ++k) { ids[k] = ids2[k]; sh[k] = sh2[k]; }
  return nf;
}

// sub-stencil patterns (stencils.py:150-186)
GKS_HD int tet_kept(int p, int q) {
  const int T[4][3] = {{0, 1, 2}, {0, 1, 3}, {1, 2, 3}, {2, 0, 3}};
  return T[p][q];
}
GKS_HD int hex_pat(int p, int q) {
  const int H[8][3] = {{0, 1, 2}, {0, 2, 3}, {0, 3, 4}, {0, 4, 1}, {5, 1, 2}, {5, 2, 3}, {5, 3, 4}, {5, 4, 1}};
  return H[p][q];
}

struct Stencil {
  int nf = 0;
  int64_t nbr[NF];
  V3 nbr_s[NF];
  int nbig = 0;
  Member big[BIGCAP];
  int nsub = 0;
  int sublen[NSUBCAP];
  Member sub[NSUBCAP][SUBCAP];
  bool weno_fallback = false, hweno_fallback = false;
  GKS_HD int present() const {
    int p = 0;
    for (int k = 0; k < nf; ++k) p += nbr[k] >= 0;
    return p;
  }
};

// build_stencils for one cell (stencils.py:119-192).  rank: optional
// reference id of each cell (the enlarged tet members sort by it; NULL =
// the ids themselves).
GKS_HD void build_stencil(const GksMeshDesc& m, int64_t c, Stencil& st) {
  st.nf = ordered_neighbors(m, c, st.nbr, st.nbr_s);
  const int nf = st.nf;
  Member nb[NF];
  int n = 0;
  st.big[n++] = {c, {0, 0, 0}};
  for (int k = 0; k < nf; ++k)
    if (st.nbr[k] >= 0) st.big[n++] = {st.nbr[k], st.nbr_s[k]};
  for (int k = 0; k < nf; ++k) {
    if (st.nbr[k] < 0) continue;
    const int nn = neighbors_of(m, st.nbr[k], nb);
    for (int q = 0; q < nn; ++q) st.big[n++] = {nb[q].id, add(st.nbr_s[k], nb[q].s)};
  }
  st.nbig = dedup(st.big, n);
  st.nsub = 0;
  if (m.cell_kind[c] == 1) {
    for (int p = 0; p < 8; ++p) {
      const int a = hex_pat(p, 0), b = hex_pat(p, 1), d = hex_pat(p, 2);
      if (st.nbr[a] < 0 || st.nbr[b] < 0 || st.nbr[d] < 0) continue;
      Member* mi = st.sub[st.nsub];
      mi[0] = {c, {0, 0, 0}};
      mi[1] = {st.nbr[a], st.nbr_s[a]};
      mi[2] = {st.nbr[b], st.nbr_s[b]};
      mi[3] = {st.nbr[d], st.nbr_s[d]};
      const int len = dedup(mi, 4);
      if (len == 4) st.sublen[st.nsub++] = len;
    }
  } else {
    for (int p = 0; p < 4; ++p) {
      const int k0 = tet_kept(p, 0), k1 = tet_kept(p, 1), k2 = tet_kept(p, 2);
      if (st.nbr[k0] < 0 || st.nbr[k1] < 0 || st.nbr[k2] < 0) continue;
      Member mi[SUBCAP];
      mi[0] = {c, {0, 0, 0}};
      mi[1] = {st.nbr[k0], st.nbr_s[k0]};
      mi[2] = {st.nbr[k1], st.nbr_s[k1]};
      mi[3] = {st.nbr[k2], st.nbr_s[k2]};
      int len = 4;
      const int64_t host = st.nbr[p];  // enlarged through face p (TET_ENL = identity)
      const V3 hs = st.nbr_s[p];
      Member added[NF];
      int na = 0;
      if (host >= 0) {
        const int nn = neighbors_of(m, host, nb);
        for (int q = 0; q < nn; ++q) {
          const V3 tot = add(hs, nb[q].s);
          const double mx = fmax(fabs(tot.x), fmax(fabs(tot.y), fabs(tot.z)));
          if (nb[q].id == c && mx < 1e-12) continue;
          added[na++] = {nb[q].id, tot};
        }
      }
      // stable sort by (reference id, rounded shift)
      for (int i = 1; i < na; ++i)
        for (int j = i; j > 0; --j) {
          const Member& x = added[j];
          const Member& y = added[j - 1];
          const int64_t rx = m.cell_rank ? m.cell_rank[x.id] : x.id;
          const int64_t ry = m.cell_rank ? m.cell_rank[y.id] : y.id;
          const bool less = rx != ry ? rx < ry : skey_less(x.s, y.s);
          if (!less) break;
          const Member t = added[j]; added[j] = added[j - 1]; added[j - 1] = t;
        }
      for (int q = 0; q < na && q < 3; ++q) mi[len++] = added[q];
      len = dedup(mi, len);
      if (len == 7) {
        for (int q = 0; q < 7; ++q) st.sub[st.nsub][q] = mi[q];
        st.sublen[st.nsub++] = 7;
      }
    }
  }
  if (st.nsub < 2) {
    st.nsub = 0;
    st.weno_fallback = true;
  } else {
    st.weno_fallback = false;
  }
  st.hweno_fallback = st.present() < 2;
}

// ---------------------------------------------------------------------------
// pseudo-inverse: one-sided Jacobi SVD (in place on a, m x n row-major,
// m >= n), singular values sorted descending (stable), then
// P = V diag(1/s) U^T over the numerical rank (recon.py:60-69).
// put(i, k, value) receives P[i][k] (n x m); nothing is written when the
// rank is below rank_needed (returns false).
// ---------------------------------------------------------------------------
template <class Put>
GKS_HD bool pinv(int m, int n, double* a, int rank_needed, Put put) {
  if (m < n || n == 0) return false;
  double V[NCOEF * NCOEF];
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
        off = fmax(off, rel);
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
  double sv[NCOEF];
  int ord[NCOEF];
  for (int j = 0; j < n; ++j) {
    double acc = 0;
    for (int i = 0; i < m; ++i) acc += a[i * n + j] * a[i * n + j];
    sv[j] = sqrt(acc);
    ord[j] = j;
  }
  for (int i = 1; i < n; ++i)  // stable sort, descending
    for (int j = i; j > 0 && sv[ord[j]] > sv[ord[j - 1]]; --j) {
      const int t = ord[j]; ord[j] = ord[j - 1]; ord[j - 1] = t;
    }
  const double s0 = sv[ord[0]];
  if (s0 == 0.0) return false;
  int rank = 0;
  for (int j = 0; j < n; ++j)
    if (sv[ord[j]] >= RANK_TOL * s0) ++rank;
  if (rank < rank_needed) return false;
  for (int i = 0; i < n; ++i)
    for (int k = 0; k < m; ++k) {
      double acc = 0;
      for (int jj = 0; jj < rank; ++jj) {
        const int j = ord[jj];
        const double u = sv[j] > 0 ? a[k * n + j] / sv[j] : 0.0;
        acc += V[i * n + j] * (1.0 / sv[j]) * u;
      }
      put(i, k, acc);
    }
  return true;
}

// ---------------------------------------------------------------------------
// geometry rows (recon.py:104-146, hweno.py:45-60)
// ---------------------------------------------------------------------------
GKS_HD void mono_rows(const double* xt, double* r) {
  const double x = xt[0], y = xt[1], z = xt[2];
  r[0] = x; r[1] = y; r[2] = z;
  r[3] = x * x; r[4] = x * y; r[5] = x * z; r[6] = y * y; r[7] = y * z; r[8] = z * z;
}

GKS_HD void mono_grad_rows(const double* xt, double g[3][NCOEF]) {
  const double x = xt[0], y = xt[1], z = xt[2];
  const double gx[9] = {1, 0, 0, 2 * x, y, z, 0, 0, 0};
  const double gy[9] = {0, 1, 0, 0, x, 0, 2 * y, z, 0};
  const double gz[9] = {0, 0, 1, 0, 0, x, 0, y, 2 * z};
  for (int d = 0; d < 9; ++d) { g[0][d] = gx[d]; g[1][d] = gy[d]; g[2][d] = gz[d]; }
}

// cell-average row of the basis over member (j, s) in the chart of c
GKS_HD void avg_row(const GksMeshDesc& m, int64_t c, int64_t j, const V3& s, double* row) {
  const double* c0 = m.cell_centroid + 3 * c;
  const double h0 = m.cell_h[c];
  for (int d = 0; d < NCOEF; ++d) row[d] = 0.0;
  for (int64_t q = m.cell_cq_start[j]; q < m.cell_cq_start[j + 1]; ++q) {
    const double* p = m.cq_point + 3 * q;
    const double xt[3] = {((p[0] + s.x) - c0[0]) / h0, ((p[1] + s.y) - c0[1]) / h0, ((p[2] + s.z) - c0[2]) / h0};
    double r[NCOEF];
    mono_rows(xt, r);
    const double w = m.cq_weight[q];
    for (int d = 0; d < NCOEF; ++d) row[d] += w * r[d];
  }
}

// h_j * mean gradient rows of the basis over member (j, s), chart of c
GKS_HD void grad_rows(const GksMeshDesc& m, int64_t c, int64_t j, const V3& s, double out[3][NCOEF]) {
  const double* c0 = m.cell_centroid + 3 * c;
  const double h0 = m.cell_h[c];
  double acc[3][NCOEF];
  for (int x = 0; x < 3; ++x)
    for (int d = 0; d < NCOEF; ++d) acc[x][d] = 0.0;
  for (int64_t q = m.cell_cq_start[j]; q < m.cell_cq_start[j + 1]; ++q) {
    const double* p = m.cq_point + 3 * q;
    const double xt[3] = {((p[0] + s.x) - c0[0]) / h0, ((p[1] + s.y) - c0[1]) / h0, ((p[2] + s.z) - c0[2]) / h0};
    double g[3][NCOEF];
    mono_grad_rows(xt, g);
    const double w = m.cq_weight[q];
    for (int x = 0; x < 3; ++x)
      for (int d = 0; d < NCOEF; ++d) acc[x][d] += w * g[x][d];
  }
  for (int x = 0; x < 3; ++x)
    for (int d = 0; d < NCOEF; ++d) out[x][d] = m.cell_h[j] * (acc[x][d] / h0);
}

// avg0 (9) and the smoothness matrix beta (81) of cell c (recon.py:104-146)
GKS_HD void cell_geometry(const GksMeshDesc& m, int64_t c, double* avg0, double* B) {
  avg_row(m, c, c, V3{0, 0, 0}, avg0);
  for (int i = 0; i < 81; ++i) B[i] = 0.0;
  const double* c0 = m.cell_centroid + 3 * c;
  const double h0 = m.cell_h[c];
  for (int64_t q = m.cell_cq_start[c]; q < m.cell_cq_start[c + 1]; ++q) {
    const double* p = m.cq_point + 3 * q;
    const double xt[3] = {(p[0] - c0[0]) / h0, (p[1] - c0[1]) / h0, (p[2] - c0[2]) / h0};
    double g[3][NCOEF];
    mono_grad_rows(xt, g);
    const double w = m.cq_weight[q];
    for (int d = 0; d < 9; ++d)
      for (int e = 0; e < 9; ++e) B[d * 9 + e] += w * (g[0][d] * g[0][e] + g[1][d] * g[1][e] + g[2][d] * g[2][e]);
  }
  // + B2 (second-derivative rows, recon.py:28-36)
  B[3 * 9 + 3] += 4.0; B[4 * 9 + 4] += 1.0; B[5 * 9 + 5] += 1.0;
  B[6 * 9 + 6] += 4.0; B[7 * 9 + 7] += 1.0; B[8 * 9 + 8] += 4.0;
}

GKS_HD void member_row(const GksMeshDesc& m, int64_t c, const Member& mb, const double* avg0c, double* row) {
  avg_row(m, c, mb.id, mb.s, row);
  for (int d = 0; d < NCOEF; ++d) row[d] -= avg0c[d];
}

// ---------------------------------------------------------------------------
// WENO operators of one cell (recon.py:216-274).  Sink receives:
//   sub_op(slot, d, k, v), sub_gather(slot, k, id), sub_active(slot),
//   drop_subs(n)   -- fewer than two candidates survived: undo slots [0, n)
//   big_op(d, k, v), big_gather(k, id), big_degree(1)
// and the return value packs the surviving count and their column width
// (nsurv | scols << 8).  Values never written stay zero.
// ---------------------------------------------------------------------------
template <class Sink>
GKS_HD int weno_cell(const GksMeshDesc& m, int64_t c, const Stencil& st, const double* avg0c, Sink& out) {
  double a[RMAX * NCOEF];
  double full[NCOEF];
  int nsurv = 0, scols = 0;
  for (int si = 0; si < st.nsub; ++si) {
    const int S1 = st.sublen[si] - 1;
    for (int k = 1; k <= S1; ++k) {
      member_row(m, c, st.sub[si][k], avg0c, full);
      for (int d = 0; d < 3; ++d) a[(k - 1) * 3 + d] = full[d];
    }
    const int slot = nsurv;
    if (!pinv(S1, 3, a, 3, [&](int d, int k, double v) { out.sub_op(slot, d, k, v); })) continue;
    for (int k = 0; k < S1; ++k) out.sub_gather(slot, k, st.sub[si][k + 1].id);
    out.sub_active(slot);
    scols = scols > S1 ? scols : S1;
    ++nsurv;
  }
  if (nsurv < 2) {
    out.drop_subs(nsurv);
    nsurv = 0;
    scols = 0;
  }
  const int R = st.nbig - 1;
  auto fill_rows = [&](int ncol) {
    for (int k = 1; k <= R; ++k) {
      member_row(m, c, st.big[k], avg0c, full);
      for (int d = 0; d < ncol; ++d) a[(k - 1) * ncol + d] = full[d];
    }
  };
  bool ok = false;
  if (nsurv && R >= NCOEF) {
    fill_rows(NCOEF);
    ok = pinv(R, NCOEF, a, NCOEF, [&](int d, int k, double v) { out.big_op(d, k, v); });
  }
  if (!ok) {
    out.big_degree(1);
    if (R >= 3) {
      fill_rows(3);
      pinv(R, 3, a, 3, [&](int d, int k, double v) { out.big_op(d, k, v); });
    }
  }
  for (int k = 1; k <= R; ++k) out.big_gather(k - 1, st.big[k].id);
  return nsurv | (scols << 8);
}

// ---------------------------------------------------------------------------
// HWENO operators of one cell (hweno.py:62-137).  Sink receives:
//   big_op(d, col, v)     col < na: average columns, else na + gradient column
//   avg_gather(k, id), grad_gather(k, id, h), big_ncols(R), big_degree(1),
//   sub_op(slot, i, v) (i < 21), sub_gather(slot, id), sub_active(slot),
//   drop_subs(n)
// Returns the surviving sub-stencil count.
// ---------------------------------------------------------------------------
template <class Sink>
GKS_HD int hweno_cell(const GksMeshDesc& m, int64_t c, const Stencil& st, const double* avg0c, Sink& out) {
  Member ids[NF + 1];
  int nid = 0;
  ids[nid++] = {c, {0, 0, 0}};
  for (int k = 0; k < st.nf; ++k)
    if (st.nbr[k] >= 0) ids[nid++] = {st.nbr[k], st.nbr_s[k]};
  const int na = nid - 1;
  const int R = na + 3 * nid;
  double a[RMAX * NCOEF];
  auto fill_rows = [&](int ncol) {
    double full[NCOEF];
    for (int k = 1; k <= na; ++k) {
      member_row(m, c, ids[k], avg0c, full);
      for (int d = 0; d < ncol; ++d) a[(k - 1) * ncol + d] = full[d];
    }
    for (int k = 0; k < nid; ++k) {
      double g[3][NCOEF];
      grad_rows(m, c, ids[k].id, ids[k].s, g);
      for (int x = 0; x < 3; ++x)
        for (int d = 0; d < ncol; ++d) a[(na + 3 * k + x) * ncol + d] = g[x][d];
    }
  };
  bool ok = false;
  if (!st.hweno_fallback && R >= NCOEF) {
    fill_rows(NCOEF);
    ok = pinv(R, NCOEF, a, NCOEF, [&](int d, int k, double v) { out.big_op(d, k, v); });
  }
  if (!ok) {
    out.big_degree(1);
    fill_rows(3);
    pinv(R, 3, a, 3, [&](int d, int k, double v) { out.big_op(d, k, v); });
  }
  out.big_ncols(R);
  out.grad_gather(0, c, m.cell_h[c]);
  for (int k = 1; k <= na; ++k) {
    out.avg_gather(k - 1, ids[k].id);
    out.grad_gather(k, ids[k].id, m.cell_h[ids[k].id]);
  }
  int nsurv = 0;
  if (!st.hweno_fallback) {
    double g0[3][NCOEF];
    grad_rows(m, c, c, V3{0, 0, 0}, g0);
    for (int k = 1; k <= na; ++k) {
      // rows: [avg row of the neighbour (3 cols); grad rows of target; grad rows of neighbour]
      double srows[7 * 3];
      double full[NCOEF];
      member_row(m, c, ids[k], avg0c, full);
      for (int d = 0; d < 3; ++d) srows[d] = full[d];
      for (int x = 0; x < 3; ++x)
        for (int d = 0; d < 3; ++d) srows[(1 + x) * 3 + d] = g0[x][d];
      double g[3][NCOEF];
      grad_rows(m, c, ids[k].id, ids[k].s, g);
      for (int x = 0; x < 3; ++x)
        for (int d = 0; d < 3; ++d) srows[(4 + x) * 3 + d] = g[x][d];
      const int slot = nsurv;
      if (!pinv(7, 3, srows, 3, [&](int i, int kk, double v) { out.sub_op(slot, i * 7 + kk, v); })) continue;
      out.sub_gather(slot, ids[k].id);
      out.sub_active(slot);
      ++nsurv;
    }
    if (nsurv < 2) {
      out.drop_subs(nsurv);
      nsurv = 0;
    }
  }
  return nsurv;
}

}  // namespace su
}  // namespace gks
