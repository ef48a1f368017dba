// Device-side gas-kinetic interface solver (FP64), one thread per face
// quadrature point.
//
// Restates the algorithm of the reference gks3d/kinetic.py and gks3d/flux.py
// (/root/reference/pkg/src/gks3d) in a form fused for the FP64 pipe:
//
//   * Maxwellian moments <u^a>, <v^b>, <w^c>, <xi^2s> by the recurrence of
//     kinetic.py:113-137 (erfc/exp seeds for the half ranges);
//   * closed-form micro-slope solve (kinetic.py:271-302) and the time slope
//     from the compatibility condition (kinetic.py:305-312);
//   * compatibility equilibrium W0 and its slopes (flux.py:69-107);
//   * the six coefficient families of flux.py:110-159 are folded, per
//     Maxwellian, into ONE polynomial weight
//         W(c) = s . psi(c) + sum_k c_k (d_k . psi(c)),  psi = (1,u,v,w,|c|^2/2)
//     so each of the three Maxwellians (g0, g_l on u>0, g_r on u<0) costs a
//     single pass over 23 weight monomials instead of the reference's
//     memoized table of psi rows.  The result is the same integral; only the
//     rounding order differs (parity bar 1e-12 relative, see tests).
#pragma once
#include <cuda_runtime.h>
#include <math.h>

#include <type_traits>

// FP64 divisions are the face kernel's most expensive single operations;
// three per face point are gone (C2 face 2.679 -> 2.570 ms): the pressure
// of a side state as rho * h (h = 1 / (2 lam) of its moment table) instead
// of rho / (2 lam) (GKS_PS_MUL), h itself as (2 / (N + 3)) e / rho from
// cons_to_prim_h's reciprocal density instead of 0.5 / lam (GKS_H_MUL), and
// the per-cell 1 / h of the face-point evaluation from a table.  Rounding-
// level changes; every parity bar holds.
// both sides of the interface in one unrolled body: with the 255-register
// budget (no spills) the compiler overlaps the two sides' work (C2 face
// 2.543 -> 2.531 ms); it was kept rolled while registers were the limit
#ifndef GKS_SIDE_UNROLL
#define GKS_SIDE_UNROLL 1
#endif
// time slopes from the Euler flux Jacobians of the conserved slopes
// (euler_axis_jvp) instead of the 13-group moment sums: C2 face 2.499 ->
// 2.330 ms, C3 2.91-3.02 -> 2.83 ms; a rounding-level change, every parity
// bar holds
#ifndef GKS_TSLOPE_EULER
#define GKS_TSLOPE_EULER 1
#endif
// the interface (equilibrium) state's flux and point terms in closed form
// (equilibrium_flux): no moment table, no micro-slope solves; C2 face 2.330 ->
// 2.203 ms
#ifndef GKS_EQ_CLOSED
#define GKS_EQ_CLOSED 1
#endif
#ifndef GKS_PS_MUL
#define GKS_PS_MUL 1
#endif
#ifndef GKS_H_MUL
#define GKS_H_MUL 1
#endif
#ifndef GKS_ERFC_SCALED
#define GKS_ERFC_SCALED 1
#endif

namespace gks {

struct Maxw {
  double U[7];  // <u^a>, full or half range, a = 0..6
  double V[6];  // <v^b>, b = 0..5
  double W[6];  // <w^c>, c = 0..5
  double X[3];  // <xi^2s>, s = 0..2
  double h;     // 1 / (2 lam)
};

struct KinConst {
  double gamma;
  double nd;   // internal dof N = (5 - 3 gamma)/(gamma - 1)
  double n3;   // N + 3
  double c4n;  // 4 / (N + 3)
  double c2n;  // 2 / (N + 3): h = 1 / (2 lam) = c2n e / rho for internal energy density e
};

__host__ __device__ inline KinConst make_kin(double gamma) {
  KinConst k;
  k.gamma = gamma;
  k.nd = (5.0 - 3.0 * gamma) / (gamma - 1.0);
  k.n3 = k.nd + 3.0;
  k.c4n = 4.0 / k.n3;
  k.c2n = 2.0 / k.n3;
  return k;
}

template <int N>
__device__ __forceinline__ void recur(double* m, double mean, double h) {
#pragma unroll
  for (int k = 2; k < N; ++k) m[k] = mean * m[k - 1] + (double)(k - 1) * h * m[k - 2];
}

// Full-range tables of a primitive state (rho, U, V, W, lam).
__device__ __forceinline__ void maxw_full(Maxw& m, const double w[5], const KinConst& kc) {
  const double h = 0.5 / w[4];
  m.h = h;
  m.U[0] = 1.0; m.U[1] = w[1]; recur<7>(m.U, w[1], h);
  m.V[0] = 1.0; m.V[1] = w[2]; recur<6>(m.V, w[2], h);
  m.W[0] = 1.0; m.W[1] = w[3]; recur<6>(m.W, w[3], h);
  m.X[0] = 1.0;
  m.X[1] = kc.nd * h;                    // N / (2 lam)
  m.X[2] = kc.nd * (kc.nd + 2.0) * h * h;  // N (N + 2) / (4 lam^2)
}

// maxw_full with h = 1 / (2 lam) supplied (cons_to_prim_h forms it without a
// division)
__device__ __forceinline__ void maxw_full_h(Maxw& m, const double w[5], const KinConst& kc, double h) {
  m.h = h;
  m.U[0] = 1.0; m.U[1] = w[1]; recur<7>(m.U, w[1], h);
  m.V[0] = 1.0; m.V[1] = w[2]; recur<6>(m.V, w[2], h);
  m.W[0] = 1.0; m.W[1] = w[3]; recur<6>(m.W, w[3], h);
  m.X[0] = 1.0;
  m.X[1] = kc.nd * h;
  m.X[2] = kc.nd * (kc.nd + 2.0) * h * h;
}

// Replace the u table by its half-range version: sign = +1 (u>0) or -1 (u<0).
// Needs m.h = 1/(2 lam) from maxw_full; exp(-lam u^2) / (2 sqrt(pi lam)) is
// formed as exp(.) sqrt(lam) h / sqrt(pi) (no division).
__device__ __forceinline__ void maxw_half_u(Maxw& m, const double w[5], double sign) {
  const double lam = w[4], u = w[1];
  const double rl = sqrt(lam);
  constexpr double kInvSqrtPi = 0.56418958354775628695;  // 1 / sqrt(pi)
  const double e = exp(-lam * u * u);
  const double g = kInvSqrtPi * e * rl * m.h;
#if GKS_ERFC_SCALED
  // erfc(x) = exp(-x^2) erfcx(x) for x >= 0 and 2 - exp(-x^2) erfcx(-x)
  // below, reusing exp(-lam u^2) of the Gaussian term: erfcx is branch-light
  // where erfc switches algorithms across |x| (warp divergence)
  const double x = -sign * rl * u;
  const double ex = e * erfcx(fabs(x));
  m.U[0] = 0.5 * (x >= 0.0 ? ex : 2.0 - ex);
#else
  m.U[0] = 0.5 * erfc(-sign * rl * u);
#endif
  m.U[1] = u * m.U[0] + sign * g;
  recur<7>(m.U, u, m.h);
}

// One group of weight monomials sharing the factor v^B w^C xi^2S, with a
// polynomial sum_a k[a] u^a in u, integrated against u^P psi.  Grouping by
// the (v, w, xi) part lets each group's u-sums be formed once (the compiler
// may not reassociate FP sums by itself).
template <int P, int B, int C, int S, int NA>
__device__ __forceinline__ void group_acc(const Maxw& m, const double (&k)[NA], double o[5]) {
  double s0 = k[0] * m.U[P], s1 = k[0] * m.U[P + 1], s2 = k[0] * m.U[P + 2];
#pragma unroll
  for (int a = 1; a < NA; ++a) {
    s0 += k[a] * m.U[a + P];
    s1 += k[a] * m.U[a + P + 1];
    s2 += k[a] * m.U[a + P + 2];
  }
  const double vw = m.V[B] * m.W[C];
  const double vwx = vw * m.X[S];
  o[0] += s0 * vwx;
  o[1] += s1 * vwx;
  o[2] += s0 * (m.V[B + 1] * m.W[C] * m.X[S]);
  o[3] += s0 * (m.V[B] * m.W[C + 1] * m.X[S]);
  o[4] += 0.5 * (s2 * vwx + s0 * (m.X[S] * (m.V[B + 2] * m.W[C] + m.V[B] * m.W[C + 2]) + vw * m.X[S + 1]));
}

// <u^P W(c) psi> with W(c) = s.psi(c) + DIR * ds * sum_k c_k d_k.psi(c).
// The 23 weight monomials (8 without DIR) fall into 13 (6) groups.  The
// directional coefficients come scaled by ds on the fly (the flux passes'
// time-coefficient factor) instead of as a materialised scaled copy: 15
// fewer live doubles across the side loop.
template <int P, bool DIR>
__device__ __forceinline__ void wmom(const Maxw& m, const double s[5], const double (*d)[5], double ds,
                                     double o[5]) {
  o[0] = o[1] = o[2] = o[3] = o[4] = 0.0;
  const double hs = 0.5 * s[4];
  // (two accumulators per output, alternating groups, to halve the add
  // chain of the 13 groups: measured slower, 2.73 vs 2.67 ms on C2 -- the
  // kernel is limited by register pressure, not by this chain)
  if (!DIR) {
    group_acc<P, 0, 0, 0, 3>(m, {s[0], s[1], hs}, o);  // 1, u, u^2
    group_acc<P, 1, 0, 0, 1>(m, {s[2]}, o);            // v
    group_acc<P, 0, 1, 0, 1>(m, {s[3]}, o);            // w
    group_acc<P, 2, 0, 0, 1>(m, {hs}, o);              // v^2
    group_acc<P, 0, 2, 0, 1>(m, {hs}, o);              // w^2
    group_acc<P, 0, 0, 1, 1>(m, {hs}, o);              // xi^2
    return;
  }
  const double hu = 0.5 * ds * d[0][4], hv = 0.5 * ds * d[1][4], hw = 0.5 * ds * d[2][4];
  group_acc<P, 0, 0, 0, 4>(m, {s[0], s[1] + ds * d[0][0], hs + ds * d[0][1], hu}, o);         // 1, u, u^2, u^3
  group_acc<P, 1, 0, 0, 3>(m, {s[2] + ds * d[1][0], ds * (d[0][2] + d[1][1]), hv}, o);       // v, uv, u^2 v
  group_acc<P, 0, 1, 0, 3>(m, {s[3] + ds * d[2][0], ds * (d[0][3] + d[2][1]), hw}, o);       // w, uw, u^2 w
  group_acc<P, 2, 0, 0, 2>(m, {hs + ds * d[1][2], hu}, o);                                   // v^2, u v^2
  group_acc<P, 0, 2, 0, 2>(m, {hs + ds * d[2][3], hu}, o);                                   // w^2, u w^2
  group_acc<P, 0, 0, 1, 2>(m, {hs, hu}, o);                                                  // xi^2, u xi^2
  group_acc<P, 1, 1, 0, 1>(m, {ds * (d[1][3] + d[2][2])}, o);                                // vw
  group_acc<P, 3, 0, 0, 1>(m, {hv}, o);                                                      // v^3
  group_acc<P, 0, 3, 0, 1>(m, {hw}, o);                                                      // w^3
  group_acc<P, 1, 2, 0, 1>(m, {hv}, o);                                                      // v w^2
  group_acc<P, 2, 1, 0, 1>(m, {hw}, o);                                                      // v^2 w
  group_acc<P, 1, 0, 1, 1>(m, {hv}, o);                                                      // v xi^2
  group_acc<P, 0, 1, 1, 1>(m, {hw}, o);                                                      // w xi^2
}

// <u^P (sum_k c_k d_k.psi) psi>: wmom<P, true> with s = 0 and ds = 1 (the
// time-slope right-hand sides and the deferred-tau slope family), without
// the zero terms IEEE arithmetic cannot fold away (0 * x, 0 + x); a group
// whose leading coefficient vanishes is the same sum started one u-order
// higher (group_acc<P + 1, ...>)
template <int P>
__device__ __forceinline__ void wmom_dir(const Maxw& m, const double (*d)[5], double o[5]) {
  o[0] = o[1] = o[2] = o[3] = o[4] = 0.0;
  const double hu = 0.5 * d[0][4], hv = 0.5 * d[1][4], hw = 0.5 * d[2][4];
  group_acc<P + 1, 0, 0, 0, 3>(m, {d[0][0], d[0][1], hu}, o);  // u, u^2, u^3
  group_acc<P, 1, 0, 0, 3>(m, {d[1][0], d[0][2] + d[1][1], hv}, o);  // v, uv, u^2 v
  group_acc<P, 0, 1, 0, 3>(m, {d[2][0], d[0][3] + d[2][1], hw}, o);  // w, uw, u^2 w
  group_acc<P, 2, 0, 0, 2>(m, {d[1][2], hu}, o);                     // v^2, u v^2
  group_acc<P, 0, 2, 0, 2>(m, {d[2][3], hu}, o);                     // w^2, u w^2
  group_acc<P + 1, 0, 0, 1, 1>(m, {hu}, o);                          // u xi^2
  group_acc<P, 1, 1, 0, 1>(m, {d[1][3] + d[2][2]}, o);               // vw
  group_acc<P, 3, 0, 0, 1>(m, {hv}, o);                              // v^3
  group_acc<P, 0, 3, 0, 1>(m, {hw}, o);                              // w^3
  group_acc<P, 1, 2, 0, 1>(m, {hv}, o);                              // v w^2
  group_acc<P, 2, 1, 0, 1>(m, {hw}, o);                              // v^2 w
  group_acc<P, 1, 0, 1, 1>(m, {hv}, o);                              // v xi^2
  group_acc<P, 0, 1, 1, 1>(m, {hw}, o);                              // w xi^2
}

// the zero-weight directional moment: wmom_dir where it measured faster
// (the non-point kernels: C2 face 2.520 -> 2.50-2.51 ms), the general
// wmom otherwise (the point-value kernels: 2.5 % slower with it)
template <int P, bool DIRFORM>
__device__ __forceinline__ void dir_moment(const Maxw& m, const double (*d)[5], double o[5]) {
  if constexpr (DIRFORM) {
    wmom_dir<P>(m, d, o);
  } else {
    const double zero5[5] = {0, 0, 0, 0, 0};
    wmom<P, true>(m, zero5, d, 1.0, o);
  }
}

// rho sum_k <c_k (a_k.psi) psi> over the three local axes for the micro-
// slopes a_k of the conserved slopes dq_k, in closed form: a Maxwellian's
// moments <c_k psi> are the Euler fluxes of the gas (gamma = (N+5)/(N+3)),
// and the conserved increment dq perturbs rho g by rho (a.psi) g, so the sum
// is sum_k (dF_k/dq) dq_k -- the Euler flux Jacobians applied to the slopes
// (the time slope's right-hand side, kinetic.py:305-312, at ~70 operations
// instead of the 13-group moment sum's ~230).  h = 1 / (2 lam) = p / rho.
__device__ __forceinline__ void euler_axis_jvp(const double w[5], double h, const KinConst& kc,
                                               const double (*dq)[5], double out[5]) {
  const double vel[3] = {w[1], w[2], w[3]};
  const double ke = 0.5 * (vel[0] * vel[0] + vel[1] * vel[1] + vel[2] * vel[2]);
  const double gm1 = kc.c2n;                       // gamma - 1 = 2 / (N + 3)
  const double H = ke + 0.5 * (kc.n3 + 2.0) * h;   // (E + p) / rho
#pragma unroll
  for (int i = 0; i < 5; ++i) out[i] = 0.0;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const double* d = dq[k];
    const double a = d[1 + k] - vel[k] * d[0];
    const double b = gm1 * (ke * d[0] - (vel[0] * d[1] + vel[1] * d[2] + vel[2] * d[3]) + d[4]);
    out[0] += d[1 + k];
#pragma unroll
    for (int i = 0; i < 3; ++i) out[1 + i] += vel[i] * a + vel[k] * d[1 + i] + (i == k ? b : 0.0);
    out[4] += H * a + vel[k] * (b + d[4]);
  }
}

// The equilibrium part of the interface flux (kinetic.py:110-159, the g0
// terms) in closed form:  rho0 <u psi (c1 + c3 Ab.psi + c2 sum_k c_k ab_k.psi)>_0.
// rho0 <u psi>_0 is the Euler flux along the normal axis; rho0 <u (Ab.psi) psi>_0
// is its Jacobian applied to D = rho0 <(Ab.psi) psi>_0 (the time slope's
// right-hand side); and rho0 <u c_k (ab_k.psi) psi>_0 is the derivative of the
// Gaussian moment vector T_k = rho <u c_k psi> along the conserved slope dq_k:
//   T_k[0]   = rho (U0 Uk + th d0k)
//   T_k[1+i] = rho (U0 Uk Ui + th (U0 dki + Uk d0i + Ui d0k))
//   T_k[4]   = rho/2 (U0 Uk |U|^2 + th ((Kt+4) U0 Uk + |U|^2 d0k) + (Kt+2) th^2 d0k)
// with th = h = 1 / (2 lam) and Kt = N + 3.  Differentiated through
// e = rho dU = dm - U drho and b = dp = (gamma-1)(dE - U.dm + ke drho):
// ~180 operations instead of the full moment table and the 13-group sums
// (plus the four micro-slope solves the sums need).
__device__ __forceinline__ void equilibrium_flux(const double w[5], double h, const KinConst& kc, const double D[5],
                                                 const double (*dq)[5], double c1, double c3, double c2,
                                                 double out[5]) {
  const double rho = w[0];
  const double U[3] = {w[1], w[2], w[3]};
  const double U2 = U[0] * U[0] + U[1] * U[1] + U[2] * U[2];
  const double ke = 0.5 * U2;
  const double gm1 = kc.c2n;
  const double kt4 = kc.n3 + 4.0, kt2 = kc.n3 + 2.0;
  const double H = ke + 0.5 * kt2 * h;
  const double mn = rho * U[0];
  // c1 F_x + c3 (dF_x/dq) D
  const double a = D[1] - U[0] * D[0];
  const double bD = gm1 * (ke * D[0] - (U[0] * D[1] + U[1] * D[2] + U[2] * D[3]) + D[4]);
  out[0] = c1 * mn + c3 * D[1];
#pragma unroll
  for (int i = 0; i < 3; ++i)
    out[1 + i] = c1 * (mn * U[i] + (i == 0 ? rho * h : 0.0)) + c3 * (U[i] * a + U[0] * D[1 + i] + (i == 0 ? bD : 0.0));
  out[4] = c1 * mn * H + c3 * (H * a + U[0] * (bD + D[4]));
  // c2 sum_k dT_k . dq_k
  double t[5] = {0, 0, 0, 0, 0};
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const double* d = dq[k];
    const double d0 = d[0];
    const double e[3] = {d[1] - U[0] * d0, d[2] - U[1] * d0, d[3] - U[2] * d0};
    const double Ue = U[0] * e[0] + U[1] * e[1] + U[2] * e[2];
    const double b = gm1 * (d[4] - Ue - ke * d0);
    const double UU = U[0] * U[k];
    const double p1 = d0 * UU + e[0] * U[k] + U[0] * e[k];
    t[0] += p1 + (k == 0 ? b : 0.0);
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      double v = U[i] * p1 + UU * e[i];
      if (k == i) v += b * U[0] + h * e[0];
      if (i == 0) v += b * U[k] + h * e[k];
      if (k == 0) v += b * U[i] + h * e[i];
      t[1 + i] += v;
    }
    double v4 = U2 * p1 + 2.0 * UU * Ue + kt4 * (b * UU + h * (e[0] * U[k] + U[0] * e[k]));
    if (k == 0) v4 += b * U2 + 2.0 * h * Ue + kt2 * h * (2.0 * b - h * d0);
    t[4] += 0.5 * v4;
  }
#pragma unroll
  for (int i = 0; i < 5; ++i) out[i] += c2 * t[i];
}

// Gram matrix G_ij = <u^P psi_i psi_j> of one Maxwellian.  Every weight
// without the directional part is a product with it: wmom<P,false>(m, s) = G s,
// so the several such weights of one Maxwellian share one G.
template <int P>
__device__ __forceinline__ void gram(const Maxw& m, double G[5][5]) {
  const double* U = m.U + P;
  const double* V = m.V;
  const double* W = m.W;
  const double x1 = m.X[1];
  const double r = V[2] + W[2] + x1;  // <v^2 + w^2 + xi^2>
  G[0][0] = U[0];
  G[0][1] = U[1];
  G[0][2] = U[0] * V[1];
  G[0][3] = U[0] * W[1];
  G[0][4] = 0.5 * (U[2] + U[0] * r);
  G[1][1] = U[2];
  G[1][2] = U[1] * V[1];
  G[1][3] = U[1] * W[1];
  G[1][4] = 0.5 * (U[3] + U[1] * r);
  G[2][2] = U[0] * V[2];
  G[2][3] = U[0] * V[1] * W[1];
  G[2][4] = 0.5 * (U[2] * V[1] + U[0] * (V[3] + V[1] * (W[2] + x1)));
  G[3][3] = U[0] * W[2];
  G[3][4] = 0.5 * (U[2] * W[1] + U[0] * (W[3] + W[1] * (V[2] + x1)));
  G[4][4] = 0.25 * (U[4] + 2.0 * U[2] * r +
                    U[0] * (V[4] + W[4] + m.X[2] + 2.0 * (V[2] * W[2] + (V[2] + W[2]) * x1)));
#pragma unroll
  for (int i = 1; i < 5; ++i)
#pragma unroll
    for (int j = 0; j < i; ++j) G[i][j] = G[j][i];
}

// For the NS vectors s_k: acc_k += scale * G s_k and q0 += scale * G e_0
// (the first column), with G = <u^P psi psi^T> formed one unique entry at a
// time and scattered into both of its symmetric positions at once: no
// 25-entry matrix is ever live (ncu r01: the materialised G was the face
// kernel's largest spill site).  Same products as gram + gram_acc, summed in
// a different order.
template <int P, int NS>
__device__ __forceinline__ void gram_scatter(const Maxw& m, double scale, const double* const (&sv)[NS],
                                             double* const (&av)[NS], double q0[5]) {
  const double* U = m.U + P;
  const double* V = m.V;
  const double* W = m.W;
  const double x1 = m.X[1];
  const double r = V[2] + W[2] + x1;  // <v^2 + w^2 + xi^2>
  auto put = [&](int i, int j, double g) {
    g *= scale;
    if (j == 0) q0[i] += g;
    else if (i == 0) q0[j] += g;
#pragma unroll
    for (int k = 0; k < NS; ++k) {
      av[k][i] += g * sv[k][j];
      if (i != j) av[k][j] += g * sv[k][i];
    }
  };
  put(0, 0, U[0]);
  put(0, 1, U[1]);
  put(0, 2, U[0] * V[1]);
  put(0, 3, U[0] * W[1]);
  put(0, 4, 0.5 * (U[2] + U[0] * r));
  put(1, 1, U[2]);
  put(1, 2, U[1] * V[1]);
  put(1, 3, U[1] * W[1]);
  put(1, 4, 0.5 * (U[3] + U[1] * r));
  put(2, 2, U[0] * V[2]);
  put(2, 3, U[0] * V[1] * W[1]);
  put(2, 4, 0.5 * (U[2] * V[1] + U[0] * (V[3] + V[1] * (W[2] + x1))));
  put(3, 3, U[0] * W[2]);
  put(3, 4, 0.5 * (U[2] * W[1] + U[0] * (W[3] + W[1] * (V[2] + x1))));
  put(4, 4, 0.25 * (U[4] + 2.0 * U[2] * r + U[0] * (V[4] + W[4] + m.X[2] + 2.0 * (V[2] * W[2] + (V[2] + W[2]) * x1))));
}

// acc += scale * G s
__device__ __forceinline__ void gram_acc(const double G[5][5], const double s[5], double scale, double acc[5]) {
#pragma unroll
  for (int i = 0; i < 5; ++i)
    acc[i] += scale * (G[i][0] * s[0] + G[i][1] * s[1] + G[i][2] * s[2] + G[i][3] * s[3] + G[i][4] * s[4]);
}

// Per-state constants of the micro-slope solve (shared by the 4 solves of
// one Maxwellian: 3 spatial slopes + the time slope).
struct SlopeConst {
  double U, V, W, lam, ir, k2, c4;  // ir = 1/rho, k2 = |u|^2 + (N+3)/(2 lam), c4 = 4 lam^2 / (N+3)
};

// h = 1 / (2 lam) (Maxw::h)
__device__ __forceinline__ SlopeConst slope_const(const double w[5], const KinConst& kc, double h) {
  SlopeConst s;
  s.U = w[1]; s.V = w[2]; s.W = w[3]; s.lam = w[4];
  s.ir = 1.0 / w[0];
  s.k2 = s.U * s.U + s.V * s.V + s.W * s.W + kc.n3 * h;
  s.c4 = kc.c4n * s.lam * s.lam;
  return s;
}

__device__ __forceinline__ SlopeConst slope_const(const double w[5], const KinConst& kc) {
  return slope_const(w, kc, 0.5 / w[4]);
}

// kinetic.py:271-302 closed-form solve of <a psi> = dq / rho.
__device__ __forceinline__ void micro_slope(const SlopeConst& s, const double dq[5], double a[5]) {
  const double b0 = dq[0] * s.ir, b1 = dq[1] * s.ir, b2 = dq[2] * s.ir, b3 = dq[3] * s.ir, b4 = dq[4] * s.ir;
  const double U = s.U, V = s.V, W = s.W, lam = s.lam;
  const double r1 = b1 - U * b0, r2 = b2 - V * b0, r3 = b3 - W * b0;
  const double r4 = 2.0 * b4 - s.k2 * b0;
  a[4] = s.c4 * (r4 - 2.0 * U * r1 - 2.0 * V * r2 - 2.0 * W * r3);
  a[3] = 2.0 * lam * r3 - W * a[4];
  a[2] = 2.0 * lam * r2 - V * a[4];
  a[1] = 2.0 * lam * r1 - U * a[4];
  a[0] = b0 - U * a[1] - V * a[2] - W * a[3] - 0.5 * a[4] * s.k2;
}

__device__ __forceinline__ void micro_slope(const double w[5], const double dq[5], const KinConst& kc, double a[5]) {
  micro_slope(slope_const(w, kc), dq, a);
}

// Conserved -> primitive; returns false on rho <= 0 / e <= 0 / non-finite
// (kinetic.py:35-51).
__device__ __forceinline__ bool cons_to_prim(const double q[5], const KinConst& kc, double w[5]) {
  const double rho = q[0];
  if (!(rho > 0.0) || !isfinite(rho)) return false;
  const double ir = 1.0 / rho;
  const double u = q[1] * ir, v = q[2] * ir, ww = q[3] * ir;
  const double e = q[4] - 0.5 * (q[1] * u + q[2] * v + q[3] * ww);
  if (!(e > 0.0) || !isfinite(e)) return false;
  w[0] = rho; w[1] = u; w[2] = v; w[3] = ww;
  w[4] = kc.n3 * rho / (4.0 * e);
  return true;
}

// cons_to_prim that also returns h = 1 / (2 lam) = (2 / (N + 3)) e / rho from
// the reciprocal density it already has: one FP64 division less per state
// than 0.5 / lam (the two agree to rounding)
__device__ __forceinline__ bool cons_to_prim_h(const double q[5], const KinConst& kc, double w[5], double& h) {
  const double rho = q[0];
  if (!(rho > 0.0) || !isfinite(rho)) return false;
  const double ir = 1.0 / rho;
  const double u = q[1] * ir, v = q[2] * ir, ww = q[3] * ir;
  const double e = q[4] - 0.5 * (q[1] * u + q[2] * v + q[3] * ww);
  if (!(e > 0.0) || !isfinite(e)) return false;
  w[0] = rho; w[1] = u; w[2] = v; w[3] = ww;
  w[4] = kc.n3 * rho / (4.0 * e);
  h = kc.c2n * e * ir;
  return true;
}

__device__ __forceinline__ void prim_to_cons(const double w[5], const KinConst& kc, double q[5]) {
  const double rho = w[0];
  q[0] = rho;
  q[1] = rho * w[1]; q[2] = rho * w[2]; q[3] = rho * w[3];
  q[4] = 0.5 * rho * (w[1] * w[1] + w[2] * w[2] + w[3] * w[3]) + kc.n3 * rho / (4.0 * w[4]);
}

__device__ __forceinline__ bool prim_ok(const double w[5]) {
  return (w[0] > 0.0) && (w[4] > 0.0) && isfinite(w[0]) && isfinite(w[1]) && isfinite(w[2]) &&
         isfinite(w[3]) && isfinite(w[4]);
}

enum : int { MODEL_INVISCID = 0, MODEL_VISCOUS = 1 };

struct FluxIn {
  double wl[5], wr[5];      // local-frame primitive states
  double sl[3][5], sr[3][5];  // local-frame conserved slopes along (n, t1, t2)
};

// time coefficients of flux.py:162-179 (divided by dt) and of the point
// value at time tp (flux.py:182-188)
struct TimeCoef {
  double c1, c2, c3, c4, c5, c6;  // flux families (g base/slope/time, f base/slope/time)
  double g1, g2, g3, f1, f2, f3;  // point-value families
};

__device__ __forceinline__ TimeCoef time_coefficients(double tau, double dt, double tp) {
  TimeCoef t;
  if (isinf(tau)) {
    // collisionless limit with slopes dropped: the KFVS split flux
    t.c1 = t.c2 = t.c3 = t.c5 = t.c6 = 0.0;
    t.c4 = 1.0;
  } else {
    const double x = dt / tau;
    const double em1 = -expm1(-x);
    const double e = exp(-x);
    const double idt = 1.0 / dt;
    t.c1 = (dt - tau * em1) * idt;
    t.c2 = (2.0 * tau * tau * em1 - tau * dt * e - tau * dt) * idt;
    t.c3 = (0.5 * dt * dt - tau * dt + tau * tau * em1) * idt;
    const double c4r = tau * em1;
    const double c5r = tau * tau * em1 - tau * dt * e;
    t.c4 = c4r * idt;
    t.c5 = -(tau * c4r + c5r) * idt;
    t.c6 = -tau * c4r * idt;
  }
  if (isinf(tau)) {
    // collisionless point value: the initial (half-range) distribution itself
    t.g1 = t.g2 = t.g3 = t.f2 = t.f3 = 0.0;
    t.f1 = 1.0;
    return t;
  }
  const double e = exp(-tp / tau);
  t.g1 = 1.0 - e;
  t.g2 = (tp + tau) * e - tau;
  t.g3 = tp - tau + tau * e;
  t.f1 = e;
  t.f2 = -(tau + tp) * e;
  t.f3 = -tau * e;
  return t;
}

__device__ __forceinline__ double collision_tau(double pl, double pr, double dt, bool viscous, double mu,
                                                const double w0[5]) {
  const double jump = fabs(pl - pr) / (pl + pr) * dt;
  if (viscous) return mu / (w0[0] / (2.0 * w0[4])) + jump;
  return 0.1 * dt + jump;
}

// Interface distribution -> time-averaged flux over [0, dt] (p = 1) and,
// optionally (POINT), the point value at time tp (p = 0).
//   get_side(side, w, s)   : local primitive state and conserved slopes of side 0 (left) / 1 (right)
//   get_pressures(pl, pr)  : both side pressures, needed before the side loop when tau_in < 0
// Returns 0 on success, 1 if an intermediate state is unphysical.
//
// Register plan: the two transport sides run through ONE loop body (not
// unrolled).  When tau is known before the loop (inviscid, or given) the
// six families of flux.py:110-159 are folded per side into one polynomial
// weight, so a side leaves behind only
//   q0  = sum_s rho_s <psi>_s                     (compatibility, flux.py:94)
//   dqa = sum_s rho_s <(a_s,k . psi) psi>_s        (equilibrium slopes, :99)
//   F   = sum_s rho_s <u (c4 + c5 a_s.c + c6 A_s) psi>_s  (transport part of the flux)
// (+ the point-value analogue).  Viscous tau needs W0, so that path keeps
// the three transport families separate until tau is known.
//
// TAU (inviscid, tau_in < 0) chooses where the collision time comes from:
//   0: get_pressures(pl, pr) before the loop (both sides re-evaluated);
//   1 (DEFER): keep the three transport families separate like the viscous
//      path and take both pressures from the loop's own states; tau after
//      the loop;
//   2 (PRE_R): get_pressures(pl, pr) provides the RIGHT pressure only
//      (one side re-evaluated before the loop); the left one comes from
//      side 0's loop state, so tau is known before any transport moment and
//      both sides take the folded single-weight path (10 fewer doubles live
//      across the loop, one Gram pass per side less than DEFER).
// dt: the time window, or a callable returning it (evaluated where it is
// first needed, so its loads need not complete before the side loop).
template <class DT>
__device__ __forceinline__ double dt_value(const DT& d) {
  if constexpr (std::is_arithmetic<DT>::value) return d;
  else return d();
}

// INSTANT: the moment flux of the distribution at the instant tp instead of
// its average over [0, dt] (flux.py:191-197 instantaneous_flux): the flux
// families take the point-value time coefficients
__device__ __forceinline__ TimeCoef instant_coefficients(TimeCoef t) {
  t.c1 = t.g1; t.c2 = t.g2; t.c3 = t.g3;
  t.c4 = t.f1; t.c5 = t.f2; t.c6 = t.f3;
  return t;
}

template <bool VISCOUS, bool POINT, int TAU = 0, bool INSTANT = false, class SideFn, class PressFn, class DT = double>
__device__ __forceinline__ int interface_flux_t(const SideFn& get_side, const PressFn& get_pressures, double tau_in,
                                                const DT& dt_in, double mu, const KinConst& kc, double flux[5], double tp,
                                                double point[5]) {
  double dt = -1.0;  // dt_value(dt_in) once needed
  double q0[5] = {0, 0, 0, 0, 0};
  double dqa[3][5] = {};
  double F[5] = {0, 0, 0, 0, 0};   // folded transport flux (known tau) / base family (viscous)
  double F5[5] = {0, 0, 0, 0, 0};  // viscous only: slope family
  double F6[5] = {0, 0, 0, 0, 0};  // viscous only: time family
  double P[5] = {0, 0, 0, 0, 0};   // point value transport part (known tau) / slope family (viscous)
  double P6[5] = {0, 0, 0, 0, 0};  // viscous only
  double pl = 0.0, pr = 0.0;
  constexpr bool DEFER = TAU == 1;
  constexpr bool PRE_R = TAU == 2 && !VISCOUS;
  TimeCoef tc;
  double tau = tau_in;
  const bool tau_known = (!VISCOUS && !DEFER) || tau_in >= 0.0;
  if (!VISCOUS) {
    if (PRE_R && tau < 0.0) {
      if (!get_pressures(pl, pr)) return 1;
    } else if (!DEFER && tau < 0.0) {
      if (!get_pressures(pl, pr)) return 1;
      dt = dt_value(dt_in);
      tau = collision_tau(pl, pr, dt, false, mu, nullptr);
    }
    if (tau_known && !(PRE_R && tau < 0.0)) {
      dt = dt_value(dt_in);
      tc = time_coefficients(tau, dt, tp);
      if (INSTANT) tc = instant_coefficients(tc);
    }
  }
#if GKS_SIDE_UNROLL
#pragma unroll
#else
#pragma unroll 1
#endif
  for (int side = 0; side < 2; ++side) {
    double w[5], a[3][5];
    double hside = 0.0;  // 1 / (2 lam) when the side callback supplies it
    constexpr bool SIDE_H = std::is_invocable<const SideFn&, int, double*, double (*)[5], double&>::value;
    if constexpr (SIDE_H) {
      if (!get_side(side, w, a, hside)) return 1;
    } else {
      if (!get_side(side, w, a)) return 1;
    }
    if (!prim_ok(w)) return 1;
    const double rho = w[0];
#if !GKS_PS_MUL
    if (VISCOUS || DEFER) {
      const double ps = rho / (2.0 * w[4]);
      pl = side ? pl : ps;
      pr = side ? ps : pr;
    }
#endif
    if (PRE_R && tau < 0.0) {
      // (first pass only: side 0)  the right pressure came from the
      // pre-pass: tau from side 0's state.  A data condition, not side == 0,
      // so the compiler keeps one copy of the loop body
      pl = rho / (2.0 * w[4]);
      dt = dt_value(dt_in);
      tau = collision_tau(pl, pr, dt, false, mu, nullptr);
      tc = time_coefficients(tau, dt, tp);
      if (INSTANT) tc = instant_coefficients(tc);
    }
    double A[5];
    Maxw m;
    if constexpr (SIDE_H) maxw_full_h(m, w, kc, hside);
    else maxw_full(m, w, kc);
#if GKS_PS_MUL
    if (VISCOUS || DEFER) {
      // p = rho / (2 lam) = rho * h with h = 1 / (2 lam) of the moment table
      const double ps = rho * m.h;
      pl = side ? pl : ps;
      pr = side ? ps : pr;
    }
#endif
    const SlopeConst sc = slope_const(w, kc, m.h);
#if GKS_TSLOPE_EULER
    // time slope from the compatibility condition (kinetic.py:305-312): the
    // right-hand side from the conserved slopes before they become micro-slopes
    double D[5];
    euler_axis_jvp(w, m.h, kc, a, D);
#pragma unroll
    for (int i = 0; i < 5; ++i) D[i] = -D[i];
#pragma unroll
    for (int k = 0; k < 3; ++k) micro_slope(sc, a[k], a[k]);  // slopes -> micro-slopes in place
    micro_slope(sc, D, A);
#else
#pragma unroll
    for (int k = 0; k < 3; ++k) micro_slope(sc, a[k], a[k]);  // slopes -> micro-slopes in place
    {
      // time slope from the compatibility condition (kinetic.py:305-312)
      double D[5];
      dir_moment<0, !POINT>(m, a, D);
#pragma unroll
      for (int i = 0; i < 5; ++i) D[i] = -rho * D[i];
      micro_slope(sc, D, A);
    }
#endif
    maxw_half_u(m, w, side ? -1.0 : 1.0);
    double t[5];
    if ((VISCOUS || DEFER) && POINT) {
      const double* const sv[4] = {a[0], a[1], a[2], A};
      double* const av[4] = {dqa[0], dqa[1], dqa[2], P6};
      gram_scatter<0, 4>(m, rho, sv, av, q0);
    } else {
      const double* const sv[3] = {a[0], a[1], a[2]};
      double* const av[3] = {dqa[0], dqa[1], dqa[2]};
      gram_scatter<0, 3>(m, rho, sv, av, q0);
    }
    if (tau_known && !VISCOUS) {
      double sw[5];
#pragma unroll
      for (int i = 0; i < 5; ++i) sw[i] = tc.c6 * A[i];
      sw[0] += tc.c4;
      wmom<1, true>(m, sw, a, tc.c5, t);
#pragma unroll
      for (int i = 0; i < 5; ++i) F[i] += rho * t[i];
      if (POINT) {
#pragma unroll
        for (int i = 0; i < 5; ++i) sw[i] = tc.f3 * A[i];
        wmom<0, true>(m, sw, a, tc.f2, t);
#pragma unroll
        for (int i = 0; i < 5; ++i) P[i] += rho * t[i];
      }
    } else {
      const double zero5[5] = {0, 0, 0, 0, 0};
      {
        // F += rho G_u e_0, F6 += rho G_u A with G_u = <u psi psi^T>, one
        // unique entry at a time (no 25-entry matrix live across the loop body)
        const double* const sv[1] = {A};
        double* const av[1] = {F6};
        gram_scatter<1, 1>(m, rho, sv, av, F);
      }
      dir_moment<1, !POINT>(m, a, t);
#pragma unroll
      for (int i = 0; i < 5; ++i) F5[i] += rho * t[i];
      if (POINT) {
        dir_moment<0, !POINT>(m, a, t);
#pragma unroll
        for (int i = 0; i < 5; ++i) P[i] += rho * t[i];
      }
    }
  }
  double w0[5];
#if GKS_EQ_CLOSED
  // closed-form equilibrium part: no moment table, no micro-slopes at the interface
  double h0, D0[5];
  if (!cons_to_prim_h(q0, kc, w0, h0)) return 1;
  euler_axis_jvp(w0, h0, kc, dqa, D0);
#pragma unroll
  for (int i = 0; i < 5; ++i) D0[i] = -D0[i];
#else
  double ab[3][5], Ab[5];
  Maxw m0;
#if GKS_H_MUL
  {
    double h0;
    if (!cons_to_prim_h(q0, kc, w0, h0)) return 1;
    maxw_full_h(m0, w0, kc, h0);
  }
#else
  if (!cons_to_prim(q0, kc, w0)) return 1;
  maxw_full(m0, w0, kc);
#endif
  const SlopeConst sc0 = slope_const(w0, kc, m0.h);
#pragma unroll
  for (int k = 0; k < 3; ++k) micro_slope(sc0, dqa[k], ab[k]);
  {
    double D[5];
#if GKS_TSLOPE_EULER
    euler_axis_jvp(w0, m0.h, kc, dqa, D);
#pragma unroll
    for (int i = 0; i < 5; ++i) D[i] = -D[i];
#else
    dir_moment<0, !POINT>(m0, ab, D);
#pragma unroll
    for (int i = 0; i < 5; ++i) D[i] = -w0[0] * D[i];
#endif
    micro_slope(sc0, D, Ab);
  }
#endif
  if (VISCOUS || !tau_known) {
    dt = dt_value(dt_in);
    if (tau < 0.0) tau = collision_tau(pl, pr, dt, VISCOUS, mu, w0);
    tc = time_coefficients(tau, dt, tp);
    if (INSTANT) tc = instant_coefficients(tc);
#pragma unroll
    for (int i = 0; i < 5; ++i) {
      F[i] = tc.c4 * F[i] + tc.c5 * F5[i] + tc.c6 * F6[i];
      if (POINT) P[i] = tc.f2 * P[i] + tc.f3 * P6[i];
    }
  }
#if GKS_EQ_CLOSED
  {
    double o[5];
    equilibrium_flux(w0, h0, kc, D0, dqa, tc.c1, tc.c3, tc.c2, o);
#pragma unroll
    for (int i = 0; i < 5; ++i) flux[i] = o[i] + F[i];
  }
  if (POINT) {
    // rho0 <psi (g1 + g3 Ab.psi + g2 sum_k c_k ab_k.psi)>_0 = g1 q0 + g3 D0 - g2 D0
    // (the compatibility condition makes the directional sum -D0)
    const double gd = tc.g3 - tc.g2;
#pragma unroll
    for (int i = 0; i < 5; ++i) point[i] = tc.f1 * q0[i] + P[i] + (tc.g1 * q0[i] + gd * D0[i]);
  }
#else
  {
    double s[5], o[5];
#pragma unroll
    for (int i = 0; i < 5; ++i) s[i] = tc.c3 * Ab[i];
    s[0] += tc.c1;
    wmom<1, true>(m0, s, ab, tc.c2, o);
#pragma unroll
    for (int i = 0; i < 5; ++i) flux[i] = w0[0] * o[i] + F[i];
  }
  if (POINT) {
#pragma unroll
    for (int i = 0; i < 5; ++i) point[i] = tc.f1 * q0[i] + P[i];
    if (tc.g1 != 0.0 || tc.g2 != 0.0 || tc.g3 != 0.0) {
      double s[5], o[5];
#pragma unroll
      for (int i = 0; i < 5; ++i) s[i] = tc.g3 * Ab[i];
      s[0] += tc.g1;
      wmom<0, true>(m0, s, ab, tc.g2, o);
#pragma unroll
      for (int i = 0; i < 5; ++i) point[i] += w0[0] * o[i];
    }
  }
#endif
  return 0;
}

// Convenience form on explicit left/right inputs (inviscid or given tau).
__device__ __forceinline__ int interface_flux(const FluxIn& in, double tau_in, double dt, int model, double mu,
                                              const KinConst& kc, double flux[5], bool want_point, double tp,
                                              double point[5], double* tau_out) {
  auto get = [&](int side, double w[5], double sl[3][5]) {
#pragma unroll
    for (int i = 0; i < 5; ++i) w[i] = side ? in.wr[i] : in.wl[i];
#pragma unroll
    for (int k = 0; k < 3; ++k)
#pragma unroll
      for (int i = 0; i < 5; ++i) sl[k][i] = side ? in.sr[k][i] : in.sl[k][i];
    return true;
  };
  auto press = [&](double& pl, double& pr) {
    pl = in.wl[0] / (2.0 * in.wl[4]);
    pr = in.wr[0] / (2.0 * in.wr[4]);
    return true;
  };
  if (!prim_ok(in.wl) || !prim_ok(in.wr)) return 1;
  (void)tau_out;
  if (model == MODEL_VISCOUS)
    return want_point ? interface_flux_t<true, true>(get, press, tau_in, dt, mu, kc, flux, tp, point)
                      : interface_flux_t<true, false>(get, press, tau_in, dt, mu, kc, flux, tp, point);
  return want_point ? interface_flux_t<false, true>(get, press, tau_in, dt, mu, kc, flux, tp, point)
                    : interface_flux_t<false, false>(get, press, tau_in, dt, mu, kc, flux, tp, point);
}

}  // namespace gks
