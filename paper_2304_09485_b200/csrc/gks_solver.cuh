// Device-resident solver state (one handle per GPU) and the device helpers
// shared by the residual and implicit kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "gks_common.cuh"
#include "gks_kinetic.cuh"
#include "gks_reduce.cuh"

namespace gks {

enum PatchKind : int {
  PK_NONE = -1,
  PK_WALL_NOSLIP_ISOTHERMAL = 0,
  PK_WALL_NOSLIP_ADIABATIC = 1,
  PK_WALL_SLIP_ADIABATIC = 2,
  PK_FARFIELD_RIEMANN = 3,
  PK_SUPERSONIC_INLET = 4,
  PK_SUPERSONIC_OUTLET = 5,
};

struct DevPatch {
  int kind;
  int wall;           // kind in WALL_KINDS (boundary.py:18)
  int wall_moving;    // any(velocity != 0)
  double ref[5];      // reference primitive (rho, U, V, W, lam)
  double lambda_wall;
  double vel[3];
};

// Scalars shared between kernels without host round trips.
struct DevScalars {
  double red[8];        // reduction results (norms, dots)
  double stat[4];       // sum|res_rho|, sum res^2, #bad cells, min dt (allreduced)
  double sigma;
};

// Halo exchange map: per peer, local ids sent (owned cells) / received (ghosts)
struct HaloMap {
  std::vector<int> peers;
  std::vector<int64_t> soff{0}, roff{0};
  int* sids = nullptr;  // device
  int* rids = nullptr;  // device
  int64_t ns = 0, nr = 0;
};

template <class T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
};

struct Handle {
  int device = 0;
  cudaStream_t stream = nullptr;
  // sizes
  int64_t nc = 0, nf = 0, nfq = 0, nfi = 0, nbf = 0, nnz = 0;
  // domain decomposition: local cells = [owned | layer-1 ghosts | deeper ghosts]
  int64_t n_owned = 0, n_recon = 0, nc_global = 0;
  HaloMap hq, hx;                    // Q(+grad) halo (all layers), x/dt halo (layer 1)
  double *hsend = nullptr, *hrecv = nullptr;
  int64_t hsend_half = 0;            // hsend holds two buffers of this many doubles
  Comm* comm = nullptr;              // NCCL or in-process loopback transport (gks_comm.cu)
  int nranks = 1, rank = 0;
  int64_t cell_first = 0;            // canonical index of the first owned cell (reductions)
  int nfpc = 4;
  // options
  int scheme = 0, model = 0, compact = 0, linear_weights = 0, global_dt = 0, jac_mode = 0;
  int first_order = 0;  // KFVS on piecewise-constant states (no reconstruction, tau = inf)
  int ortho = 0;        // GMRES orthogonalisation: 0 MGS, 1 CGS2
  double mu = 0, gamma = 1.4, cfl = 2, eps = 1e-6, lw = 0.025;
  KinConst kc;
  int krylov_dim = 10, restarts = 3, jacobi_sweeps = 2;
  double gmres_rtol = 0;
  std::vector<DevPatch> patches_h;
  std::vector<std::string> patch_names;
  DevPatch* patches = nullptr;
  int npatch = 0;
  // cell geometry
  double *vol = nullptr, *h = nullptr, *cen = nullptr, *avg0 = nullptr;
  double* ih = nullptr;  // 1 / h per cell (face-point evaluation)
  // faces
  int *f_own = nullptr, *f_nbr = nullptr, *f_patch = nullptr;
  double *f_area = nullptr, *f_normal = nullptr, *f_frame = nullptr, *f_shift = nullptr;
  // fq points
  int* fq_face = nullptr;
  int fq_nq = 0;  // > 0: fq_face[i] == i / fq_nq (uniform points per face)
  double *fq_point = nullptr, *fq_ws = nullptr;
  // cell -> fq CSR (assembly order), entries fq<<1 | is_neighbor
  int *cfq_start = nullptr, *cfq = nullptr;
  int asm_tile = 0;  // every 32-cell tile's list segment fits k_assemble_tile's staging
  // slot assembly: per fq point the CSR positions of its owner / neighbour
  // entries (int2, -1 = none or not an owned cell); the face kernel writes
  // its signed contribution into both, the assembly is a contiguous
  // segmented sum (same order and signs as the CSR walk: bitwise equal)
  int2* fq_slot = nullptr;
  double* slots = nullptr;  // (nent, 5)
  int64_t nent = 0;
  // cell -> face CSR for local dt (owner faces then neighbour faces), face<<1 | is_neighbor
  int *cdt_start = nullptr, *cdt = nullptr;
  // cell -> face CSR for the Jacobian diagonal, face<<1 | is_neighbor (interior own, interior nbr, boundary own)
  int *cjd_start = nullptr, *cjd = nullptr;
  // Jacobian off-diagonal CSR (row-sorted), per interior face the two CSR slots
  int* face_slot = nullptr;  // (2*nf) CSR slot of (face, side) off block, -1 for boundary faces
  int* bidx = nullptr;       // (nf) index into boundary_faces, -1 for interior faces
  int* interior_faces = nullptr;  // list of interior face ids (nfi)
  int* boundary_faces = nullptr;  // list of boundary face ids (nbf)
  // reconstruction operators
  int K = 0, M = 0, S = 0;          // WENO widths
  int HA = 0, HG = 0, HM = 0;       // HWENO widths
  int Kt = 0, Mt = 0, St = 0;       // padded record shape of the K2 kernel (K,M,S) / (HA,HG,M)
  double *big_op = nullptr, *sub_op = nullptr, *beta = nullptr, *grad_scale = nullptr;
  int *big_gather = nullptr, *sub_gather = nullptr, *avg_gather = nullptr, *grad_gather = nullptr;
  int8_t* sub_active = nullptr;
  // state and work
  double *q = nullptr, *grad = nullptr, *dt = nullptr, *coef = nullptr;
  double *contrib = nullptr, *qpt = nullptr, *res = nullptr, *grad_new = nullptr;
  double *ghosts = nullptr;
  double *diag = nullptr, *dinv = nullptr, *off = nullptr;
  double *q_new = nullptr, *dq = nullptr, *qtmp = nullptr, *res2 = nullptr;
  // Krylov work
  double *V = nullptr, *w = nullptr, *r = nullptr, *t1 = nullptr, *t2 = nullptr, *x = nullptr;
  double* partial = nullptr;     // reduction partials
  unsigned int* counter = nullptr;
  void* gm = nullptr;            // GmresDev state (device)
  DevScalars* scal = nullptr;
  int* status = nullptr;         // device error word (4 ints)
  int8_t* bad = nullptr;
  int red_blocks = 0;
  // timing / evidence
  int64_t launches = 0;
  cudaEvent_t ev[8];
  int ev_ready = 0;
  std::vector<void*> allocs;
};

// ---------------------------------------------------------------------------
// boundary ghost states (boundary.py:66-171), primitive in / conserved out
// ---------------------------------------------------------------------------

__device__ __forceinline__ double half_mass_flux(double un, double lam, double sign) {
  const double g = 0.5 * exp(-lam * un * un) / sqrt(M_PI * lam);
  if (sign > 0) return un * 0.5 * erfc(-sqrt(lam) * un) + g;
  return -(un * 0.5 * erfc(sqrt(lam) * un) - g);
}

// Returns false if the interior state is unphysical.
__device__ __forceinline__ bool ghost_state(const double qi[5], const DevPatch& P, const double n[3],
                                            const KinConst& kc, double qg[5]) {
  double w[5];
  if (!cons_to_prim(qi, kc, w)) return false;
  double o[5] = {w[0], w[1], w[2], w[3], w[4]};
  const double gam = kc.gamma;
  switch (P.kind) {
    case PK_WALL_SLIP_ADIABATIC: {
      const double un = w[1] * n[0] + w[2] * n[1] + w[3] * n[2];
      o[1] = w[1] - 2.0 * un * n[0];
      o[2] = w[2] - 2.0 * un * n[1];
      o[3] = w[3] - 2.0 * un * n[2];
    } break;
    case PK_WALL_NOSLIP_ADIABATIC:
      o[1] = 2.0 * P.vel[0] - w[1];
      o[2] = 2.0 * P.vel[1] - w[2];
      o[3] = 2.0 * P.vel[2] - w[3];
      break;
    case PK_WALL_NOSLIP_ISOTHERMAL: {
      o[1] = 2.0 * P.vel[0] - w[1];
      o[2] = 2.0 * P.vel[1] - w[2];
      o[3] = 2.0 * P.vel[2] - w[3];
      o[4] = P.lambda_wall;
      const double un = w[1] * n[0] + w[2] * n[1] + w[3] * n[2];
      const double ung = o[1] * n[0] + o[2] * n[1] + o[3] * n[2];
      o[0] = w[0] * half_mass_flux(un, w[4], 1.0) / half_mass_flux(ung, P.lambda_wall, -1.0);
    } break;
    case PK_SUPERSONIC_INLET:
      for (int i = 0; i < 5; ++i) o[i] = P.ref[i];
      break;
    case PK_SUPERSONIC_OUTLET:
      break;
    case PK_FARFIELD_RIEMANN: {
      const double rho = w[0], lam = w[4];
      const double p = rho / (2.0 * lam);
      const double a = sqrt(gam * p / rho);
      const double un = w[1] * n[0] + w[2] * n[1] + w[3] * n[2];
      const double rinf = P.ref[0], laminf = P.ref[4];
      const double pinf = rinf / (2.0 * laminf);
      const double ainf = sqrt(gam * pinf / rinf);
      const double uninf = P.ref[1] * n[0] + P.ref[2] * n[1] + P.ref[3] * n[2];
      const double g1 = gam - 1.0;
      const double rp = un + 2.0 * a / g1;
      const double rm = uninf - 2.0 * ainf / g1;
      const double unb = 0.5 * (rp + rm);
      const double ab = 0.25 * g1 * (rp - rm);
      const bool outflow = unb > 0.0;
      const double s = outflow ? p / pow(rho, gam) : pinf / pow(rinf, gam);
      double ut[3];
      for (int i = 0; i < 3; ++i)
        ut[i] = outflow ? w[1 + i] - un * n[i] : P.ref[1 + i] - uninf * n[i];
      const double rhob = pow(ab * ab / (gam * s), 1.0 / g1);
      const double pb = rhob * ab * ab / gam;
      const double mach = un / a;
      const bool sup_out = mach >= 1.0, sup_in = mach <= -1.0;
      if (sup_out) {
        // interior state unchanged
      } else if (sup_in) {
        for (int i = 0; i < 5; ++i) o[i] = P.ref[i];
      } else {
        o[0] = rhob;
        for (int i = 0; i < 3; ++i) o[1 + i] = ut[i] + unb * n[i];
        o[4] = rhob / (2.0 * pb);
      }
    } break;
    default:
      break;
  }
  prim_to_cons(o, kc, qg);
  return true;
}

// ghost_gradients (boundary.py:144-171); g[x][k]
__device__ __forceinline__ void ghost_gradients(const double g[3][5], const DevPatch& P, const double n[3],
                                                double out[3][5]) {
  if (!P.wall) {
    for (int x = 0; x < 3; ++x)
      for (int k = 0; k < 5; ++k) out[x][k] = g[x][k];
    return;
  }
  double gn[5];
  for (int k = 0; k < 5; ++k) gn[k] = g[0][k] * n[0] + g[1][k] * n[1] + g[2][k] * n[2];
  double mir[3][5];
  for (int x = 0; x < 3; ++x)
    for (int k = 0; k < 5; ++k) mir[x][k] = g[x][k] - 2.0 * n[x] * gn[k];
  for (int x = 0; x < 3; ++x) {
    out[x][0] = mir[x][0];
    out[x][4] = mir[x][4];
  }
  if (P.kind == PK_WALL_SLIP_ADIABATIC) {
    for (int x = 0; x < 3; ++x) {
      const double mn = mir[x][1] * n[0] + mir[x][2] * n[1] + mir[x][3] * n[2];
      for (int c = 0; c < 3; ++c) out[x][1 + c] = mir[x][1 + c] - 2.0 * mn * n[c];
    }
  } else {
    for (int x = 0; x < 3; ++x)
      for (int c = 0; c < 3; ++c) {
        out[x][1 + c] = -mir[x][1 + c];
        if (P.wall_moving) out[x][1 + c] += 2.0 * mir[x][0] * P.vel[c];
      }
  }
}

// ---------------------------------------------------------------------------
// Euler flux Jacobian / spectral radius (jacobian.py:37-71)
// ---------------------------------------------------------------------------

__device__ __forceinline__ void euler_jacobian(const double q[5], const double n[3], double gam,
                                               double J[5][5]) {
  const double g1 = gam - 1.0;
  const double rho = q[0];
  const double v[3] = {q[1] / rho, q[2] / rho, q[3] / rho};
  const double un = v[0] * n[0] + v[1] * n[1] + v[2] * n[2];
  const double ke = 0.5 * (v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
  const double p = g1 * (q[4] - rho * ke);
  const double ht = (q[4] + p) / rho;
  J[0][0] = 0.0;
  J[0][1] = n[0]; J[0][2] = n[1]; J[0][3] = n[2];
  J[0][4] = 0.0;
  for (int i = 0; i < 3; ++i) {
    J[1 + i][0] = g1 * ke * n[i] - v[i] * un;
    for (int j = 0; j < 3; ++j) J[1 + i][1 + j] = v[i] * n[j] - g1 * v[j] * n[i];
    J[1 + i][1 + i] += un;
    J[1 + i][4] = g1 * n[i];
  }
  J[4][0] = (g1 * ke - ht) * un;
  for (int j = 0; j < 3; ++j) J[4][1 + j] = ht * n[j] - g1 * v[j] * un;
  J[4][4] = gam * un;
}

__device__ __forceinline__ double spectral_radius(const double q[5], const double n[3], double gam) {
  const double rho = q[0];
  const double v[3] = {q[1] / rho, q[2] / rho, q[3] / rho};
  const double p = (gam - 1.0) * (q[4] - 0.5 * rho * (v[0] * v[0] + v[1] * v[1] + v[2] * v[2]));
  return fabs(v[0] * n[0] + v[1] * n[1] + v[2] * n[2]) + sqrt(gam * p / rho);
}

// host-side entry points shared across translation units
// Frechet epilogue of the assembly (stepping.py:298-313): instead of the
// residual r1 write out = (r1 - r0)/s (mode 0) or V/dt v - (r1 - r0)/s (mode 1)
struct FrechetEpi {
  const double* r0 = nullptr;
  const double* sigma = nullptr;
  const double* v = nullptr;
  const double* dt = nullptr;
  int mode = 0;
  double* out = nullptr;
};
int residual_device(Handle* H, const double* q, double* res, bool with_gradients, const int* gate,
                    const FrechetEpi* fe = nullptr);
void reset_status(Handle* H);
int halo_exchange(Handle* H, HaloMap& X, double* arr, int width, cudaStream_t s);
int allreduce(Handle* H, void* dev, int64_t count, int dtype, int op, cudaStream_t s);  // dtype 0 f64 1 i32; op 0 sum 1 min 2 max
int comm_init(Handle* H, const void* uid, int nranks, int rank);
struct LoopGroup;
LoopGroup* loopback_group(GksLoopback* lb);
int comm_init_loopback(Handle* H, LoopGroup* g, int rank);
void comm_destroy(Handle* H);
// reductions: the group-partial buffer for the next reduction, and the
// exchange + final fold after it (gks_reduce.cuh; ns sums then nm mins)
struct KrylovWS;
double* comm_red_buffer(Comm* c, KrylovWS* W);
int comm_red_final(Comm* c, KrylovWS* W, int ns, int nm, const RedOut& out, const int* gate, cudaStream_t s);
int comm_red_final_n(Comm* c, KrylovWS* W, int nc, const RedOutN& out, const int* gate, cudaStream_t s);
int local_dt_device(Handle* H);
int boundary_ghosts_device(Handle* H, const double* q);
int gauss_gradients_device(Handle* H, const double* qpt, double* grad_out);
int ghost_batch_device(int64_t n, const DevPatch& P, const double* q, const double* nrm, const double* grad,
                       const KinConst& kc, double* q_out, double* grad_out);
int jacobian_device(Handle* H, const double* q, bool ghosts_given);
int assemble_tile_fits(const int* cfq_start_host, int64_t n_owned);
// reconstruction pieces of the host API (gks_solver.cu)
int recon_coeffs_device(Handle* H, const double* q, int linear);  // -> H->coef
int recon_candidates_device(Handle* H, const double* q, int Mout, double* cbig, double* bsub);
int combine_batch_device(int64_t n, int nk, int M, const double* cbig, const double* bsub, const int8_t* act,
                         const double* beta, double eps, double lw, double* out, double* w0n, double* wmn,
                         cudaStream_t s);
int face_values_device(Handle* H, const double* q, const double* coef, double* vo, double* go, double* vn,
                       double* gn);
void count_launch(int n);
void set_error_index(int64_t i);
int check_status(Handle* H, const char* what);
// message + code for a host copy of a device error word (0: no error)
int status_report(Handle* H, const char* what, const int* st);

}  // namespace gks
