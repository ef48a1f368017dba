// Multi-GPU plumbing behind one interface (Comm), two transports:
//
//  * NCCL (loaded with dlopen so the library never pins an NCCL build --
//    inside a torch process it binds to the one torch loaded): grouped
//    ncclSend/ncclRecv halo exchange of cell data, in-place scalar
//    allreduces (error words, min dt) and the group-partial exchange of the
//    partition-invariant reductions (gks_reduce.cuh).  One process per GPU.
//
//  * loopback: R rank-local handles in ONE process (one host thread per rank,
//    all on one device), exchanging through device-to-device copies.  A
//    collective is a host barrier between the rank threads plus CUDA events:
//    each rank records an event after producing its side, every rank's stream
//    waits on its peers' events before consuming.  No kernel ever waits for
//    another (nothing spins), so the ranks may share a GPU.  It runs the same
//    pack / exchange / unpack and reduction code paths as NCCL, which lets a
//    single-GPU test step 2-4 ranks of a partitioned mesh.  Buffers read by
//    peers alternate between two parity halves: a rank can only overwrite a
//    half two collectives later, after every peer's stream has passed the
//    collective in between.
//
// With no communicator every call is a no-op: the single-GPU path.
#include <dlfcn.h>
#include <nccl.h>

#include <chrono>
#include <condition_variable>
#include <mutex>
#include <vector>

#include "gks_implicit.cuh"

namespace gks {

namespace {
struct NcclApi {
  bool ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};
NcclApi g_nccl;
std::mutex g_nccl_mu;

bool nccl_load() {
  std::lock_guard<std::mutex> lk(g_nccl_mu);
  if (g_nccl.ok) return true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return false;
#define LOAD(name) g_nccl.name = reinterpret_cast<decltype(g_nccl.name)>(dlsym(h, "nccl" #name))
  LOAD(GetUniqueId);
  LOAD(CommInitRank);
  LOAD(CommDestroy);
  LOAD(GroupStart);
  LOAD(GroupEnd);
  LOAD(Send);
  LOAD(Recv);
  LOAD(AllReduce);
  LOAD(GetErrorString);
#undef LOAD
  g_nccl.ok = g_nccl.GetUniqueId && g_nccl.CommInitRank && g_nccl.GroupStart && g_nccl.GroupEnd && g_nccl.Send &&
              g_nccl.Recv && g_nccl.AllReduce;
  return g_nccl.ok;
}

int nccl_fail(ncclResult_t r, const char* what) {
  set_error("NCCL error in %s: %s", what, g_nccl.GetErrorString ? g_nccl.GetErrorString(r) : "?");
  return GKS_ERR_NCCL;
}
}  // namespace

#define GKS_NCCL(call)                                       \
  do {                                                       \
    ncclResult_t _r = (call);                                \
    if (_r != ncclSuccess) return nccl_fail(_r, #call);      \
  } while (0)

#define TRY_LB(x)        \
  do {                   \
    int _r = (x);        \
    if (_r) return _r;   \
  } while (0)

constexpr int LB_MAXR = 16;     // loopback ranks (RedSrc capacity)
constexpr int LB_SLOT = 64;     // doubles per rank per scalar collective

struct LoopGroup;

struct Comm {
  int kind = 0;  // 1 NCCL, 2 loopback
  int nranks = 1, rank = 0;
  ncclComm_t nccl = nullptr;
  // loopback
  LoopGroup* grp = nullptr;
  Handle* H = nullptr;
  int64_t seq = 0;  // collectives issued (parity of the peer-visible buffers)
  cudaEvent_t ev[2] = {nullptr, nullptr};
  KrylovWS* ws = nullptr;  // this rank's reduction buffers (set at the first reduction)
  // per halo map (0: q, 1: x) and peer index: offset of this rank's data in
  // the peer's send buffer
  std::vector<int64_t> src_off[2];
};

struct LoopGroup {
  int R = 0;
  std::vector<Comm*> ranks;
  int registered = 0;
  bool ready = false;
  double* slots = nullptr;  // device [2][R][LB_SLOT] scalar staging
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  int64_t generation = 0;
  bool broken = false;
};

namespace {

// Host barrier of the loopback ranks (timeout: a rank that errored out of
// the step would otherwise leave its peers waiting forever).
int lb_barrier(LoopGroup* g) {
  std::unique_lock<std::mutex> lk(g->mu);
  if (g->broken) {
    set_error("loopback group broken (a rank failed or timed out)");
    return GKS_ERR_NCCL;
  }
  const int64_t gen = g->generation;
  if (++g->arrived == g->R) {
    g->arrived = 0;
    g->generation++;
    g->cv.notify_all();
    return GKS_OK;
  }
  if (!g->cv.wait_for(lk, std::chrono::seconds(120), [&] { return g->generation != gen || g->broken; })) {
    g->broken = true;
    g->cv.notify_all();
    set_error("loopback barrier timed out");
    return GKS_ERR_NCCL;
  }
  if (g->broken) {
    set_error("loopback group broken (a rank failed or timed out)");
    return GKS_ERR_NCCL;
  }
  return GKS_OK;
}

// record this rank's event for parity p, meet the peers, wait on theirs
int lb_sync(Comm* c, int p, cudaStream_t s) {
  GKS_CUDA(cudaEventRecord(c->ev[p], s));
  if (int rc = lb_barrier(c->grp)) return rc;
  for (Comm* o : c->grp->ranks)
    if (o != c) GKS_CUDA(cudaStreamWaitEvent(s, o->ev[p], 0));
  return GKS_OK;
}

__global__ void k_lb_scalar(const double* slots, int R, int64_t count, int dtype, int op, void* dev) {
  const int i = threadIdx.x;
  if (i >= count) return;
  if (dtype == 0) {
    double v = slots[i];
    for (int r = 1; r < R; ++r) {
      const double x = slots[r * LB_SLOT + i];
      v = op == 0 ? v + x : (op == 1 ? fmin(v, x) : fmax(v, x));
    }
    ((double*)dev)[i] = v;
  } else {
    const int* si = (const int*)slots;
    int v = si[i];
    for (int r = 1; r < R; ++r) {
      const int x = si[r * 2 * LB_SLOT + i];
      v = op == 0 ? v + x : (op == 1 ? min(v, x) : max(v, x));
    }
    ((int*)dev)[i] = v;
  }
}

}  // namespace

__global__ void k_pack(int64_t n, int width, const int* __restrict__ ids, const double* __restrict__ arr,
                       double* __restrict__ buf) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n * width) return;
  const int64_t k = t / width;
  const int j = (int)(t - k * width);
  buf[t] = arr[(int64_t)ids[k] * width + j];
}

__global__ void k_unpack(int64_t n, int width, const int* __restrict__ ids, const double* __restrict__ buf,
                         double* __restrict__ arr) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n * width) return;
  const int64_t k = t / width;
  const int j = (int)(t - k * width);
  arr[(int64_t)ids[k] * width + j] = buf[t];
}

template <int NS, int NM>
__global__ void k_red_final(RedSrc src, int64_t ngrp_g, RedOut out, const int* gate);

int halo_exchange(Handle* H, HaloMap& X, double* arr, int width, cudaStream_t s) {
  Comm* c = H->comm;
  if (!c) return GKS_OK;
  if (c->kind == 1) {
    if (X.peers.empty()) return GKS_OK;
    if (X.ns) GKS_LAUNCH(KC_VEC, k_pack, blocks_for(X.ns * width, 256), 256, 0, s, X.ns, width, X.sids, arr, H->hsend);
    GKS_NCCL(g_nccl.GroupStart());
    for (size_t p = 0; p < X.peers.size(); ++p) {
      const int64_t sc = X.soff[p + 1] - X.soff[p], rc = X.roff[p + 1] - X.roff[p];
      if (sc) GKS_NCCL(g_nccl.Send(H->hsend + X.soff[p] * width, sc * width, ncclDouble, X.peers[p], c->nccl, s));
      if (rc) GKS_NCCL(g_nccl.Recv(H->hrecv + X.roff[p] * width, rc * width, ncclDouble, X.peers[p], c->nccl, s));
    }
    GKS_NCCL(g_nccl.GroupEnd());
    if (X.nr) GKS_LAUNCH(KC_VEC, k_unpack, blocks_for(X.nr * width, 256), 256, 0, s, X.nr, width, X.rids, H->hrecv, arr);
    return GKS_OK;
  }
  // loopback: every rank takes part in every collective (even with no peers)
  const int p = (int)(c->seq++ & 1);
  const int mi = &X == &H->hq ? 0 : 1;
  double* mine = H->hsend + p * H->hsend_half;
  if (X.ns) GKS_LAUNCH(KC_VEC, k_pack, blocks_for(X.ns * width, 256), 256, 0, s, X.ns, width, X.sids, arr, mine);
  TRY_LB(lb_sync(c, p, s));
  for (size_t k = 0; k < X.peers.size(); ++k) {
    const int64_t rc = X.roff[k + 1] - X.roff[k];
    if (!rc) continue;
    const Comm* o = c->grp->ranks[X.peers[k]];
    const double* src = o->H->hsend + p * o->H->hsend_half + c->src_off[mi][k] * width;
    GKS_CUDA(cudaMemcpyAsync(H->hrecv + X.roff[k] * width, src, rc * width * sizeof(double),
                             cudaMemcpyDeviceToDevice, s));
  }
  if (X.nr) GKS_LAUNCH(KC_VEC, k_unpack, blocks_for(X.nr * width, 256), 256, 0, s, X.nr, width, X.rids, H->hrecv, arr);
  return GKS_OK;
}

int allreduce(Handle* H, void* dev, int64_t count, int dtype, int op, cudaStream_t s) {
  Comm* c = H->comm;
  if (!c) return GKS_OK;
  if (c->kind == 1) {
    const ncclDataType_t t = dtype == 0 ? ncclDouble : ncclInt32;
    const ncclRedOp_t o = op == 0 ? ncclSum : (op == 1 ? ncclMin : ncclMax);
    GKS_NCCL(g_nccl.AllReduce(dev, dev, count, t, o, c->nccl, s));
    return GKS_OK;
  }
  if (count > LB_SLOT) {
    set_error("loopback allreduce of %lld values exceeds the staging slot", (long long)count);
    return GKS_ERR_BAD_ARG;
  }
  LoopGroup* g = c->grp;
  const int p = (int)(c->seq++ & 1);
  double* base = g->slots + (size_t)p * g->R * LB_SLOT;
  GKS_CUDA(cudaMemcpyAsync(base + (size_t)c->rank * LB_SLOT, dev, count * (dtype == 0 ? 8 : 4),
                           cudaMemcpyDeviceToDevice, s));
  TRY_LB(lb_sync(c, p, s));
  GKS_LAUNCH(KC_SCALAR, k_lb_scalar, 1, LB_SLOT, 0, s, base, g->R, count, dtype, op, dev);
  return GKS_OK;
}

double* comm_red_buffer(Comm* c, KrylovWS* W) {
  if (c->kind == 1) return W->gpart[0];
  c->ws = W;
  return W->gpart[c->seq & 1];
}

int comm_red_final(Comm* c, KrylovWS* W, int ns, int nm, const RedOut& out, const int* gate, cudaStream_t s) {
  const int64_t ng = W->red.ngrp_g;
  RedSrc src{};
  if (c->kind == 1) {
    // exact: every group partial is non-zero (non-inf) on its owner only
    if (ns) GKS_NCCL(g_nccl.AllReduce(W->gpart[0], W->gall, ns * ng, ncclDouble, ncclSum, c->nccl, s));
    if (nm)
      GKS_NCCL(g_nccl.AllReduce(W->gpart[0] + RED_MIN_SLOT * ng, W->gall + RED_MIN_SLOT * ng, nm * ng, ncclDouble,
                                ncclMin, c->nccl, s));
    src.p[0] = W->gall;
    src.n = 1;
  } else {
    const int p = (int)(c->seq++ & 1);
    c->ws = W;
    TRY_LB(lb_sync(c, p, s));
    src.n = c->grp->R;
    for (int r = 0; r < src.n; ++r) src.p[r] = c->grp->ranks[r]->ws->gpart[p];
  }
  if (ns == 1 && nm == 0) GKS_LAUNCH(KC_REDUCE, (k_red_final<1, 0>), 1, RED_T, 0, s, src, ng, out, gate);
  else if (ns == 2 && nm == 0) GKS_LAUNCH(KC_REDUCE, (k_red_final<2, 0>), 1, RED_T, 0, s, src, ng, out, gate);
  else if (ns == 3 && nm == 1) GKS_LAUNCH(KC_REDUCE, (k_red_final<3, 1>), 1, RED_T, 0, s, src, ng, out, gate);
  else {
    set_error("no final reduction kernel for %d sums + %d mins", ns, nm);
    return GKS_ERR_BAD_ARG;
  }
  return GKS_OK;
}

__global__ void k_red_final_n(RedSrc src, int64_t ngrp_g, int nc, RedOutN out, const int* gate);

int comm_red_final_n(Comm* c, KrylovWS* W, int nc, const RedOutN& out, const int* gate, cudaStream_t s) {
  const int64_t ng = W->red.ngrp_g;
  RedSrc src{};
  if (c->kind == 1) {
    GKS_NCCL(g_nccl.AllReduce(W->gpart[0], W->gall, nc * ng, ncclDouble, ncclSum, c->nccl, s));
    src.p[0] = W->gall;
    src.n = 1;
  } else {
    const int p = (int)(c->seq++ & 1);
    c->ws = W;
    TRY_LB(lb_sync(c, p, s));
    src.n = c->grp->R;
    for (int r = 0; r < src.n; ++r) src.p[r] = c->grp->ranks[r]->ws->gpart[p];
  }
  GKS_LAUNCH(KC_REDUCE, k_red_final_n, 1, RED_T, 0, s, src, ng, nc, out, gate);
  return GKS_OK;
}

int comm_init(Handle* H, const void* uid, int nranks, int rank) {
  if (!nccl_load()) {
    set_error("libnccl.so.2 could not be loaded");
    return GKS_ERR_NCCL;
  }
  ncclUniqueId id;
  memcpy(&id, uid, sizeof(id));
  ncclComm_t nc;
  GKS_CUDA(cudaSetDevice(H->device));
  GKS_NCCL(g_nccl.CommInitRank(&nc, nranks, id, rank));
  Comm* c = new Comm();
  c->kind = 1;
  c->nccl = nc;
  c->nranks = nranks;
  c->rank = rank;
  H->comm = c;
  H->nranks = nranks;
  H->rank = rank;
  return GKS_OK;
}

void comm_destroy(Handle* H) {
  Comm* c = H->comm;
  if (!c) return;
  if (c->kind == 1 && c->nccl && g_nccl.CommDestroy) g_nccl.CommDestroy(c->nccl);
  if (c->kind == 2) {
    for (int k = 0; k < 2; ++k)
      if (c->ev[k]) cudaEventDestroy(c->ev[k]);
    if (c->grp) {
      std::lock_guard<std::mutex> lk(c->grp->mu);
      c->grp->ranks[c->rank] = nullptr;
      c->grp->ready = false;
    }
  }
  delete c;
  H->comm = nullptr;
}

// Loopback: register rank `rank` of group g; the last registration checks
// that every halo map pairs up and computes each receiver's source offsets.
int comm_init_loopback(Handle* H, LoopGroup* g, int rank) {
  if (rank < 0 || rank >= g->R) {
    set_error("loopback rank %d out of range [0, %d)", rank, g->R);
    return GKS_ERR_BAD_ARG;
  }
  std::lock_guard<std::mutex> lk(g->mu);
  if (g->ranks[rank]) {
    set_error("loopback rank %d registered twice", rank);
    return GKS_ERR_BAD_ARG;
  }
  Comm* c = new Comm();
  c->kind = 2;
  c->grp = g;
  c->H = H;
  c->nranks = g->R;
  c->rank = rank;
  GKS_CUDA(cudaSetDevice(H->device));
  for (int k = 0; k < 2; ++k) GKS_CUDA(cudaEventCreateWithFlags(&c->ev[k], cudaEventDisableTiming));
  g->ranks[rank] = c;
  H->comm = c;
  H->nranks = g->R;
  H->rank = rank;
  if (++g->registered < g->R) return GKS_OK;
  // all ranks present: pair the maps
  for (Comm* r : g->ranks) {
    for (int mi = 0; mi < 2; ++mi) {
      const HaloMap& X = mi == 0 ? r->H->hq : r->H->hx;
      r->src_off[mi].assign(X.peers.size(), 0);
      for (size_t k = 0; k < X.peers.size(); ++k) {
        const int pr = X.peers[k];
        if (pr < 0 || pr >= g->R || pr == r->rank) {
          set_error("loopback: bad peer %d of rank %d", pr, r->rank);
          return GKS_ERR_BAD_ARG;
        }
        const HaloMap& Y = mi == 0 ? g->ranks[pr]->H->hq : g->ranks[pr]->H->hx;
        size_t j = 0;
        while (j < Y.peers.size() && Y.peers[j] != r->rank) ++j;
        const int64_t want = X.roff[k + 1] - X.roff[k];
        const int64_t have = j < Y.peers.size() ? Y.soff[j + 1] - Y.soff[j] : 0;
        if (want != have) {
          set_error("loopback: rank %d expects %lld cells from rank %d, which sends %lld", r->rank, (long long)want,
                    pr, (long long)have);
          return GKS_ERR_BAD_ARG;
        }
        r->src_off[mi][k] = j < Y.peers.size() ? Y.soff[j] : 0;
      }
    }
  }
  GKS_CUDA(cudaMalloc(&g->slots, (size_t)2 * g->R * LB_SLOT * sizeof(double)));
  g->ready = true;
  return GKS_OK;
}

}  // namespace gks

using namespace gks;

struct GksLoopback {
  LoopGroup g;
};

namespace gks {
LoopGroup* loopback_group(GksLoopback* lb) { return lb ? &lb->g : nullptr; }
}  // namespace gks

extern "C" {

int gks_comm_unique_id(void* out, int64_t nbytes) {
  if (nbytes < (int64_t)sizeof(ncclUniqueId)) {
    set_error("unique id buffer needs %d bytes", (int)sizeof(ncclUniqueId));
    return GKS_ERR_BAD_ARG;
  }
  if (!nccl_load()) {
    set_error("libnccl.so.2 could not be loaded");
    return GKS_ERR_NCCL;
  }
  ncclUniqueId id;
  GKS_NCCL(g_nccl.GetUniqueId(&id));
  memcpy(out, &id, sizeof(id));
  return GKS_OK;
}

int gks_loopback_create(int nranks, GksLoopback** out) {
  if (nranks < 1 || nranks > LB_MAXR || !out) {
    set_error("loopback group size must be in [1, %d]", LB_MAXR);
    return GKS_ERR_BAD_ARG;
  }
  GksLoopback* lb = new GksLoopback();
  lb->g.R = nranks;
  lb->g.ranks.assign(nranks, nullptr);
  *out = lb;
  return GKS_OK;
}

void gks_loopback_destroy(GksLoopback* lb) {
  if (!lb) return;
  if (lb->g.slots) cudaFree(lb->g.slots);
  delete lb;
}

}  // extern "C"
