// Multi-GPU plumbing: NCCL (loaded with dlopen so the library never pins an
// NCCL build -- inside a torch process it binds to the one torch loaded),
// halo exchange of cell data over grouped ncclSend/ncclRecv, and in-place
// device allreduces used by the GMRES reductions, the step norms and the
// status word.  With no communicator every call is a no-op, which is the
// single-GPU path.
#include <dlfcn.h>
#include <nccl.h>

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

int halo_exchange(Handle* H, HaloMap& X, double* arr, int width, cudaStream_t s) {
  if (!H->comm || X.peers.empty()) return GKS_OK;
  if (X.ns) GKS_LAUNCH(KC_VEC, k_pack, blocks_for(X.ns * width, 256), 256, 0, s, X.ns, width, X.sids, arr, H->hsend);
  GKS_NCCL(g_nccl.GroupStart());
  for (size_t p = 0; p < X.peers.size(); ++p) {
    const int64_t sc = X.soff[p + 1] - X.soff[p], rc = X.roff[p + 1] - X.roff[p];
    if (sc)
      GKS_NCCL(g_nccl.Send(H->hsend + X.soff[p] * width, sc * width, ncclDouble, X.peers[p], (ncclComm_t)H->comm, s));
    if (rc)
      GKS_NCCL(g_nccl.Recv(H->hrecv + X.roff[p] * width, rc * width, ncclDouble, X.peers[p], (ncclComm_t)H->comm, s));
  }
  GKS_NCCL(g_nccl.GroupEnd());
  if (X.nr) GKS_LAUNCH(KC_VEC, k_unpack, blocks_for(X.nr * width, 256), 256, 0, s, X.nr, width, X.rids, H->hrecv, arr);
  return GKS_OK;
}

int allreduce(Handle* H, void* dev, int64_t count, int dtype, int op, cudaStream_t s) {
  if (!H->comm) return GKS_OK;
  const ncclDataType_t t = dtype == 0 ? ncclDouble : ncclInt32;
  const ncclRedOp_t o = op == 0 ? ncclSum : (op == 1 ? ncclMin : ncclMax);
  GKS_NCCL(g_nccl.AllReduce(dev, dev, count, t, o, (ncclComm_t)H->comm, s));
  return GKS_OK;
}

int comm_init(Handle* H, const void* uid, int nranks, int rank) {
  if (!nccl_load()) {
    set_error("libnccl.so.2 could not be loaded");
    return GKS_ERR_NCCL;
  }
  ncclUniqueId id;
  memcpy(&id, uid, sizeof(id));
  ncclComm_t c;
  GKS_CUDA(cudaSetDevice(H->device));
  GKS_NCCL(g_nccl.CommInitRank(&c, nranks, id, rank));
  H->comm = c;
  H->nranks = nranks;
  H->rank = rank;
  return GKS_OK;
}

void comm_destroy(Handle* H) {
  if (H->comm && g_nccl.CommDestroy) g_nccl.CommDestroy((ncclComm_t)H->comm);
  H->comm = nullptr;
}

}  // namespace gks

using namespace gks;

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

}  // extern "C"
