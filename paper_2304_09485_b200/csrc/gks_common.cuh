// Shared host/device plumbing for libgks: status codes, error text, CUDA
// checks, a device-side error word that kernels raise without host syncs.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string>

#include "../../include/gks.h"

// Minimum resident CTAs per SM (register budgets), chosen by measurement:
// the 128-thread face kernel runs best at 255 regs/thread (2 CTAs, 8
// warps/SM, nearly spill-free) since round 2 removed three FP64 divisions
// per point -- C2 2.570 -> 2.558 ms, C3 (viscous + point value) 3.202 ->
// 3.009 ms; it was 168 regs / 3 CTAs before (profiles/r01); 4 CTAs / 128
// regs: 2.93 ms.  The closed-form time slopes and equilibrium terms shrank
// the live state enough that 168 regs / 3 CTAs (12 warps/SM) spill only
// 80 B/thread: C2 face 2.203 -> 1.867 ms, C1 2.55 -> 2.06, C3 2.68 -> 2.58,
// C5 19.1 -> 18.0 ms (4 CTAs / 128 regs: 2.18 ms; 160 threads x 3: 2.28 ms;
// the side loop rolled at 3 CTAs: 2.00 ms).  The 160-thread reconstruction
// kernels run at 96 (4 CTAs).
#ifndef GKS_FACE_MINB
#define GKS_FACE_MINB 3
#endif
#ifndef GKS_FLUX_MINB
#define GKS_FLUX_MINB 3
#endif
#ifndef GKS_RECON_MINB
#define GKS_RECON_MINB 4
#endif

#include <nvtx3/nvToolsExt.h>

namespace gks {

// NVTX range over a host API call (header-only NVTX3: a no-op unless a
// profiler such as nsys / ncu --nvtx injects itself)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
#define GKS_NVTX_CAT2(a, b) a##b
#define GKS_NVTX_CAT(a, b) GKS_NVTX_CAT2(a, b)
#define GKS_NVTX(name) ::gks::NvtxRange GKS_NVTX_CAT(gks_nvtx_, __LINE__)(name)

void set_error(const char* fmt, ...);
int cuda_fail(cudaError_t e, const char* what, const char* file, int line);

#define GKS_CUDA(call)                                                  \
  do {                                                                  \
    cudaError_t _e = (call);                                            \
    if (_e != cudaSuccess) return ::gks::cuda_fail(_e, #call, __FILE__, __LINE__); \
  } while (0)

// Device error word layout: status[0] = first error code (atomicCAS from 0),
// status[1] = smallest offending index (atomicMin), status[2..] = aux.
struct DevStatus {
  int* word;  // device pointer, 4 ints
};

__device__ __forceinline__ void raise_dev(int* status, int code, int index) {
  atomicCAS(status, 0, code);
  atomicMin(status + 1, index);
}

inline int blocks_for(int64_t n, int threads) { return (int)((n + threads - 1) / threads); }

// --- launch accounting and the optional per-kernel-class profiler ----------
// Kernel classes reported by gks_profile_read (names in gks_flux.cu).
enum KClass : int {
  KC_DT = 0, KC_RECON, KC_FACE, KC_ASSEMBLE, KC_GHOST, KC_JAC_FACE, KC_JAC_DIAG, KC_SPMV, KC_JACOBI,
  KC_REDUCE, KC_VEC, KC_SCALAR, KC_UPDATE, KC_FLUXBATCH, KC_COUNT
};
void count_launch(int n);
extern bool g_prof_on;
cudaEvent_t prof_begin(cudaStream_t s);
void prof_end(int cls, cudaStream_t s, cudaEvent_t start);
void prof_harvest();

#define GKS_LAUNCH(cls, kern, grid, block, smem, stream, ...)              \
  do {                                                                     \
    cudaEvent_t _pa = ::gks::g_prof_on ? ::gks::prof_begin(stream) : nullptr; \
    kern<<<(grid), (block), (smem), (stream)>>>(__VA_ARGS__);              \
    ::gks::count_launch(1);                                                \
    if (_pa) ::gks::prof_end((cls), (stream), _pa);                        \
  } while (0)

}  // namespace gks
