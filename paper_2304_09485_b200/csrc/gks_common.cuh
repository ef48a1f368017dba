// Shared host/device plumbing for libgks: status codes, error text, CUDA
// checks, a device-side error word that kernels raise without host syncs.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string>

#include "../../include/gks.h"

namespace gks {

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

}  // namespace gks
