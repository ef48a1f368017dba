// Per-tile staging of per-cell operator records into shared memory with the
// Blackwell bulk-copy engine (cp.async.bulk global -> shared, completion on
// an mbarrier; no registers, no per-thread address math).
//
// Why: the reconstruction kernels run one thread per (cell, component), so
// the five threads of a cell read the same operator entries.  Read straight
// from global memory every warp-wide load touches ~7 cells' records (7 L1
// wavefronts per instruction; ncu r01: L1 wavefronts 71 % of peak, DRAM
// 28 %).  Staged, the same loads are shared-memory broadcasts with one
// wavefront each, and HBM sees one coalesced stream per operator array.
// (A tile-transposed HBM layout read through L1 instead was measured 3.5x
// slower: every entry then starts a new cache line, so each load waits on
// DRAM; the bulk copy keeps the whole record stream in flight.)
//
// Record strides in shared memory are chosen so the ~7 distinct cells a warp
// touches fall into distinct banks: a stride of s doubles is conflict-free
// when s is odd or s = 2 (mod 4).  Records whose natural stride is not get
// copied cell by cell into a padded stride (needs 16-byte aligned records).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace gks {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  }
}

// bytes must be a multiple of 16, dst/src 16-byte aligned
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__host__ __device__ constexpr uint32_t round16(uint32_t b) { return (b + 15u) & ~15u; }

// Shared-memory stride (bytes) for a record of `bytes` bytes: natural when
// conflict-free (odd or 2 mod 4 doubles, or not a whole number of doubles),
// else padded by 16 bytes (s = 0 mod 4 doubles -> s + 2; such records are
// multiples of 32 bytes, so per-record copies stay 16-byte aligned).
__host__ __device__ constexpr uint32_t stage_stride(uint32_t bytes) {
  return (bytes % 8 != 0 || ((bytes / 8) & 3u) != 0) ? bytes : bytes + 16u;
}

// Record strides in HBM: the handle stores every per-cell record with a
// stride that is already conflict-free in shared memory (doubles: odd or
// 2 mod 4; 32-bit words: odd), so each array is one chunk copy per tile.
__host__ __device__ constexpr int rec_stride_f64(int e) { return e % 4 == 0 ? e + 2 : e; }
__host__ __device__ constexpr int rec_stride_i32(int e) { return e % 2 == 0 ? e + 1 : e; }

// One staged array of the tile: record bytes, smem stride, smem offset.
struct StageArr {
  const unsigned char* src;  // global base of record 0
  uint32_t rec;              // record bytes in HBM
  uint32_t bytes;            // record bytes staged (0: not staged)
  uint32_t stride;           // smem record stride
  uint32_t off;              // smem offset of the tile's record 0
};

// Bytes the bulk engine delivers for n records of one array.
__device__ __forceinline__ uint32_t stage_tx(const StageArr& a, int n) {
  return a.stride == a.bytes ? round16(a.bytes * (uint32_t)n) : a.bytes * (uint32_t)n;
}

// Issue the copies of records [c0, c0+n) of one array; called by every lane
// of warp 0 (lane l copies record l when padded; lane 0 the whole chunk
// otherwise).  Chunk copies may read up to 15 bytes past the last record:
// device allocations carry 64 bytes of tail padding (gks_api.cu upload).
__device__ __forceinline__ void stage_issue(unsigned char* smem, const StageArr& a, int64_t c0, int n, int lane,
                                            uint64_t* bar) {
  if (a.stride == a.bytes) {
    if (lane == 0) bulk_g2s(smem + a.off, a.src + (size_t)c0 * a.bytes, round16(a.bytes * (uint32_t)n), bar);
  } else {
    for (int c = lane; c < n; c += 32)
      bulk_g2s(smem + a.off + (uint32_t)c * a.stride, a.src + (size_t)(c0 + c) * a.bytes, a.bytes, bar);
  }
}

// A tile of N staged arrays, laid out back to back for `rt` cells.
template <int N>
struct Tile {
  StageArr a[N];
  uint32_t smem;
};

template <int N>
struct TileBuilder {
  Tile<N> t{};
  uint32_t off = 0;
  int rt;
  explicit TileBuilder(int rt_) : rt(rt_) {}
  void add(int i, const void* src, uint32_t bytes, bool on = true) {
    StageArr& a = t.a[i];
    a.src = (const unsigned char*)src;
    a.rec = bytes;
    a.bytes = on ? bytes : 0;
    a.stride = on ? stage_stride(bytes) : 0;
    a.off = off;
    off += round16(a.stride * (uint32_t)rt);
    t.smem = off;
  }
};

// Thread 0 arms the tile's mbarrier, the CTA synchronises once (nobody may
// wait on an uninitialised barrier), then warp 0 issues the bulk copies
// while the other warps go on to their first global loads.
template <int N>
__device__ __forceinline__ void stage_tile(unsigned char* sm, uint64_t* bar, const Tile<N>& T, int64_t c0, int n) {
  if (threadIdx.x == 0) {
    uint32_t tx = 0;
#pragma unroll
    for (int a = 0; a < N; ++a)
      if (T.a[a].bytes) tx += stage_tx(T.a[a], n);
    mbar_init(bar, 1);
    mbar_expect_tx(bar, tx);
  }
  __syncthreads();
  if (threadIdx.x < 32) {
#pragma unroll
    for (int a = 0; a < N; ++a)
      if (T.a[a].bytes) stage_issue(sm, T.a[a], c0, n, threadIdx.x, bar);
  }
}

}  // namespace gks
