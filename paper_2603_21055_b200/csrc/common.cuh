// Shared helpers for the sm_100a kernels of libsgad.so.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <atomic>

#include "../../include/sgad.h"
#include "../../include/sgad_numerics.h"

namespace sgad {

void set_error(const char* fmt, ...);

// kernels of this library launched so far (sgad_launch_count)
extern std::atomic<long long> g_launches;

#define SGAD_CHECK_CUDA(x)                                                                  \
  do {                                                                                      \
    cudaError_t e_ = (x);                                                                   \
    if (e_ != cudaSuccess) {                                                                \
      ::sgad::set_error("%s:%d %s: %s", __FILE__, __LINE__, #x, cudaGetErrorString(e_));    \
      return SGAD_E_CUDA;                                                                   \
    }                                                                                       \
  } while (0)

#define SGAD_REQUIRE(cond, ...)          \
  do {                                   \
    if (!(cond)) {                       \
      ::sgad::set_error(__VA_ARGS__);    \
      return SGAD_E_INVALID;             \
    }                                    \
  } while (0)

// SGAD_DEBUG_SYNC=1 (debugging): synchronise after every launch so a fault is
// reported at the kernel that caused it
extern int g_debug_sync;

#define SGAD_LAUNCH_CHECK()                                                                 \
  do {                                                                                      \
    ::sgad::g_launches.fetch_add(1, std::memory_order_relaxed);                             \
    cudaError_t e_ = cudaGetLastError();                                                    \
    if (e_ == cudaSuccess && ::sgad::g_debug_sync) e_ = cudaDeviceSynchronize();            \
    if (e_ != cudaSuccess) {                                                                \
      ::sgad::set_error("%s:%d launch: %s", __FILE__, __LINE__, cudaGetErrorString(e_));    \
      return SGAD_E_CUDA;                                                                   \
    }                                                                                       \
  } while (0)

// Grow-only device scratch.  Growing frees the old block (cudaFree
// synchronises the device), which only happens while sizes are warming up.
struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  cudaError_t ensure(size_t bytes) {
    if (bytes <= cap && p) return cudaSuccess;
    if (p) {
      cudaFree(p);
      p = nullptr;
    }
    size_t want = bytes + bytes / 4 + 256;
    cudaError_t e = cudaMalloc(&p, want);
    cap = e == cudaSuccess ? want : 0;
    return e;
  }
  template <class T>
  T* as() const {
    return reinterpret_cast<T*>(p);
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
};

__device__ __forceinline__ uint32_t ld_volatile_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

__device__ __forceinline__ void st_volatile_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.volatile.global.u32 [%0], %1;" ::"l"(p), "r"(v));
}

__device__ __forceinline__ int ceil_div(int a, int b) { return (a + b - 1) / b; }

// ---------------------------------------------------------------------------
// Ordered stream compaction: decoupled look-back over 256-item tiles.
// status word: bits 31..30 = flag (0 empty, 1 aggregate, 2 inclusive prefix),
// bits 29..0 = value (counts < 2^30).
constexpr uint32_t LB_FLAG_A = 1u << 30;
constexpr uint32_t LB_FLAG_P = 2u << 30;
constexpr uint32_t LB_VALUE = (1u << 30) - 1;

// Called by warp 0 of the tile after thread 0 published the aggregate.
// Returns the exclusive prefix of this tile (valid on all lanes of warp 0).
__device__ __forceinline__ uint32_t lookback_exclusive(uint32_t* status, int tile) {
  const int lane = threadIdx.x & 31;
  uint32_t excl = 0;
  int pred = tile - 1;
  while (true) {
    const int idx = pred - lane;
    uint32_t s = idx >= 0 ? ld_volatile_u32(status + idx) : LB_FLAG_P;
    while (__any_sync(0xffffffffu, (s >> 30) == 0)) {
      if ((s >> 30) == 0) s = ld_volatile_u32(status + idx);
    }
    const uint32_t pmask = __ballot_sync(0xffffffffu, (s >> 30) == 2);
    const int stop = pmask ? __ffs(pmask) - 1 : 31;
    uint32_t v = lane <= stop ? (s & LB_VALUE) : 0u;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    excl += v;
    if (pmask) break;
    pred -= 32;
  }
  return excl;
}

}  // namespace sgad
