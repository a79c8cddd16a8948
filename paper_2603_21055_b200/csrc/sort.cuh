// Hand-written LSD radix sort (onesweep: one read and one write of the
// pairs per digit pass, partitions ordered by a decoupled look-back), the
// pair-count scan and their helpers for the mapping preparation (K2, K3).
//
// Replaces np.lexsort (rasterizer.py:157-158) and the stable tile binning of
// _build_tile_lists (:178-218).  Every kernel reads its element count from
// device memory (no host round trip between the passes), so a view is
// prepared without host synchronisation.
//
// Pass structure (one launch per digit):
//   * the partition index comes from an atomic counter, so a partition's
//     predecessors were all scheduled before it (forward progress of the
//     look-back);
//   * each warp ranks its 512 keys (16 per lane, warp-striped so a warp's
//     keys are consecutive) with __match_any_sync per round of 32 -- stable;
//   * per digit: exclusive sums over the warps, the partition's count is
//     published (flag A), the look-back over earlier partitions gives the
//     exclusive global offset, the inclusive one is published (flag P);
//   * keys and values are reordered through shared memory so the global
//     writes of a digit's run are consecutive.
#pragma once

#include "common.cuh"

namespace sgad {

constexpr int OS_THREADS = 256;
constexpr int OS_WARPS = OS_THREADS / 32;
#ifndef SGAD_OS_ITEMS
#define SGAD_OS_ITEMS 16
#endif
#ifndef SGAD_OS_MATCH
#define SGAD_OS_MATCH 0  // warp ranks: 0 = RB ballots per round, 1 = __match_any_sync
#endif
constexpr int OS_ITEMS = SGAD_OS_ITEMS;
constexpr int OS_PART = OS_THREADS * OS_ITEMS;  // 4096 keys per partition

// partitions needed for n keys
__host__ __device__ __forceinline__ uint32_t os_parts(uint32_t n) {
  return (n + OS_PART - 1) / OS_PART;
}

// Depth bucket of a survivor (monotone in z): floor((z - zmin) * scale),
// capped at top = 2^bits - 2; culled ids carry 2^bits - 1 (never sorted).
struct DepthBucket {
  double zmin, scale, top;
  __device__ __forceinline__ void init(const unsigned long long* zrange, int kbits) {
    const double zlo = __longlong_as_double((long long)zrange[0]);
    const double zhi = __longlong_as_double((long long)zrange[1]);
    top = (double)(uint32_t)((kbits == 32 ? 0u : (1u << kbits)) - 2u);
    zmin = zlo;
    scale = zhi > zlo ? top / (zhi - zlo) : 0.0;
  }
  __device__ __forceinline__ uint32_t operator()(unsigned long long zk) const {
    const double b = floor((__longlong_as_double((long long)zk) - zmin) * scale);
    return b >= top ? (uint32_t)top : (uint32_t)b;
  }
};

// ---------------------------------------------------------------- block scans
// Exclusive scan of one value per thread over the first R threads of the
// block (R <= OS_THREADS, a multiple of 32); returns the exclusive prefix,
// *total receives the sum.  Every thread of the block must call it.
template <int R>
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* warp_tot,
                                                    uint32_t* total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t x = threadIdx.x < R ? v : 0u;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[w] = x;
  __syncthreads();
  uint32_t before = 0, all = 0;
#pragma unroll
  for (int i = 0; i < R / 32; ++i) {
    const uint32_t t = warp_tot[i];
    before += i < w ? t : 0u;
    all += t;
  }
  __syncthreads();  // warp_tot may be reused by the caller
  *total = all;
  return before + x - (threadIdx.x < R ? v : 0u);
}

// ---------------------------------------------------------------- histograms
// Digit histograms of every pass of the depth sort in one read of the keys.
template <int PASSES>
__global__ void __launch_bounds__(256)
k_depth_hist(const unsigned long long* __restrict__ zkeys, uint32_t n,
             const unsigned long long* __restrict__ zrange, int kbits,
             uint32_t* __restrict__ hist) {
  __shared__ uint32_t sh[PASSES][256];
  for (int i = threadIdx.x; i < PASSES * 256; i += blockDim.x) (&sh[0][0])[i] = 0u;
  DepthBucket bk;
  bk.init(zrange, kbits);
  __syncthreads();
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const unsigned long long zk = zkeys[i];
    if (zk == ~0ull) continue;
    const uint32_t k = bk(zk);
#pragma unroll
    for (int p = 0; p < PASSES; ++p) atomicAdd(&sh[p][(k >> (8 * p)) & 255u], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < PASSES * 256; i += blockDim.x) {
    const uint32_t c = (&sh[0][0])[i];
    if (c) atomicAdd(hist + i, c);
  }
}

// ---------------------------------------------------------------- onesweep pass
// MODE 0: keys/values from kin/vin; MODE 1: the depth sort's first pass --
// keys are the depth buckets of zkeys[i], values the emission index i,
// culled ids (zkeys == ~0) are dropped.
//
// Order of work inside a partition ("early counts"): the partition's digit
// counts (shared-memory atomics) are published before the warps rank their
// keys, so a successor's look-back rarely waits; the stable warp ranks come
// from RB ballots per round of 32 keys (the lanes sharing a digit).
// blocks per SM: 4 for the 6-bit passes (64 registers), 3 for the 8-bit ones
// (their 64-register build spills)
template <int RB, int MODE>
__global__ void __launch_bounds__(OS_THREADS, RB <= 6 ? 4 : 3)
k_onesweep(const uint32_t* __restrict__ kin, const uint32_t* __restrict__ vin,
           const unsigned long long* __restrict__ zkeys,
           const unsigned long long* __restrict__ zrange, int kbits, uint32_t n_static,
           const uint32_t* __restrict__ n_dev, uint32_t* __restrict__ kout,
           uint32_t* __restrict__ vout, const uint32_t* __restrict__ hist,
           uint32_t* __restrict__ status, uint32_t* __restrict__ ctr, int shift) {
  constexpr int R = 1 << RB;
  constexpr uint32_t DMASK = R - 1;
  static_assert(R <= OS_THREADS && R % 32 == 0, "radix");
  __shared__ uint32_t s_keys[OS_PART];
  __shared__ uint32_t s_vals[OS_PART];
  __shared__ uint32_t whist[OS_WARPS][R];
  __shared__ uint32_t s_cnt[R];      // the partition's digit counts
  __shared__ uint32_t s_bstart[R];   // first smem slot of each digit
  __shared__ int32_t s_goff[R];      // global position of smem slot 0 of each digit's run
  __shared__ uint32_t s_wt[OS_WARPS];
  __shared__ uint32_t s_part, s_nvalid;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (tid == 0) s_part = atomicAdd(ctr, 1u);
  for (int i = tid; i < OS_WARPS * R; i += OS_THREADS) (&whist[0][0])[i] = 0u;
  if (tid < R) s_cnt[tid] = 0u;
  // n_dev above n_static: the pairs overflowed their capacity (the view is
  // discarded); the digit histograms count every pair, so nothing is moved
  const uint32_t gh = tid < R ? hist[tid] : 0u;  // (this pass's global digit counts)
  const uint32_t nd = n_dev ? *n_dev : n_static;
  const uint32_t n = nd > n_static ? 0u : nd;
  __syncthreads();
  const uint32_t p = s_part;
  if (p >= os_parts(n)) return;  // block-uniform

  // keys in registers; values are read (MODE 0) or formed (MODE 1: the
  // index) when they are placed, so they do not hold registers meanwhile
  uint32_t key[OS_ITEMS];
  uint32_t vbits = 0;  // valid items of this lane
  const uint32_t base = p * OS_PART + (uint32_t)w * (OS_ITEMS * 32) + (uint32_t)lane;
  if (MODE == 1) {
    DepthBucket bk;
    bk.init(zrange, kbits);
#pragma unroll
    for (int k = 0; k < OS_ITEMS; ++k) {
      const uint32_t i = base + 32u * k;
      const unsigned long long zk = i < n ? zkeys[i] : ~0ull;
      const bool ok = zk != ~0ull;
      key[k] = ok ? bk(zk) : 0u;
      vbits |= ok ? (1u << k) : 0u;
    }
  } else {
#pragma unroll
    for (int k = 0; k < OS_ITEMS; ++k) {
      const uint32_t i = base + 32u * k;
      const bool ok = i < n;
      key[k] = ok ? kin[i] : 0u;
      vbits |= ok ? (1u << k) : 0u;
    }
  }
  // early counts, published as the partition's aggregate
#pragma unroll
  for (int k = 0; k < OS_ITEMS; ++k)
    if ((vbits >> k) & 1u) atomicAdd(&s_cnt[(key[k] >> shift) & DMASK], 1u);
  __syncthreads();
  // publish the aggregate; with fewer digits than threads the look-back runs
  // right away on the digit warps (the inclusive prefix is out early, so
  // successors' look-backs stay short) while the other warps rank their keys;
  // with a digit per thread it runs after the ranking, which hides its wait
  constexpr bool EARLY_LB = R < OS_THREADS;
  uint32_t cnt = 0, excl = 0;
  if (tid < R) {
    cnt = s_cnt[tid];
    st_volatile_u32(status + (size_t)p * R + tid, (p == 0 ? LB_FLAG_P : LB_FLAG_A) | cnt);
  }
  auto lookback = [&]() {
    if (tid < R && p > 0) {
      for (int q = (int)p - 1; q >= 0; --q) {
        uint32_t s;
        do {
          s = ld_volatile_u32(status + (size_t)q * R + tid);
        } while ((s >> 30) == 0u);
        excl += s & LB_VALUE;
        if ((s >> 30) == 2u) break;
      }
      st_volatile_u32(status + (size_t)p * R + tid, LB_FLAG_P | (excl + cnt));
    }
  };
  if (EARLY_LB) lookback();
  // warp-local stable ranks (16-bit, two per register)
  const uint32_t lt = (1u << lane) - 1u;
  uint32_t rank2[(OS_ITEMS + 1) / 2];
#pragma unroll
  for (int k = 0; k < OS_ITEMS; ++k) {
    const bool ok = (vbits >> k) & 1u;
    const uint32_t d = (key[k] >> shift) & DMASK;
    uint32_t peers = __ballot_sync(0xffffffffu, ok);
#if SGAD_OS_MATCH
    if (ok) peers = __match_any_sync(peers, d);
#else
#pragma unroll
    for (int b = 0; b < RB; ++b) {
      const uint32_t bal = __ballot_sync(0xffffffffu, (d >> b) & 1u);
      peers &= ((d >> b) & 1u) ? bal : ~bal;
    }
#endif
    const uint32_t old = ok ? whist[w][d] : 0u;
    __syncwarp();
    if (ok && (peers & lt) == 0u) whist[w][d] = old + __popc(peers);
    __syncwarp();
    const uint32_t rk = old + __popc(peers & lt);
    if (k & 1) rank2[k >> 1] |= rk << 16;
    else rank2[k >> 1] = rk;
  }
  __syncthreads();
  // per digit: exclusive over warps
  if (tid < R) {
    uint32_t c = 0;
#pragma unroll
    for (int i = 0; i < OS_WARPS; ++i) {
      const uint32_t x = whist[i][tid];
      whist[i][tid] = c;
      c += x;
    }
  }
  if (!EARLY_LB) lookback();
  uint32_t nvalid;
  const uint32_t bstart = block_excl_scan<R>(cnt, s_wt, &nvalid);
  uint32_t gtot;
  const uint32_t gstart = block_excl_scan<R>(gh, s_wt, &gtot);
  if (tid < R) {
    s_bstart[tid] = bstart;
    s_goff[tid] = (int32_t)(gstart + excl) - (int32_t)bstart;
  }
  if (tid == 0) s_nvalid = nvalid;
  __syncthreads();
#pragma unroll
  for (int k = 0; k < OS_ITEMS; ++k) {
    if ((vbits >> k) & 1u) {
      const uint32_t d = (key[k] >> shift) & DMASK;
      const uint32_t rk = (rank2[k >> 1] >> (16 * (k & 1))) & 0xFFFFu;
      const uint32_t pos = s_bstart[d] + whist[w][d] + rk;
      const uint32_t i = base + 32u * k;
      s_keys[pos] = key[k];
      s_vals[pos] = MODE == 1 ? i : vin[i];
    }
  }
  __syncthreads();
  const uint32_t nv = s_nvalid;
  for (uint32_t j = tid; j < nv; j += OS_THREADS) {
    const uint32_t kk = s_keys[j];
    const uint32_t o = (uint32_t)(s_goff[(kk >> shift) & DMASK] + (int32_t)j);
    kout[o] = kk;
    vout[o] = s_vals[j];
  }
}

// ---------------------------------------------------------------- pair scan + emit
// The tile pairs of the survivors in depth order (rasterizer.py:187-217):
// each partition of 4096 survivors counts its pairs (tile boxes), takes its
// exclusive offset from the decoupled look-back, and emits its (tile, value)
// pairs at their final positions in emission order, accumulating the digit
// histograms of the tile sort.  *n_pairs receives the total; pairs at or past
// cap are dropped and flag *overflow (and *ext_flag).
template <class Box, class Emit>
__global__ void __launch_bounds__(OS_THREADS, 4)
k_pair_emit(const uint32_t* __restrict__ perm, const Box* __restrict__ box,
            const uint32_t* __restrict__ n_dev, uint32_t n_static,
            uint32_t* __restrict__ status, uint32_t* __restrict__ ctr,
            uint32_t* __restrict__ n_pairs, Emit emit) {
  __shared__ uint32_t s_wt[OS_WARPS];
  __shared__ uint32_t s_part, s_excl;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (tid == 0) s_part = atomicAdd(ctr, 1u);
  const uint32_t n = min(*n_dev, n_static);
  __syncthreads();
  const uint32_t p = s_part;
  if (p >= os_parts(n)) return;
  const uint32_t base = p * OS_PART + (uint32_t)w * (OS_ITEMS * 32) + (uint32_t)lane;
  uint32_t off[OS_ITEMS];  // this item's offset within the warp's pairs
  uint32_t ee[OS_ITEMS];   // its survivor id
  uint32_t run = 0;
#pragma unroll
  for (int k = 0; k < OS_ITEMS; ++k) {
    const uint32_t i = base + 32u * k;
    uint32_t c = 0;
    ee[k] = i < n ? perm[i] : 0u;
    if (i < n) {
      const Box b = box[ee[k]];
      c = (uint32_t)(b.tx1 - b.tx0 + 1) * (uint32_t)(b.ty1 - b.ty0 + 1);
    }
    uint32_t x = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    off[k] = run + x - c;
    run += __shfl_sync(0xffffffffu, x, 31);
  }
  if (lane == 0) s_wt[w] = run;
  __syncthreads();
  uint32_t wbefore = 0, total = 0;
#pragma unroll
  for (int i = 0; i < OS_WARPS; ++i) {
    const uint32_t t = s_wt[i];
    wbefore += i < w ? t : 0u;
    total += t;
  }
  if (tid == 0) {
    if (p == 0) st_volatile_u32(status, LB_FLAG_P | total);
    else st_volatile_u32(status + p, LB_FLAG_A | total);
  }
  if (w == 0) {
    uint32_t excl = 0;
    if (p > 0) {
      excl = lookback_exclusive(status, (int)p);
      if (lane == 0) st_volatile_u32(status + p, LB_FLAG_P | (excl + total));
    }
    if (lane == 0) s_excl = excl;
  }
  __syncthreads();
  const uint32_t o0 = s_excl + wbefore;
  if (p + 1 == os_parts(n) && w == OS_WARPS - 1 && lane == 31) *n_pairs = s_excl + total;
  // emit, four items at a time with their boxes loaded together
  static_assert(OS_ITEMS % 4 == 0, "items per thread");
#pragma unroll 1
  for (int k0 = 0; k0 < OS_ITEMS; k0 += 4) {
    Box bb[4];
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (base + 32u * (k0 + k) < n) bb[k] = box[ee[k0 + k]];
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (base + 32u * (k0 + k) < n) emit(ee[k0 + k], bb[k], o0 + off[k0 + k]);
  }
}

// ---------------------------------------------------------------- long runs
// Runs of equal depth buckets longer than 64 (queued by k_depth_fixup) are
// put in exact (z bits, emission index) order here, one block per run (two
// blocks per SM: ~300 runs per C4 view; already-ordered runs, e.g. a plane
// seen head-on, are never queued): runs of up to LONG_RUN_SMEM_N are sorted
// bitonically in shared memory, longer ones by a block merge sort through a
// global scratch (each element finds its place in the other half by binary
// search; the keys are unique).
constexpr uint32_t LONG_RUN_SMEM_N = 8192;

__device__ __forceinline__ bool zlt(unsigned long long za, uint32_t ea, unsigned long long zb,
                                    uint32_t eb) {
  return za < zb || (za == zb && ea < eb);
}

__global__ void __launch_bounds__(1024)
k_long_runs(const uint2* __restrict__ long_runs, const uint32_t* __restrict__ n_long,
            const unsigned long long* __restrict__ zkeys, uint32_t* __restrict__ perm,
            unsigned long long* __restrict__ zscr, uint32_t* __restrict__ escr) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  unsigned long long* zs = reinterpret_cast<unsigned long long*>(smem_raw);  // [LONG_RUN_SMEM_N]
  uint32_t* es = reinterpret_cast<uint32_t*>(zs + LONG_RUN_SMEM_N);           // [LONG_RUN_SMEM_N]
  const uint32_t nr = *n_long;
  for (uint32_t r = blockIdx.x; r < nr; r += gridDim.x) {
    // (queued by k_depth_fixup only after an out-of-order pair: never sorted)
    const uint2 ru = long_runs[r];
    if (ru.y <= LONG_RUN_SMEM_N) {
      uint32_t P = 1;
      while (P < ru.y) P <<= 1;
      for (uint32_t i = threadIdx.x; i < P; i += blockDim.x) {
        if (i < ru.y) {
          const uint32_t e = perm[ru.x + i];
          zs[i] = zkeys[e];
          es[i] = e;
        } else {
          zs[i] = ~0ull;
          es[i] = ~0u;
        }
      }
      __syncthreads();
      for (uint32_t k = 2; k <= P; k <<= 1) {
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
          for (uint32_t i = threadIdx.x; i < P; i += blockDim.x) {
            const uint32_t x = i ^ j;
            if (x > i) {
              const bool gt = zlt(zs[x], es[x], zs[i], es[i]);
              if (((i & k) == 0) == gt) {
                const unsigned long long tz = zs[i];
                zs[i] = zs[x];
                zs[x] = tz;
                const uint32_t te = es[i];
                es[i] = es[x];
                es[x] = te;
              }
            }
          }
          __syncthreads();
        }
      }
      for (uint32_t i = threadIdx.x; i < ru.y; i += blockDim.x) perm[ru.x + i] = es[i];
      __syncthreads();
      continue;
    }
    // block merge sort through the scratch (zscr/escr at the run's own offset)
    unsigned long long* za = zscr + ru.x;
    uint32_t* ea = escr + ru.x;
    for (uint32_t i = threadIdx.x; i < ru.y; i += blockDim.x) {
      const uint32_t e = perm[ru.x + i];
      za[i] = zkeys[e];
      ea[i] = e;
    }
    __syncthreads();
    bool in_scr = true;  // current data in (za, ea); the other buffer is perm (+ zkeys)
    for (uint32_t wdt = 1; wdt < ru.y; wdt <<= 1) {
      for (uint32_t i = threadIdx.x; i < ru.y; i += blockDim.x) {
        const uint32_t s0 = (i / (2 * wdt)) * (2 * wdt);
        const uint32_t mid = min(s0 + wdt, ru.y), end = min(s0 + 2 * wdt, ru.y);
        const bool left = i < mid;
        const uint32_t e = in_scr ? ea[i] : perm[ru.x + i];
        const unsigned long long z = in_scr ? za[i] : zkeys[e];
        // position within the other half: elements strictly before (z, e)
        uint32_t lo = left ? mid : s0, hi = left ? end : mid;
        while (lo < hi) {
          const uint32_t m = (lo + hi) >> 1;
          const uint32_t em = in_scr ? ea[m] : perm[ru.x + m];
          const unsigned long long zm = in_scr ? za[m] : zkeys[em];
          if (zlt(zm, em, z, e)) lo = m + 1; else hi = m;
        }
        const uint32_t pos = s0 + (i - (left ? s0 : mid)) + (lo - (left ? mid : s0));
        if (in_scr) perm[ru.x + pos] = e; else { ea[pos] = e; za[pos] = z; }
      }
      __syncthreads();
      in_scr = !in_scr;
    }
    if (in_scr)
      for (uint32_t i = threadIdx.x; i < ru.y; i += blockDim.x) perm[ru.x + i] = ea[i];
    __syncthreads();
  }
}

}  // namespace sgad
