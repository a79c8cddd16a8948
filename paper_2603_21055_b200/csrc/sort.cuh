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
constexpr int OS_ITEMS = 16;
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
template <int RB, int MODE>
__global__ void __launch_bounds__(OS_THREADS)
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
  __shared__ uint32_t s_bstart[R];   // first smem slot of each digit
  __shared__ int32_t s_goff[R];      // global position of smem slot 0 of each digit's run
  __shared__ uint32_t s_wt[OS_WARPS];
  __shared__ uint32_t s_part, s_nvalid;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (tid == 0) s_part = atomicAdd(ctr, 1u);
  for (int i = tid; i < OS_WARPS * R; i += OS_THREADS) (&whist[0][0])[i] = 0u;
  __syncthreads();
  const uint32_t p = s_part;
  const uint32_t n = n_dev ? min(*n_dev, n_static) : n_static;
  if (p >= os_parts(n)) return;  // block-uniform

  uint32_t key[OS_ITEMS], val[OS_ITEMS];
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
      val[k] = i;
      vbits |= ok ? (1u << k) : 0u;
    }
  } else {
#pragma unroll
    for (int k = 0; k < OS_ITEMS; ++k) {
      const uint32_t i = base + 32u * k;
      const bool ok = i < n;
      key[k] = ok ? kin[i] : 0u;
      val[k] = ok ? vin[i] : 0u;
      vbits |= ok ? (1u << k) : 0u;
    }
  }
  // warp-local stable ranks
  const uint32_t lt = (1u << lane) - 1u;
  uint32_t rank[OS_ITEMS];
#pragma unroll
  for (int k = 0; k < OS_ITEMS; ++k) {
    const bool ok = (vbits >> k) & 1u;
    const uint32_t vm = __ballot_sync(0xffffffffu, ok);
    const uint32_t d = (key[k] >> shift) & DMASK;
    uint32_t old = 0, peers = 0;
    if (ok) {
      peers = __match_any_sync(vm, d);
      old = whist[w][d];
    }
    __syncwarp();
    if (ok && (peers & lt) == 0u) whist[w][d] = old + __popc(peers);
    __syncwarp();
    rank[k] = old + __popc(peers & lt);
  }
  __syncthreads();
  // per digit: exclusive over warps, partition count, publish the aggregate
  uint32_t cnt = 0;
  if (tid < R) {
#pragma unroll
    for (int i = 0; i < OS_WARPS; ++i) {
      const uint32_t x = whist[i][tid];
      whist[i][tid] = cnt;
      cnt += x;
    }
    st_volatile_u32(status + (size_t)p * R + tid, (p == 0 ? LB_FLAG_P : LB_FLAG_A) | cnt);
  }
  uint32_t nvalid;
  const uint32_t bstart = block_excl_scan<R>(cnt, s_wt, &nvalid);
  uint32_t gh = 0;
  if (tid < R) gh = hist[tid];
  uint32_t gtot;
  const uint32_t gstart = block_excl_scan<R>(gh, s_wt, &gtot);
  if (tid < R) {
    uint32_t excl = 0;
    if (p > 0) {
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
    s_bstart[tid] = bstart;
    s_goff[tid] = (int32_t)(gstart + excl) - (int32_t)bstart;
  }
  if (tid == 0) s_nvalid = nvalid;
  __syncthreads();
#pragma unroll
  for (int k = 0; k < OS_ITEMS; ++k) {
    if ((vbits >> k) & 1u) {
      const uint32_t d = (key[k] >> shift) & DMASK;
      const uint32_t pos = s_bstart[d] + whist[w][d] + rank[k];
      s_keys[pos] = key[k];
      s_vals[pos] = val[k];
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

// ---------------------------------------------------------------- pair-count scan
// poff[i] = sum of tile counts of survivors 0..i-1 in depth order (exclusive
// scan, decoupled look-back over 4096-item partitions); poff[ns] = total
// pairs, also stored at *n_pairs.
struct TileBoxView {  // the fields of TileBox the scan reads
  uint16_t tx0, tx1, ty0, ty1;
};

template <class Box>
__global__ void __launch_bounds__(OS_THREADS)
k_pair_scan(const uint32_t* __restrict__ perm, const Box* __restrict__ box,
            const uint32_t* __restrict__ n_dev, uint32_t n_static, uint32_t* __restrict__ poff,
            uint32_t* __restrict__ status, uint32_t* __restrict__ ctr,
            uint32_t* __restrict__ n_pairs) {
  __shared__ uint32_t s_wt[OS_WARPS];
  __shared__ uint32_t s_part, s_excl;
  const int tid = threadIdx.x, lane = tid & 31;
  if (tid == 0) s_part = atomicAdd(ctr, 1u);
  __syncthreads();
  const uint32_t p = s_part;
  const uint32_t n = min(*n_dev, n_static);
  if (p >= os_parts(n)) return;
  const uint32_t i0 = p * OS_PART + (uint32_t)tid * OS_ITEMS;
  uint32_t c[OS_ITEMS];
  uint32_t sum = 0;
#pragma unroll
  for (int k = 0; k < OS_ITEMS; ++k) {
    const uint32_t i = i0 + k;
    uint32_t v = 0;
    if (i < n) {
      const Box b = box[perm[i]];
      v = (uint32_t)(b.tx1 - b.tx0 + 1) * (uint32_t)(b.ty1 - b.ty0 + 1);
    }
    c[k] = v;
    sum += v;
  }
  uint32_t total;
  const uint32_t mine = block_excl_scan<OS_THREADS>(sum, s_wt, &total);
  if (tid == 0) {
    if (p == 0) st_volatile_u32(status, LB_FLAG_P | total);
    else st_volatile_u32(status + p, LB_FLAG_A | total);
  }
  if (tid < 32) {
    uint32_t excl = 0;
    if (p > 0) {
      excl = lookback_exclusive(status, (int)p);
      if (lane == 0) st_volatile_u32(status + p, LB_FLAG_P | (excl + total));
    }
    if (lane == 0) s_excl = excl;
  }
  __syncthreads();
  uint32_t run = s_excl + mine;
#pragma unroll
  for (int k = 0; k < OS_ITEMS; ++k) {
    const uint32_t i = i0 + k;
    if (i < n) poff[i] = run;
    run += c[k];
    if (i + 1 == n) {
      poff[n] = run;
      *n_pairs = run;
    }
  }
}

// ---------------------------------------------------------------- long runs
// Runs of equal depth buckets longer than 64 (queued by k_depth_fixup) are
// put in exact (z bits, emission index) order here, one block per run:
// already-ordered runs (a plane seen head-on: equal z, emission order kept by
// the stable sort) are skipped, runs of up to LONG_RUN_SMEM_N are sorted
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
  __shared__ int s_unsorted;
  const uint32_t nr = *n_long;
  for (uint32_t r = blockIdx.x; r < nr; r += gridDim.x) {
    const uint2 ru = long_runs[r];
    if (threadIdx.x == 0) s_unsorted = 0;
    __syncthreads();
    for (uint32_t i = threadIdx.x; i + 1 < ru.y; i += blockDim.x) {
      const uint32_t ea = perm[ru.x + i], eb = perm[ru.x + i + 1];
      if (!zlt(zkeys[ea], ea, zkeys[eb], eb)) s_unsorted = 1;
    }
    __syncthreads();
    if (!s_unsorted) continue;
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
