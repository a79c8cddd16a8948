// Mapping hot path: projection (K1), depth sort (K2), tile binning (K3),
// front-to-back compositing with optional fused L1 loss (K4) and the
// backward sweep with chain rule (K5).
//
// Restates /root/reference/pkg/src/raysplat/rasterizer.py:
//   K1 <- _prepare :86-135      K2 <- lexsort :157-158
//   K3 <- _build_tile_lists :178-218
//   K4 <- _forward_kernel :221-269 (+ mapper.py:118-152 loss, tau = 0)
//   K5 <- _backward_kernel :272-363 + chain rule :462-483
//
// Layout (HBM): survivors live in EMISSION order (frame, pixel) as 64-byte
// records; the depth sort produces a permutation, tile lists hold emission
// indices in depth order (plus, in the top bits, the warp rectangles each
// entry reaches).  A forward that keeps state writes per-warp compact lists
// (entries reaching the warp's 8x4 pixels + exact masks) that the backward
// walks instead of the tile lists.  Per-view scratch is owned by the
// sgad_raster handle.  DESIGN.md section 4 has the measured design notes.
#include <stdarg.h>
#include <stddef.h>
#include <stdlib.h>
#include <algorithm>
#include <vector>

#include "common.cuh"
#include "sort.cuh"

namespace sgad {

struct __align__(16) Record {
  double u0, v0, sigma, opacity, z;
  double nh;             // -0.5 / sigma^2 (the compositing exponent scale)
  float r, g, b;
  uint32_t gid;          // bit 31: learnable
};

struct TileBox {         // inclusive tile bbox of a survivor (rasterizer.py:187-199)
  uint16_t tx0, tx1, ty0, ty1;
  int16_t px0, px1, py0, py1;  // pixel centres its 3-sigma disc may reach (conservative)
};

// Tile list values: the record index in the low 26 bits and, above it, which
// of the tile's 8x4 warp rectangles the Gaussian's (conservative) 3-sigma box
// reaches -- 2 column bits, 4 row bits -- so K4 culls a list entry against
// its rectangle without loading the record.  Views with 2^26 or more
// Gaussians store the bare index and K4 culls nothing at this stage.
constexpr int LIST_IDX_BITS = 26;
constexpr uint32_t LIST_IDX_MASK = (1u << LIST_IDX_BITS) - 1u;
static_assert(sizeof(Record) == 64, "record must be one 64-byte line");
// K4/K5 read the record as four 16-byte vectors: (u0, v0) (sigma, opacity) (z, nh) (r, g, b, gid)
static_assert(offsetof(Record, sigma) == 16 && offsetof(Record, z) == 32 &&
              offsetof(Record, nh) == 40 && offsetof(Record, r) == 48 && offsetof(Record, gid) == 60,
              "record field offsets");

// The window backward's record (one 64-byte line, two 32-byte loads): the
// fields a contribution needs and the view-dependent chain-rule coefficients
// of rasterizer.py:462-483, so K5 adds parameter gradients directly.  The
// compositing fields stay fp64: the backward reconstructs T and the suffix
// sums from the forward's fp64 state, and c T_b - S / (1 - a) cancels
// heavily (neighbouring Gaussians share colour and depth), so fp32 opacity
// or exponent scale cost 1e-3 of a gradient (measured).  The remaining
// coefficients follow from these: d delta / d(sigma g_sigma) = -a_z / z,
// d radius / d(sigma g_sigma) = fx sqrt(-2 nh) / z, d logit / d op =
// op (1 - op).
struct __align__(16) BwdRecord {
  double u0, v0, op, nh;       // nh = -0.5 / sigma^2
  double z;
  float r, g, b;
  float a_u, a_v, a_z;         // d delta / d (u0, v0, z)
};
static_assert(sizeof(BwdRecord) == 64, "backward record must be one 64-byte line");

#ifndef SGAD_K1_TMA
#define SGAD_K1_TMA 1  // K1 writes its staged records with bulk copies (TMA)
#endif

constexpr uint32_t GID_LEARN = 0x80000000u;
#ifdef SGAD_K5_COUNT
__device__ unsigned long long g_k5_count[4];
#endif
constexpr int PROJ_THREADS = 256;
constexpr int RASTER_THREADS = 256;

}  // namespace sgad

struct sgad_raster {
  sgad::DevBuf frames, counters, records, coef, keys0, keys1, vals0, vals1;
  sgad::DevBuf pkeys0, pkeys1, pvals0, pvals1, ranges, sortws, pairws;
  sgad::DevBuf trans_final, last_idx, signs, raw_grads, rank_of, scratch, col64, zrange, k32a, k32b, bbox, runs, cl_e, cl_m, cl_n;
  int any_f64 = 0;
  std::vector<sgad_frame> host_frames;
  sgad_camera cam{};
  // n_surv / n_pairs: host copies, valid after a synchronous prepare (-1
  // after an asynchronous one: the counts live in `counters` on the device)
  int64_t n_total = 0, n_surv = 0, n_pairs = 0;
  int64_t cap_pairs = 0;  // capacity of the pair / compact-list buffers
  int32_t n_tiles = 0, ntx = 0, nty = 0;
  int prepared = 0, forwarded = 0, have_coef = 0, fused_ready = 0;
  int packed = 0;  // tile list values carry the warp-rectangle bits (n_total < 2^26)
  int kbits = 24, dpasses = 3, tpasses = 2;
  double rho = 0, sigma_d = 0;
  int64_t n_depth = 0;
  uint32_t* pinned = nullptr;  // host-pinned counters
};

// counters[] slots (device, per prepared view)
enum : int { C_NSURV = 1, C_NLONG = 3, C_NPAIRS = 4, C_OVERFLOW = 5 };

namespace sgad {

static thread_local char g_err[1024] = "";
std::atomic<long long> g_launches{0};
int g_debug_sync = [] {
  const char* e = getenv("SGAD_DEBUG_SYNC");
  return e && e[0] == '1' ? 1 : 0;
}();

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
}

// ------------------------------------------------------------------ K1
__device__ __forceinline__ int find_frame(const sgad_frame* frames, int n, uint32_t gid) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if ((uint64_t)frames[mid].gauss_offset <= gid) lo = mid; else hi = mid - 1;
  }
  return lo;
}

__device__ __forceinline__ double plane_ld(const sgad_frame& f, int64_t i) {
  return f.planes_f64 ? reinterpret_cast<const double*>(f.planes)[i]
                      : (double)reinterpret_cast<const float*>(f.planes)[i];
}

struct Proj {
  double u0, v0, z, sig, op, bd;
  double dir[3], y[3];
};

// The seven parameter planes of pixel p, loaded together up front (the loads
// are independent, so they are all in flight before the first use).
struct Params {
  double base, delta, logr, logit, r, g, b;
};

__device__ __forceinline__ Params load_params(const sgad_frame& f, int64_t p, int64_t hw) {
  Params q;
  if (f.planes_f64) {
    const double* P = reinterpret_cast<const double*>(f.planes) + p;
    q.base = __ldg(P);
    q.delta = __ldg(P + hw);
    q.logr = __ldg(P + 2 * hw);
    q.logit = __ldg(P + 3 * hw);
    q.r = __ldg(P + 4 * hw);
    q.g = __ldg(P + 5 * hw);
    q.b = __ldg(P + 6 * hw);
  } else {
    const float* P = reinterpret_cast<const float*>(f.planes) + p;
    q.base = (double)__ldg(P);
    q.delta = (double)__ldg(P + hw);
    q.logr = (double)__ldg(P + 2 * hw);
    q.logit = (double)__ldg(P + 3 * hw);
    q.r = (double)__ldg(P + 4 * hw);
    q.g = (double)__ldg(P + 5 * hw);
    q.b = (double)__ldg(P + 6 * hw);
  }
  return q;
}

// rasterizer.py:86-116 for one active pixel p of frame f; true if it survives
// the near-plane and on-screen culls.  Operation order matches the reference.
__device__ __forceinline__ bool project_point(const sgad_frame& f, int64_t p, const Params& q,
                                              const sgad_camera& cam, Proj& o) {
  const int pi = (int)p;  // < 2^30 (checked in sgad_raster_prepare)
  const double xx = (double)(pi % f.width), yy = (double)(pi / f.width);
  const double r0 = SG_DIV(SG_SUB(xx, f.cx), f.fx);
  const double r1 = SG_DIV(SG_SUB(yy, f.cy), f.fy);
  o.bd = SG_ADD(q.base, q.delta);
  const double dadj = fabs(o.bd);
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    // rays @ R.T as OpenBLAS evaluates it: fma(r1, R[j,1], r0 * R[j,0]) + R[j,2]
    o.dir[j] = SG_ADD(SG_FMA(r1, f.rot[3 * j + 1], SG_MUL(r0, f.rot[3 * j])), f.rot[3 * j + 2]);
    o.y[j] = SG_ADD(SG_MUL(o.dir[j], dadj), f.trans[j]);
  }
  o.z = o.y[2];
  if (!(o.z > SGAD_Z_NEAR)) return false;
  const double radius = sgad_exp(q.logr);
  o.u0 = SG_ADD(SG_DIV(SG_MUL(cam.fx, o.y[0]), o.z), cam.cx);
  o.v0 = SG_ADD(SG_DIV(SG_MUL(cam.fy, o.y[1]), o.z), cam.cy);
  o.sig = SG_DIV(SG_MUL(radius, cam.fx), o.z);
  const double margin = SG_MUL(3.0, o.sig);
  const double wlim = SG_SUB((double)cam.width, 1.0), hlim = SG_SUB((double)cam.height, 1.0);
  if (!(SG_ADD(o.u0, margin) >= 0.0 && SG_SUB(o.u0, margin) <= wlim &&
        SG_ADD(o.v0, margin) >= 0.0 && SG_SUB(o.v0, margin) <= hlim))
    return false;
  o.op = sgad_sigmoid(q.logit);
  return true;
}

#ifndef SGAD_PROJ_MINB
#define SGAD_PROJ_MINB 4  // 64 registers: 4 blocks per SM (289 -> 260 us at C4)
#endif
__global__ void __launch_bounds__(PROJ_THREADS, SGAD_PROJ_MINB)
k_project(const sgad_frame* __restrict__ frames, sgad_camera cam, int ntx, int nty,
          int want_coef, Record* __restrict__ rec, TileBox* __restrict__ box,
          BwdRecord* __restrict__ coef, double* __restrict__ col64,
          unsigned long long* __restrict__ zkey, uint32_t* __restrict__ counters,
          unsigned long long* __restrict__ zrange, uint32_t* __restrict__ tile_count) {
  // one block = 256 consecutive pixels of frame blockIdx.y; the frame
  // descriptor is copied to shared memory (no per-thread frame search), and
  // the 64-byte records and 32-byte chain coefficients are staged in shared
  // memory so the global stores are whole contiguous lines
  __shared__ sgad_frame fsh;
  __shared__ __align__(16) Record rs[PROJ_THREADS];
  __shared__ __align__(16) BwdRecord cs[PROJ_THREADS];
  __shared__ unsigned long long red_z[2][PROJ_THREADS / 32];
  __shared__ uint32_t red_n[PROJ_THREADS / 32];
  constexpr int FW = (int)(sizeof(sgad_frame) / 4);
  static_assert(sizeof(sgad_frame) % 4 == 0, "frame descriptor size");
  for (int i = threadIdx.x; i < FW; i += PROJ_THREADS)
    reinterpret_cast<uint32_t*>(&fsh)[i] = reinterpret_cast<const uint32_t*>(frames + blockIdx.y)[i];
  __syncthreads();
  const sgad_frame& f = fsh;
  const int64_t hw = (int64_t)f.height * f.width;
  const int64_t p0 = (int64_t)blockIdx.x * PROJ_THREADS;
  if (p0 >= hw) return;  // block-uniform
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t p = p0 + threadIdx.x;
  const uint32_t gid = (uint32_t)(f.gauss_offset + p);

  bool keep = false;
  Proj o;
  TileBox bx{};
  if (p < hw) {
    const bool active = f.mask[p] != 0;
    const Params q = load_params(f, p, hw);
    if (active && project_point(f, p, q, cam, o)) {
      keep = true;
      Record r;
      r.u0 = o.u0;
      r.v0 = o.v0;
      r.sigma = o.sig;
      r.opacity = o.op;
      r.z = o.z;
      r.nh = SG_DIV(-0.5, SG_MUL(o.sig, o.sig));
      r.r = (float)q.r;
      r.g = (float)q.g;
      r.b = (float)q.b;
      if (col64) {
        col64[3 * (size_t)gid] = q.r;
        col64[3 * (size_t)gid + 1] = q.g;
        col64[3 * (size_t)gid + 2] = q.b;
      }
      r.gid = gid | (f.learnable ? GID_LEARN : 0u);
      rs[threadIdx.x] = r;
      // tile bbox (rasterizer.py:187-199); (x) / 16 is exact as (x) * 0.0625
      const double rr = SG_MUL(3.0, o.sig), it16 = 1.0 / (double)SGAD_TILE;
      long long x0 = (long long)floor(SG_MUL(SG_SUB(o.u0, rr), it16));
      long long x1 = (long long)floor(SG_MUL(SG_ADD(o.u0, rr), it16));
      long long y0 = (long long)floor(SG_MUL(SG_SUB(o.v0, rr), it16));
      long long y1 = (long long)floor(SG_MUL(SG_ADD(o.v0, rr), it16));
      x0 = x0 < 0 ? 0 : x0;
      y0 = y0 < 0 ? 0 : y0;
      x1 = x1 > ntx - 1 ? ntx - 1 : x1;
      y1 = y1 > nty - 1 ? nty - 1 : y1;
      bx.tx0 = (uint16_t)x0;
      bx.tx1 = (uint16_t)x1;
      bx.ty0 = (uint16_t)y0;
      bx.ty1 = (uint16_t)y1;
      {  // pixel-centre range of the disc, grown by a margin far above fp rounding
        const double R = SG_ADD(SG_MUL(rr, 1.0001), 0.01);
        const double lim_x = (double)cam.width, lim_y = (double)cam.height;
        bx.px0 = (int16_t)fmin(fmax(ceil(SG_SUB(o.u0, R)), -1.0), lim_x);
        bx.px1 = (int16_t)fmin(fmax(floor(SG_ADD(o.u0, R)), -1.0), lim_x);
        bx.py0 = (int16_t)fmin(fmax(ceil(SG_SUB(o.v0, R)), -1.0), lim_y);
        bx.py1 = (int16_t)fmin(fmax(floor(SG_ADD(o.v0, R)), -1.0), lim_y);
      }
      box[gid] = bx;
      if (want_coef) {
        BwdRecord c;
        const double sgn = o.bd >= 0.0 ? 1.0 : -1.0;
        const double iz = 1.0 / o.z;
        c.u0 = o.u0;
        c.v0 = o.v0;
        c.op = o.op;
        c.nh = r.nh;
        c.z = o.z;
        c.r = r.r;
        c.g = r.g;
        c.b = r.b;
        c.a_u = (float)(sgn * cam.fx * iz * (o.dir[0] - o.dir[2] * o.y[0] * iz));
        c.a_v = (float)(sgn * cam.fy * iz * (o.dir[1] - o.dir[2] * o.y[1] * iz));
        c.a_z = (float)(sgn * o.dir[2]);
        cs[threadIdx.x] = c;
      }
    }
  }
  // pairs per tile (the tile lists' sizes): the lanes of a warp hold
  // neighbouring pixels whose boxes share tiles, so each round of tiles is
  // aggregated over the lanes naming the same tile (one atomic per tile)
  {
    const int bw = keep ? bx.tx1 - bx.tx0 + 1 : 0, bh = keep ? bx.ty1 - bx.ty0 + 1 : 0;
    const int cnt_t = bw * bh;
    int most = cnt_t;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) most = max(most, __shfl_xor_sync(0xffffffffu, most, off));
    for (int j = 0; j < most; ++j) {
      const bool has = j < cnt_t;
      const uint32_t t = has ? (uint32_t)((bx.ty0 + j / bw) * ntx + bx.tx0 + j % bw) : ~0u;
      const uint32_t act = __ballot_sync(0xffffffffu, has);
      if (has) {
        const uint32_t peers = __match_any_sync(act, t);
        if ((peers & ((1u << lane) - 1u)) == 0u) atomicAdd(tile_count + t, (uint32_t)__popc(peers));
      }
    }
  }
  // depth keys: records stay at their Gaussian id; culled ids carry the
  // sentinel and sort behind every survivor
  const unsigned long long zk = keep ? (unsigned long long)__double_as_longlong(o.z) : ~0ull;
  if (p < hw) zkey[gid] = zk;
  // survivors and their depth range (positive doubles order like their
  // bits): warp shuffles, then one atomic per block
  unsigned long long zmn = zk, zmx = keep ? zk : 0ull;
  uint32_t ns = keep ? 1u : 0u;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    zmn = min(zmn, __shfl_xor_sync(0xffffffffu, zmn, off));
    zmx = max(zmx, __shfl_xor_sync(0xffffffffu, zmx, off));
    ns += __shfl_xor_sync(0xffffffffu, ns, off);
  }
  if (lane == 0) {
    red_z[0][warp] = zmn;
    red_z[1][warp] = zmx;
    red_n[warp] = ns;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < PROJ_THREADS / 32; ++w) {
      zmn = min(zmn, red_z[0][w]);
      zmx = max(zmx, red_z[1][w]);
      ns += red_n[w];
    }
    if (ns) {
      atomicAdd(&counters[1], ns);
      atomicMin(zrange, zmn);
      atomicMax(zrange + 1, zmx);
    }
  }
  // coalesced stores of the staged records (culled slots carry stale bytes;
  // nothing reads a record whose depth key is the sentinel)
  const int nvalid = (int)min((int64_t)PROJ_THREADS, hw - p0);
  const uint32_t gid0 = (uint32_t)(f.gauss_offset + p0);
#if SGAD_K1_TMA
  // one thread hands both staged arrays to the bulk-copy engine (TMA,
  // cp.async.bulk shared -> global) and waits until they have been read
  if (threadIdx.x == 0) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    const uint32_t bytes = (uint32_t)nvalid * (uint32_t)sizeof(Record);
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                 ::"l"(rec + gid0), "r"((uint32_t)__cvta_generic_to_shared(rs)), "r"(bytes)
                 : "memory");
    if (want_coef)
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                   ::"l"(coef + gid0), "r"((uint32_t)__cvta_generic_to_shared(cs)), "r"(bytes)
                   : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  }
#else
  {
    const uint4* src = reinterpret_cast<const uint4*>(rs);
    uint4* dst = reinterpret_cast<uint4*>(rec + gid0);
    for (int i = threadIdx.x; i < nvalid * 4; i += PROJ_THREADS) dst[i] = src[i];
  }
  if (want_coef) {
    const uint4* src = reinterpret_cast<const uint4*>(cs);
    uint4* dst = reinterpret_cast<uint4*>(coef + gid0);
    for (int i = threadIdx.x; i < nvalid * 4; i += PROJ_THREADS) dst[i] = src[i];
  }
#endif
}

// ------------------------------------------------------------------ K2
// Depth order = np.lexsort((pixel, frame, z)) (rasterizer.py:157-158).
// Survivors are sorted stably by a 24-bit monotone depth bucket,
// floor((z - zmin) * scale) (3 onesweep passes of sort.cuh; the first pass
// computes the buckets from the fp64 z bits and drops culled ids), so equal
// buckets keep emission (frame, pixel) order; the runs of equal buckets are
// then put in exact (z, emission) order by k_depth_fixup / k_long_runs.
static int depth_key_bits() {  // SGAD_DEPTH_BITS (A/B): 16..32, default 24
  const char* v = getenv("SGAD_DEPTH_BITS");
  const int b = v ? atoi(v) : 24;
  return b < 16 ? 16 : (b > 32 ? 32 : b);
}

// Runs of equal buckets whose exact (z bits, emission index) order differs
// from the stable bucket order: every adjacent pair of equal buckets is
// checked in parallel (runs of exactly equal z -- a plane seen head-on -- are
// already in order: the sort is stable); an out-of-order pair claims its
// run's head in a bitmap, and the claiming thread sorts a run of up to 64 by
// insertion or queues it for k_long_runs (sort.cuh; any length).
__global__ void k_depth_fixup(const uint32_t* __restrict__ k32, const uint32_t* __restrict__ n_dev,
                              const unsigned long long* __restrict__ zkeys,
                              uint32_t* __restrict__ perm, uint32_t* __restrict__ claim,
                              uint32_t* __restrict__ n_long, uint2* __restrict__ long_runs) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t n = *n_dev;
  if (i + 1 >= n) return;
  const uint32_t kk = k32[i];
  if (k32[i + 1] != kk) return;
  {
    const uint32_t e0 = perm[i], e1 = perm[i + 1];
    if (zlt(zkeys[e0], e0, zkeys[e1], e1)) return;  // in order
  }
  // the run [h, end) of bucket kk: galloping searches in the sorted buckets
  uint32_t h = i, step = 1;
  while (h > 0 && k32[h - 1] == kk) {  // k32[h] == kk; find lo with k32[lo] < kk
    const uint32_t lo = h > step ? h - step : 0;
    if (k32[lo] == kk) {
      h = lo;
      step <<= 1;
    } else {
      uint32_t a = lo, b = h;  // k32[a] < kk == k32[b]
      while (b - a > 1) {
        const uint32_t m = (a + b) >> 1;
        if (k32[m] == kk) b = m; else a = m;
      }
      h = b;
      break;
    }
  }
  if (atomicOr(claim + (h >> 5), 1u << (h & 31)) & (1u << (h & 31))) return;  // claimed
  uint32_t end = i + 1;
  step = 1;
  while (end + 1 < n && k32[end + 1] == kk) {  // k32[end] == kk
    const uint32_t hi = end + step < n - 1 ? end + step : n - 1;
    if (k32[hi] == kk) {
      end = hi;
      step <<= 1;
    } else {
      uint32_t a = end, b = hi;  // k32[a] == kk < k32[b]
      while (b - a > 1) {
        const uint32_t m = (a + b) >> 1;
        if (k32[m] == kk) a = m; else b = m;
      }
      end = a;
      break;
    }
  }
  ++end;
  if (end - h > 64) {
    long_runs[atomicAdd(n_long, 1u)] = make_uint2(h, end - h);
    return;
  }
  for (uint32_t a = h + 1; a < end; ++a) {  // insertion sort on (z, e)
    const uint32_t e = perm[a];
    const unsigned long long z = zkeys[e];
    uint32_t b = a;
    while (b > h) {
      const uint32_t pe = perm[b - 1];
      if (zlt(zkeys[pe], pe, z, e)) break;
      perm[b] = pe;
      --b;
    }
    perm[b] = e;
  }
}

// ------------------------------------------------------------------ K3
// Tile lists = _build_tile_lists (rasterizer.py:178-218): the pair count of
// every survivor in depth order is scanned (k_pair_emit, sort.cuh), each
// survivor emits its (tile, value) pairs in (ty, tx) order at its offset, and
// a stable radix sort on the tile key (6-bit digits) bins them: every tile's
// list ends up in depth order.  Pairs past the handle's capacity are dropped
// and flag *overflow (the caller grows the capacity and prepares again).
constexpr int TILE_RB = 6;

struct TileEmit {
  int ntx, packed;
  uint32_t cap;
  uint32_t* pkeys;
  uint32_t* pvals;
  uint32_t* overflow;
  int32_t* ext_flag;
  // the (tile, value) pairs of survivor e from offset o, in (ty, tx) order
  __device__ __forceinline__ void operator()(uint32_t e, const TileBox& r, uint32_t o) const {
    for (int ty = r.ty0; ty <= r.ty1; ++ty) {
      uint32_t rows = 0;  // 4-row bands [by + 4b, by + 4b + 3] the box reaches
      const int by = ty * SGAD_TILE;
#pragma unroll
      for (int b = 0; b < 4; ++b)
        rows |= (r.py0 <= by + 4 * b + 3 && r.py1 >= by + 4 * b) ? (1u << b) : 0u;
      for (int tx = r.tx0; tx <= r.tx1; ++tx) {
        const int bx = tx * SGAD_TILE;
        const uint32_t cols = ((r.px0 <= bx + 7 && r.px1 >= bx) ? 1u : 0u) |
                              ((r.px0 <= bx + 15 && r.px1 >= bx + 8) ? 2u : 0u);
        if (o < cap) {
          pkeys[o] = (uint32_t)(ty * ntx + tx);
          pvals[o] = packed ? e | ((cols | rows << 2) << LIST_IDX_BITS) : e;
        } else {
          *overflow = 1u;
          if (ext_flag) *ext_flag = 1;
        }
        ++o;
      }
    }
  }
};

// Per-tile list ranges (exclusive scan of K1's per-tile pair counts) and the
// digit histograms of the tile sort's passes -- one block.
__global__ void __launch_bounds__(1024)
k_tile_scan(const uint32_t* __restrict__ tile_count, int n_tiles, int tpasses, uint32_t cap,
            uint2* __restrict__ ranges, uint32_t* __restrict__ hist) {
  __shared__ uint32_t s_wt[32];
  __shared__ uint32_t s_carry;
  __shared__ uint32_t sh[6 << TILE_RB];
  for (int j = threadIdx.x; j < (6 << TILE_RB); j += blockDim.x) sh[j] = 0u;
  if (threadIdx.x == 0) s_carry = 0u;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int b0 = 0; b0 < n_tiles; b0 += 1024) {
    const int t = b0 + (int)threadIdx.x;
    const uint32_t c = t < n_tiles ? tile_count[t] : 0u;
    uint32_t x = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s_wt[w] = x;
    __syncthreads();
    uint32_t before = s_carry;
    for (int i = 0; i < w; ++i) before += s_wt[i];
    const uint32_t start = before + x - c;
    if (t < n_tiles) {
      // (clamped to the capacity: an overflowed view is discarded, never read out of bounds)
      ranges[t] = make_uint2(min(start, cap), min(start + c, cap));
      for (int p = 0; p < tpasses; ++p)
        atomicAdd(&sh[(p << TILE_RB) + (((uint32_t)t >> (TILE_RB * p)) & ((1u << TILE_RB) - 1u))], c);
    }
    __syncthreads();
    if (threadIdx.x == 1023) s_carry = start + c;
    __syncthreads();
  }
  // more pairs than the capacity: the tile sort is skipped (sort.cuh), so the
  // lists hold stale entries -- every tile renders empty and the view is discarded
  if (s_carry > cap)
    for (int t = threadIdx.x; t < n_tiles; t += blockDim.x) ranges[t] = make_uint2(0u, 0u);
  for (int j = threadIdx.x; j < (tpasses << TILE_RB); j += blockDim.x) hist[j] = sh[j];
}

// ------------------------------------------------------------------ K4 / K5 shared
struct TileGeom {
  int tile, tx, ty, warp, lane, px, py;
  bool valid;
};

__device__ __forceinline__ TileGeom tile_geom(int ntx, int width, int height) {
  TileGeom g;
  g.tile = blockIdx.x;
  g.ty = g.tile / ntx;
  g.tx = g.tile - g.ty * ntx;
  g.warp = threadIdx.x >> 5;
  g.lane = threadIdx.x & 31;
  // warp w covers an 8x4 sub-tile: columns (w&1)*8.., rows (w>>1)*4..
  g.px = g.tx * SGAD_TILE + (g.warp & 1) * 8 + (g.lane & 7);
  g.py = g.ty * SGAD_TILE + (g.warp >> 1) * 4 + (g.lane >> 3);
  g.valid = g.px < width && g.py < height;
  return g;
}

// Each warp owns one 8x4 sub-tile and walks the tile's depth-ordered list on
// its own (no block barriers: sub-tiles finish at different list positions).
// Forward (K4):
//   1. lane i reads list value i of a 32-entry chunk (two chunks ahead) and
//      keeps it if its warp-rectangle bits say the entry's 3-sigma box reaches
//      the sub-tile; kept entries queue up in shared memory;
//   2. 32 queued entries at a time, one per lane: the record is loaded and the
//      reference test d2 > 9 s2 evaluated at all 32 pixels (fp32 row
//      intervals outside a guard band, fp64 inside it) -> exact pixel mask;
//   3. entries with pixels fill a window of 33..64 slots (fields staged in
//      shared memory; with state, also appended to the warp's compact list),
//      and two 32x32 bit transposes give each lane (pixel) its 64 bits;
//   4. every lane pops its own bits in list order and composites in fp64.
// Backward (K5): windows are staged from the compact list in reverse into a
// per-warp ring of RING windows, each lane consumes them at its own pace and
// reads the entry's record through L1.  Depth order sweeps across a surface,
// so a pixel's contributors arrive in bursts that differ from lane to lane;
// with one window at a time the warp paid every window's busiest lane (8 of
// 32 lanes busy at C4), with the ring the lanes stay busy (K4/K5).
// A window is staged when a lane has run dry and the slot it needs is no
// longer read by any lane.
constexpr int NWARP = RASTER_THREADS / 32;
constexpr int WIN = 64;
#ifndef SGAD_RING
#define SGAD_RING 10
#endif
constexpr int RING = SGAD_RING;

struct WarpRing {
  uint32_t e[RING][WIN];                  // record index of each slot
  unsigned long long mask[RING][32];      // per-lane bits over the slots
};

// 32x32 bit transpose across the warp: lane i holds row i on entry, column i
// on exit.
__device__ __forceinline__ uint32_t transpose32(uint32_t x, int lane) {
  const uint32_t masks[5] = {0x0000FFFFu, 0x00FF00FFu, 0x0F0F0F0Fu, 0x33333333u, 0x55555555u};
#pragma unroll
  for (int r = 0; r < 5; ++r) {
    const int s = 16 >> r;
    const uint32_t m = masks[r];
    const uint32_t y = __shfl_xor_sync(0xffffffffu, x, s);
    x = (lane & s) ? ((x & ~m) | ((y >> s) & m)) : ((x & m) | ((y << s) & ~m));
  }
  return x;
}

// Pixel mask of one Gaussian over the warp's 8x4 rectangle: bit (ly*8 + lx)
// is set if the reference test d2 > 9 s2 may fail at pixel (xlo+lx, ylo+ly).
// Per row, fp32 gives the column interval of possible passes, grown by a
// guard band of 2e-4 (thr + 1) in d2; the fp32 error is < 1e-6 (thr + 400)
// for any Gaussian that survived the rectangle cull, so no pass is missed
// (K4), and the exact fp64 test is made where d2 is computed.
__device__ __forceinline__ uint32_t col_range(float a, float b) {
  // columns c in [ceil(a), floor(b)] intersected with [0, 7], as an 8-bit mask
  const int lo = max((int)ceilf(a), 0), hi = min((int)floorf(b), 7);
  return lo > hi ? 0u : ((0xFFu >> (7 - hi + lo)) << lo);
}

__device__ __forceinline__ uint32_t pixel_mask(double u0, double v0, double thr, double xlo,
                                               double ylo) {
  // superset of the pixels passing the test: fp32 column intervals grown by
  // the guard band; the compositing loops decide the exact test in fp64 for
  // every bit (they compute d2 anyway), so the mask never drops a pass
  const float ru = (float)(u0 - xlo), rv = (float)(v0 - ylo), thrf = (float)thr;
  const float band = 2e-4f * (thrf + 1.0f);
  uint32_t maybe = 0;
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const float dyf = rv - (float)r;
    const float rem_hi = thrf + band - dyf * dyf;
    if (rem_hi >= 0.0f) {
      const float h_hi = sqrtf(rem_hi) * 1.000001f + 1e-5f;
      maybe |= col_range(ru - h_hi, ru + h_hi) << (8 * r);
    }
  }
  return maybe;
}

// Exact variant for the backward (its contributions are expensive to start,
// so no superset bits): columns between the fp32 intervals of certain and of
// possible passes are decided by the fp64 test.
__device__ __forceinline__ uint32_t pixel_mask_exact(double u0, double v0, double thr, double xlo,
                                                     double ylo) {
  const float ru = (float)(u0 - xlo), rv = (float)(v0 - ylo), thrf = (float)thr;
  const float band = 2e-4f * (thrf + 1.0f);
  uint32_t sure = 0, maybe = 0;
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const float dyf = rv - (float)r;
    const float dy2 = dyf * dyf;
    const float rem_hi = thrf + band - dy2;
    if (rem_hi < 0.0f) continue;
    const float h_hi = sqrtf(rem_hi) * 1.000001f + 1e-5f;
    maybe |= col_range(ru - h_hi, ru + h_hi) << (8 * r);
    const float rem_lo = thrf - band - dy2;
    if (rem_lo > 0.0f) {
      const float h_lo = sqrtf(rem_lo) * 0.999999f - 1e-5f;
      sure |= col_range(ru - h_lo, ru + h_lo) << (8 * r);
    }
  }
  uint32_t unsure = maybe & ~sure;
  while (unsure) {
    const int bit = __ffs(unsure) - 1;
    unsure &= unsure - 1;
    const double dx = SG_SUB(u0, xlo + (bit & 7)), dy = SG_SUB(v0, ylo + (bit >> 3));
    if (!(SG_ADD(SG_MUL(dx, dx), SG_MUL(dy, dy)) > thr)) sure |= 1u << bit;
  }
  return sure;
}

// position of the q-th (0-based) set bit of m (q < popc(m))
__device__ __forceinline__ int nth_set_bit(uint32_t m, int q) {
  int pos = 0, c;
  c = __popc(m & 0xFFFFu);
  if (q >= c) { q -= c; m >>= 16; pos += 16; }
  c = __popc(m & 0xFFu);
  if (q >= c) { q -= c; m >>= 8; pos += 8; }
  c = __popc(m & 0xFu);
  if (q >= c) { q -= c; m >>= 4; pos += 4; }
  c = __popc(m & 0x3u);
  if (q >= c) { q -= c; m >>= 2; pos += 2; }
  if (q >= (int)(m & 1u)) pos += 1;
  return pos;
}

// 32-byte read-only load (one LDG.256: a record is two of them)
__device__ __forceinline__ void ld256(const void* p, double& a, double& b, double& c, double& d) {
  asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
      : "=d"(a), "=d"(b), "=d"(c), "=d"(d)
      : "l"(p));
}

#ifndef FWD_PREFETCH
#define FWD_PREFETCH 2
#endif
// the list value of entry base + lane (0 past the range)
__device__ __forceinline__ uint32_t load_value(const uint32_t* __restrict__ lists, int64_t base,
                                               int64_t hi, int lane) {
  const int64_t k = base + lane;
  return k < hi ? __ldg(lists + k) : 0u;
}

// ---- forward: window-synchronous, entry data staged in shared memory ----
// The forward's per-contribution work is light, so it keeps one window at a
// time with the entries' fields in shared memory (short-latency loads); the
// backward's heavy contributions pay for the ring below (K4/K5).
struct FwdStage {
  double u0[WIN], v0[WIN], nh[WIN], op[WIN], z[WIN], rgb[3][WIN], thr[WIN];
  // cull queue (ring of WIN): record ids of list entries whose 3-sigma box
  // reaches the warp's rectangle, waiting for their pixel masks
  uint32_t qe[WIN];
};

// Per-warp compact lists written by a forward that keeps state for the
// backward: every list entry that reaches the warp's rectangle, in list
// order, with its exact pixel mask -- the backward stages its windows from
// these instead of culling the tile list again.  Warp w of a tile with list
// range [x, y) owns slots [8x + w (y - x), 8x + (w + 1)(y - x)).  A pixel's
// last contributor is kept as its index in this list.
struct CList {
  uint32_t* e;
  uint32_t* m;
  uint32_t* count;  // [n_tiles * 8] entries written per warp
};

__device__ __forceinline__ int64_t clist_base(uint2 rg, int warp) {
  return 8 * (int64_t)rg.x + (int64_t)warp * (int64_t)(rg.y - rg.x);
}

// Pixel masks of up to 32 queued entries (one per lane, all lanes busy),
// staged into window slots n.. in list order; returns how many had pixels.
template <bool EXACT>
__device__ __forceinline__ int stage_from_queue(FwdStage& s, int qh, int take,
                                                const Record* __restrict__ rec,
                                                const double* __restrict__ col64, double xlo,
                                                double ylo, int lane, int n, uint32_t& mlo,
                                                uint32_t& mhi, const CList& cl, int64_t cbase) {
  uint32_t m = 0, e = 0;
  double u0 = 0.0, v0 = 0.0, sig = 0.0, op = 0.0;
  const double2* rp = nullptr;
  if (lane < take) {
    const int qi = (qh + lane) & (WIN - 1);
    e = s.qe[qi];
    rp = reinterpret_cast<const double2*>(rec + e);
    ld256(rp, u0, v0, sig, op);
    const double thr = SG_MUL(9.0, SG_MUL(sig, sig));
    m = EXACT ? pixel_mask_exact(u0, v0, thr, xlo, ylo) : pixel_mask(u0, v0, thr, xlo, ylo);
  }
  const uint32_t keep = __ballot_sync(0xffffffffu, m != 0);
  const int c = __popc(keep);
#ifdef SGAD_K5_COUNT
  if (EXACT && lane == 0) {  // (diagnostics) queued entries vs entries with pixels
    atomicAdd(&g_k5_count[2], (unsigned long long)take);
    atomicAdd(&g_k5_count[3], (unsigned long long)c);
  }
#endif
  if (m) {
    const int j = n + __popc(keep & ((1u << lane) - 1u));
    if (EXACT) {  // the backward's compact list (cbase = this batch's first slot - n)
      cl.e[cbase + j] = e;
      cl.m[cbase + j] = m;
    }
    double zz, nh, rg_, bgid;                                                // z, nh | r, g, b, gid
    ld256(rp + 2, zz, nh, rg_, bgid);
    const double2 zn = make_double2(zz, nh);
    const float2 c01 = *reinterpret_cast<const float2*>(&rg_);
    const float2 c2g = *reinterpret_cast<const float2*>(&bgid);
    const float4 cg = make_float4(c01.x, c01.y, c2g.x, c2g.y);
    if (!EXACT) s.thr[j] = SG_MUL(9.0, SG_MUL(sig, sig));
    s.u0[j] = u0;
    s.v0[j] = v0;
    s.nh[j] = zn.y;
    s.op[j] = op;
    s.z[j] = zn.x;
    if (col64) {  // fp64 drop-in maps keep exact fp64 colours
      s.rgb[0][j] = __ldg(col64 + 3 * (size_t)e);
      s.rgb[1][j] = __ldg(col64 + 3 * (size_t)e + 1);
      s.rgb[2][j] = __ldg(col64 + 3 * (size_t)e + 2);
    } else {
      s.rgb[0][j] = cg.x;
      s.rgb[1][j] = cg.y;
      s.rgb[2][j] = cg.z;
    }
  }
  const int q = (lane - n) & 31;
  const int src = q < c ? nth_set_bit(keep, q) : 0;
  const uint32_t val = __shfl_sync(0xffffffffu, m, src);
  if (q < c) {
    if (n + q < 32) mlo = val; else mhi = val;
  }
  return c;
}

// One contribution's record fields.
struct Contrib {
  double u0, v0, sig, op, z, nh;
  float r, g, b;
  uint32_t gid, e;
  float a_u, a_v, a_z;  // chain coefficients (window backward)
};

// the window backward's 64-byte record (BwdRecord) as two 256-bit loads
__device__ __forceinline__ void load_contrib_bwd(Contrib& q, const WarpRing& rg, int slot, int j,
                                                 const BwdRecord* __restrict__ brec) {
  q.e = rg.e[slot][j];
  const double* rp = reinterpret_cast<const double*>(brec + q.e);
  double r_g, b_au, av_az;
  ld256(rp, q.u0, q.v0, q.op, q.nh);
  ld256(rp + 4, q.z, r_g, b_au, av_az);
  const float2 c = *reinterpret_cast<const float2*>(&r_g);
  const float2 d = *reinterpret_cast<const float2*>(&b_au);
  const float2 e = *reinterpret_cast<const float2*>(&av_az);
  q.r = c.x;
  q.g = c.y;
  q.b = d.x;
  q.a_u = d.y;
  q.a_v = e.x;
  q.a_z = e.y;
}

__device__ __forceinline__ void load_contrib(Contrib& q, const WarpRing& rg, int slot, int j,
                                             const Record* __restrict__ rec) {
  q.e = rg.e[slot][j];
  const double* rp = reinterpret_cast<const double*>(rec + q.e);
  double rg_, bgid;
  ld256(rp, q.u0, q.v0, q.sig, q.op);
  ld256(rp + 4, q.z, q.nh, rg_, bgid);
  const float2 c01 = *reinterpret_cast<const float2*>(&rg_);
  const float2 c2g = *reinterpret_cast<const float2*>(&bgid);
  q.r = c01.x;
  q.g = c01.y;
  q.b = c2g.x;
  q.gid = __float_as_uint(c2g.y);
}

__device__ const double kExp2Table[SGAD_EXP2_TABLE_N] = {SGAD_EXP2_TABLE};

__device__ __forceinline__ void load_exp_table(double* tab) {
  for (int i = threadIdx.x; i < SGAD_EXP2_TABLE_N; i += blockDim.x) tab[i] = kExp2Table[i];
  __syncthreads();
}

// Per-lane ring cursor: the lane's current window (cw) and its remaining bits.
struct Cursor {
  unsigned long long cur;
  int cw;    // window index
  int slot;  // cw % RING, kept incrementally
};

// advance a dry lane to the next staged window that has bits for it
__device__ __forceinline__ void advance(Cursor& c, const WarpRing& rg, int w_head, int lane,
                                        bool done) {
  if (done || c.cur != 0ull) return;
  while (c.cw + 1 < w_head) {
    ++c.cw;
    c.slot = c.slot + 1 == RING ? 0 : c.slot + 1;
    c.cur = rg.mask[c.slot][lane];
    if (c.cur) break;
  }
}

// ------------------------------------------------------------------ K4
// Per-pixel compositing state carried from the forward sweep to the loss
// epilogue (and, in the fused kernel, into the backward sweep).
struct PixState {
  double T, C0, C1, C2, D, A;
  int cnt, last;
};

struct SweepGeom {
  double pxd, pyd, xlo, ylo;
};

__device__ __forceinline__ SweepGeom sweep_geom(const TileGeom& g) {
  SweepGeom q;
  q.pxd = (double)g.px;
  q.pyd = (double)g.py;
  q.xlo = (double)(g.tx * SGAD_TILE + (g.warp & 1) * 8);
  q.ylo = (double)(g.ty * SGAD_TILE + (g.warp >> 1) * 4);
  return q;
}

// rasterizer.py:221-269 for the warp's 8x4 pixels over the tile list rg;
// with EXACT the masks are exact and the warp's compact list is written
template <bool EXACT>
__device__ __forceinline__ PixState fwd_sweep(FwdStage& s, const TileGeom& g, const SweepGeom& q,
                                              uint2 rg, const uint32_t* __restrict__ lists,
                                              int packed, const Record* __restrict__ rec,
                                              const double* __restrict__ col64,
                                              const double* tab, const CList& cl) {
  PixState st{1.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0, -1};
  bool done = !g.valid;
  int64_t pos = rg.x;
  const int64_t cbase = clist_base(rg, g.warp);
  int64_t nw = 0;  // compact entries written so far
  int qh = 0, qn = 0;  // cull queue head and fill (warp-uniform)
  // list-value bits of this warp's rectangle (column g.warp & 1, band g.warp >> 1)
  const uint32_t need =
      packed ? (1u << (LIST_IDX_BITS + (g.warp & 1))) | (1u << (LIST_IDX_BITS + 2 + (g.warp >> 1)))
             : 0u;
  const uint32_t idx_mask = packed ? LIST_IDX_MASK : ~0u;
  uint32_t nx[FWD_PREFETCH];  // list values FWD_PREFETCH chunks ahead
#pragma unroll
  for (int i = 0; i < FWD_PREFETCH; ++i) nx[i] = load_value(lists, pos + 32 * i, rg.y, g.lane);
  while ((pos < (int64_t)rg.y || qn > 0) && !__all_sync(0xffffffffu, done)) {
    int n = 0;
    uint32_t mlo = 0, mhi = 0;
    while (n <= 32) {
      // cull whole chunks into the queue until 32 wait (the masks are then
      // computed with every lane busy)
      while (qn < 32 && pos < (int64_t)rg.y) {
        const uint32_t cur = nx[0];
#pragma unroll
        for (int i = 0; i + 1 < FWD_PREFETCH; ++i) nx[i] = nx[i + 1];
        nx[FWD_PREFETCH - 1] = load_value(lists, pos + 32 * FWD_PREFETCH, rg.y, g.lane);
        const bool hit = pos + g.lane < (int64_t)rg.y && (cur & need) == need;
        const uint32_t b = __ballot_sync(0xffffffffu, hit);
        if (hit) {
          const int qi = (qh + qn + __popc(b & ((1u << g.lane) - 1u))) & (WIN - 1);
          s.qe[qi] = cur & idx_mask;
        }
        qn += __popc(b);
        pos += 32;
      }
      if (qn == 0) break;
      __syncwarp();
      const int take = min(qn, 32);
      n += stage_from_queue<EXACT>(s, qh, take, rec, col64, q.xlo, q.ylo, g.lane, n, mlo, mhi,
                                   cl, cbase + nw);
      qh = (qh + take) & (WIN - 1);
      qn -= take;
      __syncwarp();  // queue slots read above may be refilled next
    }
    const int wbase = (int)nw;  // compact-list index of slot 0
    nw += n;
    __syncwarp();
    // this lane's bits over the window: slots 0..31, then 32..63 (list order)
    uint32_t mine_lo = transpose32(mlo, g.lane), mine_hi = transpose32(mhi, g.lane);
    if (done) mine_lo = mine_hi = 0u;
    int base = 0;
    uint32_t mine = mine_lo;
    while (true) {
      if (!mine) {
        if (base || !mine_hi) break;
        base = 32;
        mine = mine_hi;
      }
      const int j = base + __ffs(mine) - 1;
      mine &= mine - 1;
      const double dx = SG_SUB(s.u0[j], q.pxd), dy = SG_SUB(s.v0[j], q.pyd);
      const double d2 = SG_ADD(SG_MUL(dx, dx), SG_MUL(dy, dy));
      if (!EXACT && d2 > s.thr[j]) continue;  // rasterizer.py:248 (superset masks only;
                                              // exact masks already made this test)
      const double w = sgad_exp_neg(SG_MUL(d2, s.nh[j]), tab);
      double a = SG_MUL(s.op[j], w);
      if (a > SGAD_ALPHA_MAX) a = SGAD_ALPHA_MAX;
      const double at = SG_MUL(a, st.T);
      st.C0 = SG_FMA(s.rgb[0][j], at, st.C0);
      st.C1 = SG_FMA(s.rgb[1][j], at, st.C1);
      st.C2 = SG_FMA(s.rgb[2][j], at, st.C2);
      st.D = SG_FMA(s.z[j], at, st.D);
      st.A = SG_ADD(st.A, at);
      ++st.cnt;
      st.last = wbase + j;
      st.T = SG_MUL(st.T, SG_SUB(1.0, a));
      if (st.T < SGAD_TRANSMITTANCE_MIN) {
        done = true;
        break;
      }
    }
    __syncwarp();
  }
  if (EXACT && g.lane == 0) cl.count[(int64_t)g.tile * NWARP + g.warp] = (uint32_t)nw;
  return st;
}

// mapper.py:118-152 (tau = 0): per-pixel L1 residual signs (2 bits per
// channel) and the warp's |residual| sums added into loss_accum
__device__ __forceinline__ uint8_t loss_epilogue(const PixState& st, const TileGeom& g, int64_t p,
                                                 const sgad_loss_target& tgt) {
  double lc = 0.0, ld = 0.0;
  uint8_t code = 0;
  if (g.valid) {
    const double rc[3] = {SG_SUB(st.C0, (double)tgt.color[3 * p]),
                          SG_SUB(st.C1, (double)tgt.color[3 * p + 1]),
                          SG_SUB(st.C2, (double)tgt.color[3 * p + 2])};
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
      lc += fabs(rc[ch]);
      code |= (uint8_t)((rc[ch] > 0.0 ? 1u : (rc[ch] < 0.0 ? 2u : 0u)) << (2 * ch));
    }
    if (tgt.mask[p]) {
      const double rd = SG_SUB(st.D, (double)tgt.depth[p]);
      ld = fabs(rd);
      code |= (uint8_t)((rd > 0.0 ? 1u : (rd < 0.0 ? 2u : 0u)) << 6);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lc += __shfl_xor_sync(0xffffffffu, lc, o);
    ld += __shfl_xor_sync(0xffffffffu, ld, o);
  }
  if (g.lane == 0) {
    atomicAdd(tgt.loss_accum, lc);
    atomicAdd(tgt.loss_accum + 1, ld);
  }
  return code;
}

#ifndef SGAD_FWD_MINB
#define SGAD_FWD_MINB 4  // 64 registers: 3 blocks/SM 1.10 ms, 5 blocks 1.06 ms, 4 blocks 0.98 ms (C4 view)
#endif
template <bool IMAGES, bool STATE, bool LOSS>
__global__ void __launch_bounds__(RASTER_THREADS, SGAD_FWD_MINB)
k_forward(const uint2* __restrict__ ranges, const uint32_t* __restrict__ lists, int packed,
          const Record* __restrict__ rec, const double* __restrict__ col64, int ntx, int width,
          int height, double* __restrict__ out_color, double* __restrict__ out_depth,
          double* __restrict__ out_alpha, int32_t* __restrict__ out_count,
          double* __restrict__ t_final, int32_t* __restrict__ last_out,
          uint8_t* __restrict__ signs, sgad_loss_target tgt, CList cl) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  FwdStage& s = reinterpret_cast<FwdStage*>(smem_raw)[threadIdx.x >> 5];
  __shared__ double tab[SGAD_EXP2_TABLE_N];
  load_exp_table(tab);
  const TileGeom g = tile_geom(ntx, width, height);
  const SweepGeom q = sweep_geom(g);
  const PixState st = fwd_sweep<STATE>(s, g, q, ranges[g.tile], lists, packed, rec, col64, tab, cl);
  const int64_t p = (int64_t)g.py * width + g.px;
  if (g.valid) {
    if (IMAGES) {
      if (out_color) {
        out_color[3 * p] = st.C0;
        out_color[3 * p + 1] = st.C1;
        out_color[3 * p + 2] = st.C2;
      }
      if (out_depth) out_depth[p] = st.D;
      if (out_alpha) out_alpha[p] = st.A;
      if (out_count) out_count[p] = st.cnt;
    }
    if (STATE) {
      t_final[p] = st.T;
      last_out[p] = st.last;
    }
  }
  if (LOSS) {
    const uint8_t code = loss_epilogue(st, g, p, tgt);
    if (g.valid) signs[p] = code;
  }
}

// ------------------------------------------------------------------ K5
// The exact drop-in backward sums its per-Gaussian fp64 gradients in 128-bit
// fixed point (resolution 2^-100, |sum| < 2^27): integer addition is
// associative, so the sums -- and the map gradients, map_frame's
// trajectories and map files -- are bit-identical run to run whatever order
// the atomics land in (the reference's gradients are deterministic,
// reference tests/test_pipeline.py:76-85).  Each contribution loses at most
// 2^-100 absolute (8e-31: the chain rule multiplies the image-space sums by
// up to fx y / z^2 and subtracts them, so the sums need resolution far below
// the gradients' own ulp); the window engine's fp32 path keeps fp32 atomics.
struct Fx128 {
  unsigned long long lo;
  long long hi;  // value = (hi 2^64 + lo) 2^-100
};

__device__ __forceinline__ void fx_add(Fx128* dst, double x) {
  const double t = x * 0x1p36;  // x 2^36 (exact)
  const double hf = floor(t);
  long long hi = (long long)hf;
  const unsigned long long lo = (unsigned long long)((t - hf) * 18446744073709551616.0);
  if (lo) {
    const unsigned long long old = atomicAdd(&dst->lo, lo);
    if (old + lo < old) ++hi;  // the low word wrapped: carry
  }
  if (hi) atomicAdd(reinterpret_cast<unsigned long long*>(&dst->hi), (unsigned long long)hi);
}

__device__ __forceinline__ double fx_value(const Fx128& v) {
  return (double)v.hi * 0x1p-36 + (double)v.lo * 0x1p-100;
}

struct Upstream {  // fused-loss upstream scales: rho / (3HW), sigma / |U|; camera fx
  double kc, kd;
  float fx;
};

__device__ __forceinline__ double sign_of(uint32_t code) {
  return code == 1u ? 1.0 : (code == 2u ? -1.0 : 0.0);
}

// 1/x: approximate fp32 seed (one MUFU.RCP) + two Newton steps in fp64
// (full fp64 accuracy for x within the fp32 range, a fraction of the IEEE
// division's cost; gradients carry a 1e-3 bar, the exact drop-in backward 1e-9)
__device__ __forceinline__ double fast_rcp(double x) {
  float r32;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r32) : "f"((float)x));
  double r = (double)r32;
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

__device__ __forceinline__ void red_add_v4(float* addr, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "f"(a), "f"(b),
               "f"(c), "f"(d)
               : "memory");
}
__device__ __forceinline__ void red_add_v2(float* addr, float a, float b) {
  asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" ::"l"(addr), "f"(a), "f"(b) : "memory");
}

struct PixUpstream {
  double gc0, gc1, gc2, gd, ga;
  float fx;  // target camera fx (the window backward's radius coefficient)
};

// rasterizer.py:272-363 (+ the fused chain of :462-483) for the warp's
// pixels: reverse sweep from each pixel's last contributor with transmittance
// T_final, walking a ring of windows per warp (K5)
template <bool FUSED>
__device__ __forceinline__ void bwd_sweep(WarpRing& ring, const TileGeom& g, const SweepGeom& q,
                                          uint2 rg, const CList& cl,
                                          const Record* __restrict__ rec,
                                          const BwdRecord* __restrict__ brec,
                                          const double* __restrict__ col64, const double* tab,
                                          const PixUpstream& u, double T, int mylast,
                                          Fx128* __restrict__ raw,
                                          float* __restrict__ grad_accum) {
  int wend = mylast + 1;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) wend = max(wend, __shfl_xor_sync(0xffffffffu, wend, o));
  const bool done = mylast < 0;  // nothing to propagate for this pixel
  double sc0 = 0.0, sc1 = 0.0, sc2 = 0.0, sd = 0.0, sa = 0.0;
  // the warp's compact list (written by the forward): entries [0, cpos) are
  // not staged yet; entries past the warp's last contributor are skipped
  const int64_t cbase = clist_base(rg, g.warp);
  // (plain loads: in k_forward_backward the same kernel wrote them)
  __syncwarp();
  int64_t cpos = (int64_t)cl.count[(int64_t)g.tile * NWARP + g.warp];
  if (cpos > wend) cpos = wend;  // entries past every lane's last contributor
  Cursor c{0ull, -1, RING - 1};
  int w_head = 0, head_slot = 0;  // head_slot = w_head % RING
  Contrib cc;
  while (true) {
    advance(c, ring, w_head, g.lane, done);
    if (cpos > 0 && __any_sync(0xffffffffu, !done && c.cur == 0ull) &&
        !__any_sync(0xffffffffu, !done && c.cw == w_head - RING)) {
      const int slot = head_slot;
      // the next (up to) 64 compact entries below cpos, descending: lane i
      // takes slots i and 32 + i, whose masks are already exact
      const int n = (int)min(cpos, (int64_t)WIN);
      uint32_t mlo = 0, mhi = 0;
      {
        const int64_t i0 = cbase + cpos - 1 - g.lane, i1 = i0 - 32;
        if (g.lane < n) {
          ring.e[slot][g.lane] = cl.e[i0];
          mlo = cl.m[i0];
        }
        if (32 + g.lane < n) {
          ring.e[slot][32 + g.lane] = cl.e[i1];
          mhi = cl.m[i1];
        }
      }
      // slot i holds compact entry cpos - 1 - i (descending): the leading
      // slots above this lane's last contributor are dropped
      const int lo_s = (int)max((int64_t)0, min((int64_t)n, cpos - 1 - (int64_t)mylast));
      cpos -= n;
      __syncwarp();
      unsigned long long bits = ((unsigned long long)transpose32(mhi, g.lane) << 32) |
                                transpose32(mlo, g.lane);
      if (lo_s >= 64) bits = 0ull;
      else bits &= ~((1ull << lo_s) - 1ull);
      ring.mask[slot][g.lane] = done ? 0ull : bits;
      __syncwarp();
      ++w_head;
      head_slot = head_slot + 1 == RING ? 0 : head_slot + 1;
      continue;
    }
    if (!__any_sync(0xffffffffu, c.cur != 0ull)) break;
    if (!c.cur) continue;
    {
      const int j = __ffsll((long long)c.cur) - 1;
      c.cur &= c.cur - 1;
      if (FUSED) load_contrib_bwd(cc, ring, c.slot, j, brec);
      else load_contrib(cc, ring, c.slot, j, rec);
    }
    {
      const uint32_t e = cc.e;
      const double dx = SG_SUB(cc.u0, q.pxd), dy = SG_SUB(cc.v0, q.pyd);
      const double d2 = SG_ADD(SG_MUL(dx, dx), SG_MUL(dy, dy));
      const double nh = cc.nh, op = cc.op, z = cc.z;
      const double w = sgad_exp_neg(SG_MUL(d2, nh), tab);
      const double aw = SG_MUL(op, w);
      const bool clamped = aw > SGAD_ALPHA_MAX;
      const double a = clamped ? SGAD_ALPHA_MAX : aw;
      const double iom = fast_rcp(1.0 - a);
      const double tb = T * iom;
      const double at = a * tb;
      double c0 = cc.r, c1 = cc.g, c2 = cc.b;
      if (col64) {
        c0 = __ldg(col64 + 3 * (size_t)e);
        c1 = __ldg(col64 + 3 * (size_t)e + 1);
        c2 = __ldg(col64 + 3 * (size_t)e + 2);
      }
      if (FUSED || (cc.gid & GID_LEARN)) {  // (the window: every Gaussian learnable)
        // (the fused loss has no alpha upstream: its term is compiled out)
        double d_alpha = u.gc0 * (c0 * tb - sc0 * iom) + u.gc1 * (c1 * tb - sc1 * iom) +
                         u.gc2 * (c2 * tb - sc2 * iom) + u.gd * (z * tb - sd * iom);
        if (!FUSED) d_alpha += u.ga * (tb - sa * iom);
        const double gcol0 = u.gc0 * at, gcol1 = u.gc1 * at, gcol2 = u.gc2 * at, gz = u.gd * at;
        double gop = 0.0, gsig = 0.0, gu = 0.0, gv = 0.0;
        if (!clamped) {
          const double gw = d_alpha * op;
          gop = d_alpha * w;
          // gw w d2 / (s2 sigma) = gw w d2 (-2 nh) / sigma: the fused path
          // keeps sigma g_sigma (its coefficients carry the 1 / sigma)
          gsig = gw * w * d2 * (-2.0 * nh);
          if (!FUSED) gsig *= fast_rcp(cc.sig);
          const double gd2 = gw * w * nh;  // gw (-0.5 w / s2)
          gu = 2.0 * gd2 * dx;
          gv = 2.0 * gd2 * dy;
        }
        if (FUSED) {
          // rasterizer.py:462-483 with this view's coefficients: window
          // gradients (delta, radius, logit, R, G, B) straight into grad_accum
          // (gsig holds sigma g_sigma)
          const float gs = (float)gsig, iz = __frcp_rn((float)z);
          const float g_delta = cc.a_u * (float)gu + cc.a_v * (float)gv + cc.a_z * (float)gz -
                                cc.a_z * iz * gs;
          const float g_radius = u.fx * sqrtf(-2.0f * (float)nh) * iz * gs;
          float* dst = grad_accum + (size_t)e * 8;
#ifdef SGAD_K5_COUNT
          {  // (diagnostics) contributions and distinct entries per warp iteration
            const unsigned act = __activemask(), grp = __match_any_sync(act, e);
            const int ln = threadIdx.x & 31;
            if (ln == __ffs(act) - 1) atomicAdd(&g_k5_count[0], (unsigned long long)__popc(act));
            if (ln == __ffs(grp) - 1) atomicAdd(&g_k5_count[1], 1ull);
          }
#endif
          red_add_v4(dst, g_delta, g_radius, (float)(op * (1.0 - op) * gop), (float)gcol0);
          red_add_v2(dst + 4, (float)gcol1, (float)gcol2);
        } else {
          Fx128* dst = raw + (size_t)e * 8;
          fx_add(dst + 0, gcol0);
          fx_add(dst + 1, gcol1);
          fx_add(dst + 2, gcol2);
          fx_add(dst + 3, gop);
          fx_add(dst + 4, gu);
          fx_add(dst + 5, gv);
          fx_add(dst + 6, gsig);
          fx_add(dst + 7, gz);
        }
      }
      sc0 = fma(c0, at, sc0);
      sc1 = fma(c1, at, sc1);
      sc2 = fma(c2, at, sc2);
      sd = fma(z, at, sd);
      if (!FUSED) sa += at;
      T = tb;
    }
  }
}

__device__ __forceinline__ PixUpstream fused_upstream(uint32_t code, const double* g_color,
                                                      int64_t p, const Upstream& up) {
  // mapper.py:145-152: rho * sign / n_color; sigma * sign * mask / n_depth
  PixUpstream u;
  if (g_color) {  // tau != 0: colour upstream with the SSIM term (sgad_ssim)
    u.gc0 = g_color[3 * p];
    u.gc1 = g_color[3 * p + 1];
    u.gc2 = g_color[3 * p + 2];
  } else {
    u.gc0 = SG_MUL(up.kc, sign_of(code & 3u));
    u.gc1 = SG_MUL(up.kc, sign_of((code >> 2) & 3u));
    u.gc2 = SG_MUL(up.kc, sign_of((code >> 4) & 3u));
  }
  u.gd = SG_MUL(up.kd, sign_of((code >> 6) & 3u));
  u.ga = 0.0;
  u.fx = up.fx;
  return u;
}

__device__ __forceinline__ bool any_upstream(const PixUpstream& u) {
  return !(u.gc0 == 0.0 && u.gc1 == 0.0 && u.gc2 == 0.0 && u.gd == 0.0 && u.ga == 0.0);
}

template <bool FUSED>
__global__ void __launch_bounds__(RASTER_THREADS)
k_backward(const uint2* __restrict__ ranges, const uint32_t* __restrict__ lists,
           const Record* __restrict__ rec, const BwdRecord* __restrict__ coef,
           const double* __restrict__ col64, int ntx, int width, int height,
           const double* __restrict__ t_final, const int32_t* __restrict__ last_idx,
           const uint8_t* __restrict__ signs, Upstream up, const double* __restrict__ g_color,
           const double* __restrict__ g_depth, const double* __restrict__ g_alpha,
           Fx128* __restrict__ raw, float* __restrict__ grad_accum, CList cl) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  WarpRing& ring = reinterpret_cast<WarpRing*>(smem_raw)[threadIdx.x >> 5];
  __shared__ double tab[SGAD_EXP2_TABLE_N];
  load_exp_table(tab);
  const TileGeom g = tile_geom(ntx, width, height);
  const SweepGeom q = sweep_geom(g);
  const int64_t p = (int64_t)g.py * width + g.px;
  PixUpstream u{0.0, 0.0, 0.0, 0.0, 0.0, 0.0f};
  double T = 0.0;
  int mylast = -1;
  if (g.valid) {
    if (FUSED) {
      u = fused_upstream(signs[p], g_color, p, up);
    } else {
      u.gc0 = g_color[3 * p];
      u.gc1 = g_color[3 * p + 1];
      u.gc2 = g_color[3 * p + 2];
      u.gd = g_depth[p];
      u.ga = g_alpha[p];
    }
    if (any_upstream(u)) {
      mylast = last_idx[p];
      T = t_final[p];
    }
  }
  bwd_sweep<FUSED>(ring, g, q, ranges[g.tile], cl, rec, coef, col64, tab, u, T, mylast,
                         raw, grad_accum);
}

// K4+K5 fused (tau = 0 window step): the tile's forward sweep, the L1 loss
// epilogue, then its backward sweep from the state still in registers --
// no per-pixel state round trip through HBM, and the tile's list entries and
// records are re-read while still in L2.  Each warp's shared memory holds
// first its forward staging window, then its backward ring.
constexpr size_t FB_SLAB = sizeof(WarpRing) > sizeof(FwdStage) ? sizeof(WarpRing)
                                                                : sizeof(FwdStage);

__global__ void __launch_bounds__(RASTER_THREADS)
k_forward_backward(const uint2* __restrict__ ranges, const uint32_t* __restrict__ lists,
                   int packed, const Record* __restrict__ rec, const BwdRecord* __restrict__ coef, int ntx,
                   int width, int height, sgad_loss_target tgt, Upstream up,
                   float* __restrict__ grad_accum, CList cl) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  unsigned char* slab = smem_raw + FB_SLAB * (threadIdx.x >> 5);
  __shared__ double tab[SGAD_EXP2_TABLE_N];
  load_exp_table(tab);
  const TileGeom g = tile_geom(ntx, width, height);
  const SweepGeom q = sweep_geom(g);
  const uint2 rg = ranges[g.tile];
  const PixState st = fwd_sweep<true>(*reinterpret_cast<FwdStage*>(slab), g, q, rg, lists, packed, rec,
                                      nullptr, tab, cl);
  const int64_t p = (int64_t)g.py * width + g.px;
  const uint8_t code = loss_epilogue(st, g, p, tgt);
  __syncwarp();
  PixUpstream u{0.0, 0.0, 0.0, 0.0, 0.0, 0.0f};
  int mylast = -1;
  if (g.valid) {
    u = fused_upstream(code, nullptr, p, up);
    if (any_upstream(u)) mylast = st.last;
  }
  bwd_sweep<true>(*reinterpret_cast<WarpRing*>(slab), g, q, rg, cl, rec, coef, nullptr, tab, u,
                  st.T, mylast, nullptr, grad_accum);
}

// Exact-mode chain rule (rasterizer.py:462-483) from per-survivor fp64 sums.
__global__ void k_chain_exact(const Record* __restrict__ rec, const Fx128* __restrict__ raw,
                              const uint32_t* __restrict__ perm, uint32_t n_surv,
                              const sgad_frame* __restrict__ frames, int n_frames,
                              sgad_camera cam, double* const* __restrict__ map_grads) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_surv) return;
  const uint32_t e = perm[i];
  const uint32_t gidw = rec[e].gid;
  if (!(gidw & GID_LEARN)) return;
  const uint32_t gid = gidw & ~GID_LEARN;
  const int fi = find_frame(frames, n_frames, gid);
  double* out = map_grads[fi];
  if (!out) return;
  const sgad_frame& f = frames[fi];
  const int64_t hw = (int64_t)f.height * f.width;
  const int64_t p = (int64_t)gid - f.gauss_offset;
  Proj o;
  project_point(f, p, load_params(f, p, hw), cam, o);
  const Fx128* rf = raw + (size_t)e * 8;
  double rg[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) rg[k] = fx_value(rf[k]);
  const double g_op = rg[3], g_u0 = rg[4], g_v0 = rg[5], g_sig = rg[6], g_z = rg[7];
  const double z = o.z, z2 = SG_MUL(z, z);
  const double g_radius = SG_DIV(SG_MUL(g_sig, cam.fx), z);
  double g_zt = SG_SUB(g_z, SG_DIV(SG_MUL(g_sig, o.sig), z));
  g_zt = SG_SUB(g_zt, SG_DIV(SG_MUL(SG_MUL(g_u0, cam.fx), o.y[0]), z2));
  g_zt = SG_SUB(g_zt, SG_DIV(SG_MUL(SG_MUL(g_v0, cam.fy), o.y[1]), z2));
  const double g_y0 = SG_DIV(SG_MUL(g_u0, cam.fx), z);
  const double g_y1 = SG_DIV(SG_MUL(g_v0, cam.fy), z);
  const double g_dadj =
      SG_ADD(SG_ADD(SG_MUL(g_y0, o.dir[0]), SG_MUL(g_y1, o.dir[1])), SG_MUL(g_zt, o.dir[2]));
  const double sgn = o.bd >= 0.0 ? 1.0 : -1.0;
  out[p] += SG_MUL(g_dadj, sgn);
  out[hw + p] += g_radius;
  out[2 * hw + p] += SG_MUL(SG_MUL(g_op, o.op), SG_SUB(1.0, o.op));
  out[3 * hw + p] += rg[0];
  out[4 * hw + p] += rg[1];
  out[5 * hw + p] += rg[2];
}

__global__ void k_rank_of(const uint32_t* __restrict__ perm, uint32_t n, uint32_t* __restrict__ rank) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) rank[perm[i]] = i;
}

__global__ void k_export_lists(const uint32_t* __restrict__ pvals, const uint32_t* __restrict__ rank,
                               uint32_t n, uint32_t idx_mask, int64_t* __restrict__ out) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = rank[pvals[i] & idx_mask];
}

__global__ void k_export_ranges(const uint2* __restrict__ r, int n, int64_t* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    out[2 * i] = r[i].x;
    out[2 * i + 1] = r[i].y;
  }
}

__global__ void k_export_surv(const uint32_t* __restrict__ perm, const Record* __restrict__ rec,
                              uint32_t n, int64_t* gid, double* u0, double* v0, double* z,
                              double* sigma, double* opacity) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const Record& r = rec[perm[i]];
  if (gid) gid[i] = r.gid & ~GID_LEARN;
  if (u0) u0[i] = r.u0;
  if (v0) v0[i] = r.v0;
  if (z) z[i] = r.z;
  if (sigma) sigma[i] = r.sigma;
  if (opacity) opacity[i] = r.opacity;
}

constexpr size_t FWD_SMEM = sizeof(FwdStage) * NWARP;
constexpr size_t FB_SMEM = FB_SLAB * NWARP;
constexpr size_t BWD_SMEM = sizeof(WarpRing) * NWARP;

constexpr size_t LONG_RUN_SMEM = (sizeof(unsigned long long) + sizeof(uint32_t)) * LONG_RUN_SMEM_N;

// opt in to >48 KB dynamic shared memory once per process
static int smem_attrs() {
  static int done = 0;
  if (done) return SGAD_OK;
  SGAD_CHECK_CUDA(cudaFuncSetAttribute(k_forward<true, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)FWD_SMEM));
  SGAD_CHECK_CUDA(cudaFuncSetAttribute(k_forward<true, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)FWD_SMEM));
  SGAD_CHECK_CUDA(cudaFuncSetAttribute(k_forward<true, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)FWD_SMEM));
  SGAD_CHECK_CUDA(cudaFuncSetAttribute(k_forward<false, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)FWD_SMEM));
  SGAD_CHECK_CUDA(cudaFuncSetAttribute(k_forward<false, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)FWD_SMEM));
  SGAD_CHECK_CUDA(cudaFuncSetAttribute(k_backward<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)BWD_SMEM));
  SGAD_CHECK_CUDA(cudaFuncSetAttribute(k_backward<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)BWD_SMEM));
  SGAD_CHECK_CUDA(cudaFuncSetAttribute(k_forward_backward, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)FB_SMEM));
  SGAD_CHECK_CUDA(cudaFuncSetAttribute(k_long_runs, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)LONG_RUN_SMEM));
  done = 1;
  return SGAD_OK;
}

static inline unsigned blocks_for(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

static int bits_for(uint32_t maxval) {
  int b = 1;
  while (b < 32 && (maxval >> b) != 0) ++b;
  return b;
}

}  // namespace sgad

using namespace sgad;

// the per-warp compact lists of the prepared view (sized at the forward)
static int ensure_clist(sgad_raster* h) {
  const size_t n = 8 * (size_t)(h->cap_pairs > 0 ? h->cap_pairs : 1);
  SGAD_CHECK_CUDA(h->cl_e.ensure(sizeof(uint32_t) * n));
  SGAD_CHECK_CUDA(h->cl_m.ensure(sizeof(uint32_t) * n));
  SGAD_CHECK_CUDA(h->cl_n.ensure(sizeof(uint32_t) * 8 * (size_t)(h->n_tiles > 0 ? h->n_tiles : 1)));
  return SGAD_OK;
}

static CList clist_of(sgad_raster* h) {
  return CList{h->cl_e.as<uint32_t>(), h->cl_m.as<uint32_t>(),
               h->cl_n.as<uint32_t>()};
}

extern "C" {

const char* sgad_last_error(void) { return g_err; }
int sgad_version(void) { return 1; }

int sgad_launch_count(int64_t* out) {
  SGAD_REQUIRE(out != nullptr, "sgad_launch_count: null out");
  *out = (int64_t)g_launches.load(std::memory_order_relaxed);
  return SGAD_OK;
}

int sgad_raster_create(sgad_raster** out) {
  SGAD_REQUIRE(out != nullptr, "sgad_raster_create: null out");
  sgad_raster* h = new sgad_raster();
  cudaError_t e = cudaMallocHost(&h->pinned, 16 * sizeof(uint32_t));
  if (e != cudaSuccess) {
    delete h;
    set_error("cudaMallocHost: %s", cudaGetErrorString(e));
    return SGAD_E_CUDA;
  }
  *out = h;
  return SGAD_OK;
}

int sgad_raster_destroy(sgad_raster* h) {
  if (!h) return SGAD_OK;
  DevBuf* bufs[] = {&h->frames, &h->counters, &h->records, &h->coef, &h->keys0, &h->keys1,
                    &h->vals0, &h->vals1, &h->pkeys0, &h->pkeys1, &h->pvals0,
                    &h->pvals1, &h->ranges, &h->sortws, &h->pairws, &h->trans_final, &h->last_idx, &h->signs,
                    &h->raw_grads, &h->rank_of, &h->scratch, &h->col64, &h->zrange, &h->k32a,
                    &h->k32b, &h->bbox, &h->runs, &h->cl_e, &h->cl_m, &h->cl_n};
  for (DevBuf* b : bufs) b->release();
  if (h->pinned) cudaFreeHost(h->pinned);
  delete h;
  return SGAD_OK;
}

int sgad_raster_tile_count(sgad_raster* h, int64_t* n_tiles) {
  SGAD_REQUIRE(h && n_tiles, "sgad_raster_tile_count: null argument");
  *n_tiles = h->n_tiles;
  return SGAD_OK;
}

// ---- preparation (K1-K3), all on the stream, element counts on the device
//
// Workspaces: h->sortws (zeroed once per preparation) and h->pairws (zeroed
// before every binning attempt; resized when the pair capacity grows).
//   sortws: [0, 16) partition counters (depth passes 0..7, pair emit 8, tile
//           passes 9..15), depth_hist[dpasses][256], tile_count[n_tiles],
//           claim bitmap[n_total / 32 + 1], depth_status[dpasses][parts(n_total)][256]
//   pairws: tile_hist[tpasses][64], emit_status[parts(n_total)],
//           tile_status[tpasses][parts(cap_pairs)][64]
struct PrepWs {
  uint32_t* ctr;
  uint32_t* dhist;
  uint32_t* tcount;
  uint32_t* claim;
  uint32_t* dstat;
  size_t words;
};

struct PairWs {
  uint32_t* thist;
  uint32_t* sstat;
  uint32_t* tstat;
  size_t words;
};

static PrepWs prep_layout(uint32_t* base, int dpasses, uint32_t n_total, uint32_t n_tiles) {
  PrepWs w{};
  size_t o = 0;
  w.ctr = base + o;
  o += 16;
  w.dhist = base + o;
  o += (size_t)dpasses * 256;
  w.tcount = base + o;
  o += n_tiles;
  w.claim = base + o;
  o += n_total / 32 + 1;
  w.dstat = base + o;
  o += (size_t)dpasses * os_parts(n_total) * 256;
  w.words = o;
  return w;
}

static PairWs pair_layout(uint32_t* base, int tpasses, uint32_t n_total, uint32_t cap) {
  PairWs w{};
  size_t o = 0;
  w.thist = base + o;
  o += (size_t)tpasses * (1u << TILE_RB);
  w.sstat = base + o;
  o += os_parts(n_total);
  w.tstat = base + o;
  o += (size_t)tpasses * os_parts(cap) * (1u << TILE_RB);
  w.words = o;
  return w;
}

static int ensure_pair_buffers(sgad_raster* h) {
  const size_t n = (size_t)h->cap_pairs + 1;
  SGAD_CHECK_CUDA(h->pkeys0.ensure(sizeof(uint32_t) * n));
  SGAD_CHECK_CUDA(h->pkeys1.ensure(sizeof(uint32_t) * n));
  SGAD_CHECK_CUDA(h->pvals0.ensure(sizeof(uint32_t) * n));
  SGAD_CHECK_CUDA(h->pvals1.ensure(sizeof(uint32_t) * n));
  return SGAD_OK;
}

// K1 + K2 + the pair-count scan: independent of the pair capacity
static int prepare_front(sgad_raster* h, const sgad_frame* frames, int32_t n_frames,
                         const sgad_camera* cam, int32_t want_coef, const sgad_frame* frames_dev,
                         cudaStream_t st) {
  SGAD_REQUIRE(h && cam && n_frames >= 0 && (n_frames == 0 || frames), "sgad_raster_prepare: bad args");
  SGAD_REQUIRE(cam->width > 0 && cam->height > 0, "sgad_raster_prepare: empty camera");
  if (int rc = smem_attrs()) return rc;
  h->prepared = h->forwarded = h->fused_ready = 0;
  h->cam = *cam;
  h->ntx = (cam->width + SGAD_TILE - 1) / SGAD_TILE;
  h->nty = (cam->height + SGAD_TILE - 1) / SGAD_TILE;
  h->n_tiles = h->ntx * h->nty;
  SGAD_REQUIRE(h->ntx <= 65535 && h->nty <= 65535, "image too large");
  h->host_frames.assign(frames, frames + n_frames);
  int64_t n_total = 0, max_hw = 0;
  for (int i = 0; i < n_frames; ++i) {
    SGAD_REQUIRE(frames[i].gauss_offset == n_total, "frames must be packed: gauss_offset[%d]", i);
    const int64_t hw = (int64_t)frames[i].height * frames[i].width;
    n_total += hw;
    max_hw = hw > max_hw ? hw : max_hw;
  }
  SGAD_REQUIRE(n_total < (1ll << 30), "too many Gaussians (%lld)", (long long)n_total);
  h->n_total = n_total;
  // (SGAD_PACK=0 forces the bare-index lists of very large views: tests)
  const char* pack_env = getenv("SGAD_PACK");
  h->packed = n_total < (int64_t)(1u << sgad::LIST_IDX_BITS) && !(pack_env && pack_env[0] == '0')
                  ? 1 : 0;
  h->have_coef = want_coef != 0;
  h->any_f64 = 0;
  for (int i = 0; i < n_frames; ++i) h->any_f64 |= frames[i].planes_f64 ? 1 : 0;
  h->kbits = depth_key_bits();
  h->dpasses = (h->kbits + 7) / 8;
  h->tpasses = (bits_for((uint32_t)(h->n_tiles > 1 ? h->n_tiles - 1 : 1)) + TILE_RB - 1) / TILE_RB;
  SGAD_REQUIRE(h->tpasses <= 6, "too many tiles");
  // pair capacity: at least 2 x Gaussians (C4: 1.6 pairs per survivor); a
  // synchronous prepare grows it on overflow, the window engine reserves it
  if (h->cap_pairs < 2 * n_total + 4096) h->cap_pairs = 2 * n_total + 4096;
  SGAD_REQUIRE(h->cap_pairs < (1ll << 30), "too many tile pairs");
  const int64_t nt = h->n_tiles;
  SGAD_CHECK_CUDA(h->ranges.ensure(sizeof(uint2) * nt));
  SGAD_CHECK_CUDA(h->counters.ensure(sizeof(uint32_t) * 8));
  SGAD_CHECK_CUDA(cudaMemsetAsync(h->ranges.p, 0, sizeof(uint2) * nt, st));
  SGAD_CHECK_CUDA(cudaMemsetAsync(h->counters.p, 0, sizeof(uint32_t) * 8, st));
  h->prepared = 1;
  if (n_total == 0) return SGAD_OK;
  const uint32_t ntot = (uint32_t)n_total;
  if (!frames_dev) SGAD_CHECK_CUDA(h->frames.ensure(sizeof(sgad_frame) * n_frames));
  SGAD_CHECK_CUDA(h->records.ensure(sizeof(Record) * n_total));
  SGAD_CHECK_CUDA(h->bbox.ensure(sizeof(TileBox) * n_total));
  if (want_coef) SGAD_CHECK_CUDA(h->coef.ensure(sizeof(BwdRecord) * n_total));
  if (h->any_f64) SGAD_CHECK_CUDA(h->col64.ensure(sizeof(double) * 3 * n_total));
  SGAD_CHECK_CUDA(h->keys0.ensure(sizeof(unsigned long long) * n_total));
  SGAD_CHECK_CUDA(h->keys1.ensure(sizeof(unsigned long long) * n_total));
  SGAD_CHECK_CUDA(h->vals0.ensure(sizeof(uint32_t) * n_total));
  SGAD_CHECK_CUDA(h->vals1.ensure(sizeof(uint32_t) * n_total));
  SGAD_CHECK_CUDA(h->k32a.ensure(sizeof(uint32_t) * n_total));
  SGAD_CHECK_CUDA(h->k32b.ensure(sizeof(uint32_t) * n_total));
  SGAD_CHECK_CUDA(h->runs.ensure(sizeof(uint2) * (n_total / 65 + 1)));
  if (int rc = ensure_pair_buffers(h)) return rc;
  PrepWs w = prep_layout(nullptr, h->dpasses, ntot, (uint32_t)h->n_tiles);
  SGAD_CHECK_CUDA(h->sortws.ensure(sizeof(uint32_t) * w.words));
  w = prep_layout(h->sortws.as<uint32_t>(), h->dpasses, ntot, (uint32_t)h->n_tiles);
  SGAD_CHECK_CUDA(cudaMemsetAsync(w.ctr, 0, sizeof(uint32_t) * w.words, st));
  // the frame table: the caller's device copy (resident: a step captured in a
  // CUDA graph), or uploaded here
  const sgad_frame* dframes = frames_dev;
  if (!dframes) {
    SGAD_CHECK_CUDA(cudaMemcpyAsync(h->frames.p, frames, sizeof(sgad_frame) * n_frames,
                                    cudaMemcpyHostToDevice, st));
    dframes = h->frames.as<sgad_frame>();
  }
  SGAD_CHECK_CUDA(h->zrange.ensure(sizeof(unsigned long long) * 2));
  SGAD_CHECK_CUDA(cudaMemsetAsync(h->zrange.p, 0xff, sizeof(unsigned long long), st));
  SGAD_CHECK_CUDA(cudaMemsetAsync(h->zrange.as<unsigned long long>() + 1, 0, sizeof(unsigned long long), st));
  uint32_t* cnt = h->counters.as<uint32_t>();
  const unsigned long long* zkeys = h->keys0.as<unsigned long long>();
  const unsigned long long* zr = h->zrange.as<unsigned long long>();
  // K1
  const dim3 pgrid((unsigned)((max_hw + PROJ_THREADS - 1) / PROJ_THREADS), (unsigned)n_frames);
  k_project<<<pgrid, PROJ_THREADS, 0, st>>>(
      dframes, *cam, h->ntx, h->nty, want_coef, h->records.as<Record>(),
      h->bbox.as<TileBox>(), h->coef.as<BwdRecord>(), h->any_f64 ? h->col64.as<double>() : nullptr,
      h->keys0.as<unsigned long long>(), cnt, h->zrange.as<unsigned long long>(), w.tcount);
  SGAD_LAUNCH_CHECK();
  // K2: digit histograms, onesweep passes (the permutation lands in vals0
  // and the sorted buckets in k32a), run fix-up
  const unsigned hist_grid = (unsigned)std::min<int64_t>(148 * 8, (n_total + 255) / 256);
  switch (h->dpasses) {
    case 2: k_depth_hist<2><<<hist_grid, 256, 0, st>>>(zkeys, ntot, zr, h->kbits, w.dhist); break;
    case 3: k_depth_hist<3><<<hist_grid, 256, 0, st>>>(zkeys, ntot, zr, h->kbits, w.dhist); break;
    default: k_depth_hist<4><<<hist_grid, 256, 0, st>>>(zkeys, ntot, zr, h->kbits, w.dhist); break;
  }
  SGAD_LAUNCH_CHECK();
  const unsigned dparts = os_parts(ntot);
  uint32_t* kb[2] = {h->k32a.as<uint32_t>(), h->k32b.as<uint32_t>()};
  uint32_t* vb[2] = {h->vals0.as<uint32_t>(), h->vals1.as<uint32_t>()};
  int cur = (h->dpasses & 1) ? 0 : 1;  // the last pass writes buffer 0
  for (int pss = 0; pss < h->dpasses; ++pss) {
    uint32_t* st_p = w.dstat + (size_t)pss * dparts * 256;
    if (pss == 0) {
      k_onesweep<8, 1><<<dparts, OS_THREADS, 0, st>>>(
          nullptr, nullptr, zkeys, zr, h->kbits, ntot, nullptr, kb[cur], vb[cur], w.dhist,
          st_p, w.ctr + pss, 0);
    } else {
      k_onesweep<8, 0><<<dparts, OS_THREADS, 0, st>>>(
          kb[cur ^ 1], vb[cur ^ 1], nullptr, nullptr, h->kbits, ntot, cnt + C_NSURV, kb[cur],
          vb[cur], w.dhist + 256 * pss, st_p, w.ctr + pss, 8 * pss);
    }
    SGAD_LAUNCH_CHECK();
    cur ^= 1;
  }
  uint32_t* perm = h->vals0.as<uint32_t>();
  k_depth_fixup<<<blocks_for(n_total, 256), 256, 0, st>>>(
      h->k32a.as<uint32_t>(), cnt + C_NSURV, zkeys, perm, w.claim, cnt + C_NLONG,
      h->runs.as<uint2>());
  SGAD_LAUNCH_CHECK();
  k_long_runs<<<2 * 148, 1024, LONG_RUN_SMEM, st>>>(h->runs.as<uint2>(), cnt + C_NLONG, zkeys, perm,
                                                h->keys1.as<unsigned long long>(),
                                                h->vals1.as<uint32_t>());
  SGAD_LAUNCH_CHECK();
  return SGAD_OK;
}

// K3: pair counts in depth order -> offsets (look-back scan) and the
// (tile, value) pairs at their offsets, stable tile sort, per-tile ranges.
// The pair region of the workspace is zeroed here (a retry after an
// overflow re-runs only this part).
static int prepare_pairs(sgad_raster* h, int32_t* ext_flag, cudaStream_t st) {
  if (h->n_total == 0) return SGAD_OK;
  const uint32_t ntot = (uint32_t)h->n_total, cap = (uint32_t)h->cap_pairs;
  if (int rc = ensure_pair_buffers(h)) return rc;
  const PrepWs w = prep_layout(h->sortws.as<uint32_t>(), h->dpasses, ntot, (uint32_t)h->n_tiles);
  PairWs pw = pair_layout(nullptr, h->tpasses, ntot, cap);
  SGAD_CHECK_CUDA(h->pairws.ensure(sizeof(uint32_t) * pw.words));
  pw = pair_layout(h->pairws.as<uint32_t>(), h->tpasses, ntot, cap);
  uint32_t* cnt = h->counters.as<uint32_t>();
  SGAD_CHECK_CUDA(cudaMemsetAsync(w.ctr + 8, 0, sizeof(uint32_t) * 8, st));
  SGAD_CHECK_CUDA(cudaMemsetAsync(pw.thist, 0, sizeof(uint32_t) * pw.words, st));
  SGAD_CHECK_CUDA(cudaMemsetAsync(cnt + C_OVERFLOW, 0, sizeof(uint32_t), st));
  k_tile_scan<<<1, 1024, 0, st>>>(w.tcount, h->n_tiles, h->tpasses, cap, h->ranges.as<uint2>(),
                                  pw.thist);
  SGAD_LAUNCH_CHECK();
  uint32_t* kb[2] = {h->pkeys0.as<uint32_t>(), h->pkeys1.as<uint32_t>()};
  uint32_t* vb[2] = {h->pvals0.as<uint32_t>(), h->pvals1.as<uint32_t>()};
  int cur = (h->tpasses & 1) ? 1 : 0;  // emit here; the last pass lands in buffer 0
  const uint32_t* perm = h->vals0.as<uint32_t>();
  const unsigned dparts = os_parts(ntot);
  k_pair_emit<TileBox, TileEmit><<<dparts, OS_THREADS, 0, st>>>(
      perm, h->bbox.as<TileBox>(), cnt + C_NSURV, ntot, pw.sstat, w.ctr + 8, cnt + C_NPAIRS,
      TileEmit{h->ntx, h->packed, cap, kb[cur], vb[cur], cnt + C_OVERFLOW, ext_flag});
  SGAD_LAUNCH_CHECK();
  const unsigned tparts = os_parts(cap);
  for (int pss = 0; pss < h->tpasses; ++pss) {
    k_onesweep<TILE_RB, 0><<<tparts, OS_THREADS, 0, st>>>(
        kb[cur], vb[cur], nullptr, nullptr, 0, cap, cnt + C_NPAIRS, kb[cur ^ 1], vb[cur ^ 1],
        pw.thist + (1u << TILE_RB) * pss, pw.tstat + (size_t)pss * tparts * (1u << TILE_RB),
        w.ctr + 9 + pss, TILE_RB * pss);
    SGAD_LAUNCH_CHECK();
    cur ^= 1;
  }
  return SGAD_OK;
}

int sgad_raster_prepare(sgad_raster* h, const sgad_frame* frames, int32_t n_frames,
                        const sgad_camera* cam, int32_t want_coef, void* stream_,
                        int64_t* n_survivors, int64_t* n_pairs) {
  cudaStream_t st = (cudaStream_t)stream_;
  if (int rc = prepare_front(h, frames, n_frames, cam, want_coef, nullptr, st)) return rc;
  if (int rc = prepare_pairs(h, nullptr, st)) return rc;
  h->n_surv = h->n_pairs = 0;
  if (h->n_total > 0) {
    for (int attempt = 0; attempt < 2; ++attempt) {
      SGAD_CHECK_CUDA(cudaMemcpyAsync(h->pinned, h->counters.p, sizeof(uint32_t) * 8,
                                      cudaMemcpyDeviceToHost, st));
      SGAD_CHECK_CUDA(cudaStreamSynchronize(st));
      h->n_surv = h->pinned[C_NSURV];
      h->n_pairs = h->pinned[C_NPAIRS];
      if (h->n_pairs <= h->cap_pairs) break;
      SGAD_REQUIRE(attempt == 0, "sgad_raster_prepare: pair capacity");
      h->cap_pairs = h->n_pairs + h->n_pairs / 4 + 4096;  // grow and bin again
      SGAD_REQUIRE(h->cap_pairs < (1ll << 30), "too many tile pairs (%lld)", (long long)h->n_pairs);
      if (int rc = prepare_pairs(h, nullptr, st)) return rc;
    }
  }
  if (getenv("SGAD_DEBUG_RUNS") && h->n_total > 0) {  // (diagnostics: the depth fix-up's long runs)
    uint32_t nl = 0;
    SGAD_CHECK_CUDA(cudaMemcpy(&nl, h->counters.as<uint32_t>() + C_NLONG, 4, cudaMemcpyDeviceToHost));
    std::vector<uint2> runs(nl);
    if (nl) SGAD_CHECK_CUDA(cudaMemcpy(runs.data(), h->runs.p, sizeof(uint2) * nl, cudaMemcpyDeviceToHost));
    unsigned long long tot = 0, mx = 0;
    for (auto& r : runs) { tot += r.y; mx = std::max<unsigned long long>(mx, r.y); }
    fprintf(stderr, "depth runs: survivors %lld long runs %u elements %llu longest %llu\n",
            (long long)h->n_surv, nl, tot, mx);
  }
  if (n_survivors) *n_survivors = h->n_surv;
  if (n_pairs) *n_pairs = h->n_pairs;
  return SGAD_OK;
}

int sgad_raster_prepare_async(sgad_raster* h, const sgad_frame* frames, int32_t n_frames,
                              const sgad_camera* cam, int32_t want_coef,
                              const sgad_frame* frames_dev, uint32_t* counts_out,
                              int32_t* overflow_flag, void* stream_) {
  cudaStream_t st = (cudaStream_t)stream_;
  if (int rc = prepare_front(h, frames, n_frames, cam, want_coef, frames_dev, st)) return rc;
  if (int rc = prepare_pairs(h, overflow_flag, st)) return rc;
  h->n_surv = h->n_pairs = -1;
  if (counts_out) {
    SGAD_CHECK_CUDA(cudaMemcpyAsync(counts_out, h->counters.as<uint32_t>() + C_NSURV,
                                    sizeof(uint32_t), cudaMemcpyDeviceToDevice, st));
    SGAD_CHECK_CUDA(cudaMemcpyAsync(counts_out + 1, h->counters.as<uint32_t>() + C_NPAIRS,
                                    sizeof(uint32_t), cudaMemcpyDeviceToDevice, st));
  }
  return SGAD_OK;
}

int sgad_raster_reserve(sgad_raster* h, int64_t pair_capacity) {
  SGAD_REQUIRE(h && pair_capacity >= 0 && pair_capacity < (1ll << 30),
               "sgad_raster_reserve: bad capacity");
  if (pair_capacity > h->cap_pairs) h->cap_pairs = pair_capacity;
  return SGAD_OK;
}

int sgad_raster_forward(sgad_raster* h, double* out_color, double* out_depth, double* out_alpha,
                        int32_t* out_count, int32_t save_state, const sgad_loss_target* target,
                        void* stream_) {
  SGAD_REQUIRE(h && h->prepared, "sgad_raster_forward: view not prepared");
  cudaStream_t st = (cudaStream_t)stream_;
  const int64_t npx = (int64_t)h->cam.width * h->cam.height;
  const bool images = out_color || out_depth || out_alpha || out_count;
  const bool loss = target != nullptr;
  const bool state = save_state || loss;
  if (state) {
    SGAD_CHECK_CUDA(h->trans_final.ensure(sizeof(double) * npx));
    SGAD_CHECK_CUDA(h->last_idx.ensure(sizeof(int32_t) * npx));
  }
  sgad_loss_target tg{};
  if (loss) {
    SGAD_REQUIRE(target->color && target->depth && target->mask && target->loss_accum,
                 "sgad_raster_forward: incomplete loss target");
    SGAD_CHECK_CUDA(h->signs.ensure(npx));
    tg = *target;
    h->rho = target->rho;
    h->sigma_d = target->sigma;
    h->n_depth = target->n_depth;
  }
  const dim3 grid((unsigned)h->n_tiles), block(RASTER_THREADS);
  const double* col64 = h->any_f64 ? h->col64.as<double>() : nullptr;
  if (int rc = smem_attrs()) return rc;
  if (state)
    if (int rc = ensure_clist(h)) return rc;
  const CList cl = clist_of(h);
#define SGAD_FWD(I, S, L)                                                                      \
  k_forward<I, S, L><<<grid, block, FWD_SMEM, st>>>(                                                \
      h->ranges.as<uint2>(), h->pvals0.as<uint32_t>(), h->packed, h->records.as<Record>(),     \
      col64, h->ntx,                                                                         \
      h->cam.width, h->cam.height, out_color, out_depth, out_alpha, out_count,               \
      h->trans_final.as<double>(), h->last_idx.as<int32_t>(), h->signs.as<uint8_t>(), tg, cl)
  if (images && state && loss) SGAD_FWD(true, true, true);
  else if (images && state) SGAD_FWD(true, true, false);
  else if (images) SGAD_FWD(true, false, false);
  else if (loss) SGAD_FWD(false, true, true);
  else if (state) SGAD_FWD(false, true, false);
  else SGAD_FWD(true, false, false);
#undef SGAD_FWD
  SGAD_LAUNCH_CHECK();
  h->forwarded = state ? 1 : 0;
  h->fused_ready = loss ? 1 : 0;
  return SGAD_OK;
}

int sgad_raster_backward(sgad_raster* h, int32_t mode, const double* g_color,
                         const double* g_depth, const double* g_alpha, double* const* map_grads,
                         float* grad_accum, void* stream_) {
  SGAD_REQUIRE(h && h->prepared && h->forwarded, "sgad_raster_backward: run forward with state first");
  cudaStream_t st = (cudaStream_t)stream_;
  if (h->n_surv == 0) return SGAD_OK;
  if (int rc = smem_attrs()) return rc;
  const dim3 grid((unsigned)h->n_tiles), block(RASTER_THREADS);
  const int64_t npx = (int64_t)h->cam.width * h->cam.height;
  if (mode == 1) {
    SGAD_REQUIRE(h->fused_ready && h->have_coef && grad_accum,
                 "fused backward needs a loss forward, chain coefficients and grad_accum");
    Upstream up;
    up.kc = h->rho / (double)(3 * npx);
    up.kd = h->n_depth > 0 ? h->sigma_d / (double)h->n_depth : 0.0;
    up.fx = (float)h->cam.fx;
    k_backward<true><<<grid, block, BWD_SMEM, st>>>(
        h->ranges.as<uint2>(), h->pvals0.as<uint32_t>(), h->records.as<Record>(),
        h->coef.as<BwdRecord>(), h->any_f64 ? h->col64.as<double>() : nullptr, h->ntx,
        h->cam.width, h->cam.height,
        h->trans_final.as<double>(), h->last_idx.as<int32_t>(), h->signs.as<uint8_t>(), up,
        g_color, nullptr, nullptr, nullptr, grad_accum, clist_of(h));
    SGAD_LAUNCH_CHECK();
#ifdef SGAD_K5_COUNT
    {
      unsigned long long c[4];
      SGAD_CHECK_CUDA(cudaStreamSynchronize(st));
      SGAD_CHECK_CUDA(cudaMemcpyFromSymbol(c, g_k5_count, sizeof c));
      fprintf(stderr, "k5 contributions %llu distinct (entry, iteration) %llu ratio %.3f; "
              "k4 queued %llu with pixels %llu\n", c[0], c[1],
              c[1] ? (double)c[0] / (double)c[1] : 0.0, c[2], c[3]);
      memset(c, 0, sizeof c);
      SGAD_CHECK_CUDA(cudaMemcpyToSymbol(g_k5_count, c, sizeof c));
    }
#endif
    return SGAD_OK;
  }
  SGAD_REQUIRE(mode == 0 && g_color && g_depth && g_alpha && map_grads,
               "exact backward needs upstream images and map_grads");
  SGAD_REQUIRE(h->n_surv >= 0, "exact backward needs a synchronous sgad_raster_prepare");
  const int n_frames = (int)h->host_frames.size();
  SGAD_CHECK_CUDA(h->raw_grads.ensure(sizeof(Fx128) * 8 * h->n_total));
  SGAD_CHECK_CUDA(cudaMemsetAsync(h->raw_grads.p, 0, sizeof(Fx128) * 8 * h->n_total, st));
  SGAD_CHECK_CUDA(h->scratch.ensure(sizeof(double*) * n_frames));
  SGAD_CHECK_CUDA(cudaMemcpyAsync(h->scratch.p, map_grads, sizeof(double*) * n_frames,
                                  cudaMemcpyHostToDevice, st));
  Upstream up{0.0, 0.0, 0.0f};
  k_backward<false><<<grid, block, BWD_SMEM, st>>>(
      h->ranges.as<uint2>(), h->pvals0.as<uint32_t>(), h->records.as<Record>(), nullptr,
      h->any_f64 ? h->col64.as<double>() : nullptr, h->ntx, h->cam.width, h->cam.height, h->trans_final.as<double>(), h->last_idx.as<int32_t>(),
      nullptr, up, g_color, g_depth, g_alpha, h->raw_grads.as<Fx128>(), nullptr, clist_of(h));
  SGAD_LAUNCH_CHECK();
  k_chain_exact<<<blocks_for(h->n_surv, 256), 256, 0, st>>>(
      h->records.as<Record>(), h->raw_grads.as<Fx128>(), h->vals0.as<uint32_t>(),
      (uint32_t)h->n_surv, h->frames.as<sgad_frame>(), n_frames, h->cam, h->scratch.as<double*>());
  SGAD_LAUNCH_CHECK();
  // the pointer table is read by the kernel; keep the host copy alive until done
  SGAD_CHECK_CUDA(cudaStreamSynchronize(st));
  return SGAD_OK;
}

int sgad_raster_forward_backward(sgad_raster* h, const sgad_loss_target* target,
                                 float* grad_accum, void* stream_) {
  SGAD_REQUIRE(h && h->prepared && target && grad_accum && h->have_coef,
               "sgad_raster_forward_backward: prepare with chain coefficients, a target and "
               "grad_accum are required");
  SGAD_REQUIRE(!h->any_f64, "sgad_raster_forward_backward: fp32 window parameters only");
  SGAD_REQUIRE(target->color && target->depth && target->mask && target->loss_accum,
               "sgad_raster_forward_backward: incomplete loss target");
  cudaStream_t st = (cudaStream_t)stream_;
  if (h->n_surv == 0) return SGAD_OK;
  if (int rc = smem_attrs()) return rc;
  if (int rc = ensure_clist(h)) return rc;
  const int64_t npx = (int64_t)h->cam.width * h->cam.height;
  Upstream up;
  up.kc = target->rho / (double)(3 * npx);
  up.kd = target->n_depth > 0 ? target->sigma / (double)target->n_depth : 0.0;
  up.fx = (float)h->cam.fx;
  k_forward_backward<<<dim3((unsigned)h->n_tiles), dim3(RASTER_THREADS), FB_SMEM, st>>>(
      h->ranges.as<uint2>(), h->pvals0.as<uint32_t>(), h->packed, h->records.as<Record>(),
      h->coef.as<BwdRecord>(), h->ntx, h->cam.width, h->cam.height, *target, up, grad_accum,
      clist_of(h));
  SGAD_LAUNCH_CHECK();
  h->forwarded = 0;
  h->fused_ready = 0;
  return SGAD_OK;
}

int sgad_raster_get_survivors(sgad_raster* h, int64_t* gid, double* u0, double* v0, double* z,
                              double* sigma, double* opacity, void* stream_) {
  SGAD_REQUIRE(h && h->prepared && h->n_surv >= 0,
               "sgad_raster_get_survivors: view not prepared (synchronously)");
  if (h->n_surv == 0) return SGAD_OK;
  k_export_surv<<<blocks_for(h->n_surv, 256), 256, 0, (cudaStream_t)stream_>>>(
      h->vals0.as<uint32_t>(), h->records.as<Record>(), (uint32_t)h->n_surv, gid, u0, v0, z,
      sigma, opacity);
  SGAD_LAUNCH_CHECK();
  return SGAD_OK;
}

int sgad_raster_get_tiles(sgad_raster* h, int64_t* ranges, int64_t* lists, void* stream_) {
  SGAD_REQUIRE(h && h->prepared && h->n_surv >= 0,
               "sgad_raster_get_tiles: view not prepared (synchronously)");
  cudaStream_t st = (cudaStream_t)stream_;
  if (ranges) {
    k_export_ranges<<<blocks_for(h->n_tiles, 256), 256, 0, st>>>(h->ranges.as<uint2>(),
                                                                 h->n_tiles, ranges);
    SGAD_LAUNCH_CHECK();
  }
  if (lists && h->n_pairs > 0) {
    SGAD_CHECK_CUDA(h->rank_of.ensure(sizeof(uint32_t) * h->n_surv));
    k_rank_of<<<blocks_for(h->n_surv, 256), 256, 0, st>>>(h->vals0.as<uint32_t>(),
                                                          (uint32_t)h->n_surv,
                                                          h->rank_of.as<uint32_t>());
    SGAD_LAUNCH_CHECK();
    k_export_lists<<<blocks_for(h->n_pairs, 256), 256, 0, st>>>(
        h->pvals0.as<uint32_t>(), h->rank_of.as<uint32_t>(), (uint32_t)h->n_pairs,
        h->packed ? LIST_IDX_MASK : ~0u, lists);
    SGAD_LAUNCH_CHECK();
  }
  return SGAD_OK;
}

}  // extern "C"
