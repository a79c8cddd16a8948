// Tracking hot path: local geometry Gaussian fit (K7), exact 1-NN grid
// (K10), fused GICP normal equations (K8) and frozen-weight cost (K9).
//
// Restates /root/reference/pkg/src/raysplat/tracker.py and geometry.py:
//   K7  <- build_local_set :193-230 / _fit_oriented_gaussians :144-170 with the
//          5x5 window neighbourhood of north_star (delta D2), sym_eigh3_batch
//          geometry.py:275-353
//   K10 <- GlobalGeomSet.query_nearest :125-128 (scipy cKDTree exact 1-NN)
//   K8  <- gicp_align :286-321 (gate, C_b + R C_a R^T, W = C^-1, H, g, cost)
//   K9  <- gicp_align :312-314,329-333 (cost_at for step halving)
// Everything is fp64: the sizes are small (M ~ 1e5) and the passes are
// latency-bound, so fp64 costs nothing measurable and keeps H within the
// 1e-3 parity bar with margin.  Reductions are two-stage and deterministic.
#include <cub/cub.cuh>
#include <stdlib.h>

#include "common.cuh"

namespace sgad {

constexpr int TRK_THREADS = 256;
constexpr double EIG_GAP_FALLBACK = 1e-8;
constexpr double EIGVAL_FLOOR_REL = 1e-6;

// ---------------------------------------------------------------- 3x3 eig
__device__ __forceinline__ double det3(const double* a) {
  return a[0] * (a[4] * a[8] - a[5] * a[7]) - a[1] * (a[3] * a[8] - a[5] * a[6]) +
         a[2] * (a[3] * a[7] - a[4] * a[6]);
}

__device__ __forceinline__ void matmul3(const double* a, const double* b, double* c) {
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      c[3 * i + j] = a[3 * i] * b[j] + a[3 * i + 1] * b[3 + j] + a[3 * i + 2] * b[6 + j];
}

// column of `a` with the largest norm, normalised (geometry.py:339-343)
__device__ __forceinline__ void principal_column(const double* a, double* v) {
  double best = -1.0;
  int idx = 0;
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const double n = sqrt(a[c] * a[c] + a[3 + c] * a[3 + c] + a[6 + c] * a[6 + c]);
    if (n > best) {
      best = n;
      idx = c;
    }
  }
  const double n = sqrt(a[idx] * a[idx] + a[3 + idx] * a[3 + idx] + a[6 + idx] * a[6 + idx]);
  v[0] = a[idx] / n;
  v[1] = a[3 + idx] / n;
  v[2] = a[6 + idx] / n;
}

// Cyclic Jacobi for the near-degenerate cases the reference hands to LAPACK
// (geometry.py:320-324); eigenvalues descending, vectors in columns.
__device__ void jacobi_eig3(const double* m, double* rot, double* vals) {
  double a[9], v[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
#pragma unroll
  for (int i = 0; i < 9; ++i) a[i] = m[i];
  for (int sweep = 0; sweep < 32; ++sweep) {
    const double off = a[1] * a[1] + a[2] * a[2] + a[5] * a[5];
    if (off == 0.0) break;
    for (int pq = 0; pq < 3; ++pq) {
      const int p = pq == 2 ? 1 : 0, q = pq == 0 ? 1 : 2;
      const double apq = a[3 * p + q];
      if (apq == 0.0) continue;
      const double theta = (a[3 * q + q] - a[3 * p + p]) / (2.0 * apq);
      const double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
      const double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
      for (int k = 0; k < 3; ++k) {  // A <- A J
        const double akp = a[3 * k + p], akq = a[3 * k + q];
        a[3 * k + p] = c * akp - s * akq;
        a[3 * k + q] = s * akp + c * akq;
      }
      for (int k = 0; k < 3; ++k) {  // A <- J^T A
        const double apk = a[3 * p + k], aqk = a[3 * q + k];
        a[3 * p + k] = c * apk - s * aqk;
        a[3 * q + k] = s * apk + c * aqk;
      }
      for (int k = 0; k < 3; ++k) {
        const double vkp = v[3 * k + p], vkq = v[3 * k + q];
        v[3 * k + p] = c * vkp - s * vkq;
        v[3 * k + q] = s * vkp + c * vkq;
      }
    }
  }
  int order[3] = {0, 1, 2};
  double d[3] = {a[0], a[4], a[8]};
  for (int i = 0; i < 2; ++i)
    for (int j = 0; j < 2 - i; ++j)
      if (d[order[j]] < d[order[j + 1]]) {
        int t = order[j];
        order[j] = order[j + 1];
        order[j + 1] = t;
      }
  for (int c = 0; c < 3; ++c) {
    vals[c] = d[order[c]];
    for (int r = 0; r < 3; ++r) rot[3 * r + c] = v[3 * r + order[c]];
  }
}

// geometry.py:275-332 for one matrix; rot row-major with eigenvectors as columns.
__device__ void sym_eigh3(const double* m, double* rot, double* vals) {
  const double q = (m[0] + m[4] + m[8]) / 3.0;
  const double off = m[1] * m[1] + m[2] * m[2] + m[5] * m[5];
  const double d0 = m[0] - q, d1 = m[4] - q, d2 = m[8] - q;
  const double p2 = (d0 * d0 + d1 * d1 + d2 * d2) + 2.0 * off;
  double scale = 0.0;
#pragma unroll
  for (int i = 0; i < 9; ++i) scale = fmax(scale, fabs(m[i]));
  scale = fmax(scale, 1e-300);
  if (p2 <= (1e-14 * scale) * (1e-14 * scale)) {
    vals[0] = vals[1] = vals[2] = q;
#pragma unroll
    for (int i = 0; i < 9; ++i) rot[i] = (i % 4 == 0) ? 1.0 : 0.0;
  } else {
    const double p = sqrt(p2 / 6.0);
    double b[9];
#pragma unroll
    for (int i = 0; i < 9; ++i) b[i] = (m[i] - ((i % 4 == 0) ? q : 0.0)) / p;
    const double detb = det3(b);
    const double phi = acos(fmin(fmax(detb / 2.0, -1.0), 1.0)) / 3.0;
    const double e1 = q + 2.0 * p * cos(phi);
    const double e3 = q + 2.0 * p * cos(phi + 2.0 * 3.141592653589793 / 3.0);
    const double e2 = 3.0 * q - e1 - e3;
    const double gap = fmin(e1 - e2, e2 - e3) / scale;
    if (gap > EIG_GAP_FALLBACK) {
      double m1[9], m2[9], m3[9], t[9], v1[3], v3[3];
#pragma unroll
      for (int i = 0; i < 9; ++i) {
        const double dg = (i % 4 == 0) ? 1.0 : 0.0;
        m1[i] = m[i] - e1 * dg;
        m2[i] = m[i] - e2 * dg;
        m3[i] = m[i] - e3 * dg;
      }
      matmul3(m2, m3, t);
      principal_column(t, v1);
      matmul3(m1, m2, t);
      principal_column(t, v3);
      const double dt = v3[0] * v1[0] + v3[1] * v1[1] + v3[2] * v1[2];
      v3[0] -= dt * v1[0];
      v3[1] -= dt * v1[1];
      v3[2] -= dt * v1[2];
      const double n3 = sqrt(v3[0] * v3[0] + v3[1] * v3[1] + v3[2] * v3[2]);
      v3[0] /= n3;
      v3[1] /= n3;
      v3[2] /= n3;
      const double v2[3] = {v3[1] * v1[2] - v3[2] * v1[1], v3[2] * v1[0] - v3[0] * v1[2],
                            v3[0] * v1[1] - v3[1] * v1[0]};
      for (int r = 0; r < 3; ++r) {
        rot[3 * r] = v1[r];
        rot[3 * r + 1] = v2[r];
        rot[3 * r + 2] = v3[r];
      }
      vals[0] = e1;
      vals[1] = e2;
      vals[2] = e3;
    } else {
      jacobi_eig3(m, rot, vals);
    }
  }
  if (det3(rot) < 0.0) {
    rot[2] = -rot[2];
    rot[5] = -rot[5];
    rot[8] = -rot[8];
  }
}

__global__ void k_sym_eigh3(const double* __restrict__ mats, int64_t n, double* __restrict__ rot,
                            double* __restrict__ vals) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double m[9], r[9], v[3];
#pragma unroll
  for (int k = 0; k < 9; ++k) m[k] = mats[9 * i + k];
  sym_eigh3(m, r, v);
#pragma unroll
  for (int k = 0; k < 9; ++k) rot[9 * i + k] = r[k];
#pragma unroll
  for (int k = 0; k < 3; ++k) vals[3 * i + k] = v[k];
}

// ---------------------------------------------------------------- K7 fit
struct FitArgs {
  const float* depth;
  const uint8_t* mask;
  int height, width, stride, win, k_min, scale_mode;
  double fx, fy, cx, cy;
};

__device__ __forceinline__ void backproject(const FitArgs& a, int u, int v, double z, double* p) {
  // tracker.py:210-212: ((u - cx) / fx) * z, ((v - cy) / fy) * z, z
  p[0] = SG_MUL(SG_DIV(SG_SUB((double)u, a.cx), a.fx), z);
  p[1] = SG_MUL(SG_DIV(SG_SUB((double)v, a.cy), a.fy), z);
  p[2] = z;
}

__global__ void __launch_bounds__(TRK_THREADS)
k_track_fit(FitArgs a, double* __restrict__ centers, double* __restrict__ cov,
            double* __restrict__ normals, double* __restrict__ rot_out,
            double* __restrict__ scales_out, int64_t* __restrict__ pixel_out,
            uint32_t* __restrict__ status, uint32_t* __restrict__ counters,
            int64_t* __restrict__ count_out) {
  typedef cub::BlockScan<uint32_t, TRK_THREADS> Scan;
  __shared__ typename Scan::TempStorage scan_tmp;
  __shared__ uint32_t s_tile, s_prefix;
  if (threadIdx.x == 0) s_tile = atomicAdd(&counters[0], 1u);
  __syncthreads();
  const int tile = (int)s_tile;
  const int64_t npx = (int64_t)a.height * a.width;
  const int64_t pix = (int64_t)tile * TRK_THREADS + threadIdx.x;
  bool keep = false;
  double c[3], rot[9], s[3], nrm[3];
  if (pix < npx) {
    const int v = (int)(pix / a.width), u = (int)(pix % a.width);
    if (v % a.stride == 0 && u % a.stride == 0 && a.mask[pix]) {
      backproject(a, u, v, (double)a.depth[pix], c);
      const int r = a.win / 2;
      double sum[3] = {0, 0, 0};
      int k = 0;
      for (int dv = -r; dv <= r; ++dv)
        for (int du = -r; du <= r; ++du) {
          if (dv == 0 && du == 0) continue;
          const int y = v + dv, x = u + du;
          if (y < 0 || y >= a.height || x < 0 || x >= a.width) continue;
          const int64_t q = (int64_t)y * a.width + x;
          if (!a.mask[q]) continue;
          double pt[3];
          backproject(a, x, y, (double)a.depth[q], pt);
          sum[0] += pt[0];
          sum[1] += pt[1];
          sum[2] += pt[2];
          ++k;
        }
      if (k >= a.k_min) {
        const double mean[3] = {sum[0] / k, sum[1] / k, sum[2] / k};
        double cv[6] = {0, 0, 0, 0, 0, 0};
        for (int dv = -r; dv <= r; ++dv)
          for (int du = -r; du <= r; ++du) {
            if (dv == 0 && du == 0) continue;
            const int y = v + dv, x = u + du;
            if (y < 0 || y >= a.height || x < 0 || x >= a.width) continue;
            const int64_t q = (int64_t)y * a.width + x;
            if (!a.mask[q]) continue;
            double pt[3];
            backproject(a, x, y, (double)a.depth[q], pt);
            const double d0 = pt[0] - mean[0], d1 = pt[1] - mean[1], d2 = pt[2] - mean[2];
            cv[0] += d0 * d0;
            cv[1] += d0 * d1;
            cv[2] += d0 * d2;
            cv[3] += d1 * d1;
            cv[4] += d1 * d2;
            cv[5] += d2 * d2;
          }
        double m[9] = {cv[0] / k, cv[1] / k, cv[2] / k, cv[1] / k, cv[3] / k,
                       cv[4] / k, cv[2] / k, cv[4] / k, cv[5] / k};
        double vals[3];
        sym_eigh3(m, rot, vals);
        // tracker.py:162-169
        const double fl = EIGVAL_FLOOR_REL * vals[0];
        for (int i = 0; i < 3; ++i) s[i] = sqrt(fmax(vals[i], fl));
        if (a.scale_mode == 0) {
          const double nn = sqrt(s[0] * s[0] + s[1] * s[1] + s[2] * s[2]);
          s[0] /= nn;
          s[1] /= nn;
          s[2] /= nn;
        } else if (a.scale_mode == 1) {
          s[0] = 1.0;
          s[1] = 1.0;
          s[2] = 1e-3;
        }
        nrm[0] = rot[2];
        nrm[1] = rot[5];
        nrm[2] = rot[8];
        if (nrm[0] * -c[0] + nrm[1] * -c[1] + nrm[2] * -c[2] < 0.0) {
          for (int i = 0; i < 3; ++i) {
            nrm[i] = -nrm[i];
            rot[3 * i + 2] = -rot[3 * i + 2];
            rot[3 * i + 1] = -rot[3 * i + 1];
          }
        }
        keep = true;
      }
    }
  }
  uint32_t rank, agg;
  Scan(scan_tmp).ExclusiveSum(keep ? 1u : 0u, rank, agg);
  if (threadIdx.x == 0) {
    if (tile == 0) {
      st_volatile_u32(status, LB_FLAG_P | agg);
      s_prefix = 0;
    } else {
      st_volatile_u32(status + tile, LB_FLAG_A | agg);
    }
  }
  if (tile > 0 && threadIdx.x < 32) {
    const uint32_t excl = lookback_exclusive(status, tile);
    if (threadIdx.x == 0) {
      st_volatile_u32(status + tile, LB_FLAG_P | (excl + agg));
      s_prefix = excl;
    }
  }
  __syncthreads();
  if (keep) {
    const int64_t o = s_prefix + rank;
    for (int i = 0; i < 3; ++i) {
      centers[3 * o + i] = c[i];
      normals[3 * o + i] = nrm[i];
      if (scales_out) scales_out[3 * o + i] = s[i];
    }
    if (rot_out)
      for (int i = 0; i < 9; ++i) rot_out[9 * o + i] = rot[i];
    if (pixel_out) pixel_out[o] = pix;
    // covariance R diag(s^2) R^T (tracker.py:76-78), upper triangle
    const double s2[3] = {s[0] * s[0], s[1] * s[1], s[2] * s[2]};
    double cc[6];
    int t = 0;
    for (int i = 0; i < 3; ++i)
      for (int j = i; j < 3; ++j) {
        cc[t++] = rot[3 * i] * s2[0] * rot[3 * j] + rot[3 * i + 1] * s2[1] * rot[3 * j + 1] +
                  rot[3 * i + 2] * s2[2] * rot[3 * j + 2];
      }
    for (int i = 0; i < 6; ++i) cov[6 * o + i] = cc[i];
  }
  if (threadIdx.x == 0 && (int64_t)(tile + 1) * TRK_THREADS >= npx) *count_out = s_prefix + agg;
}

// ---------------------------------------------------------------- K10 exact 1-NN
// Uniform hash grid over the target centres.  The cell size adapts to the
// point density (surfaces: ~3 points per occupied cell).  A query searches
// Chebyshev rings of cells around its (clamped) cell, pruning cells whose box
// is farther than the best distance so far, and stops when no unvisited cell
// can hold a closer point.  A query not settled within MAX_RINGS rings moves
// to the next, 4x coarser grid level (keeping its best candidate); queries
// still unresolved after the coarsest level (far from every surface)
// (far from every surface) fall back to an exact block-parallel scan, so the
// result is always the exact Euclidean nearest neighbour (ties -> lower index),
// as scipy cKDTree gives the reference (tracker.py:125-128).
#ifndef SGAD_NN_RINGS
#define SGAD_NN_RINGS 2
#endif
constexpr int MAX_RINGS = SGAD_NN_RINGS;
#ifndef SGAD_NN_LEVELS
#define SGAD_NN_LEVELS 10
#endif
#ifndef SGAD_NN_FACTOR
#define SGAD_NN_FACTOR 1.6
#endif
// levels of cells SGAD_NN_FACTOR x larger each (10 levels x 1.6 span 68x,
// round 1's 4 x 4.0 spanned 64x): the level the warm-start reach picks has
// cells within 1.6x of what the reach needs, so the ring search scans fewer
// surface points (measured at 816 k queries: factor 4 660, 2 666, 1.6 792,
// 1.4 785, 1.25 772 GN iterations/s; one ring instead of two: 375-521)
constexpr int NLEV = SGAD_NN_LEVELS;
constexpr unsigned long long HASH_EMPTY = ~0ull;

__device__ __forceinline__ unsigned long long dkey(double x) {
  unsigned long long b = (unsigned long long)__double_as_longlong(x);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// bounding box of the centres as order-preserving keys: per-thread, then warp
// (shuffles) and block (shared memory) reductions, one atomic per block and
// value (a per-thread atomic on six addresses serialised: ~1 ms at 816 k)
__global__ void __launch_bounds__(256) k_bbox(const double* __restrict__ pts, int64_t n,
                                             unsigned long long* __restrict__ bb) {
  __shared__ unsigned long long s_v[8][6];
  unsigned long long v[6] = {~0ull, ~0ull, ~0ull, 0, 0, 0};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    for (int k = 0; k < 3; ++k) {
      const unsigned long long key = dkey(pts[3 * i + k]);
      v[k] = key < v[k] ? key : v[k];
      v[3 + k] = key > v[3 + k] ? key : v[3 + k];
    }
#pragma unroll
  for (int k = 0; k < 6; ++k)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long y = __shfl_xor_sync(0xffffffffu, v[k], o);
      v[k] = k < 3 ? (y < v[k] ? y : v[k]) : (y > v[k] ? y : v[k]);
    }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0)
    for (int k = 0; k < 6; ++k) s_v[w][k] = v[k];
  __syncthreads();
  if (threadIdx.x < 6) {
    const int k = threadIdx.x;
    unsigned long long r = s_v[0][k];
    for (int i = 1; i < (int)(blockDim.x >> 5); ++i) r = k < 3 ? min(r, s_v[i][k]) : max(r, s_v[i][k]);
    if (k < 3) atomicMin(bb + k, r);
    else atomicMax(bb + k, r);
  }
}

struct Grid {
  double lo[3];
  double h;
  int dim[3];
  unsigned long long hmask;  // hash table size - 1
  double inv_h;              // 1 / h (a query's starting cell only: see query_cell)
};

__device__ __forceinline__ int cell_coord(double x, double lo, double h, int dim) {
  double c = floor((x - lo) / h);
  c = fmin(fmax(c, 0.0), (double)(dim - 1));
  return (int)c;
}

// The cell a search starts from.  It need not be the cell the build put a
// point at q in: every pruning and termination test uses the exact
// geometry of the cells visited (box distances, the visited box's faces), so
// a multiplication by 1 / h (no fp64 division) is enough.
__device__ __forceinline__ int query_cell(double x, double lo, double inv_h, int dim) {
  double c = floor((x - lo) * inv_h);
  c = fmin(fmax(c, 0.0), (double)(dim - 1));
  return (int)c;
}

__device__ __forceinline__ unsigned long long cell_key(int x, int y, int z) {
  return ((unsigned long long)x << 42) | ((unsigned long long)y << 21) | (unsigned long long)z;
}

__device__ __forceinline__ unsigned long long hash64(unsigned long long k) {
  k ^= k >> 33;
  k *= 0xff51afd7ed558ccdull;
  k ^= k >> 33;
  k *= 0xc4ceb9fe1a85ec53ull;
  k ^= k >> 33;
  return k;
}

__global__ void k_cell_keys(const double* __restrict__ pts, int64_t n, Grid g,
                            unsigned long long* __restrict__ keys, uint32_t* __restrict__ idx) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  keys[i] = cell_key(cell_coord(pts[3 * i], g.lo[0], g.h, g.dim[0]),
                     cell_coord(pts[3 * i + 1], g.lo[1], g.h, g.dim[1]),
                     cell_coord(pts[3 * i + 2], g.lo[2], g.h, g.dim[2]));
  idx[i] = (uint32_t)i;
}

__global__ void k_cell_heads(const unsigned long long* __restrict__ keys, int64_t n,
                             uint32_t* __restrict__ head) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  head[i] = (i == 0 || keys[i] != keys[i - 1]) ? 1u : 0u;
}

// head_scan = inclusive scan of head: cell id of point i is head_scan[i] - 1
__global__ void k_cell_starts(const unsigned long long* __restrict__ keys, int64_t n,
                              const uint32_t* __restrict__ head_scan, uint32_t* __restrict__ start) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (i == 0 || keys[i] != keys[i - 1]) start[head_scan[i] - 1] = (uint32_t)i;
  if (i == n - 1) start[head_scan[i]] = (uint32_t)n;
}

// One 16-byte hash slot per occupied cell: the key and the cell's range in
// the cell-ordered point array, so a probe that hits yields the range in the
// same load.
struct __align__(16) CellSlot {
  unsigned long long key;
  uint32_t start, count;
};

__global__ void k_cell_slots(const unsigned long long* __restrict__ keys,
                             const uint32_t* __restrict__ start, int64_t n_cells,
                             CellSlot* __restrict__ slots, unsigned long long hmask) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n_cells) return;
  const uint32_t s0 = start[c], s1 = start[c + 1];
  const unsigned long long k = keys[s0];
  unsigned long long s = hash64(k) & hmask;
  while (true) {
    const unsigned long long prev = atomicCAS(&slots[s].key, HASH_EMPTY, k);
    if (prev == HASH_EMPTY) {
      slots[s].start = s0;
      slots[s].count = s1 - s0;
      break;
    }
    s = (s + 1) & hmask;
  }
}

// the points of each level in cell order, one 32-byte record each: x, y, z
// and the point's index (as the bits of the 4th double)
__global__ void k_cell_points(const uint32_t* __restrict__ order, const double* __restrict__ pts,
                              int64_t n, double4* __restrict__ out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const uint32_t j = order[t];
  out[t] = make_double4(pts[3 * (int64_t)j], pts[3 * (int64_t)j + 1], pts[3 * (int64_t)j + 2],
                        __longlong_as_double((long long)j));
}

struct LevelView {
  Grid g;
  const CellSlot* slots;
  const double4* cpts;
};

struct GridView {
  LevelView lv[NLEV];
  const double* pts;
  int64_t n;
};

#ifdef SGAD_NN_COUNT
// (diagnostics) [searches, level calls, cells tested, cells probed, empty cells, points, probes]
__device__ unsigned long long g_nn_count[8];
#define NN_COUNT(k, x) atomicAdd(&g_nn_count[k], (unsigned long long)(x))
#else
#define NN_COUNT(k, x) ((void)0)
#endif

// the cell's (start, count) in the cell-ordered points, or count 0 if empty
__device__ __forceinline__ uint2 hash_find(const LevelView& v, unsigned long long k) {
  unsigned long long s = hash64(k) & v.g.hmask;
  while (true) {
    ulonglong2 sl;
    NN_COUNT(6, 1);
    asm("ld.global.nc.v2.u64 {%0, %1}, [%2];" : "=l"(sl.x), "=l"(sl.y) : "l"(v.slots + s));
    if (sl.x == k) return make_uint2((uint32_t)sl.y, (uint32_t)(sl.y >> 32));
    if (sl.x == HASH_EMPTY) return make_uint2(0u, 0u);
    s = (s + 1) & v.g.hmask;
  }
}

// Bounded ring search on one level, refining (best_j, best_d2); returns
// false if MAX_RINGS rings did not settle it.  `second` accumulates a lower
// bound on the squared distance of every point other than best_j: exact
// distances of the points scanned, the cell bound of every pruned cell and,
// once settled, the distance to the unvisited region.
__device__ bool grid_nearest(const LevelView& v, const double* pts, const double* q,
                             int64_t& best_j, double& best_d2, double& second) {
  const Grid& g = v.g;
  NN_COUNT(1, 1);
  int c0[3];
  for (int k = 0; k < 3; ++k) c0[k] = query_cell(q[k], g.lo[k], g.inv_h, g.dim[k]);
  for (int r = 0; r <= MAX_RINGS; ++r) {
    const int x0 = max(c0[0] - r, 0), x1 = min(c0[0] + r, g.dim[0] - 1);
    const int y0 = max(c0[1] - r, 0), y1 = min(c0[1] + r, g.dim[1] - 1);
    const int z0 = max(c0[2] - r, 0), z1 = min(c0[2] + r, g.dim[2] - 1);
    for (int x = x0; x <= x1; ++x) {
      const double bx0 = g.lo[0] + x * g.h, bx = fmax(fmax(bx0 - q[0], q[0] - (bx0 + g.h)), 0.0);
      for (int y = y0; y <= y1; ++y) {
        const double by0 = g.lo[1] + y * g.h, by = fmax(fmax(by0 - q[1], q[1] - (by0 + g.h)), 0.0);
        const bool edge_xy = abs(x - c0[0]) == r || abs(y - c0[1]) == r;
        for (int z = z0; z <= z1; ++z) {
          if (!edge_xy && abs(z - c0[2]) != r) {
            if (z < c0[2] + r) z = c0[2] + r - 1;  // skip the interior of the ring cube
            continue;
          }
          const double bz0 = g.lo[2] + z * g.h, bz = fmax(fmax(bz0 - q[2], q[2] - (bz0 + g.h)), 0.0);
          const double bmin = bx * bx + by * by + bz * bz;
          NN_COUNT(2, 1);
          if (bmin > best_d2) {
            second = fmin(second, bmin);  // (a non-empty pruned cell: all its points beyond bmin)
            continue;
          }
          const uint2 rg = hash_find(v, cell_key(x, y, z));
          NN_COUNT(3, 1);
          NN_COUNT(4, rg.y == 0);
          NN_COUNT(5, rg.y);
          for (uint32_t t = rg.x; t < rg.x + rg.y; ++t) {
            double px, py, pz, pj;
            asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
                : "=d"(px), "=d"(py), "=d"(pz), "=d"(pj) : "l"(v.cpts + t));
            const int64_t j = (int64_t)__double_as_longlong(pj);
            if (j == best_j) continue;
            const double dx = q[0] - px, dy = q[1] - py, dz = q[2] - pz;
            const double d2 = dx * dx + dy * dy + dz * dz;
            if (d2 < best_d2 || (d2 == best_d2 && j < best_j)) {
              second = fmin(second, best_d2);
              best_d2 = d2;
              best_j = j;
            } else {
              second = fmin(second, d2);
            }
          }
        }
      }
    }
    // distance to any cell outside the visited box (faces at the grid border
    // are saturated: nothing lies beyond them)
    double lb = INFINITY;
    bool all_sat = true;
    const int lo_c[3] = {x0, y0, z0}, hi_c[3] = {x1, y1, z1};
    for (int k = 0; k < 3; ++k) {
      if (lo_c[k] > 0) {
        all_sat = false;
        lb = fmin(lb, fmax(q[k] - (g.lo[k] + lo_c[k] * g.h), 0.0));
      }
      if (hi_c[k] < g.dim[k] - 1) {
        all_sat = false;
        lb = fmin(lb, fmax((g.lo[k] + (hi_c[k] + 1) * g.h) - q[k], 0.0));
      }
    }
    if (all_sat) return true;
    if (best_j >= 0 && best_d2 < lb * lb) {
      second = fmin(second, lb * lb);
      return true;
    }
  }
  return false;
}

// Warp-cooperative version of grid_nearest for one query (every lane of the
// warp calls it with the same q, best and second): each ring's cells are
// dealt round robin to the lanes, each lane keeps its own best and bound,
// and the warp merges them (lexicographic (d2, index) minimum; a lane's best
// that lost is another point's exact distance, so it bounds `second`) before
// the ring's termination test.  Same result and bound as grid_nearest: the
// lanes prune with their own (at least as good) best, the termination test
// is the same.  Used when few queries search, so that a search's chain of
// dependent slot and point loads is split over 32 lanes.
template <int G>
__device__ bool grid_nearest_warp(const LevelView& v, const double* q, int64_t& best_j,
                                  double& best_d2, double& second) {
  static_assert(G >= 4 && G <= 32 && (G & (G - 1)) == 0, "group size");
  const Grid& g = v.g;
  const int lane = threadIdx.x & (G - 1);
  const unsigned gm = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << ((threadIdx.x & 31) & ~(G - 1)));
  int c0[3];
  for (int k = 0; k < 3; ++k) c0[k] = query_cell(q[k], g.lo[k], g.inv_h, g.dim[k]);
  // the query's cell and its first ring together (27 cells: one round for
  // the warp; ring 0 alone almost never settles a query), then ring by ring
  for (int r = 1; r <= MAX_RINGS; ++r) {
    const int x0 = max(c0[0] - r, 0), x1 = min(c0[0] + r, g.dim[0] - 1);
    const int y0 = max(c0[1] - r, 0), y1 = min(c0[1] + r, g.dim[1] - 1);
    const int z0 = max(c0[2] - r, 0), z1 = min(c0[2] + r, g.dim[2] - 1);
    const int ny = y1 - y0 + 1, nz = z1 - z0 + 1, total = (x1 - x0 + 1) * ny * nz;
    // ci / (ny nz) and rem / nz by multiply-shift: exact for ci < 128 and
    // divisors <= 25 (the error ci (ceil(2^16 / d) - 2^16 / d) / 2^16 < 1 / d)
    const uint32_t mul_yz = (65535u + (uint32_t)(ny * nz)) / (uint32_t)(ny * nz),
                   mul_z = (65535u + (uint32_t)nz) / (uint32_t)nz;
    double lb2 = best_d2, lsec = INFINITY;
    int64_t lj = best_j;
    for (int cb = 0; cb < total; cb += G) {  // (uniform trip count: shuffles below)
      // each lane probes one cell of the round ...
      const int ci = cb + lane;
      uint32_t cstart = 0, ccount = 0;
      if (ci < total) {
        const int qx = (int)(((uint32_t)ci * mul_yz) >> 16), rem = ci - qx * ny * nz,
                  qy = (int)(((uint32_t)rem * mul_z) >> 16);
        const int x = x0 + qx, y = y0 + qy, z = z0 + (rem - qy * nz);
        if (r == 1 || abs(x - c0[0]) == r || abs(y - c0[1]) == r || abs(z - c0[2]) == r) {
          const double bx0 = g.lo[0] + x * g.h, bx = fmax(fmax(bx0 - q[0], q[0] - (bx0 + g.h)), 0.0);
          const double by0 = g.lo[1] + y * g.h, by = fmax(fmax(by0 - q[1], q[1] - (by0 + g.h)), 0.0);
          const double bz0 = g.lo[2] + z * g.h, bz = fmax(fmax(bz0 - q[2], q[2] - (bz0 + g.h)), 0.0);
          const double bmin = bx * bx + by * by + bz * bz;
          if (bmin > lb2) {
            lsec = fmin(lsec, bmin);
          } else {
            const uint2 rg = hash_find(v, cell_key(x, y, z));
            cstart = rg.x;
            ccount = rg.y;
          }
        }
      }
      // ... then the round's points are dealt to the lanes (one load each)
      uint32_t incl = ccount;
#pragma unroll
      for (int o = 1; o < G; o <<= 1) {
        const uint32_t y = __shfl_up_sync(gm, incl, o, G);
        if (lane >= o) incl += y;
      }
      const uint32_t excl = incl - ccount, npts = __shfl_sync(gm, incl, G - 1, G);
      for (uint32_t pb = 0; pb < npts; pb += G) {
        const uint32_t pi = pb + lane;
        int own = 0;  // the lane whose cell holds point pi: last lane with excl <= pi
#pragma unroll
        for (int bit = G / 2; bit > 0; bit >>= 1) {
          const uint32_t e = __shfl_sync(gm, excl, own | bit, G);
          if (e <= pi) own |= bit;
        }
        const uint32_t t = __shfl_sync(gm, cstart, own, G) +
                           (pi - __shfl_sync(gm, excl, own, G));
        if (pi < npts) {
          double px, py, pz, pj;
          asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
              : "=d"(px), "=d"(py), "=d"(pz), "=d"(pj) : "l"(v.cpts + t));
          const int64_t j = (int64_t)__double_as_longlong(pj);
          if (j != lj) {
            const double dx = q[0] - px, dy = q[1] - py, dz = q[2] - pz;
            const double d2 = dx * dx + dy * dy + dz * dz;
            if (d2 < lb2 || (d2 == lb2 && j < lj)) {
              lsec = fmin(lsec, lb2);
              lb2 = d2;
              lj = j;
            } else {
              lsec = fmin(lsec, d2);
            }
          }
        }
      }
    }
    // merge the lanes' bests (ties -> lower index) and bounds
    double wb = lb2;
    int64_t wj = lj;
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(gm, wb, o, G);
      const int64_t oj = __shfl_xor_sync(gm, wj, o, G);
      if (ob < wb || (ob == wb && oj < wj)) {
        wb = ob;
        wj = oj;
      }
    }
    double sc = (lj != wj) ? fmin(lsec, lb2) : lsec;
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) sc = fmin(sc, __shfl_xor_sync(gm, sc, o, G));
    second = fmin(second, sc);
    best_d2 = wb;
    best_j = wj;
    double lb = INFINITY;
    bool all_sat = true;
    const int lo_c[3] = {x0, y0, z0}, hi_c[3] = {x1, y1, z1};
    for (int k = 0; k < 3; ++k) {
      if (lo_c[k] > 0) {
        all_sat = false;
        lb = fmin(lb, fmax(q[k] - (g.lo[k] + lo_c[k] * g.h), 0.0));
      }
      if (hi_c[k] < g.dim[k] - 1) {
        all_sat = false;
        lb = fmin(lb, fmax((g.lo[k] + (hi_c[k] + 1) * g.h) - q[k], 0.0));
      }
    }
    if (all_sat) return true;
    if (best_j >= 0 && best_d2 < lb * lb) {
      second = fmin(second, lb * lb);
      return true;
    }
  }
  return false;
}

struct NNArgs {
  const double* queries;  // [m, 3]
  int64_t m;
  int warm;               // idx[] holds a previous nearest neighbour per query
  int transform;          // apply pose P to the queries first
  double r[9], t[3];
  const double* pose_dev; // [12] device pose (R row-major, t) overriding r, t, or null
  const int32_t* skip;    // nonzero: nothing to do (a finished device GN loop), or null
  int64_t* idx;
  double* d2;
  uint32_t* unresolved;   // [m] list, count in *n_unres
  uint32_t* n_unres;
  // persistence test (GICP iterations): the query position of the last full
  // search and a lower bound on its second-nearest squared distance
  double* q_prev;         // [m, 3] or null
  double* second;         // [m]
  // few searching queries (late GN iterations): warp-cooperative searches
  uint32_t* mode;         // [1] 1: k_nearest only triages, k_nn_warp searches
  uint32_t* list;         // [m] queries left to search (warp mode)
  uint32_t* n_list;       // [1]
  uint32_t* n_search;     // [1] queries searched in thread mode (the next call's mode)
};

__device__ __forceinline__ void query_point(const NNArgs& a, int64_t i, double* p) {
  const double* s = a.queries + 3 * i;
  if (a.transform) {
    // pts @ R.T + t in OpenBLAS dgemm order: fma(a2, R[j,2], fma(a1, R[j,1], a0 * R[j,0])) + t[j]
    const double* r = a.pose_dev ? a.pose_dev : a.r;
    const double* t = a.pose_dev ? a.pose_dev + 9 : a.t;
#pragma unroll
    for (int j = 0; j < 3; ++j)
      p[j] = SG_ADD(SG_FMA(s[2], r[3 * j + 2], SG_FMA(s[1], r[3 * j + 1], SG_MUL(s[0], r[3 * j]))),
                    t[j]);
  } else {
    p[0] = s[0];
    p[1] = s[1];
    p[2] = s[2];
  }
}

__device__ __forceinline__ void nn_commit(const NNArgs& a, int64_t i, int64_t j, double d2,
                                          const double* q, double second) {
  a.idx[i] = j;
  a.d2[i] = d2;
  if (a.q_prev) {
    double* qw = a.q_prev + 3 * i;
    qw[0] = q[0];
    qw[1] = q[1];
    qw[2] = q[2];
    a.second[i] = second;
  }
}

__device__ __forceinline__ double warm_d2(const GridView& v, const double* q, int64_t j) {
  const double dx = q[0] - v.pts[3 * j], dy = q[1] - v.pts[3 * j + 1], dz = q[2] - v.pts[3 * j + 2];
  return dx * dx + dy * dy + dz * dz;
}

// Two modes, chosen on the device from the previous call's count of
// searching queries (k_nearest_brute updates it):
//  * thread mode (nearly every query searches: a cold call, a registration's
//    first iterations): one thread per query, in query order -- neighbouring
//    queries search neighbouring cells; throughput bound, and faster there
//    than groups of lanes per query or compacted lists (which lose the
//    coherence);
//  * cooperative mode (fewer search): k_nearest only triages -- persistence
//    test, the rest listed -- and k_nn_warp gives each listed query a group
//    of SGAD_NN_GROUP lanes (grid_nearest_warp): a lone search is a chain
//    of dependent slot and point loads, which the group splits.
#ifndef SGAD_NN_COOP_BELOW
// cooperative searches when fewer than this fraction of the queries searched
// the call before (816 k queries: 0.98 ~ thread mode for a registration's
// first five iterations, measured best; 0: never)
#define SGAD_NN_COOP_BELOW 0.98
#endif
#ifndef SGAD_NN_GROUP
#define SGAD_NN_GROUP 16  // lanes per query in the cooperative mode (2 queries per warp)
#endif
#ifndef SGAD_NN_MINB
#define SGAD_NN_MINB 10  // 48 registers: +11 % GN iterations/s over the unbounded 56 (816 k queries)
#endif
__global__ void __launch_bounds__(128, SGAD_NN_MINB) k_nearest(GridView v, NNArgs a) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.m || (a.skip && *a.skip)) return;
  double q[3];
  query_point(a, i, q);
  int64_t j = -1;
  double d2 = INFINITY;
  int l0 = 0;
  bool search = true;
  if (a.warm) {
    j = a.idx[i];
    d2 = warm_d2(v, q, j);
    if (a.q_prev) {
      // persistence: the query moved by delta since its last full search,
      // where every other point was at least sqrt(second) away; so they are
      // now at least sqrt(second) - delta away, and if the old neighbour is
      // strictly closer than that it is still the unique nearest (exact)
      const double* qp = a.q_prev + 3 * i;
      const double ex = q[0] - qp[0], ey = q[1] - qp[1], ez = q[2] - qp[2];
      const double low = sqrt(a.second[i]) - sqrt(ex * ex + ey * ey + ez * ez);
      if (low > 0.0 && sqrt(d2) < low * (1.0 - 1e-12)) {
        nn_commit(a, i, j, d2, q, low * low * (1.0 - 1e-12));
        search = false;
      }
    }
    // the old neighbour's distance bounds the answer: start at the finest
    // level whose ring reach covers it
    const double reach = sqrt(d2);
    while (l0 < NLEV - 1 && MAX_RINGS * v.lv[l0].g.h < reach) ++l0;
  }
  const bool warp_mode = a.warm && a.mode && *a.mode == 1u;
  if (a.mode) {  // count (thread mode) or list (warp mode) the searching queries
    const unsigned act = __activemask(), sm = __ballot_sync(act, search);
    const int lane = threadIdx.x & 31, leader = __ffs(act) - 1;
    uint32_t base = 0;
    if (lane == leader && sm)
      base = atomicAdd(warp_mode ? a.n_list : a.n_search, (uint32_t)__popc(sm));
    base = __shfl_sync(act, base, leader);
    if (warp_mode && search) a.list[base + __popc(sm & ((1u << lane) - 1u))] = (uint32_t)i;
  }
  if (!search || warp_mode) return;
  double second = INFINITY;
  NN_COUNT(0, 1);
  for (int l = l0; l < NLEV; ++l) {
    if (grid_nearest(v.lv[l], v.pts, q, j, d2, second)) {
      nn_commit(a, i, j, d2, q, second);
      return;
    }
  }
  if (a.q_prev) a.second[i] = 0.0;  // (resolved by the brute force: no bound kept)
  a.unresolved[atomicAdd(a.n_unres, 1u)] = (uint32_t)i;
}

// Warp mode: one warp per listed query (grid-stride over the list).
template <int G>
__global__ void __launch_bounds__(128) k_nn_warp(GridView v, NNArgs a) {
  if ((a.skip && *a.skip) || *a.mode != 1u) return;
  const uint32_t n = *a.n_list;
  const int lane = threadIdx.x & (G - 1);
  const uint32_t ng = gridDim.x * (blockDim.x / G);
  for (uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) / G; w < n; w += ng) {
    const int64_t i = a.list[w];
    double q[3];
    query_point(a, i, q);
    int64_t j = a.idx[i];
    double d2 = warm_d2(v, q, j);
    int l0 = 0;
    const double reach = sqrt(d2);
    while (l0 < NLEV - 1 && MAX_RINGS * v.lv[l0].g.h < reach) ++l0;
    double second = INFINITY;
    bool ok = false;
    for (int l = l0; l < NLEV && !ok; ++l) ok = grid_nearest_warp<G>(v.lv[l], q, j, d2, second);
    if (lane == 0) {
      if (ok) {
        nn_commit(a, i, j, d2, q, second);
      } else {
        if (a.q_prev) a.second[i] = 0.0;
        a.unresolved[atomicAdd(a.n_unres, 1u)] = (uint32_t)i;
      }
    }
  }
}

// Exact fallback: one block per unresolved query scans every centre.
__global__ void __launch_bounds__(256) k_nearest_brute(GridView v, NNArgs a) {
  __shared__ double s_d[8];
  __shared__ int64_t s_j[8];
  if (a.skip && *a.skip) return;
  if (a.mode && blockIdx.x == 0 && threadIdx.x == 0) {
    // the next call's mode from this call's searching queries; counts reset
    // (a cold call counts in thread mode whatever the mode says: one of the
    // two counts is zero)
    const uint32_t searched = *a.n_list + *a.n_search;
    *a.mode = (double)searched < SGAD_NN_COOP_BELOW * (double)a.m ? 1u : 0u;
    *a.n_list = 0u;
    *a.n_search = 0u;
  }
  const uint32_t nu = *a.n_unres;
  for (uint32_t u = blockIdx.x; u < nu; u += gridDim.x) {
    const int64_t i = a.unresolved[u];
    double q[3];
    query_point(a, i, q);
    double best = INFINITY;
    int64_t bj = -1;
    for (int64_t j = threadIdx.x; j < v.n; j += blockDim.x) {
      const double dx = q[0] - v.pts[3 * j], dy = q[1] - v.pts[3 * j + 1], dz = q[2] - v.pts[3 * j + 2];
      const double d2 = dx * dx + dy * dy + dz * dz;
      if (d2 < best) {
        best = d2;
        bj = j;
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int64_t oj = __shfl_xor_sync(0xffffffffu, bj, o);
      if (ob < best || (ob == best && oj >= 0 && (bj < 0 || oj < bj))) {
        best = ob;
        bj = oj;
      }
    }
    if ((threadIdx.x & 31) == 0) {
      s_d[threadIdx.x >> 5] = best;
      s_j[threadIdx.x >> 5] = bj;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
        if (s_d[w] < best || (s_d[w] == best && s_j[w] >= 0 && (bj < 0 || s_j[w] < bj))) {
          best = s_d[w];
          bj = s_j[w];
        }
      a.idx[i] = bj;
      a.d2[i] = best;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- K8 / K9
struct PoseArg {
  double r[9], t[3];
};

__device__ __forceinline__ void apply_pose(const PoseArg& P, const double* a, double* p) {
  // pts @ R.T + t, in the order OpenBLAS dgemm evaluates it:
  // fma(a2, R[j,2], fma(a1, R[j,1], a0 * R[j,0])) + t[j]
#pragma unroll
  for (int j = 0; j < 3; ++j)
    p[j] = SG_ADD(SG_FMA(a[2], P.r[3 * j + 2], SG_FMA(a[1], P.r[3 * j + 1], SG_MUL(a[0], P.r[3 * j]))),
                  P.t[j]);
}

constexpr int NE_VALS = 29;  // 21 (H upper) + 6 (g) + cost + inliers

__global__ void __launch_bounds__(TRK_THREADS)
k_normal_eqs(GridView v, const int64_t* __restrict__ nn_j, const double* __restrict__ nn_d2,
             const double* __restrict__ cov_b, const double* __restrict__ nrm_b,
             const double* __restrict__ a_c, const double* __restrict__ a_cov, int64_t m,
             PoseArg P, const PoseArg* __restrict__ P_dev, const int32_t* __restrict__ skip,
             int metric_mode, double dist_max, double* __restrict__ w_out,
             double* __restrict__ b_out, uint8_t* __restrict__ acc_out,
             double* __restrict__ partial) {
  __shared__ double s_part[TRK_THREADS / 32][NE_VALS];
  if (skip && *skip) return;
  if (P_dev) P = *P_dev;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double acc[NE_VALS];
#pragma unroll
  for (int k = 0; k < NE_VALS; ++k) acc[k] = 0.0;
  if (i < m) {
    const double a[3] = {a_c[3 * i], a_c[3 * i + 1], a_c[3 * i + 2]};
    double p[3];
    apply_pose(P, a, p);
    const int64_t j = nn_j[i];
    const double d2 = nn_d2[i];
    const double b[3] = {v.pts[3 * j], v.pts[3 * j + 1], v.pts[3 * j + 2]};
    const double d[3] = {b[0] - p[0], b[1] - p[1], b[2] - p[2]};
    double metric;
    if (metric_mode == 0)
      metric = fabs(nrm_b[3 * j] * d[0] + nrm_b[3 * j + 1] * d[1] + nrm_b[3 * j + 2] * d[2]);
    else
      metric = sqrt(d2);
    const bool ok = metric < dist_max;
    acc_out[i] = ok ? 1 : 0;
    if (ok) {
      // C = C_b + R C_a R^T (tracker.py:305-307)
      const double* cb = cov_b + 6 * j;
      const double* ca = a_cov + 6 * i;
      const double A[9] = {ca[0], ca[1], ca[2], ca[1], ca[3], ca[4], ca[2], ca[4], ca[5]};
      double RA[9], C[9];
      matmul3(P.r, A, RA);
      for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c)
          C[3 * r + c] = RA[3 * r] * P.r[3 * c] + RA[3 * r + 1] * P.r[3 * c + 1] +
                         RA[3 * r + 2] * P.r[3 * c + 2];
      const double B[9] = {cb[0], cb[1], cb[2], cb[1], cb[3], cb[4], cb[2], cb[4], cb[5]};
      for (int k = 0; k < 9; ++k) C[k] += B[k];
      // W = C^-1 (symmetric adjugate)
      const double c00 = C[4] * C[8] - C[5] * C[7], c01 = C[2] * C[7] - C[1] * C[8],
                   c02 = C[1] * C[5] - C[2] * C[4];
      const double c11 = C[0] * C[8] - C[2] * C[6], c12 = C[2] * C[3] - C[0] * C[5];
      const double c22 = C[0] * C[4] - C[1] * C[3];
      const double det = C[0] * c00 + C[1] * (C[5] * C[6] - C[3] * C[8]) + C[2] * (C[3] * C[7] - C[4] * C[6]);
      const double id = 1.0 / det;
      const double W[9] = {c00 * id, c01 * id, c02 * id, c01 * id, c11 * id,
                           c12 * id, c02 * id, c12 * id, c22 * id};
      // J = [skew(p) | -I]; S^T = -S
      const double S[9] = {0.0, -p[2], p[1], p[2], 0.0, -p[0], -p[1], p[0], 0.0};
      double WS[9], StWS[9];
      matmul3(W, S, WS);
      for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c)
          StWS[3 * r + c] = -(S[3 * r] * WS[c] + S[3 * r + 1] * WS[3 + c] + S[3 * r + 2] * WS[6 + c]);
      // H blocks: [StWS, -S^T W; -W S, W] = [StWS, (WS)^T ; -WS, W]
      double H[36];
      for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) {
          H[6 * r + c] = StWS[3 * r + c];
          H[6 * r + 3 + c] = -WS[3 * c + r];  // -S^T W = S W = -(W S)^T
          H[6 * (3 + r) + c] = -WS[3 * r + c];
          H[6 * (3 + r) + 3 + c] = W[3 * r + c];
        }
      const double Wd[3] = {W[0] * d[0] + W[1] * d[1] + W[2] * d[2],
                            W[3] * d[0] + W[4] * d[1] + W[5] * d[2],
                            W[6] * d[0] + W[7] * d[1] + W[8] * d[2]};
      // g = J^T W d = [S^T W d; -W d]
      const double gr[3] = {S[0] * Wd[0] + S[3] * Wd[1] + S[6] * Wd[2],
                            S[1] * Wd[0] + S[4] * Wd[1] + S[7] * Wd[2],
                            S[2] * Wd[0] + S[5] * Wd[1] + S[8] * Wd[2]};
      int t = 0;
      for (int r = 0; r < 6; ++r)
        for (int c = r; c < 6; ++c) acc[t++] = H[6 * r + c];
      acc[21] = gr[0];
      acc[22] = gr[1];
      acc[23] = gr[2];
      acc[24] = -Wd[0];
      acc[25] = -Wd[1];
      acc[26] = -Wd[2];
      acc[27] = d[0] * Wd[0] + d[1] * Wd[1] + d[2] * Wd[2];
      acc[28] = 1.0;
      w_out[6 * i + 0] = W[0];
      w_out[6 * i + 1] = W[1];
      w_out[6 * i + 2] = W[2];
      w_out[6 * i + 3] = W[4];
      w_out[6 * i + 4] = W[5];
      w_out[6 * i + 5] = W[8];
      b_out[3 * i] = b[0];
      b_out[3 * i + 1] = b[1];
      b_out[3 * i + 2] = b[2];
    } else {
      for (int k = 0; k < 6; ++k) w_out[6 * i + k] = 0.0;
    }
  }
#pragma unroll
  for (int k = 0; k < NE_VALS; ++k) {
    double x = acc[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
    if ((threadIdx.x & 31) == 0) s_part[threadIdx.x >> 5][k] = x;
  }
  __syncthreads();
  if (threadIdx.x < NE_VALS) {
    double x = 0.0;
    for (int w = 0; w < TRK_THREADS / 32; ++w) x += s_part[w][threadIdx.x];
    partial[(size_t)blockIdx.x * NE_VALS + threadIdx.x] = x;
  }
}

// fixed-order sum of per-block partials: deterministic results.  One block
// per value; thread t adds partials t, t + 256, ... in order, then a fixed
// shared-memory tree (the former one-thread-per-value loop took ~200 us for
// 3188 partials at 1200x680).
__global__ void __launch_bounds__(256)
k_reduce_partials(const double* __restrict__ partial, int nblocks, int nvals,
                  double* __restrict__ out, const int32_t* __restrict__ skip = nullptr) {
  __shared__ double red[256];
  if (skip && *skip) return;
  const int k = blockIdx.x;
  double x = 0.0;
  for (int b = threadIdx.x; b < nblocks; b += 256) x += partial[(size_t)b * nvals + k];
  red[threadIdx.x] = x;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[k] = red[0];
}

constexpr int MAX_CAND = 8;

__global__ void __launch_bounds__(TRK_THREADS)
k_cost(const double* __restrict__ a_c, const double* __restrict__ w, const double* __restrict__ bb,
       const uint8_t* __restrict__ acc_in, int64_t m, int n_cand, const PoseArg* __restrict__ poses,
       double* __restrict__ partial, const int32_t* __restrict__ skip = nullptr) {
  __shared__ PoseArg s_pose[MAX_CAND];
  __shared__ double s_part[TRK_THREADS / 32][MAX_CAND];
  if (skip && *skip) return;
  if (threadIdx.x < n_cand) s_pose[threadIdx.x] = poses[threadIdx.x];
  __syncthreads();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double cst[MAX_CAND];
#pragma unroll
  for (int c = 0; c < MAX_CAND; ++c) cst[c] = 0.0;
  if (i < m && acc_in[i]) {
    const double a[3] = {a_c[3 * i], a_c[3 * i + 1], a_c[3 * i + 2]};
    const double* W = w + 6 * i;
    for (int c = 0; c < n_cand; ++c) {
      double p[3];
      apply_pose(s_pose[c], a, p);
      const double r0 = bb[3 * i] - p[0], r1 = bb[3 * i + 1] - p[1], r2 = bb[3 * i + 2] - p[2];
      cst[c] = r0 * (W[0] * r0 + W[1] * r1 + W[2] * r2) + r1 * (W[1] * r0 + W[3] * r1 + W[4] * r2) +
               r2 * (W[2] * r0 + W[4] * r1 + W[5] * r2);
    }
  }
#pragma unroll
  for (int c = 0; c < MAX_CAND; ++c) {
    double x = cst[c];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
    if ((threadIdx.x & 31) == 0) s_part[threadIdx.x >> 5][c] = x;
  }
  __syncthreads();
  if (threadIdx.x < MAX_CAND) {
    double x = 0.0;
    for (int wi = 0; wi < TRK_THREADS / 32; ++wi) x += s_part[wi][threadIdx.x];
    partial[(size_t)blockIdx.x * MAX_CAND + threadIdx.x] = x;
  }
}

__global__ void k_sqrt(const double* __restrict__ x, int64_t n, double* __restrict__ y) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) y[i] = sqrt(x[i]);
}

// ---------------------------------------------------------------- GN loop on the device
// gicp_align (tracker.py:265-346) with the host steps as one-thread kernels
// between the launches, so a whole registration is enqueued at once and read
// back once: per iteration the 6x6 solve and the halving candidates
// (k_gn_solve), their frozen-weight costs (K9), the acceptance test
// (k_gn_accept) and the next linearisation (K10 + K8) at the accepted pose.
// Once the loop has stopped (failure, cost increase, convergence, last
// iteration) `done` turns every later launch into a no-op.
constexpr int GN_HALVINGS = 5;  // tracker.py MAX_STEP_HALVINGS

struct GnState {
  PoseArg pose, init;
  PoseArg cand[MAX_CAND];
  double xi_norm[MAX_CAND];
  double lin[NE_VALS];   // linearisation at `pose`: H upper 21, g 6, cost, inliers
  double costs[MAX_CAND];
  double final_cost;
  int32_t done, failed, converged, iterations, inliers, singular_it, n_systems, pad;
};

// geometry.py so3_exp / _left_jacobian (restated from the reference's
// geometry.py:72-82,144-169): R = I + a [w]x + b [w]x^2, J = I + b [w]x + c [w]x^2
__device__ void se3_exp_dev(const double* xi, double* R, double* t) {
  const double w0 = xi[0], w1 = xi[1], w2 = xi[2];
  const double theta = sqrt(w0 * w0 + w1 * w1 + w2 * w2);
  const double K[9] = {0.0, -w2, w1, w2, 0.0, -w0, -w1, w0, 0.0};
  double K2[9];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c)
      K2[3 * r + c] = K[3 * r] * K[c] + K[3 * r + 1] * K[3 + c] + K[3 * r + 2] * K[6 + c];
  double a, b, c;
  if (theta < 1e-8) {
    a = 1.0;
    b = 0.5;
    c = 1.0 / 6.0;
  } else {
    const double sn = sin(theta), cs = cos(theta), t2 = theta * theta;
    a = sn / theta;
    b = (1.0 - cs) / t2;
    c = (theta - sn) / (t2 * theta);
  }
  double J[9];
  for (int k = 0; k < 9; ++k) {
    const double id = (k % 4 == 0) ? 1.0 : 0.0;
    R[k] = id + a * K[k] + b * K2[k];
    J[k] = id + (theta < 1e-8 ? 0.5 : b) * K[k] + c * K2[k];
  }
  for (int r = 0; r < 3; ++r) t[r] = J[3 * r] * xi[3] + J[3 * r + 1] * xi[4] + J[3 * r + 2] * xi[5];
}

// np.linalg.solve(h, -g): LU with partial pivoting (LAPACK dgesv's pivot
// choice); false on an exactly singular system (numpy raises LinAlgError)
__device__ bool solve6(double A[6][6], double* x) {
  int piv[6];
  for (int k = 0; k < 6; ++k) piv[k] = k;
  for (int k = 0; k < 6; ++k) {
    int p = k;
    double best = fabs(A[k][k]);
    for (int r = k + 1; r < 6; ++r)
      if (fabs(A[r][k]) > best) {
        best = fabs(A[r][k]);
        p = r;
      }
    if (best == 0.0) return false;
    if (p != k) {
      for (int c = 0; c < 6; ++c) {
        const double tmp = A[k][c];
        A[k][c] = A[p][c];
        A[p][c] = tmp;
      }
      const double tx = x[k];
      x[k] = x[p];
      x[p] = tx;
    }
    for (int r = k + 1; r < 6; ++r) {
      const double f = A[r][k] / A[k][k];
      A[r][k] = f;
      for (int c = k + 1; c < 6; ++c) A[r][c] -= f * A[k][c];
      x[r] -= f * x[k];
    }
  }
  for (int k = 5; k >= 0; --k) {
    double v = x[k];
    for (int c = k + 1; c < 6; ++c) v -= A[k][c] * x[c];
    x[k] = v / A[k][k];
  }
  return true;
}

__global__ void k_gn_solve(GnState* __restrict__ s, double* __restrict__ systems, int it,
                           int min_inliers) {
  // thread 0: the gate and the solve; threads 0-5: one halving candidate each
  __shared__ double s_xi[6];
  __shared__ int s_go;
  if (threadIdx.x == 0) {
    s_go = 0;
    if (!s->done) {
      const int n_acc = (int)llround(s->lin[28]);
      s->inliers = n_acc;
      if (n_acc < min_inliers) {  // tracker.py: failure returns the initial pose
        s->failed = 1;
        s->done = 1;
        s->pose = s->init;
      } else {
        for (int k = 0; k < NE_VALS; ++k) systems[(size_t)it * NE_VALS + k] = s->lin[k];
        s->n_systems = it + 1;
        double A[6][6], xi[6];
        int q = 0;
        for (int r = 0; r < 6; ++r)
          for (int c = r; c < 6; ++c) A[r][c] = A[c][r] = s->lin[q++];
        for (int k = 0; k < 6; ++k) xi[k] = -s->lin[21 + k];
        if (!solve6(A, xi)) {  // numpy falls back to lstsq: the host finishes the loop
          s->singular_it = it;
          s->done = 1;
        } else {
          for (int k = 0; k < 6; ++k) s_xi[k] = xi[k];
          s_go = 1;
        }
      }
    }
  }
  __syncthreads();
  const int h = threadIdx.x;
  if (!s_go || h > GN_HALVINGS) return;
  // candidate h: se3_exp(xi / 2^h).compose(pose) (the halvings scale exactly)
  double xi[6];
  const double f = ldexp(1.0, -h);
  for (int k = 0; k < 6; ++k) xi[k] = s_xi[k] * f;
  double R[9], t[3];
  se3_exp_dev(xi, R, t);
  const PoseArg P = s->pose;
  PoseArg c;
  for (int r = 0; r < 3; ++r) {
    for (int k = 0; k < 3; ++k)
      c.r[3 * r + k] = R[3 * r] * P.r[k] + R[3 * r + 1] * P.r[3 + k] + R[3 * r + 2] * P.r[6 + k];
    c.t[r] = R[3 * r] * P.t[0] + R[3 * r + 1] * P.t[1] + R[3 * r + 2] * P.t[2] + t[r];
  }
  s->cand[h] = c;
  double nn = 0.0;
  for (int k = 0; k < 6; ++k) nn += xi[k] * xi[k];
  s->xi_norm[h] = sqrt(nn);
}

__global__ void k_gn_accept(GnState* __restrict__ s, double* __restrict__ pairs, int it,
                            int max_iters, double eps) {
  if (threadIdx.x != 0 || s->done) return;
  const double before = s->lin[27];
  int k = 0;
  while (s->costs[k] > before && k < GN_HALVINGS) ++k;
  const double after = s->costs[k];
  if (after > before) {
    s->final_cost = before;
    s->done = 1;
    return;
  }
  s->pose = s->cand[k];
  s->iterations += 1;
  s->final_cost = after;
  pairs[2 * it] = before;
  pairs[2 * it + 1] = after;
  if (s->xi_norm[k] < eps) {
    s->converged = 1;
    s->done = 1;
  } else if (it + 1 == max_iters) {
    s->done = 1;
  }

}


// ---------------------------------------------------------------- to world frame
// update_global_set (tracker.py:233-238) and the members' covariances
// (GlobalGeomSet.covariances, :130-133) in the reference's operation order:
// centres and normals as numpy's BLAS product pts @ R.T (+ t) -- fma(a2,
// R[j,2], fma(a1, R[j,1], a0 R[j,0])) -- rotations as einsum('ij,njk->nik')
// and covariances as einsum('nij,nj,nkj->nik', rot, s**2, rot), unfused.
__global__ void k_to_world(const double* __restrict__ c, const double* __restrict__ rot,
                           const double* __restrict__ sc, const double* __restrict__ nrm,
                           int64_t n, PoseArg P, double* __restrict__ oc,
                           double* __restrict__ orot, double* __restrict__ onrm,
                           double* __restrict__ ocov) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double a[3] = {c[3 * i], c[3 * i + 1], c[3 * i + 2]};
  const double m[3] = {nrm[3 * i], nrm[3 * i + 1], nrm[3 * i + 2]};
  double r[9], w[9];
  for (int k = 0; k < 9; ++k) r[k] = rot[9 * i + k];
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    oc[3 * i + j] = SG_ADD(SG_FMA(a[2], P.r[3 * j + 2], SG_FMA(a[1], P.r[3 * j + 1], SG_MUL(a[0], P.r[3 * j]))),
                           P.t[j]);
    onrm[3 * i + j] = SG_FMA(m[2], P.r[3 * j + 2], SG_FMA(m[1], P.r[3 * j + 1], SG_MUL(m[0], P.r[3 * j])));
  }
#pragma unroll
  for (int ii = 0; ii < 3; ++ii)
#pragma unroll
    for (int k = 0; k < 3; ++k)
      w[3 * ii + k] = SG_ADD(SG_ADD(SG_MUL(P.r[3 * ii], r[k]), SG_MUL(P.r[3 * ii + 1], r[3 + k])),
                             SG_MUL(P.r[3 * ii + 2], r[6 + k]));
  for (int k = 0; k < 9; ++k) orot[9 * i + k] = w[k];
  const double s2[3] = {SG_MUL(sc[3 * i], sc[3 * i]), SG_MUL(sc[3 * i + 1], sc[3 * i + 1]),
                        SG_MUL(sc[3 * i + 2], sc[3 * i + 2])};
  // packed (00, 01, 02, 11, 12, 22)
  const int pi[6] = {0, 0, 0, 1, 1, 2}, pk[6] = {0, 1, 2, 1, 2, 2};
#pragma unroll
  for (int e = 0; e < 6; ++e) {
    const int ii = pi[e], k = pk[e];
    double acc = SG_MUL(SG_MUL(w[3 * ii], s2[0]), w[3 * k]);
    acc = SG_ADD(acc, SG_MUL(SG_MUL(w[3 * ii + 1], s2[1]), w[3 * k + 1]));
    acc = SG_ADD(acc, SG_MUL(SG_MUL(w[3 * ii + 2], s2[2]), w[3 * k + 2]));
    ocov[6 * i + e] = acc;
  }
}

}  // namespace sgad

struct sgad_geomset {
  sgad::DevBuf pts, cov, nrm, bbox, keys0, keys1, idx0, idx1, head, headscan, start, hkeys, hvals,
      cub_tmp;
  sgad::DevBuf w, b, acc, partial, poses, nn_j, nn_d2, unres, counter, nn_qprev, nn_second, nn_list;
  sgad::DevBuf gn_state, gn_log;
  sgad::Grid grid[sgad::NLEV]{};
  sgad::DevBuf lslots[sgad::NLEV], lpts[sgad::NLEV];
  int64_t n = 0;
  int64_t nn_m = -1;  // queries whose neighbours nn_j holds (warm start)
  unsigned long long* pinned = nullptr;
};

using namespace sgad;

static inline unsigned nblk(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

extern "C" {

int sgad_sym_eigh3(const double* mats, int64_t n, double* rot, double* vals, void* stream) {
  SGAD_REQUIRE(n >= 0 && (n == 0 || (mats && rot && vals)), "sgad_sym_eigh3: bad arguments");
  if (n == 0) return SGAD_OK;
  k_sym_eigh3<<<nblk(n, 128), 128, 0, (cudaStream_t)stream>>>(mats, n, rot, vals);
  SGAD_LAUNCH_CHECK();
  return SGAD_OK;
}

int sgad_track_fit(const float* depth, const uint8_t* mask, int32_t height, int32_t width,
                   double fx, double fy, double cx, double cy, int32_t stride, int32_t win,
                   int32_t k_min, int32_t scale_mode, double* centers, double* cov,
                   double* normals, double* rot, double* scales, int64_t* pixel,
                   int64_t* count, void* stream_) {
  SGAD_REQUIRE(depth && mask && centers && cov && normals && count, "sgad_track_fit: null buffer");
  SGAD_REQUIRE(height > 0 && width > 0 && stride >= 1 && win >= 3 && (win & 1) && k_min >= 1 &&
                   scale_mode >= 0 && scale_mode <= 2,
               "sgad_track_fit: bad parameters");
  cudaStream_t st = (cudaStream_t)stream_;
  const int64_t npx = (int64_t)height * width;
  const int64_t tiles = (npx + TRK_THREADS - 1) / TRK_THREADS;
  static thread_local DevBuf status, counters;
  SGAD_CHECK_CUDA(status.ensure(sizeof(uint32_t) * tiles));
  SGAD_CHECK_CUDA(counters.ensure(sizeof(uint32_t) * 4));
  SGAD_CHECK_CUDA(cudaMemsetAsync(status.p, 0, sizeof(uint32_t) * tiles, st));
  SGAD_CHECK_CUDA(cudaMemsetAsync(counters.p, 0, sizeof(uint32_t) * 4, st));
  FitArgs a{depth, mask, height, width, stride, win, k_min, scale_mode, fx, fy, cx, cy};
  k_track_fit<<<(unsigned)tiles, TRK_THREADS, 0, st>>>(a, centers, cov, normals, rot, scales, pixel,
                                                      status.as<uint32_t>(), counters.as<uint32_t>(),
                                                      count);
  SGAD_LAUNCH_CHECK();
  return SGAD_OK;
}

int sgad_geomset_create(sgad_geomset** out) {
  SGAD_REQUIRE(out, "sgad_geomset_create: null out");
  sgad_geomset* g = new sgad_geomset();
  if (cudaMallocHost(&g->pinned, 8 * sizeof(unsigned long long)) != cudaSuccess) {
    delete g;
    set_error("cudaMallocHost failed");
    return SGAD_E_CUDA;
  }
  *out = g;
  return SGAD_OK;
}

int sgad_geomset_destroy(sgad_geomset* g) {
  if (!g) return SGAD_OK;
  DevBuf* bufs[] = {&g->pts, &g->cov, &g->nrm, &g->bbox, &g->keys0, &g->keys1, &g->idx0,
                    &g->idx1, &g->head, &g->headscan, &g->start, &g->hkeys, &g->hvals,
                    &g->cub_tmp, &g->w, &g->b, &g->acc, &g->partial, &g->poses, &g->nn_j,
                    &g->nn_d2, &g->unres, &g->counter, &g->nn_qprev, &g->nn_second,
                    &g->gn_state, &g->gn_log, &g->nn_list};
  for (DevBuf* b : bufs) b->release();
  for (int l = 0; l < NLEV; ++l) {
    g->lslots[l].release();
    g->lpts[l].release();
  }
  if (g->pinned) cudaFreeHost(g->pinned);

  delete g;
  return SGAD_OK;
}

// sort the cell keys of all centres for cell size h; returns the number of
// occupied cells (synchronises)
static int grid_sort(sgad_geomset* g, Grid& gr, cudaStream_t st, int64_t* n_cells,
                     unsigned long long** keys_sorted, uint32_t** idx_sorted) {
  const int64_t n = g->n;
  k_cell_keys<<<nblk(n, 256), 256, 0, st>>>(g->pts.as<double>(), n, gr,
                                            g->keys0.as<unsigned long long>(), g->idx0.as<uint32_t>());
  SGAD_LAUNCH_CHECK();
  int bits = 1;
  const unsigned long long maxkey = ((unsigned long long)(gr.dim[0] - 1) << 42) |
                                    ((unsigned long long)(gr.dim[1] - 1) << 21) |
                                    (unsigned long long)(gr.dim[2] - 1);
  while (bits < 64 && (maxkey >> bits)) ++bits;
  cub::DoubleBuffer<unsigned long long> dk(g->keys0.as<unsigned long long>(),
                                           g->keys1.as<unsigned long long>());
  cub::DoubleBuffer<uint32_t> dv(g->idx0.as<uint32_t>(), g->idx1.as<uint32_t>());
  size_t tmp = 0;
  SGAD_CHECK_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, dk, dv, (int)n, 0, bits, st));
  SGAD_CHECK_CUDA(g->cub_tmp.ensure(tmp));
  SGAD_CHECK_CUDA(cub::DeviceRadixSort::SortPairs(g->cub_tmp.p, tmp, dk, dv, (int)n, 0, bits, st));
  k_cell_heads<<<nblk(n, 256), 256, 0, st>>>(dk.Current(), n, g->head.as<uint32_t>());
  SGAD_LAUNCH_CHECK();
  tmp = 0;
  SGAD_CHECK_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tmp, g->head.as<uint32_t>(),
                                                g->headscan.as<uint32_t>(), (int)n, st));
  SGAD_CHECK_CUDA(g->cub_tmp.ensure(tmp));
  SGAD_CHECK_CUDA(cub::DeviceScan::InclusiveSum(g->cub_tmp.p, tmp, g->head.as<uint32_t>(),
                                                g->headscan.as<uint32_t>(), (int)n, st));
  uint32_t* hp = reinterpret_cast<uint32_t*>(g->pinned);
  SGAD_CHECK_CUDA(cudaMemcpyAsync(hp, g->headscan.as<uint32_t>() + n - 1, sizeof(uint32_t),
                                  cudaMemcpyDeviceToHost, st));
  SGAD_CHECK_CUDA(cudaStreamSynchronize(st));
  *n_cells = hp[0];
  *keys_sorted = dk.Current();
  *idx_sorted = dv.Current();
  return SGAD_OK;
}

static void grid_dims(Grid& gr, const double* ext, double h) {
  gr.h = h;
  gr.inv_h = 1.0 / h;
  for (int k = 0; k < 3; ++k) gr.dim[k] = (int)fmin(floor(ext[k] / h) + 1.0, (double)(1 << 21) - 1.0);
}

int sgad_geomset_set(sgad_geomset* g, const double* centers, const double* cov,
                     const double* normals, int64_t n, void* stream_) {
  SGAD_REQUIRE(g && centers && cov && normals && n > 0, "sgad_geomset_set: bad arguments");
  SGAD_REQUIRE(n < (1ll << 31), "sgad_geomset_set: too many points");
  cudaStream_t st = (cudaStream_t)stream_;
  g->n = n;
  g->nn_m = -1;
  SGAD_CHECK_CUDA(g->pts.ensure(sizeof(double) * 3 * n));
  SGAD_CHECK_CUDA(g->cov.ensure(sizeof(double) * 6 * n));
  SGAD_CHECK_CUDA(g->nrm.ensure(sizeof(double) * 3 * n));
  SGAD_CHECK_CUDA(cudaMemcpyAsync(g->pts.p, centers, sizeof(double) * 3 * n, cudaMemcpyDefault, st));
  SGAD_CHECK_CUDA(cudaMemcpyAsync(g->cov.p, cov, sizeof(double) * 6 * n, cudaMemcpyDefault, st));
  SGAD_CHECK_CUDA(cudaMemcpyAsync(g->nrm.p, normals, sizeof(double) * 3 * n, cudaMemcpyDefault, st));
  SGAD_CHECK_CUDA(g->bbox.ensure(sizeof(unsigned long long) * 6));
  unsigned long long init[6] = {~0ull, ~0ull, ~0ull, 0, 0, 0};
  memcpy(g->pinned, init, sizeof init);
  SGAD_CHECK_CUDA(cudaMemcpyAsync(g->bbox.p, g->pinned, sizeof init, cudaMemcpyHostToDevice, st));
  k_bbox<<<min(nblk(n, 256), 148u * 4u), 256, 0, st>>>(g->pts.as<double>(), n,
                                                   g->bbox.as<unsigned long long>());
  SGAD_LAUNCH_CHECK();
  SGAD_CHECK_CUDA(cudaMemcpyAsync(g->pinned, g->bbox.p, sizeof init, cudaMemcpyDeviceToHost, st));
  SGAD_CHECK_CUDA(cudaStreamSynchronize(st));
  double lo[3], hi[3];
  for (int k = 0; k < 3; ++k) {
    unsigned long long kl = g->pinned[k], kh = g->pinned[3 + k];
    uint64_t bl = (kl >> 63) ? (kl & 0x7fffffffffffffffull) : ~kl;
    uint64_t bh = (kh >> 63) ? (kh & 0x7fffffffffffffffull) : ~kh;
    memcpy(&lo[k], &bl, 8);
    memcpy(&hi[k], &bh, 8);
  }
  double ext[3], vol = 1.0, emax = 0.0;
  for (int k = 0; k < 3; ++k) {
    ext[k] = fmax(hi[k] - lo[k], 1e-9);
    vol *= ext[k];
    emax = fmax(emax, ext[k]);
  }
  SGAD_CHECK_CUDA(g->keys0.ensure(sizeof(unsigned long long) * n));
  SGAD_CHECK_CUDA(g->keys1.ensure(sizeof(unsigned long long) * n));
  SGAD_CHECK_CUDA(g->idx0.ensure(sizeof(uint32_t) * n));
  SGAD_CHECK_CUDA(g->idx1.ensure(sizeof(uint32_t) * n));
  SGAD_CHECK_CUDA(g->head.ensure(sizeof(uint32_t) * n));
  SGAD_CHECK_CUDA(g->headscan.ensure(sizeof(uint32_t) * n));
  Grid gr;
  for (int k = 0; k < 3; ++k) gr.lo[k] = lo[k];
  const double hmin = emax / (double)((1 << 21) - 2);
  double h = fmax(cbrt(vol / fmax(0.5 * (double)n, 1.0)), hmin);
  grid_dims(gr, ext, h);
  int64_t n_cells = 0;
  unsigned long long* ks;
  uint32_t* is;
  int rc = grid_sort(g, gr, st, &n_cells, &ks, &is);
  if (rc) return rc;
  // density refinement: points on surfaces -> occupancy scales with h^2
  const double occ = (double)n / (double)n_cells;
  if (occ > 6.0) {
    h = fmax(h * sqrt(3.0 / occ), hmin);
    grid_dims(gr, ext, h);
    rc = grid_sort(g, gr, st, &n_cells, &ks, &is);
    if (rc) return rc;
  }
  // level l uses cells SGAD_NN_FACTOR^l times larger; each level is an exact hash grid
  for (int l = 0; l < NLEV; ++l) {
    if (l > 0) {
      grid_dims(gr, ext, gr.h * SGAD_NN_FACTOR);
      rc = grid_sort(g, gr, st, &n_cells, &ks, &is);
      if (rc) return rc;
    }
    unsigned long long hsize = 1024;
    while (hsize < 2ull * (unsigned long long)n_cells) hsize <<= 1;
    gr.hmask = hsize - 1;
    g->grid[l] = gr;
    SGAD_CHECK_CUDA(g->start.ensure(sizeof(uint32_t) * (n_cells + 1)));
    SGAD_CHECK_CUDA(g->lslots[l].ensure(sizeof(CellSlot) * hsize));
    SGAD_CHECK_CUDA(g->lpts[l].ensure(sizeof(double4) * n));
    SGAD_CHECK_CUDA(cudaMemsetAsync(g->lslots[l].p, 0xff, sizeof(CellSlot) * hsize, st));
    k_cell_starts<<<nblk(n, 256), 256, 0, st>>>(ks, n, g->headscan.as<uint32_t>(),
                                                g->start.as<uint32_t>());
    SGAD_LAUNCH_CHECK();
    k_cell_slots<<<nblk(n_cells, 256), 256, 0, st>>>(ks, g->start.as<uint32_t>(), n_cells,
                                                     g->lslots[l].as<CellSlot>(), gr.hmask);
    SGAD_LAUNCH_CHECK();
    k_cell_points<<<nblk(n, 256), 256, 0, st>>>(is, g->pts.as<double>(), n,
                                                g->lpts[l].as<double4>());
    SGAD_LAUNCH_CHECK();
  }
  return SGAD_OK;
}

static GridView view_of(sgad_geomset* g) {
  GridView v;
  for (int l = 0; l < NLEV; ++l) {
    v.lv[l].g = g->grid[l];
    v.lv[l].slots = g->lslots[l].as<CellSlot>();
    v.lv[l].cpts = g->lpts[l].as<double4>();
  }
  v.pts = g->pts.as<double>();
  v.n = g->n;
  return v;
}

// SGAD_NN_PERSIST=0 (A/B): every GICP iteration searches every query afresh
static bool nn_persist() {
  static const bool on = [] {
    const char* e = getenv("SGAD_NN_PERSIST");
    return !(e && e[0] == '0');
  }();
  return on;
}

// exact 1-NN for m queries (optionally transformed by rot/trans) into idx/d2
static int run_nearest(sgad_geomset* g, const double* queries, int64_t m, const double* rot,
                       const double* trans, int64_t* idx, double* d2, int warm, cudaStream_t st,
                       bool persist = false, const double* pose_dev = nullptr,
                       const int32_t* skip = nullptr) {
  SGAD_CHECK_CUDA(g->unres.ensure(sizeof(uint32_t) * m));
  SGAD_CHECK_CUDA(g->nn_list.ensure(sizeof(uint32_t) * m));
  // counter: [0] unresolved (per call), [1] mode, [2] listed, [3] searched
  // (the last three carried from call to call, reset by k_nearest_brute)
  const bool fresh = g->counter.p == nullptr;
  SGAD_CHECK_CUDA(g->counter.ensure(sizeof(uint32_t) * 4));
  SGAD_CHECK_CUDA(cudaMemsetAsync(g->counter.p, 0, sizeof(uint32_t) * (fresh ? 4 : 1), st));
  NNArgs a;
  a.queries = queries;
  a.m = m;
  a.warm = warm;
  a.transform = rot != nullptr || pose_dev != nullptr;
  a.pose_dev = pose_dev;
  a.skip = skip;
  for (int k = 0; k < 9; ++k) a.r[k] = rot ? rot[k] : 0.0;
  for (int k = 0; k < 3; ++k) a.t[k] = trans ? trans[k] : 0.0;
  a.idx = idx;
  a.d2 = d2;
  a.unresolved = g->unres.as<uint32_t>();
  a.n_unres = g->counter.as<uint32_t>();
  a.mode = SGAD_NN_COOP_BELOW > 0 ? g->counter.as<uint32_t>() + 1 : nullptr;
  a.n_list = g->counter.as<uint32_t>() + 2;
  a.n_search = g->counter.as<uint32_t>() + 3;
  a.list = g->nn_list.as<uint32_t>();
  a.q_prev = nullptr;
  a.second = nullptr;
  if (persist) {
    SGAD_CHECK_CUDA(g->nn_qprev.ensure(sizeof(double) * 3 * m));
    SGAD_CHECK_CUDA(g->nn_second.ensure(sizeof(double) * m));
    a.q_prev = g->nn_qprev.as<double>();
    a.second = g->nn_second.as<double>();
  }
  const GridView v = view_of(g);
  k_nearest<<<nblk(m, 128), 128, 0, st>>>(v, a);
  SGAD_LAUNCH_CHECK();
  if (a.mode) {
    k_nn_warp<SGAD_NN_GROUP><<<148 * 16, 128, 0, st>>>(v, a);
    SGAD_LAUNCH_CHECK();
  }
  k_nearest_brute<<<256, 256, 0, st>>>(v, a);
  SGAD_LAUNCH_CHECK();
#ifdef SGAD_NN_COUNT
  {
    unsigned long long c[8];
    SGAD_CHECK_CUDA(cudaStreamSynchronize(st));
    SGAD_CHECK_CUDA(cudaMemcpyFromSymbol(c, g_nn_count, sizeof c));
    fprintf(stderr, "nn m=%lld searches=%llu levels=%llu cells=%llu probed=%llu empty=%llu "
            "points=%llu probes=%llu\n", (long long)m, c[0], c[1], c[2], c[3], c[4], c[5], c[6]);
    memset(c, 0, sizeof c);
    SGAD_CHECK_CUDA(cudaMemcpyToSymbol(g_nn_count, c, sizeof c));
  }
#endif
  return SGAD_OK;
}

int sgad_geomset_nearest(sgad_geomset* g, const double* queries, int64_t m, int64_t* idx,
                         double* dist, void* stream_) {
  SGAD_REQUIRE(g && g->n > 0, "global set is empty");
  SGAD_REQUIRE(m >= 0 && (m == 0 || (queries && idx)), "sgad_geomset_nearest: bad arguments");
  if (m == 0) return SGAD_OK;
  cudaStream_t st = (cudaStream_t)stream_;
  SGAD_CHECK_CUDA(g->nn_d2.ensure(sizeof(double) * m));
  int rc = run_nearest(g, queries, m, nullptr, nullptr, idx, g->nn_d2.as<double>(), 0, st);
  if (rc) return rc;
  if (dist) {
    k_sqrt<<<nblk(m, 256), 256, 0, st>>>(g->nn_d2.as<double>(), m, dist);
    SGAD_LAUNCH_CHECK();
  }
  return SGAD_OK;
}

}  // extern "C"

// The exact nearest neighbours of the local centres at a host pose
// (rot/trans) or a device pose (P_dev), skipped on the device when *skip.
static int nearest_at(sgad_geomset* g, const double* local_centers, int64_t m, const double* rot,
                      const double* trans, const PoseArg* P_dev, const int32_t* skip,
                      int32_t warm_start, cudaStream_t st) {
  const bool warm = warm_start && g->nn_m == m && g->nn_j.cap >= sizeof(int64_t) * m;
  SGAD_CHECK_CUDA(g->nn_j.ensure(sizeof(int64_t) * m));
  SGAD_CHECK_CUDA(g->nn_d2.ensure(sizeof(double) * m));
  g->nn_m = m;
  return run_nearest(g, local_centers, m, rot, trans, g->nn_j.as<int64_t>(), g->nn_d2.as<double>(),
                     warm ? 1 : 0, st, nn_persist(), reinterpret_cast<const double*>(P_dev), skip);
}

// K8 + reduce into out[NE_VALS] at the pose the last nearest_at used.
static int eqs_at(sgad_geomset* g, const double* local_centers, const double* local_cov, int64_t m,
                  const double* rot, const double* trans, const PoseArg* P_dev,
                  const int32_t* skip, int32_t metric_mode, double dist_max, double* out,
                  cudaStream_t st) {
  const unsigned nb = nblk(m, TRK_THREADS);
  SGAD_CHECK_CUDA(g->w.ensure(sizeof(double) * 6 * m));
  SGAD_CHECK_CUDA(g->b.ensure(sizeof(double) * 3 * m));
  SGAD_CHECK_CUDA(g->acc.ensure(m));
  SGAD_CHECK_CUDA(g->partial.ensure(sizeof(double) * NE_VALS * nb));
  PoseArg P{};
  if (rot)
    for (int k = 0; k < 9; ++k) P.r[k] = rot[k];
  if (trans)
    for (int k = 0; k < 3; ++k) P.t[k] = trans[k];
  k_normal_eqs<<<nb, TRK_THREADS, 0, st>>>(view_of(g), g->nn_j.as<int64_t>(), g->nn_d2.as<double>(),
                                           g->cov.as<double>(), g->nrm.as<double>(),
                                           local_centers, local_cov, m, P, P_dev, skip, metric_mode,
                                           dist_max, g->w.as<double>(), g->b.as<double>(),
                                           g->acc.as<uint8_t>(), g->partial.as<double>());
  SGAD_LAUNCH_CHECK();
  k_reduce_partials<<<NE_VALS, 256, 0, st>>>(g->partial.as<double>(), (int)nb, NE_VALS, out, skip);
  SGAD_LAUNCH_CHECK();
  return SGAD_OK;
}

// One linearisation (NN + K8 + reduce into out[NE_VALS]) at a host pose
// (rot/trans) or at a device pose (P_dev), skipped on the device when *skip.
static int linearize(sgad_geomset* g, const double* local_centers, const double* local_cov,
                     int64_t m, const double* rot, const double* trans, const PoseArg* P_dev,
                     const int32_t* skip, int32_t metric_mode, double dist_max, int32_t warm_start,
                     double* out, cudaStream_t st) {
  if (int rc = nearest_at(g, local_centers, m, rot, trans, P_dev, skip, warm_start, st)) return rc;
  return eqs_at(g, local_centers, local_cov, m, rot, trans, P_dev, skip, metric_mode, dist_max, out,
                st);
}

extern "C" {

int sgad_track_normal_eqs(sgad_geomset* g, const double* local_centers, const double* local_cov,
                          int64_t m, const double* rot, const double* trans, int32_t metric_mode,
                          double dist_max, int32_t warm_start, double* out, void* stream_) {
  SGAD_REQUIRE(g && g->n > 0, "global set is empty");
  SGAD_REQUIRE(local_centers && local_cov && rot && trans && out && m > 0,
               "sgad_track_normal_eqs: bad arguments");
  return linearize(g, local_centers, local_cov, m, rot, trans, nullptr, nullptr, metric_mode,
                   dist_max, warm_start, out, (cudaStream_t)stream_);
}

int sgad_track_correspondences(sgad_geomset* g, int64_t* idx, int64_t m, void* stream_) {
  SGAD_REQUIRE(g && idx && m >= 0 && g->nn_m == m, "sgad_track_correspondences: bad arguments");
  if (m == 0) return SGAD_OK;
  SGAD_CHECK_CUDA(cudaMemcpyAsync(idx, g->nn_j.p, sizeof(int64_t) * m, cudaMemcpyDeviceToDevice,
                                  (cudaStream_t)stream_));
  return SGAD_OK;
}

int sgad_track_accepted(sgad_geomset* g, uint8_t* out, int64_t m, void* stream_) {
  SGAD_REQUIRE(g && out && m >= 0 && g->acc.cap >= (size_t)m, "sgad_track_accepted: bad arguments");
  if (m == 0) return SGAD_OK;
  SGAD_CHECK_CUDA(cudaMemcpyAsync(out, g->acc.p, m, cudaMemcpyDeviceToDevice, (cudaStream_t)stream_));
  return SGAD_OK;
}

int sgad_track_cost(sgad_geomset* g, const double* local_centers, int64_t m, const double* poses,
                    int32_t n_cand, double* out, void* stream_) {
  SGAD_REQUIRE(g && local_centers && poses && out && m > 0 && n_cand > 0 && n_cand <= MAX_CAND,
               "sgad_track_cost: bad arguments");
  SGAD_REQUIRE(g->w.cap >= sizeof(double) * 6 * m, "sgad_track_cost: run normal_eqs first");
  cudaStream_t st = (cudaStream_t)stream_;
  const unsigned nb = nblk(m, TRK_THREADS);
  SGAD_CHECK_CUDA(g->partial.ensure(sizeof(double) * MAX_CAND * nb));
  SGAD_CHECK_CUDA(g->poses.ensure(sizeof(PoseArg) * MAX_CAND));
  PoseArg hp[MAX_CAND];
  for (int c = 0; c < n_cand; ++c) {
    for (int k = 0; k < 9; ++k) hp[c].r[k] = poses[12 * c + k];
    for (int k = 0; k < 3; ++k) hp[c].t[k] = poses[12 * c + 9 + k];
  }
  SGAD_CHECK_CUDA(cudaMemcpyAsync(g->poses.p, hp, sizeof(PoseArg) * n_cand, cudaMemcpyHostToDevice, st));
  k_cost<<<nb, TRK_THREADS, 0, st>>>(local_centers, g->w.as<double>(), g->b.as<double>(),
                                     g->acc.as<uint8_t>(), m, n_cand, g->poses.as<PoseArg>(),
                                     g->partial.as<double>());
  SGAD_LAUNCH_CHECK();
  k_reduce_partials<<<MAX_CAND, 256, 0, st>>>(g->partial.as<double>(), (int)nb, MAX_CAND, out);
  SGAD_LAUNCH_CHECK();
  // (hp may go: an asynchronous copy from pageable memory returns once the
  // source is staged)
  return SGAD_OK;
}

int sgad_track_gicp(sgad_geomset* g, const double* local_centers, const double* local_cov,
                    int64_t m, const double* init_pose, int32_t metric_mode, double dist_max,
                    int32_t max_iters, double convergence_eps, int32_t warm_start,
                    int32_t min_inliers, double* result, double* systems, double* cost_pairs,
                    uint8_t* accepted_first, void* stream_) {
  SGAD_REQUIRE(g && g->n > 0, "global set is empty");
  SGAD_REQUIRE(local_centers && local_cov && init_pose && result && m > 0 && max_iters > 0,
               "sgad_track_gicp: bad arguments");
  cudaStream_t st = (cudaStream_t)stream_;
  const unsigned nb = nblk(m, TRK_THREADS);
  SGAD_CHECK_CUDA(g->gn_state.ensure(sizeof(GnState)));
  SGAD_CHECK_CUDA(g->gn_log.ensure(sizeof(double) * (size_t)max_iters * (NE_VALS + 2)));
  SGAD_CHECK_CUDA(g->partial.ensure(sizeof(double) * (NE_VALS > MAX_CAND ? NE_VALS : MAX_CAND) * nb));
  GnState h{};
  for (int k = 0; k < 9; ++k) h.pose.r[k] = h.init.r[k] = init_pose[k];
  for (int k = 0; k < 3; ++k) h.pose.t[k] = h.init.t[k] = init_pose[9 + k];
  h.final_cost = NAN;
  h.singular_it = -1;
  GnState* s = g->gn_state.as<GnState>();
  double* sys = g->gn_log.as<double>();
  double* pairs = sys + (size_t)max_iters * NE_VALS;
  SGAD_CHECK_CUDA(cudaMemcpyAsync(s, &h, sizeof h, cudaMemcpyHostToDevice, st));
  const int32_t* done = &s->done;
  if (int rc = linearize(g, local_centers, local_cov, m, nullptr, nullptr, &s->pose, done,
                         metric_mode, dist_max, warm_start, s->lin, st))
    return rc;
  if (accepted_first)
    SGAD_CHECK_CUDA(cudaMemcpyAsync(accepted_first, g->acc.p, m, cudaMemcpyDefault, st));
  for (int it = 0; it < max_iters; ++it) {
    k_gn_solve<<<1, 32, 0, st>>>(s, sys, it, min_inliers);
    SGAD_LAUNCH_CHECK();
    k_cost<<<nb, TRK_THREADS, 0, st>>>(local_centers, g->w.as<double>(), g->b.as<double>(),
                                       g->acc.as<uint8_t>(), m, GN_HALVINGS + 1, s->cand,
                                       g->partial.as<double>(), done);
    SGAD_LAUNCH_CHECK();
    k_reduce_partials<<<MAX_CAND, 256, 0, st>>>(g->partial.as<double>(), (int)nb, MAX_CAND,
                                                s->costs, done);
    SGAD_LAUNCH_CHECK();
    k_gn_accept<<<1, 32, 0, st>>>(s, pairs, it, max_iters, convergence_eps);
    SGAD_LAUNCH_CHECK();
    if (it + 1 < max_iters) {
      if (int rc = linearize(g, local_centers, local_cov, m, nullptr, nullptr, &s->pose, done,
                             metric_mode, dist_max, 1, s->lin, st))
        return rc;
    }
  }
  SGAD_CHECK_CUDA(cudaMemcpyAsync(&h, s, sizeof h, cudaMemcpyDeviceToHost, st));
  if (systems)
    SGAD_CHECK_CUDA(cudaMemcpyAsync(systems, sys, sizeof(double) * (size_t)max_iters * NE_VALS,
                                    cudaMemcpyDeviceToHost, st));
  if (cost_pairs)
    SGAD_CHECK_CUDA(cudaMemcpyAsync(cost_pairs, pairs, sizeof(double) * 2 * (size_t)max_iters,
                                    cudaMemcpyDeviceToHost, st));
  SGAD_CHECK_CUDA(cudaStreamSynchronize(st));
  // result: pose (12), final cost, iterations, inliers, converged, failed,
  // singular iteration (-1: none), systems logged
  for (int k = 0; k < 9; ++k) result[k] = h.pose.r[k];
  for (int k = 0; k < 3; ++k) result[9 + k] = h.pose.t[k];
  result[12] = h.final_cost;
  result[13] = h.iterations;
  result[14] = h.inliers;
  result[15] = h.converged;
  result[16] = h.failed;
  result[17] = h.singular_it;
  result[18] = h.n_systems;
  return SGAD_OK;
}

int sgad_track_to_world(const double* centers, const double* rotations, const double* scales,
                        const double* normals, int64_t n, const double* rot, const double* trans,
                        double* out_centers, double* out_rotations, double* out_normals,
                        double* out_cov6, void* stream) {
  SGAD_REQUIRE(n >= 0 && rot && trans, "sgad_track_to_world: bad arguments");
  if (n == 0) return SGAD_OK;
  SGAD_REQUIRE(centers && rotations && scales && normals && out_centers && out_rotations &&
                   out_normals && out_cov6,
               "sgad_track_to_world: null buffer");
  PoseArg P;
  for (int k = 0; k < 9; ++k) P.r[k] = rot[k];
  for (int k = 0; k < 3; ++k) P.t[k] = trans[k];
  k_to_world<<<nblk(n, 256), 256, 0, (cudaStream_t)stream>>>(centers, rotations, scales, normals,
                                                             n, P, out_centers, out_rotations,
                                                             out_normals, out_cov6);
  SGAD_LAUNCH_CHECK();
  return SGAD_OK;
}

}  // extern "C"
