// IRLS normal equations of the render-based pose initialiser
// (/root/reference/pkg/src/raysplat/tracker.py:400-410):
//   J[:, k] = (r(+h e_k) - r(-h e_k)) / 2h          (central differences)
//   w = 1 / max(|r + J xi|, 1e-3)
//   H = J^T diag(w) J,  g = J^T (w r)
// in one pass over the residual rows (12 perturbed renders + the base
// residual, device fp64, component-major so every load is coalesced), with
// the Jacobian never materialised.  Each block reduces its rows' 27 sums
// (21 unique H entries + 6 of g) in fp64 and writes a partial; a one-block
// kernel adds the partials in a fixed order (deterministic); the 6x6
// least-squares solve stays on the host, as in the reference.

#include "common.cuh"

namespace sgad {

constexpr int IRLS_THREADS = 256;
constexpr int IRLS_BLOCKS = 592;  // 4 per SM
constexpr int IRLS_NV = 27;

struct IrlsArgs {
  double xi[6];
  double inv2h;
};

__global__ void __launch_bounds__(IRLS_THREADS)
k_irls_partial(const double* __restrict__ rows, const double* __restrict__ r, int64_t n,
               IrlsArgs a, double* __restrict__ partial) {
  double acc[IRLS_NV];
#pragma unroll
  for (int t = 0; t < IRLS_NV; ++t) acc[t] = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)IRLS_THREADS + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * IRLS_THREADS) {
    double j[6];
    double pred = r[i];
#pragma unroll
    for (int k = 0; k < 6; ++k) {
      j[k] = (rows[(2 * k) * n + i] - rows[(2 * k + 1) * n + i]) * a.inv2h;
      pred = fma(j[k], a.xi[k], pred);
    }
    const double w = 1.0 / fmax(fabs(pred), 1e-3);
    const double wr = w * r[i];
    int t = 0;
#pragma unroll
    for (int p = 0; p < 6; ++p) {
      const double wp = w * j[p];
#pragma unroll
      for (int q = p; q < 6; ++q) {
        acc[t] = fma(wp, j[q], acc[t]);
        ++t;
      }
    }
#pragma unroll
    for (int p = 0; p < 6; ++p) acc[21 + p] = fma(wr, j[p], acc[21 + p]);
  }
  __shared__ double red[IRLS_NV][IRLS_THREADS / 32];
#pragma unroll
  for (int t = 0; t < IRLS_NV; ++t) {
    double v = acc[t];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) red[t][threadIdx.x >> 5] = v;
  }
  __syncthreads();
  if (threadIdx.x < IRLS_NV) {
    double v = 0.0;
    for (int w = 0; w < IRLS_THREADS / 32; ++w) v += red[threadIdx.x][w];
    partial[blockIdx.x * IRLS_NV + threadIdx.x] = v;
  }
}

__global__ void k_irls_final(const double* __restrict__ partial, int nblk, double* __restrict__ out) {
  const int t = threadIdx.x;
  if (t >= IRLS_NV) return;
  double v = 0.0;
  for (int b = 0; b < nblk; ++b) v += partial[b * IRLS_NV + t];
  out[t] = v;
}

}  // namespace sgad

using namespace sgad;

extern "C" int sgad_irls_normal_eqs(const double* rows, const double* r, int64_t n,
                                    const double* xi, double h, double* partial, double* out,
                                    void* stream) {
  SGAD_REQUIRE(rows && r && xi && partial && out && n > 0 && h > 0.0,
               "sgad_irls_normal_eqs: bad arguments");
  IrlsArgs a;
  for (int k = 0; k < 6; ++k) a.xi[k] = xi[k];
  a.inv2h = 1.0 / (2.0 * h);
  int nblk = (int)((n + IRLS_THREADS - 1) / IRLS_THREADS);
  if (nblk > IRLS_BLOCKS) nblk = IRLS_BLOCKS;
  k_irls_partial<<<nblk, IRLS_THREADS, 0, (cudaStream_t)stream>>>(rows, r, n, a, partial);
  SGAD_LAUNCH_CHECK();
  k_irls_final<<<1, 32, 0, (cudaStream_t)stream>>>(partial, nblk, out);
  SGAD_LAUNCH_CHECK();
  return SGAD_OK;
}
