// Windowed SSIM of two images and its gradient with respect to the first
// (the tau term of the mapping objective).  Restates
// /root/reference/pkg/src/raysplat/ssim.py:31-87 (used at mapper.py:126-147):
// 11x11 Gaussian window (sigma 1.5) applied as a zero-padded correlation,
// local statistics divided by the in-bounds window mass, C1 = 0.01^2,
// C2 = 0.03^2, mean over pixels and channels.
//
// The 2-D window is the outer product of one normalised 11-tap kernel, so
// every correlation is evaluated separably (horizontal then vertical pass)
// on a shared-memory tile with a 5-pixel halo: K_ssim_stats computes the five
// local statistics, the per-pixel SSIM (block-reduced into the mean) and the
// three maps the gradient correlates again; K_ssim_grad correlates those and
// assembles d(mssim)/d(img_a) = (corr(gm/mass) + 2 x corr(dv/mass) +
// y corr(dxy/mass)) / N (ssim.py:73-81), optionally folded straight into the
// mapping loss's colour upstream  rho sign(x - y) / N - tau grad.
// fp64 throughout, like the reference; the separable order of the 121
// products differs from scipy's 2-D loop by rounding only.

#include "common.cuh"

namespace sgad {

constexpr int SS_R = 5;                 // window radius
constexpr int SS_TW = 32, SS_TH = 8;    // output tile
constexpr int SS_IW = SS_TW + 2 * SS_R, SS_IH = SS_TH + 2 * SS_R;
constexpr int SS_THREADS = 256;
constexpr double SSIM_C1 = 0.01 * 0.01;
constexpr double SSIM_C2 = 0.03 * 0.03;

__constant__ double c_win[2 * SS_R + 1];  // g / sum(g), ssim.py:21-25

// in-bounds mass of the 1-D window centred at i (the 2-D mass of
// ssim.py:48 is the product of the row and column masses)
__device__ __forceinline__ double mass1(int i, int n) {
  double m = 0.0;
#pragma unroll
  for (int k = -SS_R; k <= SS_R; ++k)
    if (i + k >= 0 && i + k < n) m += c_win[k + SS_R];
  return m;
}

template <typename TB>
__device__ __forceinline__ double ld_img(const TB* p, int H, int W, int C, int y, int x, int c) {
  return (y >= 0 && y < H && x >= 0 && x < W) ? (double)p[((size_t)y * W + x) * C + c] : 0.0;
}

// K_ssim_stats: grid (ceil(W/32), ceil(H/8), C)
template <typename TB>
__global__ void __launch_bounds__(SS_THREADS)
k_ssim_stats(const double* __restrict__ a, const TB* __restrict__ b, int H, int W, int C,
             double* __restrict__ sum_out, double* __restrict__ maps) {
  __shared__ double xs[SS_IH][SS_IW], ys[SS_IH][SS_IW];
  __shared__ double hs[5][SS_IH][SS_TW];
  __shared__ double red[SS_THREADS / 32];
  const int c = blockIdx.z;
  const int x0 = blockIdx.x * SS_TW - SS_R, y0 = blockIdx.y * SS_TH - SS_R;
  for (int i = threadIdx.x; i < SS_IH * SS_IW; i += SS_THREADS) {
    const int r = i / SS_IW, q = i % SS_IW;
    xs[r][q] = ld_img(a, H, W, C, y0 + r, x0 + q, c);
    ys[r][q] = ld_img(b, H, W, C, y0 + r, x0 + q, c);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < SS_IH * SS_TW; i += SS_THREADS) {
    const int r = i / SS_TW, q = i % SS_TW;
    double s1 = 0, s2 = 0, s11 = 0, s22 = 0, s12 = 0;
#pragma unroll
    for (int k = 0; k <= 2 * SS_R; ++k) {
      const double g = c_win[k], xv = xs[r][q + k], yv = ys[r][q + k];
      s1 = fma(g, xv, s1);
      s2 = fma(g, yv, s2);
      s11 = fma(g, xv * xv, s11);
      s22 = fma(g, yv * yv, s22);
      s12 = fma(g, xv * yv, s12);
    }
    hs[0][r][q] = s1;
    hs[1][r][q] = s2;
    hs[2][r][q] = s11;
    hs[3][r][q] = s22;
    hs[4][r][q] = s12;
  }
  __syncthreads();
  double acc = 0.0;
  const size_t plane = (size_t)H * W * C;
  for (int i = threadIdx.x; i < SS_TH * SS_TW; i += SS_THREADS) {
    const int r = i / SS_TW, q = i % SS_TW;
    const int y = blockIdx.y * SS_TH + r, x = blockIdx.x * SS_TW + q;
    if (y >= H || x >= W) continue;
    double v[5] = {0, 0, 0, 0, 0};
#pragma unroll
    for (int k = 0; k <= 2 * SS_R; ++k) {
      const double g = c_win[k];
#pragma unroll
      for (int t = 0; t < 5; ++t) v[t] = fma(g, hs[t][r + k][q], v[t]);
    }
    const double mass = mass1(y, H) * mass1(x, W);
    const double m1 = v[0] / mass, m2 = v[1] / mass;
    const double vx = v[2] / mass - m1 * m1, vy = v[3] / mass - m2 * m2;
    const double vxy = v[4] / mass - m1 * m2;
    const double a1 = 2.0 * m1 * m2 + SSIM_C1, a2 = 2.0 * vxy + SSIM_C2;
    const double b1 = m1 * m1 + m2 * m2 + SSIM_C1, b2 = vx + vy + SSIM_C2;
    const double s = (a1 * a2) / (b1 * b2);
    acc += s;
    if (maps) {  // ssim.py:74-78, divided by the mass for the second correlation
      const double dv = -s / b2;
      const double dxy = 2.0 * a1 / (b1 * b2);
      const double dm = (2.0 / b1) * (m2 * a2 / b2 - m1 * s);
      const double gm = dm - 2.0 * m1 * dv - m2 * dxy;
      const size_t o = ((size_t)y * W + x) * C + c;
      maps[o] = gm / mass;
      maps[plane + o] = dv / mass;
      maps[2 * plane + o] = dxy / mass;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < SS_THREADS / 32; ++w) t += red[w];
    atomicAdd(sum_out, t);
  }
}

// K_ssim_grad: grid (ceil(W/32), ceil(H/8), C).  out = grad (upstream == 0)
// or the colour upstream kc * sign(a - b) - tau * grad (mapper.py:145-147).
template <typename TB>
__global__ void __launch_bounds__(SS_THREADS)
k_ssim_grad(const double* __restrict__ a, const TB* __restrict__ b, int H, int W, int C,
            const double* __restrict__ maps, double inv_n, double kc, double tau,
            int upstream, double* __restrict__ out) {
  __shared__ double ms[3][SS_IH][SS_IW];
  __shared__ double hs[3][SS_IH][SS_TW];
  const int c = blockIdx.z;
  const int x0 = blockIdx.x * SS_TW - SS_R, y0 = blockIdx.y * SS_TH - SS_R;
  const size_t plane = (size_t)H * W * C;
  for (int i = threadIdx.x; i < SS_IH * SS_IW; i += SS_THREADS) {
    const int r = i / SS_IW, q = i % SS_IW;
    const int y = y0 + r, x = x0 + q;
    const bool in = y >= 0 && y < H && x >= 0 && x < W;
    const size_t o = ((size_t)y * W + x) * C + c;
#pragma unroll
    for (int t = 0; t < 3; ++t) ms[t][r][q] = in ? maps[t * plane + o] : 0.0;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < SS_IH * SS_TW; i += SS_THREADS) {
    const int r = i / SS_TW, q = i % SS_TW;
#pragma unroll
    for (int t = 0; t < 3; ++t) {
      double s = 0.0;
#pragma unroll
      for (int k = 0; k <= 2 * SS_R; ++k) s = fma(c_win[k], ms[t][r][q + k], s);
      hs[t][r][q] = s;
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < SS_TH * SS_TW; i += SS_THREADS) {
    const int r = i / SS_TW, q = i % SS_TW;
    const int y = blockIdx.y * SS_TH + r, x = blockIdx.x * SS_TW + q;
    if (y >= H || x >= W) continue;
    double v[3] = {0, 0, 0};
#pragma unroll
    for (int k = 0; k <= 2 * SS_R; ++k) {
      const double g = c_win[k];
#pragma unroll
      for (int t = 0; t < 3; ++t) v[t] = fma(g, hs[t][r + k][q], v[t]);
    }
    const size_t o = ((size_t)y * W + x) * C + c;
    const double xv = a[o], yv = (double)b[o];
    const double grad = (v[0] + 2.0 * xv * v[1] + yv * v[2]) * inv_n;
    if (upstream) {
      const double d = xv - yv;
      const double sg = d > 0.0 ? 1.0 : (d < 0.0 ? -1.0 : 0.0);
      out[o] = kc * sg - tau * grad;
    } else {
      out[o] = grad;
    }
  }
}

static int upload_window() {
  static int done[64] = {0};  // per device (constant memory lives per context)
  int dev = 0;
  SGAD_CHECK_CUDA(cudaGetDevice(&dev));
  if (dev < 64 && done[dev]) return SGAD_OK;
  double g[2 * SS_R + 1], s = 0.0;
  for (int i = 0; i <= 2 * SS_R; ++i) {
    const double ax = (double)(i - SS_R) / 1.5;
    g[i] = exp(-0.5 * ax * ax);
    s += g[i];
  }
  for (int i = 0; i <= 2 * SS_R; ++i) g[i] /= s;
  SGAD_CHECK_CUDA(cudaMemcpyToSymbol(c_win, g, sizeof g));
  if (dev < 64) done[dev] = 1;
  return SGAD_OK;
}

}  // namespace sgad

using namespace sgad;

extern "C" {

int sgad_ssim_workspace_size(int32_t height, int32_t width, int32_t channels, int64_t* bytes) {
  SGAD_REQUIRE(bytes && height >= 0 && width >= 0 && channels > 0, "sgad_ssim_workspace_size: bad args");
  *bytes = (int64_t)sizeof(double) * 3 * height * width * channels;
  return SGAD_OK;
}

int sgad_ssim(const double* img_a, const void* img_b, int32_t b_is_f32, int32_t height,
              int32_t width, int32_t channels, double* sum_out, double* grad_out,
              double* workspace, double kc, double tau, int32_t upstream, void* stream_) {
  SGAD_REQUIRE(img_a && img_b && sum_out && height > 0 && width > 0 && channels > 0,
               "sgad_ssim: bad args");
  SGAD_REQUIRE(!grad_out || workspace, "sgad_ssim: the gradient needs the workspace");
  if (int rc = upload_window()) return rc;
  cudaStream_t st = (cudaStream_t)stream_;
  const dim3 grid((unsigned)((width + SS_TW - 1) / SS_TW), (unsigned)((height + SS_TH - 1) / SS_TH),
                  (unsigned)channels);
  double* maps = grad_out ? workspace : nullptr;
  if (b_is_f32) {
    k_ssim_stats<float><<<grid, SS_THREADS, 0, st>>>(img_a, (const float*)img_b, height, width,
                                                      channels, sum_out, maps);
  } else {
    k_ssim_stats<double><<<grid, SS_THREADS, 0, st>>>(img_a, (const double*)img_b, height, width,
                                                       channels, sum_out, maps);
  }
  SGAD_LAUNCH_CHECK();
  if (!grad_out) return SGAD_OK;
  const double inv_n = 1.0 / ((double)height * width * channels);
  if (b_is_f32) {
    k_ssim_grad<float><<<grid, SS_THREADS, 0, st>>>(img_a, (const float*)img_b, height, width,
                                                     channels, maps, inv_n, kc, tau, upstream,
                                                     grad_out);
  } else {
    k_ssim_grad<double><<<grid, SS_THREADS, 0, st>>>(img_a, (const double*)img_b, height, width,
                                                      channels, maps, inv_n, kc, tau, upstream,
                                                      grad_out);
  }
  SGAD_LAUNCH_CHECK();
  return SGAD_OK;
}

}  // extern "C"
