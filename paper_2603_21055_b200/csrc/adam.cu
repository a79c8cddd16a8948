// K6: Adam over the six learnable planes of a keyframe window
// (restates /root/reference/pkg/src/raysplat/mapper.py:73-95).
//
// params [F, 7, HW] fp32 (base, delta, log_radius, logit, R, G, B)
// grads  [F*HW, 8]  (delta, radius, logit, R, G, B, -, -), consumed and zeroed
// m, v   [F, 6, HW] fp32 (delta, log_radius, logit, R, G, B)
// Arithmetic in fp64 per element, mirroring the reference's in-place numpy
// sequence; storage fp32 (BASELINE: parameters in fp32).
#include "common.cuh"

namespace sgad {

struct AdamArgs {
  double lr[6];
  double b1, b2, eps, bc1, bc2;
  int update_delta;
  const int32_t* skip;  // device flag: consume (zero) the gradients, update nothing
  const int32_t* t_dev;  // device step count (fp32 window): bc1, bc2 from it, not from the host
};

// bias corrections 1 / (1 - beta^t) of the fp32 window update
__device__ __forceinline__ void inv_bias(const AdamArgs& a, float& ib1, float& ib2) {
  if (a.t_dev) {
    const double t = (double)*a.t_dev;
    ib1 = (float)(1.0 / (1.0 - pow(a.b1, t)));
    ib2 = (float)(1.0 / (1.0 - pow(a.b2, t)));
  } else {
    ib1 = (float)(1.0 / a.bc1);
    ib2 = (float)(1.0 / a.bc2);
  }
}

template <typename P>
__global__ void __launch_bounds__(256)
k_adam(P* __restrict__ params, P* __restrict__ grads, P* __restrict__ m,
       P* __restrict__ v, int64_t n_frames, int64_t hw, AdamArgs a) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_frames * hw) return;
  const int64_t f = i / hw, p = i - f * hw;
  P* gp = grads + 8 * i;
  double gr[6];
#pragma unroll
  for (int c = 0; c < 6; ++c) {
    gr[c] = (double)gp[c];
    gp[c] = (P)0;
  }
  if (a.skip && *a.skip) return;
  P* pf = params + f * 7 * hw + p;
  P* mf = m + f * 6 * hw + p;
  P* vf = v + f * 6 * hw + p;
  // mapper.py:77: the radius gradient is chained onto log-radius
  const double radius = exp((double)pf[2 * hw]);
  const double g[6] = {gr[0], SG_MUL(gr[1], radius), gr[2], gr[3], gr[4], gr[5]};
#pragma unroll
  for (int c = 0; c < 6; ++c) {
    if (c == 0 && !a.update_delta) continue;
    // m *= b1; m += (1 - b1) g; v *= b2; v += (1 - b2) g g (in-place numpy order)
    const double mm = SG_ADD(SG_MUL((double)mf[c * hw], a.b1), SG_MUL(SG_SUB(1.0, a.b1), g[c]));
    const double vv = SG_ADD(SG_MUL((double)vf[c * hw], a.b2),
                             SG_MUL(SG_MUL(SG_SUB(1.0, a.b2), g[c]), g[c]));
    const double mhat = SG_DIV(mm, a.bc1), vhat = SG_DIV(vv, a.bc2);
    double prm = (double)pf[(c + 1) * hw];
    prm = SG_SUB(prm, SG_DIV(SG_MUL(a.lr[c], mhat), SG_ADD(sqrt(vhat), a.eps)));
    if (c >= 3) prm = fmin(fmax(prm, 0.0), 1.0);  // colour clip, mapper.py:95
    pf[(c + 1) * hw] = (P)prm;
    mf[c * hw] = (P)mm;
    vf[c * hw] = (P)vv;
  }
}

// The window engine's fp32 parameters (delta D4): the same update in fp32
// arithmetic -- reciprocals of the bias corrections precomputed, fast exp /
// sqrt -- so the step is bound by its 216 bytes per Gaussian, not by fp64
// division and square-root sequences.
// grid (ceil(hw / 256), n_frames): no 64-bit division per thread
__global__ void __launch_bounds__(256)
k_adam_f32(float* __restrict__ params, float* __restrict__ grads, float* __restrict__ m,
           float* __restrict__ v, int64_t hw, AdamArgs a) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= hw) return;
  const int64_t f = blockIdx.y, i = f * hw + p;
  float4* gp = reinterpret_cast<float4*>(grads + 8 * i);
  const float4 g0 = gp[0], g1 = gp[1];
  gp[0] = make_float4(0.f, 0.f, 0.f, 0.f);
  gp[1] = make_float4(0.f, 0.f, 0.f, 0.f);
  if (a.skip && *a.skip) return;
  float* pf = params + f * 7 * hw + p;
  float* mf = m + f * 6 * hw + p;
  float* vf = v + f * 6 * hw + p;
  const float b1 = (float)a.b1, b2 = (float)a.b2, eps = (float)a.eps;
  float ib1, ib2;
  inv_bias(a, ib1, ib2);
  // every load issued before any store (18 independent streams in flight)
  float m0[6], v0[6], p0[6];
#pragma unroll
  for (int c = 0; c < 6; ++c) {
    m0[c] = mf[c * hw];
    v0[c] = vf[c * hw];
    p0[c] = pf[(c + 1) * hw];
  }
  const float g[6] = {g0.x, g0.y * __expf(p0[1]), g0.z, g0.w, g1.x, g1.y};
#pragma unroll
  for (int c = 0; c < 6; ++c) {
    if (c == 0 && !a.update_delta) continue;
    const float mm = m0[c] * b1 + (1.0f - b1) * g[c];
    const float vv = v0[c] * b2 + (1.0f - b2) * g[c] * g[c];
    float prm = p0[c] - (float)a.lr[c] * (mm * ib1) / (sqrtf(vv * ib2) + eps);
    if (c >= 3) prm = fminf(fmaxf(prm, 0.0f), 1.0f);  // colour clip, mapper.py:95
    pf[(c + 1) * hw] = prm;
    mf[c * hw] = mm;
    vf[c * hw] = vv;
  }
}

// The same update, four consecutive Gaussians per thread (hw % 4 == 0):
// 16-byte loads and stores on every plane, a quarter of the instructions.
__global__ void __launch_bounds__(256)
k_adam_f32x4(float* __restrict__ params, float* __restrict__ grads, float* __restrict__ m,
             float* __restrict__ v, int64_t hw, AdamArgs a) {
  const int64_t p = 4 * ((int64_t)blockIdx.x * blockDim.x + threadIdx.x);
  if (p >= hw) return;
  const int64_t f = blockIdx.y, i = f * hw + p;
  float4* gp = reinterpret_cast<float4*>(grads + 8 * i);
  float4 gr[8];  // Gaussian u: gr[2u] = (delta, radius, logit, R), gr[2u + 1] = (G, B, -, -)
#pragma unroll
  for (int q = 0; q < 8; ++q) gr[q] = gp[q];
#pragma unroll
  for (int q = 0; q < 8; ++q) gp[q] = make_float4(0.f, 0.f, 0.f, 0.f);
  if (a.skip && *a.skip) return;
  float* pf = params + f * 7 * hw + p;
  float* mf = m + f * 6 * hw + p;
  float* vf = v + f * 6 * hw + p;
  const float b1 = (float)a.b1, b2 = (float)a.b2, eps = (float)a.eps;
  float ib1, ib2;
  inv_bias(a, ib1, ib2);
  float4 m0[6], v0[6], p0[6];
#pragma unroll
  for (int c = 0; c < 6; ++c) {
    m0[c] = *reinterpret_cast<const float4*>(mf + c * hw);
    v0[c] = *reinterpret_cast<const float4*>(vf + c * hw);
    p0[c] = *reinterpret_cast<const float4*>(pf + (c + 1) * hw);
  }
#pragma unroll
  for (int c = 0; c < 6; ++c) {
    if (c == 0 && !a.update_delta) continue;
    float* pm = reinterpret_cast<float*>(&m0[c]);
    float* pv = reinterpret_cast<float*>(&v0[c]);
    float* pp = reinterpret_cast<float*>(&p0[c]);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const float4 ga = gr[2 * u], gb = gr[2 * u + 1];
      float g = c == 0 ? ga.x : c == 1 ? ga.y : c == 2 ? ga.z : c == 3 ? ga.w : c == 4 ? gb.x : gb.y;
      if (c == 1) g *= __expf(pp[u]);  // radius -> log radius (old value, read before its update)
      const float mm = pm[u] * b1 + (1.0f - b1) * g;
      const float vv = pv[u] * b2 + (1.0f - b2) * g * g;
      float prm = pp[u] - (float)a.lr[c] * (mm * ib1) / (sqrtf(vv * ib2) + eps);
      if (c >= 3) prm = fminf(fmaxf(prm, 0.0f), 1.0f);  // colour clip, mapper.py:95
      pm[u] = mm;
      pv[u] = vv;
      pp[u] = prm;
    }
    *reinterpret_cast<float4*>(mf + c * hw) = m0[c];
    *reinterpret_cast<float4*>(vf + c * hw) = v0[c];
    *reinterpret_cast<float4*>(pf + (c + 1) * hw) = p0[c];
  }
}

}  // namespace sgad

extern "C" int sgad_adam_step(void* params, void* grads, void* m, void* v, int64_t n_frames,
                              int64_t hw, const double* lr, double beta1, double beta2, double eps,
                              double bc1, double bc2, int32_t update_delta, int32_t f64,
                              const int32_t* skip, const int32_t* step_dev, void* stream) {
  SGAD_REQUIRE(params && grads && m && v && lr && n_frames >= 0 && hw >= 0,
               "sgad_adam_step: bad arguments");
  const int64_t n = n_frames * hw;
  if (n == 0) return SGAD_OK;
  sgad::AdamArgs a;
  for (int c = 0; c < 6; ++c) a.lr[c] = lr[c];
  a.b1 = beta1;
  a.b2 = beta2;
  a.eps = eps;
  a.bc1 = bc1;
  a.bc2 = bc2;
  a.update_delta = update_delta;
  a.skip = skip;
  a.t_dev = f64 ? nullptr : step_dev;
  const unsigned nb = (unsigned)((n + 255) / 256);
  if (f64)
    sgad::k_adam<double><<<nb, 256, 0, (cudaStream_t)stream>>>(
        (double*)params, (double*)grads, (double*)m, (double*)v, n_frames, hw, a);
  else if (hw % 4 == 0 && ((uintptr_t)params | (uintptr_t)grads | (uintptr_t)m | (uintptr_t)v) % 16 == 0)
    sgad::k_adam_f32x4<<<dim3((unsigned)((hw / 4 + 255) / 256), (unsigned)n_frames), 256, 0,
                          (cudaStream_t)stream>>>((float*)params, (float*)grads, (float*)m,
                                                  (float*)v, hw, a);
  else
    sgad::k_adam_f32<<<dim3((unsigned)((hw + 255) / 256), (unsigned)n_frames), 256, 0,
                        (cudaStream_t)stream>>>((float*)params, (float*)grads, (float*)m,
                                                (float*)v, hw, a);
  SGAD_LAUNCH_CHECK();
  return SGAD_OK;
}
