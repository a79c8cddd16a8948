// Harmonic depth inpainting (Jacobi sweeps of the grid Laplace equation with
// the valid pixels held fixed), restating the iteration of
// /root/reference/pkg/src/raysplat/datasets.py:368-398 (inpaint_depth):
//   avg = 0.25 * (up + down + left + right)   (edge-replicated borders,
//                                              summed in that order)
//   delta = max over holes |avg - out|; out[holes] = avg[holes];
//   stop after the sweep whose delta < tol, or after max_iters sweeps.
// Each sweep is one kernel over ping-pong buffers that also max-reduces the
// sweep's delta; a one-thread kernel then raises a device flag once the
// delta is below tol, and later sweeps return immediately -- so all sweeps
// are queued without host round trips and the result is bit-identical to
// the reference's loop.  (The nearest-valid seeding that precedes the sweeps
// is scipy's distance transform, called on the host as the reference does.)

#include "common.cuh"

namespace sgad {

struct InpaintState {
  unsigned long long delta_bits;  // max |avg - out| of the running sweep (non-negative bits)
  uint32_t done;
  uint32_t applied;               // sweeps applied
};

__global__ void k_inpaint_sweep(const double* __restrict__ src, double* __restrict__ dst,
                                const uint8_t* __restrict__ hole, int H, int W,
                                InpaintState* __restrict__ st) {
  if (st->done) return;  // converged on an earlier sweep
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y * blockDim.y + threadIdx.y;
  double d = 0.0;
  if (x < W && y < H) {
    const int64_t p = (int64_t)y * W + x;
    const double c = src[p];
    if (hole[p]) {
      const double up = src[(int64_t)(y > 0 ? y - 1 : 0) * W + x];
      const double dn = src[(int64_t)(y < H - 1 ? y + 1 : H - 1) * W + x];
      const double lf = src[(int64_t)y * W + (x > 0 ? x - 1 : 0)];
      const double rt = src[(int64_t)y * W + (x < W - 1 ? x + 1 : W - 1)];
      const double avg = __dmul_rn(0.25, __dadd_rn(__dadd_rn(__dadd_rn(up, dn), lf), rt));
      d = fabs(__dsub_rn(avg, c));
      dst[p] = avg;
    } else {
      dst[p] = c;
    }
  }
  // block max, then one atomic per block (non-negative doubles order like their bits)
  unsigned long long b = (unsigned long long)__double_as_longlong(d);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) b = max(b, __shfl_xor_sync(0xffffffffu, b, o));
  __shared__ unsigned long long red[8];
  const int t = threadIdx.y * blockDim.x + threadIdx.x;
  if ((t & 31) == 0) red[t >> 5] = b;
  __syncthreads();
  if (t == 0) {
    for (int w = 1; w < (int)(blockDim.x * blockDim.y) / 32; ++w) b = max(b, red[w]);
    atomicMax(&st->delta_bits, b);
  }
}

__global__ void k_inpaint_check(InpaintState* __restrict__ st, double tol) {
  if (st->done) return;
  st->applied += 1;
  if (__longlong_as_double((long long)st->delta_bits) < tol) st->done = 1;
  st->delta_bits = 0ull;
}

}  // namespace sgad

using namespace sgad;

extern "C" {

int sgad_inpaint_jacobi(double* depth, const uint8_t* hole, int32_t height, int32_t width,
                        int32_t max_iters, double tol, double* scratch, int32_t* sweeps,
                        void* stream_) {
  SGAD_REQUIRE(depth && hole && scratch && sweeps && height > 0 && width > 0 && max_iters >= 0,
               "sgad_inpaint_jacobi: bad arguments");
  cudaStream_t st = (cudaStream_t)stream_;
  DevBuf state;
  SGAD_CHECK_CUDA(state.ensure(sizeof(InpaintState)));
  SGAD_CHECK_CUDA(cudaMemsetAsync(state.p, 0, sizeof(InpaintState), st));
  InpaintState* s = state.as<InpaintState>();
  const dim3 blk(32, 8), grid((unsigned)((width + 31) / 32), (unsigned)((height + 7) / 8));
  double* buf[2] = {depth, scratch};
  for (int it = 0; it < max_iters; ++it) {
    k_inpaint_sweep<<<grid, blk, 0, st>>>(buf[it & 1], buf[(it + 1) & 1], hole, height, width, s);
    SGAD_LAUNCH_CHECK();
    k_inpaint_check<<<1, 1, 0, st>>>(s, tol);
    SGAD_LAUNCH_CHECK();
  }
  InpaintState h;
  SGAD_CHECK_CUDA(cudaMemcpyAsync(&h, s, sizeof h, cudaMemcpyDeviceToHost, st));
  SGAD_CHECK_CUDA(cudaStreamSynchronize(st));
  state.release();
  *sweeps = (int32_t)h.applied;
  if (h.applied & 1)  // the result sits in the scratch buffer
    SGAD_CHECK_CUDA(cudaMemcpyAsync(depth, scratch, sizeof(double) * height * width,
                                    cudaMemcpyDeviceToDevice, st));
  return SGAD_OK;
}

}  // extern "C"
