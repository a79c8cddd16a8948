/*
 * sgad_numerics.h -- the fp64 operation conventions shared by the sm_100a
 * kernels and the CPU oracle.
 *
 * The reference (raysplat, /root/reference/pkg/src/raysplat/rasterizer.py)
 * evaluates projection and compositing in fp64 with no fused multiply-add:
 * numpy ufuncs round every operation, and the Numba kernels are compiled
 * without fast-math (rasterizer.py:178,221,272), so LLVM never contracts.
 * The exceptions are the BLAS products `rays @ R.T` (rasterizer.py:95),
 * which OpenBLAS evaluates as fma(r2, R[j,2], fma(r1, R[j,1], r0 * R[j,0])).
 *
 * nvcc contracts a*b+c into DFMA by default, so every order-sensitive
 * operation in the kernels goes through these macros, and the oracle is
 * compiled with -ffp-contract=off.  sgad_exp is a fixed Cody-Waite +
 * degree-13 Taylor evaluation so that the GPU and the oracle produce the
 * same bits for exp (libm and CUDA's exp both differ from numpy's SIMD exp by
 * at most an ulp; sharing one restatement makes GPU == oracle bit-exact).
 */
#ifndef SGAD_NUMERICS_H
#define SGAD_NUMERICS_H

#include <math.h>
#include <stdint.h>
#include <string.h>

#if defined(__CUDACC__)
#define SGAD_HD __host__ __device__ __forceinline__
#else
#define SGAD_HD static inline
#endif

#if defined(__CUDA_ARCH__)
#define SG_MUL(a, b) __dmul_rn((a), (b))
#define SG_ADD(a, b) __dadd_rn((a), (b))
#define SG_SUB(a, b) __dsub_rn((a), (b))
#define SG_DIV(a, b) __ddiv_rn((a), (b))
#define SG_FMA(a, b, c) __fma_rn((a), (b), (c))
#else
#define SG_MUL(a, b) ((a) * (b))
#define SG_ADD(a, b) ((a) + (b))
#define SG_SUB(a, b) ((a) - (b))
#define SG_DIV(a, b) ((a) / (b))
#define SG_FMA(a, b, c) fma((a), (b), (c))
#endif

/* Reference constants, rasterizer.py:28-31 */
#define SGAD_ALPHA_MAX 0.999
#define SGAD_TRANSMITTANCE_MIN 1e-4
#define SGAD_Z_NEAR 1e-6
#define SGAD_TILE 16

SGAD_HD double sgad_pow2i(int k) {
  /* exact 2^k for k in [-1022, 1023] */
#if defined(__CUDA_ARCH__)
  return __longlong_as_double((long long)(k + 1023) << 52);
#else
  uint64_t bits = (uint64_t)(k + 1023) << 52;
  double d;
  memcpy(&d, &bits, sizeof d);
  return d;
#endif
}

SGAD_HD double sgad_exp(double x) {
  if (x != x) return x;
  if (x > 709.782712893384) return INFINITY;
  if (x < -745.1332191019412) return 0.0;
  const double inv_ln2 = 1.4426950408889634;
  const double ln2_hi = 6.93147180369123816490e-01;
  const double ln2_lo = 1.90821492927058770002e-10;
  double k = rint(SG_MUL(x, inv_ln2));
  double r = SG_FMA(-k, ln2_hi, x);
  r = SG_FMA(-k, ln2_lo, r);
  double p = 1.6059043836821613e-10;      /* 1/13! */
  p = SG_FMA(p, r, 2.08767569878681e-09);  /* 1/12! */
  p = SG_FMA(p, r, 2.505210838544172e-08); /* 1/11! */
  p = SG_FMA(p, r, 2.755731922398589e-07); /* 1/10! */
  p = SG_FMA(p, r, 2.7557319223985893e-06);/* 1/9!  */
  p = SG_FMA(p, r, 2.48015873015873e-05);  /* 1/8!  */
  p = SG_FMA(p, r, 0.0001984126984126984); /* 1/7!  */
  p = SG_FMA(p, r, 0.001388888888888889);  /* 1/6!  */
  p = SG_FMA(p, r, 0.008333333333333333);  /* 1/5!  */
  p = SG_FMA(p, r, 0.041666666666666664);  /* 1/4!  */
  p = SG_FMA(p, r, 0.16666666666666666);   /* 1/3!  */
  p = SG_FMA(p, r, 0.5);
  p = SG_FMA(p, r, 1.0);
  p = SG_FMA(p, r, 1.0);
  int ki = (int)k;
  if (ki > 1023) return SG_MUL(SG_MUL(p, sgad_pow2i(1023)), sgad_pow2i(ki - 1023));
  if (ki < -1021) return SG_MUL(SG_MUL(p, sgad_pow2i(ki + 600)), sgad_pow2i(-600));
  return SG_MUL(p, sgad_pow2i(ki));
}

/* raysplat/gaussians.py:36-42: branch-stable logistic */
SGAD_HD double sgad_sigmoid(double x) {
  if (x >= 0.0) return SG_DIV(1.0, SG_ADD(1.0, sgad_exp(-x)));
  double ex = sgad_exp(x);
  return SG_DIV(ex, SG_ADD(1.0, ex));
}

#endif /* SGAD_NUMERICS_H */
