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

/* 2^(j/32), j = 0..31: the table of sgad_exp_neg (literal values, so the
 * GPU's shared-memory copy and the oracle's array hold identical bits) */
#define SGAD_EXP2_TABLE \
    1.0, 1.0218971486541166, 1.0442737824274138, 1.0671404006768237, \
    1.0905077326652577, 1.1143867425958924, 1.1387886347566916, 1.1637248587775775, \
    1.189207115002721, 1.215247359980469, 1.241857812073484, 1.2690509571917332, \
    1.2968395546510096, 1.3252366431597413, 1.3542555469368927, 1.383909881963832, \
    1.4142135623730951, 1.4451808069770467, 1.4768261459394993, 1.5091644275934228, \
    1.5422108254079407, 1.5759808451078865, 1.6104903319492543, 1.645755478153965, \
    1.681792830507429, 1.718619298122478, 1.7562521603732995, 1.7947090750031072, \
    1.8340080864093424, 1.8741676341103, 1.9152065613971474, 1.9571441241754002

/* Compositing weight exp(x) for -700 < x <= 0: table-driven (32 entries,
 * |r| <= ln2/64, degree-6 Taylor, error ~1 ulp).  Used by both the kernels
 * and the oracle for w = exp(-0.5 d2 / s2); differs from numpy's exp by at
 * most an ulp or two (the images' parity bar is 1e-4). */
SGAD_HD double sgad_exp_neg(double x, const double* tab) {
  const double n = rint(SG_MUL(x, 46.16624130844683));
  double r = SG_FMA(-n, 0.021660848520696163, x);
  r = SG_FMA(-n, 8.718021277417983e-10, r);
  double p = 0.001388888888888889;      /* 1/6! */
  p = SG_FMA(p, r, 0.008333333333333333);  /* 1/5! */
  p = SG_FMA(p, r, 0.041666666666666664);  /* 1/4! */
  p = SG_FMA(p, r, 0.16666666666666666);   /* 1/3! */
  p = SG_FMA(p, r, 0.5);
  p = SG_FMA(p, r, 1.0);
  p = SG_FMA(p, r, 1.0);
  const int ni = (int)n;
  const int j = ni & 31;
  const int k = ni >> 5; /* == (ni - j) / 32: ni - j is a multiple of 32 */
#if defined(__CUDA_ARCH__)
  /* x * 2^k by adding k to the exponent field: exact (identical to the
   * multiplication) while the result stays normal, i.e. x > -700 here */
  return __longlong_as_double(__double_as_longlong(SG_MUL(tab[j], p)) + ((long long)k << 52));
#else
  return SG_MUL(SG_MUL(tab[j], p), sgad_pow2i(k));
#endif
}

/* raysplat/gaussians.py:36-42: branch-stable logistic */
SGAD_HD double sgad_sigmoid(double x) {
  if (x >= 0.0) return SG_DIV(1.0, SG_ADD(1.0, sgad_exp(-x)));
  double ex = sgad_exp(x);
  return SG_DIV(ex, SG_ADD(1.0, ex));
}

#endif /* SGAD_NUMERICS_H */
