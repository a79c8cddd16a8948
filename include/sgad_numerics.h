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

/* 2^(j/128), j = 0..127 (correctly rounded): the table of sgad_exp_neg
 * (literal values, so the GPU's shared-memory copy and the oracle's array
 * hold identical bits) */
#define SGAD_EXP2_TABLE_N 128
#define SGAD_EXP2_TABLE \
    1.0, 1.0054299011128027, 1.0108892860517005, 1.016378314910953, \
    1.0218971486541166, 1.0274459491187637, 1.0330248790212284, 1.0386341019613787, \
    1.0442737824274138, 1.0499440858006872, 1.0556451783605572, 1.061377227289262, \
    1.0671404006768237, 1.0729348675259756, 1.0787607977571199, 1.0846183622133092, \
    1.0905077326652577, 1.0964290818163769, 1.102382583307841, 1.1083684117236787, \
    1.1143867425958924, 1.1204377524096067, 1.1265216186082418, 1.1326385195987192, \
    1.1387886347566916, 1.1449721444318042, 1.1511892299529827, 1.1574400736337511, \
    1.1637248587775775, 1.1700437696832502, 1.1763969916502812, 1.182784710984341, \
    1.189207115002721, 1.1956643920398273, 1.202156731452703, 1.2086843236265816, \
    1.215247359980469, 1.2218460329727576, 1.22848053610687, 1.2351510639369334, \
    1.241857812073484, 1.2486009771892048, 1.255380757024691, 1.2621973503942507, \
    1.2690509571917332, 1.275941778396392, 1.2828700160787783, 1.2898358734066657, \
    1.2968395546510096, 1.3038812651919358, 1.3109612115247644, 1.318079601266064, \
    1.3252366431597413, 1.3324325470831615, 1.339667524053303, 1.3469417862329458, \
    1.3542555469368927, 1.3616090206382248, 1.3690024229745905, 1.3764359707545302, \
    1.383909881963832, 1.3914243757719262, 1.3989796725383112, 1.4065759938190154, \
    1.4142135623730951, 1.4218926021691656, 1.42961333839197, 1.4373759974489824, \
    1.4451808069770467, 1.4530279958490526, 1.460917794180647, 1.4688504333369818, \
    1.4768261459394993, 1.4848451658727524, 1.4929077282912648, 1.5010140696264256, \
    1.5091644275934228, 1.5173590411982147, 1.5255981507445384, 1.533881997840956, \
    1.5422108254079407, 1.550584877685, 1.559004400237837, 1.567469639965553, \
    1.5759808451078865, 1.5845382652524937, 1.593142151342267, 1.6017927556826934, \
    1.6104903319492543, 1.6192351351948637, 1.6280274218573478, 1.6368674497669644, \
    1.645755478153965, 1.6546917676561943, 1.6636765803267364, 1.6727101796415966, \
    1.681792830507429, 1.6909247992693053, 1.7001063537185235, 1.709337763100463, \
    1.718619298122478, 1.7279512309618377, 1.7373338352737062, 1.746767386199169, \
    1.7562521603732995, 1.7657884359332727, 1.7753764925265212, 1.785016611318935, \
    1.7947090750031072, 1.804454167806624, 1.8142521755003989, 1.8241033854070534, \
    1.8340080864093424, 1.843966568958626, 1.8539791250833855, 1.864046048397789, \
    1.8741676341103, 1.8843441790323345, 1.8945759815869656, 1.9048633418176741, \
    1.9152065613971474, 1.925605943636125, 1.9360617934922943, 1.9465744175792332, \
    1.9571441241754002, 1.9677712232331759, 1.978456026387951, 1.9891988469672663

/* Compositing weight exp(x) for -700 < x <= 0: table-driven (128 entries,
 * |r| <= ln2/256, degree-5 Taylor, error <= 1.6 ulp).  The constants that
 * only steer the reduction (128/ln2, the high part of ln2/128) and the two
 * highest coefficients are rounded to 20-bit mantissas -- exact as 32-bit
 * immediates of DFMA/DMUL, so the GPU loop does not rematerialise them --
 * at no cost in accuracy (their terms are below 1e-11).  Used by both the
 * kernels and the oracle for w = exp(-0.5 d2 / s2); differs from numpy's
 * exp by an ulp or two (the images' parity bar is 1e-4). */
SGAD_HD double sgad_exp_neg(double x, const double* tab) {
  const double n = rint(SG_MUL(x, 184.6649169921875));     /* ~128 / ln2 */
  double r = SG_FMA(-n, 0.0054152123630046844, x);          /* ln2/128, high 20 bits */
  r = SG_FMA(-n, -1.4880111718420063e-11, r);               /* ln2/128 - high part */
  double p = 0.00833333283662796;                            /* ~1/5! */
  p = SG_FMA(p, r, 0.041666656732559204);                    /* ~1/4! */
  p = SG_FMA(p, r, 0.16666666666666666);                     /* 1/3! */
  p = SG_FMA(p, r, 0.5);
  p = SG_FMA(p, r, 1.0);
  p = SG_FMA(p, r, 1.0);
  const int ni = (int)n;
  const int j = ni & 127;
  const int k = ni >> 7; /* == (ni - j) / 128: ni - j is a multiple of 128 */
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
