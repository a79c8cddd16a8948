/*
 * raster_oracle.c -- CPU ORACLE (test infrastructure, never the product).
 *
 * A plain-C restatement of the reference rasterizer hot path,
 * /root/reference/pkg/src/raysplat/rasterizer.py, used only by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg.
 *
 *   orc_project_map     <- _prepare, rasterizer.py:86-135 (one map)
 *   orc_sort_survivors  <- np.lexsort((pixel, frame, z)), rasterizer.py:157-158
 *   orc_tile_lists      <- _build_tile_lists, rasterizer.py:178-218
 *   orc_forward         <- _forward_kernel, rasterizer.py:221-269
 *   orc_backward        <- _backward_kernel, rasterizer.py:272-363
 *   orc_chain           <- splat_backward chain rule, rasterizer.py:462-483
 *
 * Arithmetic follows the reference operation by operation (no contraction:
 * build with -ffp-contract=off); exp goes through sgad_exp so the oracle and
 * the sm_100a kernels share bits (see include/sgad_numerics.h).  Pinned against
 * golden vectors produced by the reference itself (tests/golden/make_golden.py).
 */
#include <stdint.h>
#include <stdlib.h>
#include <math.h>
#include "../include/sgad_numerics.h"

static const double TAB[SGAD_EXP2_TABLE_N] = {SGAD_EXP2_TABLE};

/* Contributor weight, shared convention with the kernels: exp(d2 * nh),
 * nh = -0.5 / s2, through sgad_exp_neg (the reference evaluates
 * exp(-0.5 * d2 / s2); the two differ by an ulp or two, far inside the 1e-4
 * image bar). */
static inline double weight(double d2, double s2) { return sgad_exp_neg(d2 * (-0.5 / s2), TAB); }

/* rasterizer.py:86-135 for one source map.  Survivors are written in pixel
 * order (np.nonzero order).  Returns the survivor count. */
int64_t orc_project_map(int64_t h, int64_t w, const double* base, const double* delta,
                        const double* log_radius, const double* logit, const double* color,
                        const uint8_t* active, double sfx, double sfy, double scx, double scy,
                        const double* R, const double* t, double tfx, double tfy, double tcx,
                        double tcy, int64_t tw, int64_t th, double* u0o, double* v0o, double* zo,
                        double* sigo, double* opo, double* colo, int64_t* pixo, double* diro,
                        double* yo, double* rado) {
  int64_t n = 0;
  const double wlim = (double)tw - 1.0, hlim = (double)th - 1.0;
  for (int64_t p = 0; p < h * w; ++p) {
    if (!active[p]) continue;
    const double uu = (double)(p % w), vv = (double)(p / w);
    const double r0 = (uu - scx) / sfx, r1 = (vv - scy) / sfy;
    const double dadj = fabs(base[p] + delta[p]);
    double dir[3], y[3];
    for (int j = 0; j < 3; ++j) {
      /* rays @ R.T through OpenBLAS: fma(r2, R[j,2], fma(r1, R[j,1], r0*R[j,0])), r2 == 1 */
      dir[j] = fma(1.0, R[3 * j + 2], fma(r1, R[3 * j + 1], r0 * R[3 * j + 0]));
      y[j] = dir[j] * dadj + t[j];
    }
    const double z = y[2];
    if (!(z > SGAD_Z_NEAR)) continue;
    const double radius = sgad_exp(log_radius[p]);
    const double u0 = tfx * y[0] / z + tcx;
    const double v0 = tfy * y[1] / z + tcy;
    const double sig = radius * tfx / z;
    const double margin = 3.0 * sig;
    if (!((u0 + margin >= 0.0) && (u0 - margin <= wlim) && (v0 + margin >= 0.0) &&
          (v0 - margin <= hlim)))
      continue;
    u0o[n] = u0;
    v0o[n] = v0;
    zo[n] = z;
    sigo[n] = sig;
    opo[n] = sgad_sigmoid(logit[p]);
    for (int j = 0; j < 3; ++j) {
      colo[3 * n + j] = color[3 * p + j];
      diro[3 * n + j] = dir[j];
      yo[3 * n + j] = y[j];
    }
    pixo[n] = p;
    rado[n] = radius;
    ++n;
  }
  return n;
}

typedef struct {
  double z;
  int64_t frame, pixel, pos;
} orc_key;

static int orc_key_cmp(const void* a, const void* b) {
  const orc_key* x = (const orc_key*)a;
  const orc_key* y = (const orc_key*)b;
  if (x->z < y->z) return -1;
  if (x->z > y->z) return 1;
  if (x->frame != y->frame) return x->frame < y->frame ? -1 : 1;
  if (x->pixel != y->pixel) return x->pixel < y->pixel ? -1 : 1;
  return x->pos < y->pos ? -1 : (x->pos > y->pos);
}

/* np.lexsort((pixel, frame, z)) -- stable, so equal keys keep input order */
void orc_sort_survivors(int64_t n, const double* z, const int64_t* frame, const int64_t* pixel,
                        int64_t* order) {
  orc_key* k = (orc_key*)malloc(sizeof(orc_key) * (size_t)(n > 0 ? n : 1));
  for (int64_t i = 0; i < n; ++i) {
    k[i].z = z[i];
    k[i].frame = frame[i];
    k[i].pixel = pixel[i];
    k[i].pos = i;
  }
  qsort(k, (size_t)n, sizeof(orc_key), orc_key_cmp);
  for (int64_t i = 0; i < n; ++i) order[i] = k[i].pos;
  free(k);
}

static void orc_bounds(double u0, double v0, double sigma, int64_t ntx, int64_t nty, int64_t tile,
                       int64_t* b) {
  const double r = 3.0 * sigma;
  int64_t x0 = (int64_t)floor((u0 - r) / (double)tile);
  int64_t x1 = (int64_t)floor((u0 + r) / (double)tile);
  int64_t y0 = (int64_t)floor((v0 - r) / (double)tile);
  int64_t y1 = (int64_t)floor((v0 + r) / (double)tile);
  if (x0 < 0) x0 = 0;
  if (y0 < 0) y0 = 0;
  if (x1 > ntx - 1) x1 = ntx - 1;
  if (y1 > nty - 1) y1 = nty - 1;
  b[0] = x0;
  b[1] = x1;
  b[2] = y0;
  b[3] = y1;
}

/* rasterizer.py:178-218.  offsets has n_tiles+1 entries; lists may be NULL
 * (count only).  Returns the total pair count. */
int64_t orc_tile_lists(int64_t n, const double* u0, const double* v0, const double* sigma,
                       int64_t height, int64_t width, int64_t tile, int64_t* offsets,
                       int64_t* lists) {
  const int64_t ntx = (width + tile - 1) / tile, nty = (height + tile - 1) / tile;
  const int64_t nt = ntx * nty;
  for (int64_t t = 0; t <= nt; ++t) offsets[t] = 0;
  int64_t b[4];
  for (int64_t g = 0; g < n; ++g) {
    orc_bounds(u0[g], v0[g], sigma[g], ntx, nty, tile, b);
    for (int64_t ty = b[2]; ty <= b[3]; ++ty)
      for (int64_t tx = b[0]; tx <= b[1]; ++tx) offsets[ty * ntx + tx + 1] += 1;
  }
  for (int64_t t = 0; t < nt; ++t) offsets[t + 1] += offsets[t];
  if (lists) {
    int64_t* cur = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nt > 0 ? nt : 1));
    for (int64_t t = 0; t < nt; ++t) cur[t] = offsets[t];
    for (int64_t g = 0; g < n; ++g) {
      orc_bounds(u0[g], v0[g], sigma[g], ntx, nty, tile, b);
      for (int64_t ty = b[2]; ty <= b[3]; ++ty)
        for (int64_t tx = b[0]; tx <= b[1]; ++tx) lists[cur[ty * ntx + tx]++] = g;
    }
    free(cur);
  }
  return offsets[nt];
}

/* rasterizer.py:221-269 */
void orc_forward(const double* u0, const double* v0, const double* z, const double* sigma,
                 const double* opacity, const double* color, const int64_t* offsets,
                 const int64_t* lists, int64_t height, int64_t width, int64_t tile,
                 double* out_color, double* out_depth, double* out_alpha, int32_t* out_count) {
  const int64_t ntx = (width + tile - 1) / tile, nty = (height + tile - 1) / tile;
  for (int64_t t = 0; t < ntx * nty; ++t) {
    const int64_t ty = t / ntx, tx = t - ty * ntx;
    const int64_t ylim = (ty + 1) * tile < height ? (ty + 1) * tile : height;
    const int64_t xlim = (tx + 1) * tile < width ? (tx + 1) * tile : width;
    for (int64_t py = ty * tile; py < ylim; ++py)
      for (int64_t px = tx * tile; px < xlim; ++px) {
        double trans = 1.0, c0 = 0.0, c1 = 0.0, c2 = 0.0, dep = 0.0, acc = 0.0;
        int32_t cnt = 0;
        for (int64_t k = offsets[t]; k < offsets[t + 1]; ++k) {
          const int64_t g = lists[k];
          const double dx = u0[g] - (double)px, dy = v0[g] - (double)py;
          const double d2 = dx * dx + dy * dy;
          const double s2 = sigma[g] * sigma[g];
          if (d2 > 9.0 * s2) continue;
          const double wgt = weight(d2, s2);
          double a = opacity[g] * wgt;
          if (a > SGAD_ALPHA_MAX) a = SGAD_ALPHA_MAX;
          const double at = a * trans;
          c0 = fma(color[3 * g + 0], at, c0);
          c1 = fma(color[3 * g + 1], at, c1);
          c2 = fma(color[3 * g + 2], at, c2);
          dep = fma(z[g], at, dep);
          acc += at;
          cnt += 1;
          trans *= 1.0 - a;
          if (trans < SGAD_TRANSMITTANCE_MIN) break;
        }
        const int64_t p = py * width + px;
        out_color[3 * p + 0] = c0;
        out_color[3 * p + 1] = c1;
        out_color[3 * p + 2] = c2;
        out_depth[p] = dep;
        out_alpha[p] = acc;
        out_count[p] = cnt;
      }
  }
}

/* rasterizer.py:272-363 (accumulates into the g_* buffers) */
void orc_backward(const double* u0, const double* v0, const double* z, const double* sigma,
                  const double* opacity, const double* color, const uint8_t* learnable,
                  const int64_t* offsets, const int64_t* lists, int64_t height, int64_t width,
                  int64_t tile, const double* g_out_color, const double* g_out_depth,
                  const double* g_out_alpha, double* g_color, double* g_opacity, double* g_u0,
                  double* g_v0, double* g_sigma, double* g_z) {
  const int64_t ntx = (width + tile - 1) / tile, nty = (height + tile - 1) / tile;
  for (int64_t t = 0; t < ntx * nty; ++t) {
    const int64_t ty = t / ntx, tx = t - ty * ntx;
    const int64_t ylim = (ty + 1) * tile < height ? (ty + 1) * tile : height;
    const int64_t xlim = (tx + 1) * tile < width ? (tx + 1) * tile : width;
    for (int64_t py = ty * tile; py < ylim; ++py)
      for (int64_t px = tx * tile; px < xlim; ++px) {
        const int64_t p = py * width + px;
        const double gc0 = g_out_color[3 * p], gc1 = g_out_color[3 * p + 1],
                     gc2 = g_out_color[3 * p + 2];
        const double gd = g_out_depth[p], ga = g_out_alpha[p];
        if (gc0 == 0.0 && gc1 == 0.0 && gc2 == 0.0 && gd == 0.0 && ga == 0.0) continue;
        double trans = 1.0;
        int64_t last = -1;
        for (int64_t k = offsets[t]; k < offsets[t + 1]; ++k) {
          const int64_t g = lists[k];
          const double dx = u0[g] - (double)px, dy = v0[g] - (double)py;
          const double d2 = dx * dx + dy * dy;
          const double s2 = sigma[g] * sigma[g];
          if (d2 > 9.0 * s2) continue;
          double a = opacity[g] * weight(d2, s2);
          if (a > SGAD_ALPHA_MAX) a = SGAD_ALPHA_MAX;
          last = k;
          trans *= 1.0 - a;
          if (trans < SGAD_TRANSMITTANCE_MIN) break;
        }
        if (last < 0) continue;
        double s_c0 = 0.0, s_c1 = 0.0, s_c2 = 0.0, s_d = 0.0, s_a = 0.0;
        double t_cur = trans;
        for (int64_t k = last; k > offsets[t] - 1; --k) {
          const int64_t g = lists[k];
          const double dx = u0[g] - (double)px, dy = v0[g] - (double)py;
          const double d2 = dx * dx + dy * dy;
          const double s2 = sigma[g] * sigma[g];
          if (d2 > 9.0 * s2) continue;
          const double wgt = weight(d2, s2);
          const double aw = opacity[g] * wgt;
          const int clamped = aw > SGAD_ALPHA_MAX;
          const double a = clamped ? SGAD_ALPHA_MAX : aw;
          const double t_before = t_cur / (1.0 - a);
          const double at = a * t_before;
          const double c0 = color[3 * g], c1 = color[3 * g + 1], c2 = color[3 * g + 2];
          if (learnable[g] != 0) {
            const double d_alpha = gc0 * (c0 * t_before - s_c0 / (1.0 - a)) +
                                   gc1 * (c1 * t_before - s_c1 / (1.0 - a)) +
                                   gc2 * (c2 * t_before - s_c2 / (1.0 - a)) +
                                   gd * (z[g] * t_before - s_d / (1.0 - a)) +
                                   ga * (t_before - s_a / (1.0 - a));
            g_color[3 * g] += gc0 * at;
            g_color[3 * g + 1] += gc1 * at;
            g_color[3 * g + 2] += gc2 * at;
            g_z[g] += gd * at;
            if (!clamped) {
              const double gw = d_alpha * opacity[g];
              g_opacity[g] += d_alpha * wgt;
              g_sigma[g] += gw * wgt * d2 / (s2 * sigma[g]);
              const double gd2 = gw * (-0.5 * wgt / s2);
              g_u0[g] += gd2 * 2.0 * dx;
              g_v0[g] += gd2 * 2.0 * dy;
            }
          }
          s_c0 += c0 * at;
          s_c1 += c1 * at;
          s_c2 += c2 * at;
          s_d += z[g] * at;
          s_a += at;
          t_cur = t_before;
        }
      }
  }
}

/* rasterizer.py:462-483 for the selected survivors (already gathered).
 * Outputs per survivor: g_radius, g_logit, g_delta. */
void orc_chain(int64_t n, double fx, double fy, const double* g_opacity, const double* g_u0,
               const double* g_v0, const double* g_sigma, const double* g_z, const double* y,
               const double* z, const double* dir, const double* sigma, const double* opac,
               const double* base, const double* delta, double* g_radius, double* g_logit,
               double* g_delta) {
  for (int64_t i = 0; i < n; ++i) {
    const double zi = z[i];
    const double z2 = zi * zi;
    g_radius[i] = g_sigma[i] * fx / zi;
    const double g_z_total = g_z[i] - g_sigma[i] * sigma[i] / zi - g_u0[i] * fx * y[3 * i] / z2 -
                             g_v0[i] * fy * y[3 * i + 1] / z2;
    const double g_y0 = g_u0[i] * fx / zi;
    const double g_y1 = g_v0[i] * fy / zi;
    const double g_dadj = g_y0 * dir[3 * i] + g_y1 * dir[3 * i + 1] + g_z_total * dir[3 * i + 2];
    const double sgn = (base[i] + delta[i] >= 0.0) ? 1.0 : -1.0;
    g_delta[i] = g_dadj * sgn;
    g_logit[i] = g_opacity[i] * opac[i] * (1.0 - opac[i]);
  }
}
