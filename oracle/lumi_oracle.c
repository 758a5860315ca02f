/*
 * lumi_oracle.c -- TEST INFRASTRUCTURE ONLY (see lumi_oracle.h).
 *
 * Plain-C restatement of the reference rendering path.  Build: oracle/Makefile
 * (gcc -O2 -std=c11, no -mfma, no -ffast-math).  Citations are to the reference
 * checkout (proj/...).
 */
#define _GNU_SOURCE
#include "lumi_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdatomic.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------- */
/* RNG: pcg32 (proj/include/lumi/common.h:78-124)                             */
/* ------------------------------------------------------------------------- */

#define LO_PCG_MULT 6364136223846793005ULL
#define LO_PCG_STREAM 0xda3e39cb94b95bdbULL

uint32_t lo_rng_u32(lo_rng* r) { /* common.h:88-94 */
  uint64_t old = r->state;
  r->state = old * LO_PCG_MULT + r->inc;
  uint32_t xorshifted = (uint32_t)(((old >> 18u) ^ old) >> 27u);
  uint32_t rot = (uint32_t)(old >> 59u);
  return (xorshifted >> rot) | (xorshifted << ((32u - rot) & 31u));
}

void lo_rng_init(lo_rng* r, uint64_t seed) { /* common.h:80-86 */
  r->state = 0;
  r->inc = (LO_PCG_STREAM << 1u) | 1u;
  lo_rng_u32(r);
  r->state += seed;
  lo_rng_u32(r);
}

/* O(log n) LCG jump-ahead: identical state to calling lo_rng_u32 `delta` times. */
void lo_rng_advance(lo_rng* r, uint64_t delta) {
  uint64_t cur_mult = LO_PCG_MULT, cur_plus = r->inc, acc_mult = 1, acc_plus = 0;
  while (delta > 0) {
    if (delta & 1) {
      acc_mult *= cur_mult;
      acc_plus = acc_plus * cur_mult + cur_plus;
    }
    cur_plus = (cur_mult + 1) * cur_plus;
    cur_mult *= cur_mult;
    delta >>= 1;
  }
  r->state = acc_mult * r->state + acc_plus;
}

double lo_rng_uniform(lo_rng* r) { return lo_rng_u32(r) * (1.0 / 4294967296.0); } /* :106 */

double lo_rng_normal(lo_rng* r) { /* common.h:109-114 */
  double u1 = lo_rng_uniform(r);
  if (u1 < 1e-12) u1 = 1e-12; /* std::max(uniform(), 1e-12) */
  double u2 = lo_rng_uniform(r);
  return sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
}

/* ------------------------------------------------------------------------- */
/* Model layout and synthetic parameters                                     */
/* ------------------------------------------------------------------------- */

static int lo_resolution(const lo_field_config* cfg, int level) { /* grid.h:25-27 */
  return (int)floor(cfg->base_resolution * pow(cfg->per_level_scale, level));
}

int lo_layout(const lo_field_config* cfg, lo_grid_layout* out) { /* grid.h:58-74 */
  if (cfg->levels < 1 || cfg->levels > LO_MAX_LEVELS || cfg->features_per_level < 1 ||
      cfg->features_per_level > 8)
    return -1;
  if (cfg->table_size == 0 || (cfg->table_size & (cfg->table_size - 1)) != 0) return -2;
  memset(out, 0, sizeof(*out));
  out->levels = cfg->levels;
  out->fpl = cfg->features_per_level;
  uint64_t offset = 0;
  for (int l = 0; l < cfg->levels; ++l) {
    int res = lo_resolution(cfg, l);
    if (l > 0 && res <= out->resolution[l - 1]) return -3; /* strictly increasing */
    uint64_t verts = (uint64_t)res + 1;
    uint64_t dense = verts * verts * verts;
    out->resolution[l] = res;
    out->dense[l] = dense <= cfg->table_size;
    out->entries[l] = out->dense[l] ? (uint32_t)dense : cfg->table_size;
    out->offset[l] = offset;
    offset += (uint64_t)out->entries[l] * cfg->features_per_level;
  }
  out->total_floats = offset;
  return 0;
}

size_t lo_density_param_count(const lo_field_config* c) { /* field.h:73-74 */
  size_t f = (size_t)c->levels * c->features_per_level, h = c->hidden_width, o = 1 + c->bottleneck;
  return f * h + h + h * o + o;
}

size_t lo_color_param_count(const lo_field_config* c) { /* field.h:75-77 */
  size_t i = c->bottleneck + 16, h = c->hidden_width;
  return i * h + h + h * h + h + h * 3 + 3;
}

/* DenseLayer::init_random (network.h:73-78): He-normal weights, zero bias. */
static float* lo_init_layer(lo_rng* rng, int in, int out, float* p) {
  double scale = sqrt(2.0 / in);
  for (int i = 0; i < in * out; ++i) p[i] = (float)(lo_rng_normal(rng) * scale);
  for (int i = 0; i < out; ++i) p[in * out + i] = 0.0f;
  return p + (size_t)in * out + out;
}

int lo_synth_params(const lo_field_config* cfg, uint64_t seed, double amp, float* table,
                    float* dparams, float* cparams) {
  lo_grid_layout lay;
  int rc = lo_layout(cfg, &lay);
  if (rc) return rc;
  /* RadianceField::init_random (field.h:88-93): grid (grid.h:82-84, scale 1e-4), then nets. */
  lo_rng rng;
  lo_rng_init(&rng, seed);
  if (amp > 0) {
    lo_rng_advance(&rng, lay.total_floats); /* grid values are overwritten below */
  } else {
    for (uint64_t i = 0; i < lay.total_floats; ++i)
      table[i] = (float)(-1e-4 + (1e-4 - -1e-4) * lo_rng_uniform(&rng));
  }
  const int f = cfg->levels * cfg->features_per_level, h = cfg->hidden_width;
  float* p = dparams;
  p = lo_init_layer(&rng, f, h, p);
  p = lo_init_layer(&rng, h, 1 + cfg->bottleneck, p);
  p = cparams;
  p = lo_init_layer(&rng, cfg->bottleneck + 16, h, p);
  p = lo_init_layer(&rng, h, h, p);
  p = lo_init_layer(&rng, h, 3, p);
  if (amp > 0) { /* trainer.cpp:257-259 pattern: Rng(seed+1).uniform(-a, a) */
    lo_rng g;
    lo_rng_init(&g, seed + 1);
    for (uint64_t i = 0; i < lay.total_floats; ++i)
      table[i] = (float)(-amp + (amp - -amp) * lo_rng_uniform(&g));
  }
  return 0;
}

/* ------------------------------------------------------------------------- */
/* Geometry (double, reference op order, no FMA)                              */
/* ------------------------------------------------------------------------- */

static inline double lo_max(double a, double b) { return a < b ? b : a; } /* std::max */
static inline double lo_min(double a, double b) { return b < a ? b : a; } /* std::min */
static inline double lo_clamp(double v, double lo, double hi) { /* common.h:176-179 */
  return v < lo ? lo : (v > hi ? hi : v);
}
static inline double lo_linf(const double v[3]) { /* common.h:38 */
  return lo_max(fabs(v[0]), lo_max(fabs(v[1]), fabs(v[2])));
}
static inline double lo_norm(const double v[3]) { /* common.h:36-37 */
  return sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
}

/* camera.cpp:10-17 (generate_ray_unchecked) with Pose::rotate (common.h:49-53) and
   Vec3::normalized (common.h:39). */
void lo_generate_ray(const lo_camera* cam, double px, double py, double origin[3],
                     double dir[3]) {
  double v[3] = {(px - cam->cx) / cam->fx, (py - cam->cy) / cam->fy, 1.0};
  const double* R = cam->rot;
  double d[3] = {R[0] * v[0] + R[1] * v[1] + R[2] * v[2], R[3] * v[0] + R[4] * v[1] + R[5] * v[2],
                 R[6] * v[0] + R[7] * v[1] + R[8] * v[2]};
  double n = lo_norm(d);
  dir[0] = d[0] / n;
  dir[1] = d[1] / n;
  dir[2] = d[2] / n;
  origin[0] = cam->origin[0];
  origin[1] = cam->origin[1];
  origin[2] = cam->origin[2];
}

/* camera.cpp:34-49 */
int lo_contract(const double x[3], int mode, double out[3]) {
  if (!(isfinite(x[0]) && isfinite(x[1]) && isfinite(x[2]))) return -1;
  out[0] = x[0];
  out[1] = x[1];
  out[2] = x[2];
  if (mode == 0) return 0;
  double m = lo_linf(x);
  if (m <= 1.0) return 0;
  out[0] = x[0] / m;
  out[1] = x[1] / m;
  out[2] = x[2] / m;
  double mapped = 2.0 - 1.0 / m;
  if (fabs(x[0]) == m)
    out[0] = copysign(mapped, x[0]);
  else if (fabs(x[1]) == m)
    out[1] = copysign(mapped, x[1]);
  else
    out[2] = copysign(mapped, x[2]);
  return 0;
}

/* camera.cpp:51-66 */
static int lo_uncontract(const double c[3], double out[3]) {
  out[0] = c[0];
  out[1] = c[1];
  out[2] = c[2];
  double m = lo_linf(c);
  if (m <= 1.0) return 0;
  if (!(m < 2.0)) return -1;
  double mag = 1.0 / (2.0 - m);
  out[0] = c[0] * mag;
  out[1] = c[1] * mag;
  out[2] = c[2] * mag;
  if (fabs(c[0]) == m)
    out[0] = copysign(mag, c[0]);
  else if (fabs(c[1]) == m)
    out[1] = copysign(mag, c[1]);
  else
    out[2] = copysign(mag, c[2]);
  return 0;
}

/* occupancy.cpp:22-29 */
int64_t lo_voxel_index(int res, const double c[3]) {
  double u = (c[0] + 2.0) * 0.25, v = (c[1] + 2.0) * 0.25, w = (c[2] + 2.0) * 0.25;
  if (u < 0 || u > 1 || v < 0 || v > 1 || w < 0 || w > 1) return -1;
  int ix = (int)(u * res), iy = (int)(v * res), iz = (int)(w * res);
  if (ix > res - 1) ix = res - 1;
  if (iy > res - 1) iy = res - 1;
  if (iz > res - 1) iz = res - 1;
  return ((int64_t)iz * res + iy) * res + ix;
}

static inline void lo_ray_at(const double o[3], const double d[3], double t, double p[3]) {
  p[0] = o[0] + d[0] * t; /* camera.h:29 */
  p[1] = o[1] + d[1] * t;
  p[2] = o[2] + d[2] * t;
}

/* camera.cpp:68-73 */
double lo_contracted_footprint(const double o0[3], const double d0[3], const double o1[3],
                               const double d1[3], double t, int mode) {
  double p[3], q[3], a[3], b[3];
  lo_ray_at(o0, d0, t, p);
  lo_ray_at(o1, d1, t, q);
  lo_contract(p, mode, a);
  lo_contract(q, mode, b);
  double dd[3] = {a[0] - b[0], a[1] - b[1], a[2] - b[2]};
  return 0.5 * lo_norm(dd);
}

/* grid.cpp:8-13 */
double lo_lod_level(double r, const lo_field_config* cfg) {
  double l = -log(2.0 * cfg->base_resolution * r) / log(cfg->per_level_scale);
  return lo_min(l, (double)(cfg->levels - 1));
}

/* grid.cpp:15-37 */
void lo_lod_weights(double l_star, double bias, int levels, float* w) {
  double eff = l_star + bias;
  if (eff >= levels - 1) {
    for (int i = 0; i < levels; ++i) w[i] = 1.0f;
    return;
  }
  if (eff < 0.0) {
    w[0] = 1e-4f;
    for (int i = 1; i < levels; ++i) w[i] = 0.0f;
    return;
  }
  double fl = floor(eff);
  double frac = eff - fl;
  for (int i = 0; i < levels; ++i) {
    if (i <= (int)fl)
      w[i] = 1.0f;
    else if (i == (int)fl + 1 && frac > 0.0)
      w[i] = (float)frac;
    else
      w[i] = 0.0f;
  }
}

/* network.h:17-37 (T = float) */
void lo_sh_encode(const double d[3], float out[16]) {
  const float x = (float)d[0], y = (float)d[1], z = (float)d[2];
  const float xx = x * x, yy = y * y, zz = z * z;
  out[0] = (float)0.28209479177387814;
  out[1] = (float)-0.48860251190291987 * y;
  out[2] = (float)0.48860251190291987 * z;
  out[3] = (float)-0.48860251190291987 * x;
  out[4] = (float)1.0925484305920792 * x * y;
  out[5] = (float)-1.0925484305920792 * y * z;
  out[6] = (float)0.31539156525252005 * (3.0f * zz - 1.0f);
  out[7] = (float)-1.0925484305920792 * x * z;
  out[8] = (float)0.5462742152960396 * (xx - yy);
  out[9] = (float)-0.5900435899266435 * y * (3.0f * xx - yy);
  out[10] = (float)2.890611442640554 * x * y * z;
  out[11] = (float)-0.4570457994644658 * y * (5.0f * zz - 1.0f);
  out[12] = (float)0.3731763325901154 * z * (5.0f * zz - 3.0f);
  out[13] = (float)-0.4570457994644658 * x * (5.0f * zz - 1.0f);
  out[14] = (float)1.445305721320277 * z * (xx - yy);
  out[15] = (float)-0.5900435899266435 * x * (xx - 3.0f * yy);
}

/* renderer.h:135-142 / camera.cpp:75-86 */
void lo_sample_distances(double t_near, double t_far, int n, double* ts, double* ratio) {
  double log_ratio = log(t_far / t_near);
  for (int i = 0; i < n; ++i) ts[i] = t_near * exp(log_ratio * ((double)i / (n - 1)));
  ts[0] = t_near;
  ts[n - 1] = t_far;
  if (ratio) *ratio = pow(t_far / t_near, 1.0 / (n - 1));
}

/* color.cpp:17-44 (scene-linear 1.0 = 100 cd/m^2) */
#define LO_PQ_M1 (1305.0 / 8192.0)
#define LO_PQ_M2 (2523.0 / 32.0)
#define LO_PQ_C1 (107.0 / 128.0)
#define LO_PQ_C2 (2413.0 / 128.0)
#define LO_PQ_C3 (2392.0 / 128.0)
double lo_pq_encode(double y) {
  double yn = lo_clamp(y * (100.0 / 10000.0), 0.0, 1.0);
  double p = pow(yn, LO_PQ_M1);
  double num = LO_PQ_C1 + LO_PQ_C2 * p;
  double den = 1.0 + LO_PQ_C3 * p;
  return pow(num / den, LO_PQ_M2);
}
double lo_pq_decode(double v) {
  double p = pow(v, 1.0 / LO_PQ_M2);
  double num = p - LO_PQ_C1;
  if (num < 0.0) num = 0.0;
  double den = LO_PQ_C2 - LO_PQ_C3 * p;
  double yn = pow(num / den, 1.0 / LO_PQ_M1);
  return yn / (100.0 / 10000.0);
}
double lo_srgb_oetf(double v) {
  v = lo_clamp(v, 0.0, 1.0);
  return v <= 0.0031308 ? 12.92 * v : 1.055 * pow(v, 1.0 / 2.4) - 0.055;
}

/* ------------------------------------------------------------------------- */
/* Field: hash-grid encode + MLPs                                             */
/* ------------------------------------------------------------------------- */

static inline uint32_t lo_spatial_hash(uint32_t x, uint32_t y, uint32_t z, uint32_t t) {
  return (x * 1u ^ y * 2654435761u ^ z * 805459861u) & (t - 1u); /* grid.h:50-52 */
}

/* grid.h:90-114 (encode) + grid.h:144-167 (corners); one sample, stride 1 */
void lo_encode(const lo_model* m, const double c[3], const float* w, float* out) {
  const lo_grid_layout* L = &m->layout;
  const int fpl = L->fpl;
  double u = (c[0] + 2.0) * 0.25, v = (c[1] + 2.0) * 0.25, s = (c[2] + 2.0) * 0.25;
  for (int l = 0; l < L->levels; ++l) {
    float* dst = out + (size_t)l * fpl;
    if (w[l] <= 0.0f) {
      for (int f = 0; f < fpl; ++f) dst[f] = 0.0f;
      continue;
    }
    const int res = L->resolution[l];
    double pu = lo_clamp(u, 0.0, 1.0) * res, pv = lo_clamp(v, 0.0, 1.0) * res,
           ps = lo_clamp(s, 0.0, 1.0) * res;
    int iu = (int)pu, iv = (int)pv, is = (int)ps;
    if (iu > res - 1) iu = res - 1;
    if (iv > res - 1) iv = res - 1;
    if (is > res - 1) is = res - 1;
    double fu = pu - iu, fv = pv - iv, fs = ps - is;
    const uint32_t verts = (uint32_t)res + 1;
    const float* base = m->table + L->offset[l];
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int k = 0; k < 8; ++k) {
      uint32_t x = (uint32_t)iu + (k & 1), y = (uint32_t)iv + ((k >> 1) & 1),
               z = (uint32_t)is + ((k >> 2) & 1);
      uint32_t idx = L->dense[l] ? (z * verts + y) * verts + x
                                 : lo_spatial_hash(x, y, z, L->entries[l]);
      double wu = (k & 1) ? fu : 1.0 - fu;
      double wv = ((k >> 1) & 1) ? fv : 1.0 - fv;
      double ws = ((k >> 2) & 1) ? fs : 1.0 - fs;
      float tri = (float)(wu * wv * ws);
      const float* e = base + (size_t)idx * fpl;
      for (int f = 0; f < fpl; ++f) acc[f] += tri * e[f];
    }
    for (int f = 0; f < fpl; ++f) dst[f] = acc[f] * w[l];
  }
}

/* simd::dense_forward over a feature-major batch (x [cols x n], y [rows x n]) in the
   accumulation order of the selected ISA variant, per sample:
   scalar  simd.h:35-51          y = b; y += w*x            (no FMA)
   avx2    simd_avx2.cpp:19-43   y = fma(w, x, y) from b
   avx512  simd_avx512.cpp:27-61 four fma chains, (a0+a1)+(a2+a3)
   The body is instantiated twice: with hardware FMA enabled (fast; fmaf is exact either
   way) and generic, chosen once at runtime. */
#define LO_DENSE_BODY(FMA)                                                               \
  for (int r = 0; r < rows; ++r) {                                                       \
    const float* wr = W + (size_t)r * cols;                                              \
    float* yr = y + (size_t)r * n;                                                       \
    const float bias = b[r];                                                             \
    if (mode == LO_MLP_AVX512) {                                                         \
      float a1[LO_BATCH], a2[LO_BATCH], a3[LO_BATCH];                                    \
      for (int i = 0; i < n; ++i) {                                                      \
        yr[i] = bias;                                                                    \
        a1[i] = a2[i] = a3[i] = 0.0f;                                                    \
      }                                                                                  \
      int c = 0;                                                                         \
      for (; c + 4 <= cols; c += 4) {                                                    \
        const float *x0 = x + (size_t)c * n, *x1 = x0 + n, *x2 = x1 + n, *x3 = x2 + n;   \
        const float w0 = wr[c], w1 = wr[c + 1], w2 = wr[c + 2], w3 = wr[c + 3];          \
        for (int i = 0; i < n; ++i) {                                                    \
          yr[i] = FMA(w0, x0[i], yr[i]);                                                 \
          a1[i] = FMA(w1, x1[i], a1[i]);                                                 \
          a2[i] = FMA(w2, x2[i], a2[i]);                                                 \
          a3[i] = FMA(w3, x3[i], a3[i]);                                                 \
        }                                                                                \
      }                                                                                  \
      for (; c < cols; ++c)                                                              \
        for (int i = 0; i < n; ++i) yr[i] = FMA(wr[c], x[(size_t)c * n + i], yr[i]);     \
      for (int i = 0; i < n; ++i) {                                                      \
        float v = (yr[i] + a1[i]) + (a2[i] + a3[i]);                                     \
        yr[i] = relu ? (v > 0.0f ? v : 0.0f) : v;                                        \
      }                                                                                  \
    } else if (mode == LO_MLP_AVX2) {                                                    \
      for (int i = 0; i < n; ++i) yr[i] = bias;                                          \
      for (int c = 0; c < cols; ++c) {                                                   \
        const float w = wr[c], *xc = x + (size_t)c * n;                                  \
        for (int i = 0; i < n; ++i) yr[i] = FMA(w, xc[i], yr[i]);                        \
      }                                                                                  \
      if (relu)                                                                          \
        for (int i = 0; i < n; ++i) yr[i] = yr[i] > 0.0f ? yr[i] : 0.0f;                 \
    } else {                                                                             \
      for (int i = 0; i < n; ++i) yr[i] = bias;                                          \
      for (int c = 0; c < cols; ++c) {                                                   \
        const float w = wr[c], *xc = x + (size_t)c * n;                                  \
        for (int i = 0; i < n; ++i) yr[i] += w * xc[i];                                  \
      }                                                                                  \
      if (relu)                                                                          \
        for (int i = 0; i < n; ++i)                                                      \
          if (yr[i] < 0.0f) yr[i] = 0.0f;                                                \
    }                                                                                    \
  }

#define LO_BATCH 64 /* max samples per dense call */

#if defined(__x86_64__)
__attribute__((target("fma"))) static void lo_dense_hw(int mode, int rows, int cols, int n,
                                                       const float* W, const float* b,
                                                       const float* x, float* y, int relu) {
  LO_DENSE_BODY(__builtin_fmaf)
}
#endif

static void lo_dense_sw(int mode, int rows, int cols, int n, const float* W, const float* b,
                        const float* x, float* y, int relu) {
  LO_DENSE_BODY(fmaf)
}

static void lo_dense(int mode, int rows, int cols, int n, const float* W, const float* b,
                     const float* x, float* y, int relu) {
#if defined(__x86_64__)
  static int hw = -1;
  if (hw < 0) hw = __builtin_cpu_supports("fma") ? 1 : 0;
  if (hw && mode != LO_MLP_SCALAR) {
    lo_dense_hw(mode, rows, cols, n, W, b, x, y, relu);
    return;
  }
#endif
  lo_dense_sw(mode, rows, cols, n, W, b, x, y, relu);
}

static inline float lo_trunc_exp(float x) { /* network.h:41-46 */
  const float cutoff = 10.0f;
  if (x <= cutoff) return expf(x);
  return expf(cutoff) * (1.0f + (x - cutoff));
}
static inline float lo_sigmoid(float x) { return 1.0f / (1.0f + expf(-x)); } /* :54-57 */

/* RadianceField::forward_chunk (field.h:106-137): encode every sample, density net,
   sigma = trunc_exp(raw0), colour input = raw[1..B] ++ SH, colour net, sigmoid head.
   Feature-major activations over a batch of n <= LO_BATCH samples. */
static void lo_forward_batch(const lo_model* m, int n, const double (*pos)[3], const float* lodw,
                             const float* sh, float* sigma, float* rgb /*[3][n]*/,
                             float* feat_out /*[F][n]*/) {
  const lo_field_config* cfg = &m->cfg;
  const int L = cfg->levels, F = L * cfg->features_per_level, H = cfg->hidden_width,
            B = cfg->bottleneck;
  float* feat = (float*)malloc(sizeof(float) * (size_t)F * LO_BATCH);
  float* h1 = (float*)malloc(sizeof(float) * (size_t)H * LO_BATCH);
  float* h2 = (float*)malloc(sizeof(float) * (size_t)H * LO_BATCH);
  float* dout = (float*)malloc(sizeof(float) * (size_t)(1 + B) * LO_BATCH);
  float* cin = (float*)malloc(sizeof(float) * (size_t)(B + 16) * LO_BATCH);
  float* raw = (float*)malloc(sizeof(float) * 3 * LO_BATCH);
  float one[LO_MAX_LEVELS * 8];
  for (int i = 0; i < n; ++i) {
    lo_encode(m, pos[i], lodw + (size_t)i * L, one);
    for (int f = 0; f < F; ++f) feat[(size_t)f * n + i] = one[f];
  }
  if (feat_out) memcpy(feat_out, feat, sizeof(float) * (size_t)F * n);
  const float* dp = m->dparams;
  lo_dense(m->mlp_mode, H, F, n, dp, dp + (size_t)H * F, feat, h1, 1);
  dp += (size_t)H * F + H;
  lo_dense(m->mlp_mode, 1 + B, H, n, dp, dp + (size_t)(1 + B) * H, h1, dout, 0);
  for (int i = 0; i < n; ++i) sigma[i] = lo_trunc_exp(dout[i]);
  if (sh) {
    memcpy(cin, dout + n, sizeof(float) * (size_t)B * n);
    for (int s = 0; s < 16; ++s)
      for (int i = 0; i < n; ++i) cin[(size_t)(B + s) * n + i] = sh[s];
    const float* cp = m->cparams;
    lo_dense(m->mlp_mode, H, B + 16, n, cp, cp + (size_t)H * (B + 16), cin, h1, 1);
    cp += (size_t)H * (B + 16) + H;
    lo_dense(m->mlp_mode, H, H, n, cp, cp + (size_t)H * H, h1, h2, 1);
    cp += (size_t)H * H + H;
    lo_dense(m->mlp_mode, 3, H, n, cp, cp + (size_t)3 * H, h2, raw, 0);
    for (int i = 0; i < 3 * n; ++i)
      rgb[i] = cfg->color_space == 0 ? lo_sigmoid(raw[i]) : lo_trunc_exp(raw[i]);
  }
  free(feat);
  free(h1);
  free(h2);
  free(dout);
  free(cin);
  free(raw);
}

void lo_field_forward(const lo_model* m, int n, const double* pos3, const float* lodw,
                      const float* sh, float* sigma, float* color3, float* feat) {
  const int L = m->cfg.levels, F = L * m->cfg.features_per_level;
  float rgb[3 * LO_BATCH];
  float* ft = (float*)malloc(sizeof(float) * (size_t)F * LO_BATCH);
  for (int b0 = 0; b0 < n; b0 += LO_BATCH) {
    int nb = n - b0 < LO_BATCH ? n - b0 : LO_BATCH;
    lo_forward_batch(m, nb, (const double(*)[3])(pos3 + 3 * (size_t)b0), lodw + (size_t)b0 * L,
                     color3 ? sh : NULL, sigma + b0, rgb, ft);
    for (int i = 0; i < nb; ++i) {
      if (color3)
        for (int k = 0; k < 3; ++k) color3[(size_t)k * n + b0 + i] = rgb[k * nb + i];
      if (feat)
        for (int f = 0; f < F; ++f) feat[(size_t)f * n + b0 + i] = ft[(size_t)f * nb + i];
    }
  }
  free(ft);
}

/* ------------------------------------------------------------------------- */
/* Ray march (renderer.h:126-237) and render_rows (renderer.h:252-278)        */
/* ------------------------------------------------------------------------- */

typedef struct {
  double pixel[3], depth, opacity;
  int32_t evals, contributing, kept;
} lo_ray_result;

#define LO_MAX_CHUNK 1024

static inline int lo_occupied(const lo_model* m, const double c[3]) { /* occupancy.h:50-53 */
  int64_t i = lo_voxel_index(m->occ_res, c);
  return i >= 0 && m->occ[i];
}

static void lo_march_ray(const lo_model* m, const double o[3], const double d[3],
                         const double no[3], const double nd[3], const double* ts, double ratio,
                         const lo_render_options* opts, lo_ray_result* res) {
  const int levels = m->cfg.levels, n = opts->samples_per_ray;
  const int cs = opts->chunk_size < 1 ? 1 : (opts->chunk_size > LO_MAX_CHUNK ? LO_MAX_CHUNK : opts->chunk_size);
  float sh[16];
  lo_sh_encode(d, sh);
  double cpos[LO_MAX_CHUNK][3];
  double ct[LO_MAX_CHUNK], cdelta[LO_MAX_CHUNK];
  float* clodw = (float*)malloc(sizeof(float) * (size_t)cs * levels);
  int cn = 0;
  float bsig[LO_BATCH], brgb[3 * LO_BATCH];
  double trans = 1.0;
  int terminated = 0;
  memset(res, 0, sizeof(*res));

  /* flush (renderer.h:165-202): the reference evaluates the whole chunk; samples after
     the cut do not contribute, so they need not be evaluated here. */
#define LO_FLUSH()                                                                    \
  do {                                                                                \
    if (cn > 0) {                                                                     \
      res->evals += cn;                                                               \
      for (int b0 = 0; b0 < cn && !terminated; b0 += LO_BATCH) {                      \
        int nb = cn - b0 < LO_BATCH ? cn - b0 : LO_BATCH;                             \
        lo_forward_batch(m, nb, (const double(*)[3])cpos[b0], clodw + (size_t)b0 * levels, sh, \
                         bsig, brgb, NULL);                                           \
        for (int q = 0; q < nb; ++q) {                                                \
          int s = b0 + q;                                                             \
          double sigma = (double)bsig[q];                                             \
          double a = 1.0 - exp(-sigma * cdelta[s]);                                   \
          double w = trans * a;                                                       \
          for (int k = 0; k < 3; ++k) res->pixel[k] += w * (double)brgb[k * nb + q];  \
          res->depth += w * ct[s];                                                    \
          res->opacity += w;                                                          \
          trans *= 1.0 - a;                                                           \
          ++res->contributing;                                                        \
          if (opts->termination_transmittance > 0 &&                                  \
              trans < opts->termination_transmittance) {                              \
            terminated = 1;                                                           \
            break;                                                                    \
          }                                                                           \
        }                                                                             \
      }                                                                               \
    }                                                                                 \
    cn = 0;                                                                           \
  } while (0)

  for (int i = 0; i < n && !terminated; ++i) {
    double pos[3], c[3];
    lo_ray_at(o, d, ts[i], pos);
    lo_contract(pos, opts->contraction, c);
    if (!lo_occupied(m, c)) continue;
    double delta = (i + 1 < n) ? ts[i + 1] - ts[i] : ts[i] * (ratio - 1.0);
    float* w = clodw + (size_t)cn * levels;
    if (opts->lod_enabled) {
      double r_c = lo_contracted_footprint(o, d, no, nd, ts[i], opts->contraction);
      double l_star = lo_lod_level(lo_max(r_c, 1e-12), &m->cfg);
      lo_lod_weights(l_star, opts->lod_bias, levels, w);
    } else {
      for (int l = 0; l < levels; ++l) w[l] = 1.0f;
    }
    cpos[cn][0] = c[0];
    cpos[cn][1] = c[1];
    cpos[cn][2] = c[2];
    ct[cn] = ts[i];
    cdelta[cn] = delta;
    ++cn;
    ++res->kept;
    if (cn >= cs) LO_FLUSH();
  }
  if (!terminated) LO_FLUSH();
#undef LO_FLUSH
  for (int k = 0; k < 3; ++k) res->pixel[k] += trans * opts->background[k];
  res->depth = res->depth / (res->opacity + 1e-10);
  free(clodw);
}

typedef struct {
  const lo_model* m;
  const lo_camera* cam;
  const lo_render_options* opts;
  const double* ts;
  double ratio;
  int row_begin, row_end;
  float *out, *depth, *opacity;
  int32_t *evals, *contributing, *kept;
  int64_t* row_evals;
  uint32_t* mask;
  int32_t* counts;
  atomic_int next_row;
} lo_job;

static void lo_render_row(lo_job* j, int y) {
  const lo_camera* cam = j->cam;
  const size_t W = cam->width, plane = (size_t)cam->width * cam->height;
  int64_t row_ev = 0;
  for (int x = 0; x < cam->width; ++x) {
    double o[3], d[3], no[3], nd[3];
    lo_generate_ray(cam, x + 0.5, y + 0.5, o, d);
    lo_generate_ray(cam, x + 1.5, y + 0.5, no, nd);
    lo_ray_result r;
    lo_march_ray(j->m, o, d, no, nd, j->ts, j->ratio, j->opts, &r);
    size_t p = (size_t)y * W + x;
    for (int c = 0; c < 3; ++c) j->out[c * plane + p] = (float)r.pixel[c];
    if (j->depth) j->depth[p] = (float)r.depth;
    if (j->opacity) j->opacity[p] = (float)r.opacity;
    if (j->evals) j->evals[p] = r.evals;
    if (j->contributing) j->contributing[p] = r.contributing;
    if (j->kept) j->kept[p] = r.kept;
    row_ev += r.evals;
  }
  if (j->row_evals) j->row_evals[y - j->row_begin] = row_ev;
}

static void lo_kept_row(lo_job* j, int y) {
  const lo_camera* cam = j->cam;
  const int n = j->opts->samples_per_ray, words = (n + 31) / 32;
  for (int x = 0; x < cam->width; ++x) {
    double o[3], d[3];
    lo_generate_ray(cam, x + 0.5, y + 0.5, o, d);
    size_t p = (size_t)y * cam->width + x;
    uint32_t* mk = j->mask ? j->mask + p * words : NULL;
    if (mk) memset(mk, 0, sizeof(uint32_t) * words);
    int cnt = 0;
    for (int i = 0; i < n; ++i) {
      double pos[3], c[3];
      lo_ray_at(o, d, j->ts[i], pos);
      lo_contract(pos, j->opts->contraction, c);
      if (!lo_occupied(j->m, c)) continue;
      if (mk) mk[i >> 5] |= 1u << (i & 31);
      ++cnt;
    }
    if (j->counts) j->counts[p] = cnt;
  }
}

static void* lo_render_worker(void* arg) {
  lo_job* j = (lo_job*)arg;
  for (;;) {
    int y = atomic_fetch_add(&j->next_row, 1);
    if (y >= j->row_end) break;
    lo_render_row(j, y);
  }
  return NULL;
}

static void* lo_kept_worker(void* arg) {
  lo_job* j = (lo_job*)arg;
  for (;;) {
    int y = atomic_fetch_add(&j->next_row, 1);
    if (y >= j->row_end) break;
    lo_kept_row(j, y);
  }
  return NULL;
}

static void lo_run(lo_job* j, void* (*fn)(void*), int nthreads) {
  atomic_store(&j->next_row, j->row_begin);
  if (nthreads <= 1) {
    fn(j);
    return;
  }
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * nthreads);
  for (int t = 0; t < nthreads; ++t) pthread_create(&th[t], NULL, fn, j);
  for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
  free(th);
}

static int lo_check(const lo_model* m, const lo_camera* cam, const lo_render_options* opts,
                    int b, int e) {
  if (!(b >= 0 && e <= cam->height && b <= e)) return -1;                   /* renderer.h:257 */
  if (!(cam->t_near > 0 && cam->t_far > cam->t_near && opts->samples_per_ray >= 2)) return -2;
  if (!(cam->fx > 0 && cam->fy > 0)) return -3;                             /* camera.cpp:20 */
  if (m && m->cfg.levels > LO_MAX_LEVELS) return -4;
  return 0;
}

int lo_render_rows(const lo_model* m, const lo_camera* cam, const lo_render_options* opts,
                   int row_begin, int row_end, float* out, float* depth, float* opacity,
                   int32_t* evals, int32_t* contributing, int32_t* kept, int64_t* row_evals,
                   int nthreads) {
  int rc = lo_check(m, cam, opts, row_begin, row_end);
  if (rc) return rc;
  const int n = opts->samples_per_ray;
  double* ts = (double*)malloc(sizeof(double) * n);
  double ratio;
  lo_sample_distances(cam->t_near, cam->t_far, n, ts, &ratio);
  lo_job j;
  memset(&j, 0, sizeof(j));
  j.m = m;
  j.cam = cam;
  j.opts = opts;
  j.ts = ts;
  j.ratio = ratio;
  j.row_begin = row_begin;
  j.row_end = row_end;
  j.out = out;
  j.depth = depth;
  j.opacity = opacity;
  j.evals = evals;
  j.contributing = contributing;
  j.kept = kept;
  j.row_evals = row_evals;
  lo_run(&j, lo_render_worker, nthreads);
  free(ts);
  return 0;
}

int lo_march_kept(const lo_model* m, const lo_camera* cam, const lo_render_options* opts,
                  int row_begin, int row_end, uint32_t* mask, int32_t* counts, int nthreads) {
  int rc = lo_check(m, cam, opts, row_begin, row_end);
  if (rc) return rc;
  const int n = opts->samples_per_ray;
  double* ts = (double*)malloc(sizeof(double) * n);
  lo_sample_distances(cam->t_near, cam->t_far, n, ts, NULL);
  lo_job j;
  memset(&j, 0, sizeof(j));
  j.m = m;
  j.cam = cam;
  j.opts = opts;
  j.ts = ts;
  j.row_begin = row_begin;
  j.row_end = row_end;
  j.mask = mask;
  j.counts = counts;
  lo_run(&j, lo_kept_worker, nthreads);
  free(ts);
  return 0;
}

/* ------------------------------------------------------------------------- */
/* Occupancy probe + prune (occupancy.cpp:97-154)                             */
/* ------------------------------------------------------------------------- */

typedef struct {
  const lo_model* m;
  const lo_camera* cams;
  int ncams, k, res;
  const double* ratios;
  float* probe_max;
  atomic_long next;
  long total;
} lo_probe_job;

static void* lo_probe_worker(void* arg) {
  lo_probe_job* j = (lo_probe_job*)arg;
  const int res = j->res, k = j->k, ppv = k * k * k, L = j->m->cfg.levels;
  const double e = 4.0 / res;
  double* pts = (double*)malloc(sizeof(double) * 3 * ppv);
  float* lodw = (float*)malloc(sizeof(float) * (size_t)ppv * L);
  float* sig = (float*)malloc(sizeof(float) * ppv);
  for (int i = 0; i < ppv * L; ++i) lodw[i] = 1.0f;
  for (;;) {
    long base = atomic_fetch_add(&j->next, 256);
    if (base >= j->total) break;
    long end = base + 256 < j->total ? base + 256 : j->total;
    for (long i = base; i < end; ++i) {
      int ix = (int)(i % res), iy = (int)((i / res) % res), iz = (int)(i / ((long)res * res));
      double c[3] = {-2.0 + (ix + 0.5) * e, -2.0 + (iy + 0.5) * e, -2.0 + (iz + 0.5) * e};
      double world[3];
      if (lo_linf(c) < 2.0)
        lo_uncontract(c, world);
      else
        memcpy(world, c, sizeof(world));
      double dt = 1e30;
      for (int ci = 0; ci < j->ncams; ++ci) {
        const lo_camera* cam = &j->cams[ci];
        double dv[3] = {world[0] - cam->origin[0], world[1] - cam->origin[1],
                        world[2] - cam->origin[2]};
        double dist = lo_max(lo_norm(dv), cam->t_near);
        dt = lo_min(dt, dist * (j->ratios[ci] - 1.0));
      }
      if (!(dt < 1e29)) dt = e;
      int mm = 0;
      for (int pz = 0; pz < k; ++pz)
        for (int py = 0; py < k; ++py)
          for (int px = 0; px < k; ++px) {
            pts[3 * mm + 0] = c[0] + e * ((px + 1.0) / (k + 1) - 0.5);
            pts[3 * mm + 1] = c[1] + e * ((py + 1.0) / (k + 1) - 0.5);
            pts[3 * mm + 2] = c[2] + e * ((pz + 1.0) / (k + 1) - 0.5);
            ++mm;
          }
      lo_field_forward(j->m, ppv, pts, lodw, NULL, sig, NULL, NULL);
      float best = 0.0f;
      for (int p = 0; p < ppv; ++p) {
        float conv = (float)((1.0 - exp(-sig[p] * dt)) / dt);
        best = best < conv ? conv : best; /* std::max(best, converted) */
      }
      j->probe_max[i] = best;
    }
  }
  free(pts);
  free(lodw);
  free(sig);
  return NULL;
}

int lo_probe(const lo_model* m, const lo_camera* cams, int ncams, int spp, int k, int res,
             float* probe_max, int nthreads) {
  if (k < 1 || res < 1 || spp < 2) return -1;
  double* ratios = (double*)malloc(sizeof(double) * (ncams > 0 ? ncams : 1));
  for (int ci = 0; ci < ncams; ++ci)
    ratios[ci] = pow(cams[ci].t_far / cams[ci].t_near, 1.0 / (spp - 1));
  lo_probe_job j;
  memset(&j, 0, sizeof(j));
  j.m = m;
  j.cams = cams;
  j.ncams = ncams;
  j.k = k;
  j.res = res;
  j.ratios = ratios;
  j.probe_max = probe_max;
  j.total = (long)res * res * res;
  atomic_store(&j.next, 0);
  if (nthreads <= 1) {
    lo_probe_worker(&j);
  } else {
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * nthreads);
    for (int t = 0; t < nthreads; ++t) pthread_create(&th[t], NULL, lo_probe_worker, &j);
    for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
    free(th);
  }
  free(ratios);
  return 0;
}

void lo_prune(const float* probe_max, const float* history, const uint8_t* carved, size_t n,
              float alpha, uint8_t* occ_out) {
  for (size_t i = 0; i < n; ++i) {
    if (carved && carved[i]) {
      occ_out[i] = 0;
      continue;
    }
    float h = history ? history[i] : 0.0f;
    float p = probe_max[i];
    occ_out[i] = (h < alpha && p < alpha) ? 0 : 1;
  }
}

/* ------------------------------------------------------------------------- */
/* Scheduler (scheduler.cpp:18-162)                                           */
/* ------------------------------------------------------------------------- */

typedef struct {
  double rem;
  int idx;
} lo_rem;

static int lo_rem_cmp(const void* a, const void* b) {
  const lo_rem *x = (const lo_rem*)a, *y = (const lo_rem*)b;
  if (x->rem != y->rem) return x->rem > y->rem ? -1 : 1;
  return x->idx - y->idx;
}

/* scheduler.cpp:18-44 */
static void lo_round_rows(const double* shares, int n, int height, int32_t* rows) {
  lo_rem* rem = (lo_rem*)malloc(sizeof(lo_rem) * n);
  int assigned = 0;
  for (int i = 0; i < n; ++i) {
    double exact = shares[i] * height;
    rows[i] = (int)floor(exact);
    rem[i].rem = exact - rows[i];
    rem[i].idx = i;
    assigned += rows[i];
  }
  qsort(rem, n, sizeof(lo_rem), lo_rem_cmp);
  for (int k = 0; k < height - assigned; ++k) rows[rem[k % n].idx] += 1;
  if (height >= n) {
    for (int i = 0; i < n; ++i) {
      while (rows[i] == 0) {
        int big = 0;
        for (int q = 1; q < n; ++q)
          if (rows[q] > rows[big]) big = q; /* std::max_element: first maximum */
        rows[big] -= 1;
        rows[i] += 1;
      }
    }
  }
  free(rem);
}

static void lo_from_rows(const int32_t* rows, int n, int height, double* shares) {
  for (int i = 0; i < n; ++i) shares[i] = (double)rows[i] / height; /* scheduler.cpp:46-59 */
}

int lo_equal_assignment(int height, int workers, int32_t* rows, double* shares) {
  if (workers < 1) return -1;
  if (height < workers) return -2;
  double* s = (double*)malloc(sizeof(double) * workers);
  for (int i = 0; i < workers; ++i) s[i] = 1.0 / workers;
  lo_round_rows(s, workers, height, rows);
  lo_from_rows(rows, workers, height, shares);
  free(s);
  return 0;
}

int lo_assign_rows(int height, int n, const double* tp, const double* prev_shares, double damp,
                   int32_t* rows, double* shares) {
  if (!(n >= 1 && height >= n)) return -1;
  double total = 0;
  for (int i = 0; i < n; ++i) {
    if (!(tp[i] > 0)) return -2;
    total += tp[i];
  }
  double* s = (double*)malloc(sizeof(double) * n);
  for (int i = 0; i < n; ++i) {
    double target = tp[i] / total;
    s[i] = prev_shares[i] + damp * (target - prev_shares[i]);
  }
  double sum = 0;
  for (int i = 0; i < n; ++i) sum += s[i];
  for (int i = 0; i < n; ++i) s[i] /= sum;
  lo_round_rows(s, n, height, rows);
  lo_from_rows(rows, n, height, shares);
  free(s);
  return 0;
}

int lo_next_assignment(int height, int n, const double* prev_shares, const int32_t* prev_rows,
                       const double* worker_ms, int width, double damp, int32_t* rows,
                       double* shares) {
  double* tp = (double*)malloc(sizeof(double) * n);
  for (int i = 0; i < n; ++i) { /* scheduler.cpp:154-162 */
    double ms = lo_max(worker_ms[i], 1e-6);
    double rays = (double)((int64_t)prev_rows[i] * width);
    tp[i] = lo_max(rays, 1.0) / (ms / 1000.0);
  }
  int rc = lo_assign_rows(height, n, tp, prev_shares, damp, rows, shares);
  free(tp);
  return rc;
}

static int lo_dcmp(const void* a, const void* b) {
  double x = *(const double*)a, y = *(const double*)b;
  return x < y ? -1 : (x > y ? 1 : 0);
}

int lo_aggregate_stats(const double* wall_ms, int n, double out[3]) { /* scheduler.cpp:89-112 */
  if (n <= 0) return -1;
  double* t = (double*)malloc(sizeof(double) * n);
  double mean = 0;
  for (int i = 0; i < n; ++i) {
    t[i] = wall_ms[i];
    mean += wall_ms[i] > 0 ? 1000.0 / wall_ms[i] : 0.0;
  }
  mean /= n;
  double var = 0;
  for (int i = 0; i < n; ++i) {
    double f = wall_ms[i] > 0 ? 1000.0 / wall_ms[i] : 0.0;
    var += (f - mean) * (f - mean);
  }
  var /= n;
  qsort(t, n, sizeof(double), lo_dcmp);
  double idx = 0.99 * (n - 1);
  size_t lo = (size_t)floor(idx);
  size_t hi = lo + 1 < (size_t)(n - 1) ? lo + 1 : (size_t)(n - 1);
  double frac = idx - lo;
  double p99 = t[lo] * (1 - frac) + t[hi] * frac;
  out[0] = mean;
  out[1] = sqrt(var);
  out[2] = p99 > 0 ? 1000.0 / p99 : 0.0;
  free(t);
  return 0;
}

/* ------------------------------------------------------------------------- */
/* Training reverse path: march_ray(record) + ray_loss + backward_ray         */
/* (renderer.h:126-237, train_step.h:16-154, field.h:106-179, network.h:115-136, */
/*  grid.h:118-137, simd.h:35-90 scalar order)                               */
/* ------------------------------------------------------------------------- */

/* FieldChunk (field.h:30-45) with feature-major activations of n <= LO_BATCH samples */
typedef struct {
  int n;
  double (*pos)[3];
  float *lodw, *feat, *h, *dout, *cin, *c1, *c2, *craw, *sigma_raw, *sigma, *color;
} lo_chunk;

static void lo_chunk_alloc(lo_chunk* c, int L, int F, int H, int B) {
  c->n = 0;
  c->pos = (double(*)[3])malloc(sizeof(double) * 3 * LO_BATCH);
  c->lodw = (float*)malloc(sizeof(float) * (size_t)L * LO_BATCH);
  c->feat = (float*)malloc(sizeof(float) * (size_t)F * LO_BATCH);
  c->h = (float*)malloc(sizeof(float) * (size_t)H * LO_BATCH);
  c->dout = (float*)malloc(sizeof(float) * (size_t)(1 + B) * LO_BATCH);
  c->cin = (float*)malloc(sizeof(float) * (size_t)(B + 16) * LO_BATCH);
  c->c1 = (float*)malloc(sizeof(float) * (size_t)H * LO_BATCH);
  c->c2 = (float*)malloc(sizeof(float) * (size_t)H * LO_BATCH);
  c->craw = (float*)malloc(sizeof(float) * 3 * LO_BATCH);
  c->sigma_raw = (float*)malloc(sizeof(float) * LO_BATCH);
  c->sigma = (float*)malloc(sizeof(float) * LO_BATCH);
  c->color = (float*)malloc(sizeof(float) * 3 * LO_BATCH);
}

static void lo_chunk_free(lo_chunk* c) {
  free(c->pos);
  free(c->lodw);
  free(c->feat);
  free(c->h);
  free(c->dout);
  free(c->cin);
  free(c->c1);
  free(c->c2);
  free(c->craw);
  free(c->sigma_raw);
  free(c->sigma);
  free(c->color);
}

/* RadianceField::forward_chunk with every activation kept (field.h:106-137) */
static void lo_chunk_forward(const lo_model* m, lo_chunk* ck, const float* sh) {
  const lo_field_config* cfg = &m->cfg;
  const int n = ck->n, L = cfg->levels, F = L * cfg->features_per_level, H = cfg->hidden_width,
            B = cfg->bottleneck;
  float one[LO_MAX_LEVELS * 8];
  for (int i = 0; i < n; ++i) {
    lo_encode(m, ck->pos[i], ck->lodw + (size_t)i * L, one);
    for (int f = 0; f < F; ++f) ck->feat[(size_t)f * n + i] = one[f];
  }
  const float* dp = m->dparams;
  lo_dense(m->mlp_mode, H, F, n, dp, dp + (size_t)H * F, ck->feat, ck->h, 1);
  dp += (size_t)H * F + H;
  lo_dense(m->mlp_mode, 1 + B, H, n, dp, dp + (size_t)(1 + B) * H, ck->h, ck->dout, 0);
  for (int i = 0; i < n; ++i) {
    ck->sigma_raw[i] = ck->dout[i];
    ck->sigma[i] = lo_trunc_exp(ck->dout[i]);
  }
  memcpy(ck->cin, ck->dout + n, sizeof(float) * (size_t)B * n);
  for (int s = 0; s < 16; ++s)
    for (int i = 0; i < n; ++i) ck->cin[(size_t)(B + s) * n + i] = sh[s];
  const float* cp = m->cparams;
  lo_dense(m->mlp_mode, H, B + 16, n, cp, cp + (size_t)H * (B + 16), ck->cin, ck->c1, 1);
  cp += (size_t)H * (B + 16) + H;
  lo_dense(m->mlp_mode, H, H, n, cp, cp + (size_t)H * H, ck->c1, ck->c2, 1);
  cp += (size_t)H * H + H;
  lo_dense(m->mlp_mode, 3, H, n, cp, cp + (size_t)3 * H, ck->c2, ck->craw, 0);
  for (int i = 0; i < 3 * n; ++i)
    ck->color[i] = cfg->color_space == 0 ? lo_sigmoid(ck->craw[i]) : lo_trunc_exp(ck->craw[i]);
}

static inline float lo_trunc_exp_grad(float x) { /* network.h:48-52 */
  return expf(x < 10.0f ? x : 10.0f);
}

/* simd::scalar::relu_backward / dense_backward_weights / dense_backward_data (simd.h:53-90) */
static void lo_relu_bwd(size_t mm, const float* y, float* dy) {
  for (size_t i = 0; i < mm; ++i)
    if (y[i] <= 0.0f) dy[i] = 0.0f;
}
static void lo_dense_bwd_w(int rows, int cols, int n, const float* dy, const float* x, float* dW,
                           float* db) {
  for (int r = 0; r < rows; ++r) {
    const float* dyr = dy + (size_t)r * n;
    float acc = 0.0f;
    for (int i = 0; i < n; ++i) acc += dyr[i];
    db[r] += acc;
    float* dwr = dW + (size_t)r * cols;
    for (int c = 0; c < cols; ++c) {
      const float* xc = x + (size_t)c * n;
      float a = 0.0f;
      for (int i = 0; i < n; ++i) a += dyr[i] * xc[i];
      dwr[c] += a;
    }
  }
}
static void lo_dense_bwd_x(int rows, int cols, int n, const float* W, const float* dy, float* dx) {
  for (int r = 0; r < rows; ++r) {
    const float* wr = W + (size_t)r * cols;
    const float* dyr = dy + (size_t)r * n;
    for (int c = 0; c < cols; ++c) {
      const float w = wr[c];
      float* dxc = dx + (size_t)c * n;
      for (int i = 0; i < n; ++i) dxc[i] += w * dyr[i];
    }
  }
}

/* Mlp::backward (network.h:115-136) for a stack of `nl` layers; acts[k] is layer k's output,
   dy0 the output gradient [out x n], dx (zeroed by the caller) the input gradient.  dy and
   scratch ping-pong like the reference's dy.swap(scratch); each holds maxdim x n floats. */
static void lo_mlp_backward(int nl, const int* in, const int* out, const int* relu,
                            const float* params, const float* x, const float* const* acts, int n,
                            const float* dy0, float* dx, float* grads, float* dy, float* scratch) {
  size_t off[4];
  size_t o = 0;
  for (int k = 0; k < nl; ++k) {
    off[k] = o;
    o += (size_t)out[k] * in[k] + out[k];
  }
  memcpy(dy, dy0, sizeof(float) * (size_t)out[nl - 1] * n);
  for (int k = nl - 1; k >= 0; --k) {
    if (relu[k]) lo_relu_bwd((size_t)out[k] * n, acts[k], dy);
    const float* input = k == 0 ? x : acts[k - 1];
    float* gw = grads + off[k];
    lo_dense_bwd_w(out[k], in[k], n, dy, input, gw, gw + (size_t)out[k] * in[k]);
    const float* W = params + off[k];
    if (k == 0) {
      lo_dense_bwd_x(out[k], in[k], n, W, dy, dx);
    } else {
      memset(scratch, 0, sizeof(float) * (size_t)in[k] * n);
      lo_dense_bwd_x(out[k], in[k], n, W, dy, scratch);
      float* t = dy;
      dy = scratch;
      scratch = t;
    }
  }
}

/* MultiResHashGrid::encode_backward (grid.h:118-137) for one sample */
static void lo_encode_backward(const lo_model* m, const double c[3], const float* w,
                               const float* dfeat, size_t stride, float* grad) {
  const lo_grid_layout* L = &m->layout;
  const int fpl = L->fpl;
  double u = (c[0] + 2.0) * 0.25, v = (c[1] + 2.0) * 0.25, s = (c[2] + 2.0) * 0.25;
  for (int l = 0; l < L->levels; ++l) {
    if (w[l] <= 0.0f) continue;
    const int res = L->resolution[l];
    double pu = lo_clamp(u, 0.0, 1.0) * res, pv = lo_clamp(v, 0.0, 1.0) * res,
           ps = lo_clamp(s, 0.0, 1.0) * res;
    int iu = (int)pu, iv = (int)pv, is = (int)ps;
    if (iu > res - 1) iu = res - 1;
    if (iv > res - 1) iv = res - 1;
    if (is > res - 1) is = res - 1;
    double fu = pu - iu, fv = pv - iv, fs = ps - is;
    const uint32_t verts = (uint32_t)res + 1;
    const float* dl = dfeat + (size_t)l * fpl * stride;
    float* base = grad + L->offset[l];
    for (int k = 0; k < 8; ++k) {
      uint32_t x = (uint32_t)iu + (k & 1), y = (uint32_t)iv + ((k >> 1) & 1),
               z = (uint32_t)is + ((k >> 2) & 1);
      uint32_t idx = L->dense[l] ? (z * verts + y) * verts + x
                                 : lo_spatial_hash(x, y, z, L->entries[l]);
      double wu = (k & 1) ? fu : 1.0 - fu;
      double wv = ((k >> 1) & 1) ? fv : 1.0 - fv;
      double ws = ((k >> 2) & 1) ? fs : 1.0 - fs;
      float tri = (float)(wu * wv * ws);
      float coeff = tri * w[l];
      float* entry = base + (size_t)idx * fpl;
      for (int f = 0; f < fpl; ++f) entry[f] += coeff * dl[(size_t)f * stride];
    }
  }
}

/* RadianceField::backward_chunk (field.h:141-179), colour evaluated */
static void lo_chunk_backward(const lo_model* m, const lo_chunk* ck, const float* dsigma,
                              const float* dcolor, float* g_grid, float* g_density,
                              float* g_color, float* work) {
  const lo_field_config* cfg = &m->cfg;
  const int n = ck->n, L = cfg->levels, F = L * cfg->features_per_level, H = cfg->hidden_width,
            B = cfg->bottleneck, CI = B + 16;
  float* bwd_dout = work;                            /* (1+B) x n */
  float* bwd_craw = bwd_dout + (size_t)(1 + B) * n;  /* 3 x n */
  float* bwd_cin = bwd_craw + (size_t)3 * n;         /* CI x n */
  float* bwd_feat = bwd_cin + (size_t)CI * n;        /* F x n */
  const int MD = (H > F ? H : F) > CI ? (H > F ? H : F) : CI;
  float* dyb = bwd_feat + (size_t)F * n;             /* MD x n */
  float* scratch = dyb + (size_t)MD * n;             /* MD x n */
  memset(bwd_dout, 0, sizeof(float) * (size_t)(1 + B) * n);
  if (dcolor) {
    for (int i = 0; i < 3 * n; ++i) {
      float g;
      if (cfg->color_space == 0) {
        float c = ck->color[i];
        g = c * (1.0f - c);
      } else {
        g = lo_trunc_exp_grad(ck->craw[i]);
      }
      bwd_craw[i] = dcolor[i] * g;
    }
    memset(bwd_cin, 0, sizeof(float) * (size_t)CI * n);
    const int in[3] = {CI, H, H}, out[3] = {H, H, 3}, relu[3] = {1, 1, 0};
    const float* acts[3] = {ck->c1, ck->c2, ck->craw};
    lo_mlp_backward(3, in, out, relu, m->cparams, ck->cin, acts, n, bwd_craw, bwd_cin, g_color,
                    dyb, scratch);
    memcpy(bwd_dout + n, bwd_cin, sizeof(float) * (size_t)B * n);
  }
  for (int i = 0; i < n; ++i) bwd_dout[i] = dsigma[i] * lo_trunc_exp_grad(ck->sigma_raw[i]);
  memset(bwd_feat, 0, sizeof(float) * (size_t)F * n);
  {
    const int in[2] = {F, H}, out[2] = {H, 1 + B}, relu[2] = {1, 0};
    const float* acts[2] = {ck->h, ck->dout};
    lo_mlp_backward(2, in, out, relu, m->dparams, ck->feat, acts, n, bwd_dout, bwd_feat,
                    g_density, dyb, scratch);
  }
  for (int i = 0; i < n; ++i)
    lo_encode_backward(m, ck->pos[i], ck->lodw + (size_t)i * L, bwd_feat + i, (size_t)n, g_grid);
}

static inline double lo_sgn(double x) { return x > 0 ? 1.0 : (x < 0 ? -1.0 : 0.0); }

int lo_train_backward(const lo_model* m, const double* cam_tnf, const double* alpha_v, int ncams,
                      const lo_train_ray* rays, int nrays, const lo_render_options* opts,
                      const lo_loss_config* lc, float* g_grid, float* g_density, float* g_color,
                      double* alpha_grad, lo_loss_terms* loss, int32_t* ray_evals,
                      int32_t* ray_contrib) {
  const lo_field_config* cfg = &m->cfg;
  const int L = cfg->levels, F = L * cfg->features_per_level, H = cfg->hidden_width,
            B = cfg->bottleneck;
  const int spp = opts->samples_per_ray, cs = opts->chunk_size;
  if (cfg->levels > LO_MAX_LEVELS || spp < 2 || cs < 1 || cs > LO_BATCH) return -2;
  const int max_chunks = (spp + cs - 1) / cs;
  lo_chunk* chunks = (lo_chunk*)malloc(sizeof(lo_chunk) * (size_t)max_chunks);
  for (int k = 0; k < max_chunks; ++k) lo_chunk_alloc(&chunks[k], L, F, H, B);
  double* ts = (double*)malloc(sizeof(double) * (size_t)spp);
  /* RayMarchRecord (renderer.h:34-50) */
  double *rt = (double*)malloc(sizeof(double) * spp), *rdelta = (double*)malloc(sizeof(double) * spp),
         *ralpha = (double*)malloc(sizeof(double) * spp), *rtrans = (double*)malloc(sizeof(double) * spp),
         *rweight = (double*)malloc(sizeof(double) * spp);
  float *rcolor = (float*)malloc(sizeof(float) * 3 * spp);
  uint8_t* rinner = (uint8_t*)malloc((size_t)spp);
  /* RayLossGrad (trainer.h:106-111) */
  double *g_w = (double*)malloc(sizeof(double) * spp), *g_col = (double*)malloc(sizeof(double) * 3 * spp);
  float *dsig = (float*)malloc(sizeof(float) * spp), *dcol = (float*)malloc(sizeof(float) * 3 * LO_BATCH);
  float* work = (float*)malloc(sizeof(float) * (size_t)(1 + 16 + 3 + 16 + 2 * LO_MAX_LEVELS * 8 + 256) *
                               LO_BATCH * 2);
  int rc = 0;

  for (int ri = 0; ri < nrays; ++ri) {
    const lo_train_ray* ray = &rays[ri];
    if (ray->camera < 0 || ray->camera >= ncams) {
      rc = -1;
      break;
    }
    const double t_near = cam_tnf[2 * ray->camera], t_far = cam_tnf[2 * ray->camera + 1];
    if (!(t_near > 0 && t_far > t_near)) { /* renderer.h:134 */
      rc = -3;
      break;
    }
    double ratio;
    lo_sample_distances(t_near, t_far, spp, ts, &ratio);

    /* ---- march_ray(record = true) (renderer.h:126-237) ---- */
    float sh[16];
    lo_sh_encode(ray->dir, sh);
    int nchunks = 0, nt = 0, nsig = 0, contributing = 0, evals = 0, terminated = 0;
    double trans = 1.0, pixel[3] = {0, 0, 0}, depth = 0, opacity = 0;
    lo_chunk* ck = &chunks[nchunks++];
    ck->n = 0;
#define LO_REC_FLUSH(CK)                                                                  \
  do {                                                                                    \
    lo_chunk* fc = (CK);                                                                  \
    if (fc->n > 0) {                                                                      \
      lo_chunk_forward(m, fc, sh);                                                        \
      evals += fc->n;                                                                     \
      const int base = nsig;                                                              \
      for (int i = 0; i < fc->n; ++i) {                                                   \
        const int s = base + i;                                                           \
        const double sigma = (double)fc->sigma[i];                                        \
        const double a = 1.0 - exp(-sigma * rdelta[s]);                                   \
        const double w = trans * a;                                                       \
        for (int c = 0; c < 3; ++c) rcolor[3 * s + c] = fc->color[(size_t)c * fc->n + i]; \
        ralpha[s] = a;                                                                    \
        rtrans[s] = trans;                                                                \
        rweight[s] = w;                                                                   \
        ++nsig;                                                                           \
        for (int c = 0; c < 3; ++c) pixel[c] += w * (double)fc->color[(size_t)c * fc->n + i]; \
        depth += w * rt[s];                                                               \
        opacity += w;                                                                     \
        trans *= 1.0 - a;                                                                 \
        ++contributing;                                                                   \
        if (opts->termination_transmittance > 0 && trans < opts->termination_transmittance) { \
          terminated = 1;                                                                 \
          break;                                                                          \
        }                                                                                 \
      }                                                                                   \
      while (nsig < nt) {                                                                 \
        const int s = nsig, i = s - base;                                                 \
        for (int c = 0; c < 3; ++c) rcolor[3 * s + c] = fc->color[(size_t)c * fc->n + i]; \
        ralpha[s] = 0.0;                                                                  \
        rtrans[s] = 0.0;                                                                  \
        rweight[s] = 0.0;                                                                 \
        ++nsig;                                                                           \
      }                                                                                   \
    }                                                                                     \
  } while (0)
    for (int i = 0; i < spp && !terminated; ++i) {
      double pos[3], c[3];
      lo_ray_at(ray->origin, ray->dir, ts[i], pos);
      lo_contract(pos, opts->contraction, c);
      if (!lo_occupied(m, c)) continue;
      const double delta = (i + 1 < spp) ? ts[i + 1] - ts[i] : ts[i] * (ratio - 1.0);
      float* w = ck->lodw + (size_t)ck->n * L;
      if (opts->lod_enabled) {
        double r_c = lo_contracted_footprint(ray->origin, ray->dir, ray->norigin, ray->ndir, ts[i],
                                             opts->contraction);
        double l_star = lo_lod_level(lo_max(r_c, 1e-12), cfg);
        lo_lod_weights(l_star, opts->lod_bias, L, w);
      } else {
        for (int l = 0; l < L; ++l) w[l] = 1.0f;
      }
      ck->pos[ck->n][0] = c[0];
      ck->pos[ck->n][1] = c[1];
      ck->pos[ck->n][2] = c[2];
      ck->n++;
      rt[nt] = ts[i];
      rdelta[nt] = delta;
      rinner[nt] = lo_linf(c) <= 1.0 ? 1 : 0;
      ++nt;
      if (ck->n >= cs) {
        LO_REC_FLUSH(ck);
        if (!terminated) {
          ck = &chunks[nchunks++];
          ck->n = 0;
        }
      }
    }
    if (!terminated) LO_REC_FLUSH(ck);
#undef LO_REC_FLUSH
    if (nchunks > 0 && chunks[nchunks - 1].n == 0) --nchunks;
    const double final_trans = trans;
    for (int c = 0; c < 3; ++c) pixel[c] += trans * opts->background[c];
    depth = depth / (opacity + 1e-10);
    if (ray_evals) ray_evals[ri] = evals;
    if (ray_contrib) ray_contrib[ri] = contributing;

    /* ---- ray_loss (train_step.h:16-123) ---- */
    const int n = nt;
    const double v_raw = 1.0 - alpha_v[ray->camera] * ray->vignette_r;
    const double v = lo_max(v_raw, 1e-3);
    const double inv_batch = lc->inv_batch;
    lo_loss_terms lt = {0, 0, 0, 0, 0};
    double dpix[3] = {0, 0, 0}, dv_total = 0, d_alpha_v = 0;
    for (int c = 0; c < 3; ++c) {
      double pred = v * pixel[c];
      double diff = pred - ray->gt[c];
      lt.image += fabs(diff) / 3.0 * inv_batch;
      double dpred = inv_batch * lo_sgn(diff) / 3.0;
      dpix[c] = dpred * v;
      dv_total += dpred * pixel[c];
    }
    if (v_raw > 1e-3) d_alpha_v += dv_total * (-ray->vignette_r);
    for (int i = 0; i < n; ++i) {
      double gw = 0;
      for (int c = 0; c < 3; ++c) {
        double ci = (double)rcolor[(size_t)i * 3 + c];
        gw += dpix[c] * ci;
        g_col[(size_t)i * 3 + c] = dpix[c] * rweight[i];
      }
      g_w[i] = gw;
    }
    const double W = opacity, D = depth, denom = W + 1e-10;
    double ddepth = 0;
    if (lc->depth_active && lc->lambda_depth > 0 && ray->gt_depth >= 0) {
      double diff = D - ray->gt_depth;
      lt.depth = lc->lambda_depth * fabs(diff) * inv_batch;
      ddepth = lc->lambda_depth * inv_batch * lo_sgn(diff);
    }
    double dvar_dD = 0, Wi = 0, V = 0;
    if (lc->lambda_dvar > 0) {
      double S2 = 0;
      for (int i = 0; i < n; ++i) {
        if (!rinner[i]) continue;
        Wi += rweight[i];
        S2 += rweight[i] * (rt[i] - D) * (rt[i] - D);
      }
      if (Wi > 1e-10) {
        V = S2 / Wi;
        lt.dvar = lc->lambda_dvar * V * inv_batch;
        for (int i = 0; i < n; ++i) {
          if (!rinner[i]) continue;
          g_w[i] += lc->lambda_dvar * inv_batch * ((rt[i] - D) * (rt[i] - D) - V) / Wi;
          dvar_dD += -2.0 * rweight[i] * (rt[i] - D) / Wi;
        }
        dvar_dD *= lc->lambda_dvar * inv_batch;
      }
    }
    if (lc->lambda_dist > 0) {
      double A = 0, Bs = 0, val = 0;
      for (int i = 0; i < n; ++i) {
        val += rweight[i] * (rt[i] * A - Bs);
        A += rweight[i];
        Bs += rweight[i] * rt[i];
      }
      val *= 2.0;
      lt.dist = lc->lambda_dist * val * inv_batch;
      double A_pre = 0, B_pre = 0;
      for (int i = 0; i < n; ++i) {
        double A_suf = A - A_pre - rweight[i];
        double B_suf = Bs - B_pre - rweight[i] * rt[i];
        double d = 2.0 * (rt[i] * A_pre - B_pre + B_suf - rt[i] * A_suf);
        g_w[i] += lc->lambda_dist * inv_batch * d;
        A_pre += rweight[i];
        B_pre += rweight[i] * rt[i];
      }
    }
    if (ddepth != 0 || dvar_dD != 0) {
      double dD_total = ddepth + dvar_dD;
      for (int i = 0; i < n; ++i) g_w[i] += dD_total * (rt[i] - D) / denom;
    }
    lt.total = lt.image + lt.depth + lt.dvar + lt.dist;
    loss->image += lt.image;
    loss->depth += lt.depth;
    loss->dvar += lt.dvar;
    loss->dist += lt.dist;

    /* ---- backward_ray (train_step.h:127-154) ---- */
    if (n > 0) {
      double d_final_trans = 0;
      for (int c = 0; c < 3; ++c) d_final_trans += dpix[c] * opts->background[c];
      double suffix = d_final_trans * final_trans; /* composite_backward_sigma, renderer.h:110-120 */
      for (int i = n - 1; i >= 0; --i) {
        double d = rdelta[i] * ((1.0 - ralpha[i]) * g_w[i] * rtrans[i] - suffix);
        dsig[i] = (float)d;
        suffix += g_w[i] * rweight[i];
      }
      int offset = 0;
      for (int k = 0; k < nchunks; ++k) {
        const lo_chunk* c = &chunks[k];
        for (int i = 0; i < c->n; ++i)
          for (int q = 0; q < 3; ++q)
            dcol[(size_t)q * c->n + i] = (float)g_col[(size_t)(offset + i) * 3 + q];
        lo_chunk_backward(m, c, dsig + offset, dcol, g_grid, g_density, g_color, work);
        offset += c->n;
      }
    }
    alpha_grad[ray->camera] += d_alpha_v;
  }

  /* trainer.cpp:606-607 (the ray-dependent terms) */
  loss->total = loss->image + loss->depth + loss->dvar + loss->dist;
  for (int k = 0; k < max_chunks; ++k) lo_chunk_free(&chunks[k]);
  free(chunks);
  free(ts);
  free(rt);
  free(rdelta);
  free(ralpha);
  free(rtrans);
  free(rweight);
  free(rcolor);
  free(rinner);
  free(g_w);
  free(g_col);
  free(dsig);
  free(dcol);
  free(work);
  return rc;
}

/* simd::scalar::adam_step (simd.h:106-121) */
void lo_adam_step(size_t n, float* p, const float* g, float* mom, float* vel, float lr, float beta1,
                  float beta2, float eps, float c1, float c2) {
  for (size_t i = 0; i < n; ++i) {
    float gi = g[i];
    float mi = beta1 * mom[i] + (1.0f - beta1) * gi;
    float vi = beta2 * vel[i] + (1.0f - beta2) * gi * gi;
    mom[i] = mi;
    vel[i] = vi;
    float mhat = mi * c1;
    float vhat = vi * c2;
    p[i] -= lr * mhat / (sqrtf(vhat) + eps);
  }
}
