/*
 * lumi_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C (C11) CPU restatement of the reference VR-NeRF ("lumifield")
 * frame-rendering path, used as the parity checker for the sm_100a CUDA
 * implementation in paper_2311_02542_b200/.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg may load this library; the product path never
 * links it and fails loudly when its CUDA extension is missing.
 *
 * Every function cites the reference file:line it restates (paths relative to
 * the reference checkout, proj/...).  The restatement is PINNED against the real
 * reference compiled from its own sources into oracle/_ref/ (see oracle/Makefile,
 * oracle/ref_wrap.cpp) and against the reference unit tests' known-answer values
 * (tests/test_oracle_*.py).
 *
 * Floating-point contract: compiled without -mfma / -ffast-math so that double
 * geometry and float field arithmetic round exactly as the reference's
 * non-SIMD translation units do (proj/CMakeLists.txt:39-47).  The dense-layer
 * inner product can replay the scalar, AVX2 or AVX-512 accumulation order of
 * proj/src/simd_*.cpp (LO_MLP_*), so the oracle is bit-identical to the
 * reference on the same host ISA.
 */
#ifndef LUMI_ORACLE_H
#define LUMI_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LO_MAX_LEVELS 32

/* proj/include/lumi/grid.h:18-29 + proj/include/lumi/field.h:22-27 */
typedef struct {
  int32_t levels;
  int32_t features_per_level;
  int32_t base_resolution;
  int32_t hidden_width;
  double per_level_scale;
  uint32_t table_size;
  int32_t bottleneck;
  int32_t color_space; /* 0 = kPq (sigmoid head), 1 = kLinear (trunc_exp head) */
  int32_t _pad;
} lo_field_config;

/* proj/include/lumi/grid.h:58-74 (MultiResHashGrid constructor layout) */
typedef struct {
  int32_t levels;
  int32_t fpl;
  int32_t resolution[LO_MAX_LEVELS];
  uint32_t entries[LO_MAX_LEVELS];
  uint8_t dense[LO_MAX_LEVELS];
  uint64_t offset[LO_MAX_LEVELS]; /* in floats */
  uint64_t total_floats;
} lo_grid_layout;

/* proj/include/lumi/camera.h:15-23 */
typedef struct {
  double rot[9]; /* row-major world <- camera */
  double origin[3];
  double fx, fy, cx, cy;
  int32_t width, height;
  double t_near, t_far;
} lo_camera;

/* proj/include/lumi/renderer.h:22-30 */
typedef struct {
  int32_t samples_per_ray;
  int32_t lod_enabled;
  double lod_bias;
  double termination_transmittance;
  double background[3];
  int32_t contraction; /* 0 = kNone, 1 = kLInfCubic (camera.h:32-38) */
  int32_t chunk_size;
} lo_render_options;

enum { LO_MLP_SCALAR = 0, LO_MLP_AVX2 = 1, LO_MLP_AVX512 = 2 };

typedef struct {
  lo_field_config cfg;
  lo_grid_layout layout;
  const float* table;   /* layout.total_floats */
  const float* dparams; /* density net, weights then bias per layer (network.h:144-151) */
  const float* cparams; /* color net, same order */
  const uint8_t* occ;   /* occ_res^3 bytes, index (iz*res+iy)*res+ix */
  int32_t occ_res;
  int32_t mlp_mode;     /* LO_MLP_* */
} lo_model;

/* ---- RNG: pcg32 (common.h:78-169) ---- */
typedef struct {
  uint64_t state, inc;
} lo_rng;
void lo_rng_init(lo_rng* r, uint64_t seed);
uint32_t lo_rng_u32(lo_rng* r);
void lo_rng_advance(lo_rng* r, uint64_t delta);
double lo_rng_uniform(lo_rng* r);
double lo_rng_normal(lo_rng* r);

/* ---- model ---- */
int lo_layout(const lo_field_config* cfg, lo_grid_layout* out);
size_t lo_density_param_count(const lo_field_config* cfg);
size_t lo_color_param_count(const lo_field_config* cfg);
/* RadianceField::init_random(seed) then grid overwrite Rng(seed+1).uniform(-amp,amp) when amp>0 */
int lo_synth_params(const lo_field_config* cfg, uint64_t seed, double amp, float* table,
                    float* dparams, float* cparams);

/* ---- scalar geometry (exposed for known-answer tests) ---- */
void lo_generate_ray(const lo_camera* cam, double px, double py, double origin[3], double dir[3]);
int lo_contract(const double x[3], int mode, double out[3]);
int64_t lo_voxel_index(int res, const double c[3]);
double lo_contracted_footprint(const double o0[3], const double d0[3], const double o1[3],
                               const double d1[3], double t, int mode);
double lo_lod_level(double r, const lo_field_config* cfg);
void lo_lod_weights(double l_star, double bias, int levels, float* w);
void lo_sh_encode(const double dir[3], float out[16]);
void lo_sample_distances(double t_near, double t_far, int n, double* ts, double* ratio);
double lo_pq_encode(double y);
double lo_pq_decode(double v);
double lo_srgb_oetf(double v);

/* ---- field ---- */
void lo_encode(const lo_model* m, const double c[3], const float* w, float* out /*L*F*/);
/* n points, lodw [n x levels], sh [16] shared or NULL (density only). */
void lo_field_forward(const lo_model* m, int n, const double* pos3, const float* lodw,
                      const float* sh, float* sigma, float* color3 /*[3 x n] or NULL*/,
                      float* feat /*[F x n] or NULL*/);

/* ---- march / render ---- */
/* Per-pixel outputs are optional (NULL).  Images are full-size planar
   (out: 3*W*H, depth/opacity: W*H); per-pixel int stats are W*H.  row_evals
   has (row_end-row_begin) entries.  Returns 0 or a negative error code. */
int lo_render_rows(const lo_model* m, const lo_camera* cam, const lo_render_options* opts,
                   int row_begin, int row_end, float* out, float* depth, float* opacity,
                   int32_t* evals, int32_t* contributing, int32_t* kept, int64_t* row_evals,
                   int nthreads);
/* Occupancy-kept sample bitmask per pixel (words_per_ray = ceil(spp/32)), independent of
   the network: every candidate that passes the occupancy test (renderer.h:205-208). */
int lo_march_kept(const lo_model* m, const lo_camera* cam, const lo_render_options* opts,
                  int row_begin, int row_end, uint32_t* mask, int32_t* counts, int nthreads);

/* ---- occupancy bake (occupancy.cpp:97-154) ---- */
int lo_probe(const lo_model* m, const lo_camera* cams, int ncams, int samples_per_ray,
             int points_per_axis, int res, float* probe_max, int nthreads);
void lo_prune(const float* probe_max, const float* history, const uint8_t* carved, size_t n,
              float alpha, uint8_t* occ_out);

/* ---- training reverse path (trainer.cpp:549-569, train_step.h, field.h:141-179) ---- */
/* TrainRay (trainer.h:90-97): the ray, its right-neighbour ray, target, depth, vignette */
typedef struct {
  double origin[3], dir[3];
  double norigin[3], ndir[3];
  float gt[3];
  int32_t camera;
  double gt_depth; /* < 0: unavailable */
  double vignette_r;
} lo_train_ray;

/* the TrainConfig fields ray_loss reads (trainer.h:18-60) + the per-iteration flags */
typedef struct {
  double lambda_depth, lambda_dvar, lambda_dist;
  double inv_batch;
  int32_t depth_active;
  int32_t _pad;
} lo_loss_config;

/* LossTerms (trainer.h:99-102), the ray-dependent part */
typedef struct {
  double total, image, depth, dvar, dist;
} lo_loss_terms;

/* For every ray: march_ray(record = true) + ray_loss + backward_ray, exactly as the
   training loop (trainer.cpp:549-561).  cam_tnf: [ncams][2] (t_near, t_far); alpha_v:
   [ncams].  Gradients are ACCUMULATED into g_grid [layout.total_floats], g_density,
   g_color (FieldGradients, weights-then-bias order) and alpha_grad [ncams]; loss terms are
   summed over the rays.  ray_evals / ray_contrib (optional, [nrays]) receive
   rec.t.size() and rec.contributing.  The dense backward replays the scalar order
   (simd.h:53-90), so it is bit-identical to the reference under LUMI_SIMD=scalar. */
int lo_train_backward(const lo_model* m, const double* cam_tnf, const double* alpha_v, int ncams,
                      const lo_train_ray* rays, int nrays, const lo_render_options* opts,
                      const lo_loss_config* lc, float* g_grid, float* g_density, float* g_color,
                      double* alpha_grad, lo_loss_terms* loss, int32_t* ray_evals,
                      int32_t* ray_contrib);
/* simd::scalar::adam_step (simd.h:106-121) */
void lo_adam_step(size_t n, float* p, const float* g, float* mom, float* vel, float lr, float beta1,
                  float beta2, float eps, float c1, float c2);

/* ---- scheduler (scheduler.cpp:18-162) ---- */
int lo_equal_assignment(int height, int workers, int32_t* rows, double* shares);
int lo_assign_rows(int height, int n, const double* throughputs, const double* prev_shares,
                   double dampening, int32_t* rows, double* shares);
int lo_next_assignment(int height, int n, const double* prev_shares, const int32_t* prev_rows,
                       const double* worker_ms, int width, double dampening, int32_t* rows,
                       double* shares);
int lo_aggregate_stats(const double* wall_ms, int n, double out[3] /*mean,std,p99 fps*/);

#ifdef __cplusplus
}
#endif
#endif
