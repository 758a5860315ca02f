// ref_wrap.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" shim over the UNMODIFIED reference library, compiled from the
// reference's own sources where they lie (see oracle/Makefile; nothing is copied
// into this repo).  It exposes the reference's rendering path with the same
// plain-array conventions as lumi_oracle.h so tests can pin the C restatement
// against the real thing, and so bench.py can time the reference CPU renderer
// (cpu_baseline "kind": "reference", and `--impl reference`).
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <sstream>
#include <string>
#include <vector>

#include "lumi/camera.h"
#include "lumi/color.h"
#include "lumi/field.h"
#include "lumi/grid.h"
#include "lumi/image.h"
#include "lumi/occupancy.h"
#include "lumi/renderer.h"
#include "lumi/scene.h"
#include "lumi/scheduler.h"
#include "lumi/simd.h"
#include "lumi/train_step.h"
#include "lumi/trainer.h"

#include "lumi_oracle.h"

using namespace lumi;

namespace {

thread_local std::string g_err;

FieldConfig to_cfg(const lo_field_config* c) {
  FieldConfig fc;
  fc.grid.levels = c->levels;
  fc.grid.features_per_level = c->features_per_level;
  fc.grid.base_resolution = c->base_resolution;
  fc.grid.per_level_scale = c->per_level_scale;
  fc.grid.table_size = c->table_size;
  fc.hidden_width = c->hidden_width;
  fc.bottleneck = c->bottleneck;
  fc.color_space = c->color_space == 0 ? ColorSpaceMode::kPq : ColorSpaceMode::kLinear;
  return fc;
}

CameraModel to_cam(const lo_camera* c) {
  CameraModel cam;
  for (int i = 0; i < 9; ++i) cam.pose.rot[i] = c->rot[i];
  cam.pose.origin = {c->origin[0], c->origin[1], c->origin[2]};
  cam.fx = c->fx;
  cam.fy = c->fy;
  cam.cx = c->cx;
  cam.cy = c->cy;
  cam.width = c->width;
  cam.height = c->height;
  cam.t_near = c->t_near;
  cam.t_far = c->t_far;
  return cam;
}

RenderOptions to_opts(const lo_render_options* o) {
  RenderOptions r;
  r.samples_per_ray = o->samples_per_ray;
  r.lod_bias = o->lod_bias;
  r.lod_enabled = o->lod_enabled != 0;
  r.termination_transmittance = o->termination_transmittance;
  for (int c = 0; c < 3; ++c) r.background[c] = o->background[c];
  r.contraction.mode = o->contraction == 0 ? ContractionMode::kNone : ContractionMode::kLInfCubic;
  r.chunk_size = o->chunk_size;
  return r;
}

// Builds an OccupancyGrid through its public serialization (occupancy.cpp:224-243):
// RLE bits, no carving, zero trackers.
OccupancyGrid make_grid(const uint8_t* occ, int res) {
  std::stringstream ss;
  auto put = [&](const auto& v) { ss.write(reinterpret_cast<const char*>(&v), sizeof(v)); };
  const size_t n = static_cast<size_t>(res) * res * res;
  std::vector<std::pair<uint8_t, uint64_t>> rle;
  size_t i = 0;
  while (i < n) {
    uint8_t v = occ[i] ? 1 : 0;
    uint64_t len = 1;
    while (i + len < n && (occ[i + len] ? 1 : 0) == v) ++len;
    rle.emplace_back(v, len);
    i += len;
  }
  put(static_cast<int32_t>(res));
  put(static_cast<uint64_t>(rle.size()));
  for (auto& [v, len] : rle) {
    put(v);
    put(len);
  }
  std::vector<uint8_t> zeros(n, 0);
  ss.write(reinterpret_cast<const char*>(zeros.data()), n);  // carved
  std::vector<float> fz(n, 0.0f);
  ss.write(reinterpret_cast<const char*>(fz.data()), n * sizeof(float));  // history
  ss.write(reinterpret_cast<const char*>(fz.data()), n * sizeof(float));  // probe
  return OccupancyGrid::load(ss);
}

struct RefModel {
  FieldConfig cfg;
  RadianceField<float> field;
  OccupancyGrid grid;
  RefModel(const FieldConfig& c, const float* table, const float* dp, const float* cp,
           const uint8_t* occ, int res)
      : cfg(c), field(c), grid(make_grid(occ, res)) {
    std::memcpy(field.grid().parameters(), table, field.grid().parameter_count() * sizeof(float));
    field.density_net().set_params(dp);
    field.color_net().set_params(cp);
  }
};

// Duck-typed field with the renderer plugin interface (renderer.h:122-129), as in the
// reference's own SlabField test double: zero density, so marching with the cut disabled
// records every occupancy-kept sample without network cost.
struct ZeroField {
  using Scalar = float;
  static constexpr int kShDim = 16;
  FieldConfig cfg;
  const FieldConfig& config() const { return cfg; }
  void forward_chunk(FieldChunk<float>& ck, const float*, bool with_color) const {
    ck.sigma.assign(ck.n, 0.0f);
    ck.sigma_raw.assign(ck.n, 0.0f);
    ck.color.assign(3 * static_cast<size_t>(ck.n), 0.0f);
    ck.color_evaluated = with_color;
  }
};

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
const char* ref_simd_name() { return simd::active().name; }

int ref_layout(const lo_field_config* c, lo_grid_layout* out) {
  return guarded([&] {
    FieldConfig fc = to_cfg(c);
    MultiResHashGrid<float> g(fc.grid);
    std::memset(out, 0, sizeof(*out));
    out->levels = fc.grid.levels;
    out->fpl = fc.grid.features_per_level;
    uint64_t off = 0;
    for (int l = 0; l < fc.grid.levels; ++l) {
      out->resolution[l] = fc.grid.resolution(l);
      out->dense[l] = g.level_is_dense(l);
      uint64_t v = static_cast<uint64_t>(out->resolution[l]) + 1;
      out->entries[l] = out->dense[l] ? static_cast<uint32_t>(v * v * v) : fc.grid.table_size;
      out->offset[l] = off;
      off += static_cast<uint64_t>(out->entries[l]) * fc.grid.features_per_level;
    }
    out->total_floats = g.parameter_count();
  });
}

// RadianceField<float>::init_random(seed) then grid overwrite Rng(seed+1).uniform(-amp, amp)
// (the pattern of trainer.cpp:257-259).
int ref_synth_params(const lo_field_config* c, uint64_t seed, double amp, float* table,
                     float* dparams, float* cparams) {
  return guarded([&] {
    RadianceField<float> f(to_cfg(c));
    f.init_random(seed);
    if (amp > 0) {
      Rng rng(seed + 1);
      float* g = f.grid().parameters();
      for (size_t i = 0; i < f.grid().parameter_count(); ++i) g[i] = rng.uniform(-amp, amp);
    }
    std::memcpy(table, f.grid().parameters(), f.grid().parameter_count() * sizeof(float));
    f.density_net().copy_params(dparams);
    f.color_net().copy_params(cparams);
  });
}

void* ref_model_create(const lo_field_config* c, const float* table, const float* dp,
                       const float* cp, const uint8_t* occ, int res) {
  RefModel* m = nullptr;
  if (guarded([&] { m = new RefModel(to_cfg(c), table, dp, cp, occ, res); })) return nullptr;
  return m;
}

void ref_model_destroy(void* h) { delete static_cast<RefModel*>(h); }

// The reference render_rows loop (renderer.h:252-278) with the per-ray march record
// exposed: evals (rec.evals), contributing, kept (= rec.t.size(), samples marched
// before the cut, chunk tail included).
int ref_render_rows(void* h, const lo_camera* c, const lo_render_options* o, int b, int e,
                    float* out, float* depth, float* opacity, int32_t* evals,
                    int32_t* contributing, int32_t* kept, int64_t* row_evals) {
  return guarded([&] {
    RefModel& m = *static_cast<RefModel*>(h);
    CameraModel cam = to_cam(c);
    RenderOptions opts = to_opts(o);
    require(b >= 0 && e <= cam.height && b <= e, "render_rows: row range outside image");
    RayMarchRecord<float> rec;
    const size_t plane = static_cast<size_t>(cam.width) * cam.height;
    for (int y = b; y < e; ++y) {
      int64_t ev = 0;
      for (int x = 0; x < cam.width; ++x) {
        Ray ray = generate_ray(cam, x + 0.5, y + 0.5);
        Ray nb = generate_ray_unchecked(cam, x + 1.5, y + 0.5);
        march_ray(m.field, m.grid, ray, nb, cam.t_near, cam.t_far, opts, false, rec);
        size_t p = static_cast<size_t>(y) * cam.width + x;
        for (int k = 0; k < 3; ++k) out[k * plane + p] = static_cast<float>(rec.pixel[k]);
        if (depth) depth[p] = static_cast<float>(rec.depth);
        if (opacity) opacity[p] = static_cast<float>(rec.opacity);
        if (evals) evals[p] = rec.evals;
        if (contributing) contributing[p] = rec.contributing;
        if (kept) kept[p] = static_cast<int32_t>(rec.t.size());
        ev += rec.evals;
      }
      if (row_evals) row_evals[y - b] = ev;
    }
  });
}

// Plain call of the reference template render_rows (renderer.h:252), for timing.
int ref_render_rows_plain(void* h, const lo_camera* c, const lo_render_options* o, int b, int e,
                          float* out, double* ms) {
  return guarded([&] {
    RefModel& m = *static_cast<RefModel*>(h);
    CameraModel cam = to_cam(c);
    RenderOptions opts = to_opts(o);
    Image<float> img(cam.width, cam.height, 3);
    auto t0 = std::chrono::steady_clock::now();
    render_rows(m.field, m.grid, cam, opts, b, e, &img, nullptr, nullptr, nullptr);
    *ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    if (out) std::memcpy(out, img.data.data(), img.data.size() * sizeof(float));
  });
}

// run_frame (scheduler.cpp:114-152) over `workers` std::threads, each calling the
// reference render_rows on its band of rows [b, e) split by equal_assignment.
int ref_run_frame(void* h, const lo_camera* c, const lo_render_options* o, int b, int e,
                  int workers, float* out, double* wall_ms) {
  return guarded([&] {
    RefModel& m = *static_cast<RefModel*>(h);
    CameraModel cam = to_cam(c);
    RenderOptions opts = to_opts(o);
    Image<float> img(cam.width, cam.height, 3);
    WorkerAssignment a = equal_assignment(e - b, workers);
    FrameStats st = run_frame(
        a, cam.width,
        [&](int, RowRange r) {
          render_rows(m.field, m.grid, cam, opts, b + r.begin, b + r.end, &img, nullptr, nullptr,
                      nullptr);
        },
        nullptr);
    *wall_ms = st.wall_ms;
    if (out) std::memcpy(out, img.data.data(), img.data.size() * sizeof(float));
  });
}

// Occupancy-kept sample indices from the reference march itself: march the ZeroField with
// the early cut disabled and map rec.t back onto the exact sample distances.
int ref_march_kept(void* h, const lo_camera* c, const lo_render_options* o, int b, int e,
                   uint32_t* mask, int32_t* counts) {
  return guarded([&] {
    RefModel& m = *static_cast<RefModel*>(h);
    CameraModel cam = to_cam(c);
    RenderOptions opts = to_opts(o);
    opts.termination_transmittance = 0;
    ZeroField zf;
    zf.cfg = m.cfg;
    const int n = opts.samples_per_ray, words = (n + 31) / 32;
    std::vector<double> ts = sample_distances(cam.t_near, cam.t_far, n);
    RayMarchRecord<float> rec;
    for (int y = b; y < e; ++y)
      for (int x = 0; x < cam.width; ++x) {
        Ray ray = generate_ray(cam, x + 0.5, y + 0.5);
        Ray nb = generate_ray_unchecked(cam, x + 1.5, y + 0.5);
        march_ray(zf, m.grid, ray, nb, cam.t_near, cam.t_far, opts, false, rec);
        size_t p = static_cast<size_t>(y) * cam.width + x;
        uint32_t* mk = mask ? mask + p * words : nullptr;
        if (mk) std::memset(mk, 0, sizeof(uint32_t) * words);
        size_t j = 0;
        for (double t : rec.t) {
          while (j < ts.size() && ts[j] != t) ++j;
          require(j < ts.size(), "ref_march_kept: sample distance not on the grid");
          if (mk) mk[j >> 5] |= 1u << (j & 31);
        }
        if (counts) counts[p] = static_cast<int32_t>(rec.t.size());
      }
  });
}

int ref_field_forward(void* h, int n, const double* pos3, const float* lodw, const float* sh,
                      float* sigma, float* color3, float* feat) {
  return guarded([&] {
    RefModel& m = *static_cast<RefModel*>(h);
    FieldChunk<float> ck;
    ck.n = n;
    for (int i = 0; i < n; ++i) ck.pos.push_back({pos3[3 * i], pos3[3 * i + 1], pos3[3 * i + 2]});
    ck.lodw.assign(lodw, lodw + static_cast<size_t>(n) * m.cfg.grid.levels);
    m.field.forward_chunk(ck, sh, sh != nullptr);
    for (int i = 0; i < n; ++i) sigma[i] = ck.sigma[i];
    if (color3 && sh) std::memcpy(color3, ck.color.data(), ck.color.size() * sizeof(float));
    if (feat) std::memcpy(feat, ck.feat.data(), ck.feat.size() * sizeof(float));
  });
}

// OccupancyGrid::probe (occupancy.cpp:97-142) with the training-time density functor
// (trainer.cpp:651-657: forward_chunk(with_color=false), all-ones LOD) then prune(alpha).
int ref_probe_prune(void* h, const lo_camera* cams, int ncams, int spp, int k, int res,
                    float alpha, float* probe_max, uint8_t* occ_out) {
  return guarded([&] {
    RefModel& m = *static_cast<RefModel*>(h);
    std::vector<CameraModel> cv;
    for (int i = 0; i < ncams; ++i) cv.push_back(to_cam(&cams[i]));
    OccupancyGrid g(res);
    FieldChunk<float> chunk;
    auto density = [&](const Vec3* pts, int count, float* outp) {
      chunk.n = count;
      chunk.pos.assign(pts, pts + count);
      chunk.lodw.assign(static_cast<size_t>(count) * m.cfg.grid.levels, 1.0f);
      m.field.forward_chunk(chunk, nullptr, false);
      for (int i = 0; i < count; ++i) outp[i] = chunk.sigma[i];
    };
    g.probe(density, cv, spp, k);
    g.prune(alpha);
    for (size_t i = 0; i < g.voxel_count(); ++i) {
      if (probe_max) probe_max[i] = g.probe_density(i);
      if (occ_out) occ_out[i] = g.occupied_bit(i) ? 1 : 0;
    }
  });
}

// save_checkpoint (scene.cpp:320-351) of the model, for the checkpoint-ingest parity test.
int ref_save_checkpoint(void* h, const char* path, int spp, const double* background,
                        int contraction) {
  return guarded([&] {
    RefModel& m = *static_cast<RefModel*>(h);
    Checkpoint ck{m.cfg, m.field, m.grid, {0.01, 0.02}, {background[0], background[1], background[2]},
                  contraction ? ContractionMode::kLInfCubic : ContractionMode::kNone, spp};
    save_checkpoint(ck, path);
  });
}

// write_pfm (image.cpp:20-35) of a planar float image, for the PFM writer parity test.
int ref_write_pfm(const char* path, const float* planar, int w, int h, int c) {
  return guarded([&] {
    Image<float> img(w, h, c);
    std::memcpy(img.data.data(), planar, sizeof(float) * static_cast<size_t>(w) * h * c);
    write_pfm(path, img);
  });
}

// ---- scalar functions for known-answer pinning ----
void ref_generate_ray(const lo_camera* c, double px, double py, double o[3], double d[3]) {
  Ray r = generate_ray_unchecked(to_cam(c), px, py);
  o[0] = r.origin.x; o[1] = r.origin.y; o[2] = r.origin.z;
  d[0] = r.dir.x; d[1] = r.dir.y; d[2] = r.dir.z;
}
void ref_contract(const double x[3], int mode, double out[3]) {
  Vec3 v = contract({x[0], x[1], x[2]},
                    ContractionSpec{mode ? ContractionMode::kLInfCubic : ContractionMode::kNone});
  out[0] = v.x; out[1] = v.y; out[2] = v.z;
}
double ref_lod_level(double r, const lo_field_config* c) { return lod_level(r, to_cfg(c).grid); }
void ref_lod_weights(double l, double bias, int levels, float* w) { lod_weights(l, bias, levels, w); }
double ref_pq_encode(double y) { return pq_encode(y); }
double ref_pq_decode(double v) { return pq_decode(v); }
double ref_srgb_oetf(double v) { return srgb_oetf(v); }
void ref_sh_encode(const double d[3], float out[16]) { sh_encode_deg3(Vec3{d[0], d[1], d[2]}, out); }

// ---- scheduler ----
int ref_equal_assignment(int height, int workers, int32_t* rows, double* shares) {
  return guarded([&] {
    auto a = equal_assignment(height, workers);
    for (int i = 0; i < workers; ++i) {
      rows[i] = a.ranges[i].count();
      shares[i] = a.shares[i];
    }
  });
}
int ref_assign_rows(int height, int n, const double* tp, const double* prev_shares,
                    const int32_t* prev_rows, double damp, int32_t* rows, double* shares) {
  return guarded([&] {
    WorkerAssignment prev;
    prev.height = height;
    int at = 0;
    for (int i = 0; i < n; ++i) {
      prev.ranges.push_back({at, at + prev_rows[i]});
      prev.shares.push_back(prev_shares[i]);
      at += prev_rows[i];
    }
    auto a = assign_rows(height, std::vector<double>(tp, tp + n), prev, damp);
    for (int i = 0; i < n; ++i) {
      rows[i] = a.ranges[i].count();
      shares[i] = a.shares[i];
    }
  });
}
int ref_aggregate_stats(const double* ms, int n, double out[3]) {
  return guarded([&] {
    std::vector<FrameStats> fr(n);
    for (int i = 0; i < n; ++i) fr[i].wall_ms = ms[i];
    auto s = aggregate_stats(fr);
    out[0] = s.mean_fps;
    out[1] = s.std_fps;
    out[2] = s.p99_fps;
  });
}

// The training loop's per-ray body (trainer.cpp:549-561): march_ray(record = true),
// ray_loss, backward_ray, accumulated into FieldGradients exactly as train() does.
int ref_train_backward(void* h, const double* cam_tnf, const double* alpha_v, int ncams,
                       const lo_train_ray* rays, int nrays, const lo_render_options* o,
                       const lo_loss_config* lc, float* g_grid, float* g_density, float* g_color,
                       double* alpha_grad, lo_loss_terms* loss, int32_t* ray_evals,
                       int32_t* ray_contrib) {
  return guarded([&] {
    RefModel& m = *static_cast<RefModel*>(h);
    RenderOptions opts = to_opts(o);
    TrainConfig cfg;
    cfg.lambda_depth = lc->lambda_depth;
    cfg.lambda_dvar = lc->lambda_dvar;
    cfg.lambda_dist = lc->lambda_dist;
    FieldGradients<float> grads = m.field.make_gradients();
    std::memcpy(grads.grid.data(), g_grid, grads.grid.size() * sizeof(float));
    std::memcpy(grads.density.data(), g_density, grads.density.size() * sizeof(float));
    std::memcpy(grads.color.data(), g_color, grads.color.size() * sizeof(float));
    RayMarchRecord<float> rec;
    RayLossGrad rg;
    std::vector<float> scratch, dcol_scratch;
    LossTerms losses;
    losses.image = loss->image;
    losses.depth = loss->depth;
    losses.dvar = loss->dvar;
    losses.dist = loss->dist;
    for (int i = 0; i < nrays; ++i) {
      const lo_train_ray& r = rays[i];
      require(r.camera >= 0 && r.camera < ncams, "ref_train_backward: camera index");
      TrainRay tr;
      tr.camera = r.camera;
      tr.ray.origin = {r.origin[0], r.origin[1], r.origin[2]};
      tr.ray.dir = {r.dir[0], r.dir[1], r.dir[2]};
      tr.neighbor.origin = {r.norigin[0], r.norigin[1], r.norigin[2]};
      tr.neighbor.dir = {r.ndir[0], r.ndir[1], r.ndir[2]};
      for (int c = 0; c < 3; ++c) tr.gt[c] = r.gt[c];
      tr.gt_depth = r.gt_depth;
      tr.vignette_r = r.vignette_r;
      march_ray(m.field, m.grid, tr.ray, tr.neighbor, cam_tnf[2 * r.camera],
                cam_tnf[2 * r.camera + 1], opts, true, rec);
      LossTerms lt = ray_loss(rec, tr, alpha_v[r.camera], opts.contraction, cfg,
                              lc->depth_active != 0, lc->inv_batch, &rg);
      losses.image += lt.image;
      losses.depth += lt.depth;
      losses.dvar += lt.dvar;
      losses.dist += lt.dist;
      backward_ray(m.field, rec, rg, opts.background, grads, scratch, dcol_scratch);
      alpha_grad[r.camera] += rg.d_alpha_v;
      if (ray_evals) ray_evals[i] = static_cast<int32_t>(rec.t.size());
      if (ray_contrib) ray_contrib[i] = rec.contributing;
    }
    loss->image = losses.image;
    loss->depth = losses.depth;
    loss->dvar = losses.dvar;
    loss->dist = losses.dist;
    loss->total = losses.image + losses.depth + losses.dvar + losses.dist;
    std::memcpy(g_grid, grads.grid.data(), grads.grid.size() * sizeof(float));
    std::memcpy(g_density, grads.density.data(), grads.density.size() * sizeof(float));
    std::memcpy(g_color, grads.color.data(), grads.color.size() * sizeof(float));
  });
}

// simd::adam_step through the active ISA table (simd.h:238-247)
void ref_adam_step(size_t n, float* p, const float* g, float* mom, float* vel, float lr, float beta1,
                   float beta2, float eps, float c1, float c2) {
  simd::adam_step<float>(n, p, g, mom, vel, lr, beta1, beta2, eps, c1, c2);
}

}  // extern "C"
