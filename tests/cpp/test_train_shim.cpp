// test_train_shim.cpp -- the training drop-in seen from the reference's side: the per-ray loop
// of trainer.cpp:549-562 (march_ray(record) + ray_loss + backward_ray, the reference
// templates, CPU) against lumi::cuda::train_rays_backward (include/lumi/cuda_train.h, B200) on
// the same model and batch, in the style of proj/tests/test_trainer.cpp.
//
//   test_train_shim <occupancy.raw (128^3 bytes)>
#include <cmath>
#include <cstdio>
#include <fstream>
#include <sstream>
#include <vector>

#include "lumi/cuda_train.h"
#include "lumi/train_step.h"

using namespace lumi;

static int g_fail = 0;
#define CHECK(cond)                                                       \
  do {                                                                    \
    if (!(cond)) {                                                        \
      std::printf("CHECK FAILED %s:%d: %s\n", __FILE__, __LINE__, #cond); \
      ++g_fail;                                                           \
    }                                                                     \
  } while (0)

static OccupancyGrid grid_from_bytes(const std::vector<uint8_t>& occ, int res) {
  std::stringstream ss;  // public RLE serialization (occupancy.cpp:200-243)
  auto put = [&](const auto& v) { ss.write(reinterpret_cast<const char*>(&v), sizeof(v)); };
  std::vector<std::pair<uint8_t, uint64_t>> rle;
  for (size_t i = 0; i < occ.size();) {
    uint64_t len = 1;
    while (i + len < occ.size() && occ[i + len] == occ[i]) ++len;
    rle.push_back({occ[i], len});
    i += len;
  }
  put(static_cast<int32_t>(res));
  put(static_cast<uint64_t>(rle.size()));
  for (auto& [v, n] : rle) {
    put(v);
    put(n);
  }
  std::vector<char> z(occ.size() * 9, 0);
  ss.write(z.data(), z.size());
  return OccupancyGrid::load(ss);
}

static double max_abs(const std::vector<float>& v) {
  double m = 0;
  for (float x : v) m = std::max(m, (double)std::fabs(x));
  return m;
}
static double max_diff(const std::vector<float>& a, const std::vector<float>& b) {
  double m = 0;
  for (size_t i = 0; i < a.size(); ++i) m = std::max(m, (double)std::fabs(a[i] - b[i]));
  return m;
}

int main(int argc, char** argv) {
  if (argc < 2) return 2;
  const int res = 128;
  std::vector<uint8_t> occ((size_t)res * res * res);
  std::ifstream(argv[1], std::ios::binary).read(reinterpret_cast<char*>(occ.data()), occ.size());
  OccupancyGrid grid = grid_from_bytes(occ, res);

  FieldConfig fc;
  fc.grid.table_size = 1u << 19;
  RadianceField<float> field(fc);
  field.init_random(1234);
  Rng g(1235);  // trainer.cpp:257-259 pattern: structured grid
  for (size_t i = 0; i < field.grid().parameter_count(); ++i)
    field.grid().parameters()[i] = static_cast<float>(g.uniform(-1.0, 1.0));

  // training views: pinhole 256^2 around the probe pose (presets.cpp:36-48 convention)
  std::vector<CameraModel> cams;
  for (int k = 0; k < 4; ++k) {
    CameraModel c;
    const double yaw = 0.3 * (k - 1.5);
    const double cy = std::cos(yaw), sy = std::sin(yaw);
    const double R[9] = {cy, sy, 0, 0, 0, -1, -sy, cy, 0};  // camera z -> world (sy, cy, 0)
    for (int i = 0; i < 9; ++i) c.pose.rot[i] = R[i];
    c.pose.origin = {0.1, -0.3, 0.05};
    c.fx = c.fy = 153.6;
    c.cx = c.cy = 128;
    c.width = c.height = 256;
    cams.push_back(c);
  }
  Rng rng(77);
  std::vector<TrainRay> batch;
  for (int k = 0; k < 4; ++k)
    for (int i = 0; i < 128; ++i) {
      TrainRay r;
      r.camera = k;
      r.px = static_cast<int>(rng.next_below(256));
      r.py = static_cast<int>(rng.next_below(256));
      r.ray = generate_ray(cams[k], r.px + 0.5, r.py + 0.5);
      r.neighbor = generate_ray_unchecked(cams[k], r.px + 1.5, r.py + 0.5);
      for (int c = 0; c < 3; ++c) r.gt[c] = static_cast<float>(rng.uniform());
      r.gt_depth = (i % 2) ? rng.uniform(0.3, 3.0) : -1.0;
      r.vignette_r = rng.uniform(0.0, 1.0);
      batch.push_back(r);
    }
  const std::vector<double> alpha_v = {0.0, 0.03, 0.06, 0.09};
  TrainConfig cfg;
  RenderOptions opts;
  opts.background[0] = 0.1;
  opts.background[1] = 0.2;
  opts.background[2] = 0.3;
  const double inv_batch = 1.0 / batch.size();

  // the reference loop (trainer.cpp:549-562)
  FieldGradients<float> gref = field.make_gradients();
  std::vector<double> aref(cams.size(), 0.0);
  LossTerms lref;
  RayMarchRecord<float> rec;
  RayLossGrad rg;
  std::vector<float> scratch, dcol;
  for (const auto& ray : batch) {
    const CameraModel& cam = cams[ray.camera];
    march_ray(field, grid, ray.ray, ray.neighbor, cam.t_near, cam.t_far, opts, true, rec);
    LossTerms lt = ray_loss(rec, ray, alpha_v[ray.camera], opts.contraction, cfg, true, inv_batch, &rg);
    lref.image += lt.image;
    lref.depth += lt.depth;
    lref.dvar += lt.dvar;
    lref.dist += lt.dist;
    backward_ray(field, rec, rg, opts.background, gref, scratch, dcol);
    aref[ray.camera] += rg.d_alpha_v;
  }
  // the drop-in
  FieldGradients<float> gdev = field.make_gradients();
  std::vector<double> adev(cams.size(), 0.0);
  LossTerms ldev = cuda::train_rays_backward(field, grid, cams, batch, alpha_v, opts, cfg, true,
                                             inv_batch, gdev, adev);
  std::printf("loss image %.9g/%.9g depth %.9g/%.9g dvar %.9g/%.9g dist %.9g/%.9g\n", lref.image,
              ldev.image, lref.depth, ldev.depth, lref.dvar, ldev.dvar, lref.dist, ldev.dist);
  auto rel = [](double a, double b) { return std::fabs(a - b) <= 1e-6 * std::fabs(b) + 1e-12; };
  CHECK(rel(ldev.image, lref.image));
  CHECK(rel(ldev.depth, lref.depth));
  CHECK(rel(ldev.dvar, lref.dvar));
  CHECK(rel(ldev.dist, lref.dist));
  const double eg = max_diff(gdev.grid, gref.grid), sg = max_abs(gref.grid);
  const double ed = max_diff(gdev.density, gref.density), sd = max_abs(gref.density);
  const double ec = max_diff(gdev.color, gref.color), sc = max_abs(gref.color);
  std::printf("grads max err grid %.3g / %.3g, density %.3g / %.3g, color %.3g / %.3g\n", eg, sg,
              ed, sd, ec, sc);
  CHECK(sg > 0 && eg <= 1e-4 * sg);
  CHECK(sd > 0 && ed <= 1e-4 * sd);
  CHECK(sc > 0 && ec <= 1e-4 * sc);
  for (size_t c = 0; c < cams.size(); ++c) CHECK(rel(adev[c], aref[c]));
  // errors surface as lumi::Error (common.h:61-70)
  bool threw = false;
  try {
    std::vector<double> bad_alpha = {0.0};
    cuda::train_rays_backward(field, grid, cams, batch, bad_alpha, opts, cfg, true, inv_batch,
                              gdev, adev);
  } catch (const Error&) {
    threw = true;
  }
  CHECK(threw);
  if (g_fail) {
    std::printf("FAILED (%d)\n", g_fail);
    return 1;
  }
  std::printf("OK\n");
  return 0;
}
