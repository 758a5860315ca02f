// test_shim.cpp -- the drop-in seen from the reference's side: the same call site
// `render_rows(field, grid, cam, opts, b, e, &out, ...)` resolves to the B200 overload of
// include/lumi/cuda_renderer.h, and is checked against the reference template
// (render_rows<RadianceField<float>>, renderer.h:252) on the same model -- in the style of
// proj/tests/test_renderer.cpp.  Built by tests/cpp/Makefile against the reference headers and
// objects (oracle/_ref); run by tests/test_shim.py on the GPU box.
//
//   test_shim <occupancy.raw (128^3 bytes)>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <fstream>
#include <sstream>
#include <vector>

#include "lumi/cuda_frame.h"
#include "lumi/cuda_renderer.h"
#include "lumi/scheduler.h"

using namespace lumi;

static int g_fail = 0;
#define CHECK(cond)                                                     \
  do {                                                                  \
    if (!(cond)) {                                                      \
      std::printf("CHECK FAILED %s:%d: %s\n", __FILE__, __LINE__, #cond); \
      ++g_fail;                                                         \
    }                                                                   \
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
  std::vector<char> z(occ.size() * 9, 0);  // carved bytes + history + probe floats
  ss.write(z.data(), z.size());
  return OccupancyGrid::load(ss);
}

static double psnr_db(const Image<float>& a, const Image<float>& b) {  // image.cpp:101-111
  double mse = 0;
  for (size_t i = 0; i < a.data.size(); ++i) {
    double d = static_cast<double>(a.data[i]) - b.data[i];
    mse += d * d;
  }
  mse /= a.data.size();
  return mse <= 0 ? 99.0 : std::min(99.0, 10.0 * std::log10(1.0 / mse));
}

int main(int argc, char** argv) {
  if (argc < 2) {
    std::printf("usage: test_shim occupancy.raw\n");
    return 2;
  }
  const int res = 128;
  std::vector<uint8_t> occ(static_cast<size_t>(res) * res * res);
  std::ifstream f(argv[1], std::ios::binary);
  f.read(reinterpret_cast<char*>(occ.data()), occ.size());
  CHECK(f.good());
  OccupancyGrid grid = grid_from_bytes(occ, res);

  // the C1 synthetic model
  FieldConfig fc;
  fc.grid.table_size = 1u << 19;
  RadianceField<float> field(fc);
  field.init_random(1234);
  Rng rng(1235);
  float* g = field.grid().parameters();
  for (size_t i = 0; i < field.grid().parameter_count(); ++i) g[i] = rng.uniform(-1.0, 1.0);

  CameraModel cam;
  cam.width = cam.height = 256;
  cam.fx = cam.fy = 0.6 * 256;
  cam.cx = cam.cy = 128;
  cam.pose.rot = {1, 0, 0, 0, 0, -1, 0, 1, 0};
  cam.pose.origin = {0.1, -0.3, 0.05};
  RenderOptions opts;

  // reference template on the CPU vs the overload on the B200, same call shape
  Image<float> ref(256, 256, 3), gpu(256, 256, 3), gdepth(256, 256, 1), gop(256, 256, 1);
  std::vector<RowStats> rs, gs;
  auto t0 = std::chrono::steady_clock::now();
  render_rows<RadianceField<float>>(field, grid, cam, opts, 0, 256, &ref, nullptr, nullptr, &rs);
  auto t1 = std::chrono::steady_clock::now();
  render_rows(field, grid, cam, opts, 0, 256, &gpu, &gdepth, &gop, &gs);  // warm + upload
  auto t2 = std::chrono::steady_clock::now();
  render_rows(field, grid, cam, opts, 0, 256, &gpu, &gdepth, &gop, nullptr);
  auto t3 = std::chrono::steady_clock::now();
  double maxerr = 0;
  for (size_t i = 0; i < ref.data.size(); ++i)
    maxerr = std::max(maxerr, std::abs(static_cast<double>(ref.data[i]) - gpu.data[i]));
  const double p = psnr_db(ref, gpu);
  std::printf("C1 256x256: max|dPQ|=%.3e PSNR=%.1f dB  cpu %.1f ms  gpu(first) %.1f ms  gpu %.2f ms\n",
              maxerr, p, std::chrono::duration<double, std::milli>(t1 - t0).count(),
              std::chrono::duration<double, std::milli>(t2 - t1).count(),
              std::chrono::duration<double, std::milli>(t3 - t2).count());
  CHECK(maxerr <= 1e-3);
  CHECK(p >= 60.0);
  CHECK(gs.size() == 256 && rs.size() == 256);
  int64_t ev_ref = 0, ev_gpu = 0;
  for (int y = 0; y < 256; ++y) {
    CHECK(gs[y].row == y && gs[y].rays == 256);
    ev_ref += rs[y].evals;
    ev_gpu += gs[y].evals;
  }
  std::printf("evals ref %lld gpu %lld\n", (long long)ev_ref, (long long)ev_gpu);
  CHECK(std::llabs(ev_ref - ev_gpu) <= ev_ref / 100);

  // split renders == full render (renderer.h:248-251 determinism contract)
  Image<float> split(256, 256, 3);
  render_rows(field, grid, cam, opts, 0, 100, &split, nullptr, nullptr, nullptr);
  render_rows(field, grid, cam, opts, 100, 256, &split, nullptr, nullptr, nullptr);
  CHECK(split.data == gpu.data);

  // run_frame workers (scheduler.cpp:114-152) on disjoint bands, concurrently
  Image<float> frame(256, 256, 3);
  WorkerAssignment a = equal_assignment(256, 3);
  run_frame(a, 256, [&](int, RowRange r) {
    render_rows(field, grid, cam, opts, r.begin, r.end, &frame, nullptr, nullptr, nullptr);
  }, nullptr);
  CHECK(frame.data == gpu.data);

  // the native multi-GPU frame driver (include/lumi/cuda_frame.h): three workers sharing this
  // box's GPU render stereo frames; each frame equals the per-eye overload renders bit for
  // bit, and the partition follows next_assignment on the measured per-worker times
  {
    const int S = 128;
    CameraModel eye[2];
    for (int e = 0; e < 2; ++e) {
      eye[e] = cam;
      eye[e].width = eye[e].height = S;
      eye[e].fx = eye[e].fy = 0.6 * S;
      eye[e].cx = eye[e].cy = S / 2.0;
      eye[e].pose.origin.x += (e ? 0.032 : -0.032);
    }
    cuda::GpuFrameDriver drv(field, grid, {0, 0, 0}, S, S, 2);
    for (int f = 0; f < 3; ++f) {
      WorkerAssignment before = drv.assignment();
      Image<float> stacked(S, 2 * S, 3);
      FrameStats st = drv.render({eye[0], eye[1]}, opts, &stacked);
      CHECK(st.worker_ms.size() == 3 && st.rays == 2 * S * S);
      for (int e = 0; e < 2; ++e) {
        Image<float> one(S, S, 3);
        render_rows(field, grid, eye[e], opts, 0, S, &one, nullptr, nullptr, nullptr);
        bool same = true;
        for (int c = 0; c < 3; ++c)
          for (int y = 0; y < S; ++y)
            for (int x = 0; x < S; ++x) same &= one.at(x, y, c) == stacked.at(x, e * S + y, c);
        CHECK(same);
      }
      WorkerAssignment want = next_assignment(before, st, 0.5);
      WorkerAssignment got = drv.assignment();
      for (int i = 0; i < 3; ++i) CHECK(got.ranges[i].begin == want.ranges[i].begin && got.ranges[i].end == want.ranges[i].end);
      std::printf("frame driver frame %d: rows %d/%d/%d, worker ms %.3f/%.3f/%.3f\n", f,
                  before.ranges[0].count(), before.ranges[1].count(), before.ranges[2].count(),
                  st.worker_ms[0], st.worker_ms[1], st.worker_ms[2]);
    }
  }

  // error behaviour: lumi::Error on a bad row range, like the reference's require()
  bool threw = false;
  try {
    render_rows(field, grid, cam, opts, 5, 257, &gpu, nullptr, nullptr, nullptr);
  } catch (const Error&) {
    threw = true;
  }
  CHECK(threw);

  // parameter edits are picked up (fingerprinted cache)
  field.color_net().layers.back().bias[0] = 3.0f;
  Image<float> ref2(256, 256, 3), gpu2(256, 256, 3);
  render_rows<RadianceField<float>>(field, grid, cam, opts, 120, 136, &ref2, nullptr, nullptr, nullptr);
  render_rows(field, grid, cam, opts, 120, 136, &gpu2, nullptr, nullptr, nullptr);
  double e2 = 0;
  for (size_t i = 0; i < ref2.data.size(); ++i)
    e2 = std::max(e2, std::abs(static_cast<double>(ref2.data[i]) - gpu2.data[i]));
  CHECK(e2 <= 1e-3);
  cuda::release_all();
  std::printf(g_fail ? "FAILED (%d)\n" : "OK\n", g_fail);
  return g_fail ? 1 : 0;
}
