// lumi/cuda_renderer.h -- drop-in B200 backend for the reference renderer.
//
// Include this after (or instead of) "lumi/renderer.h" from the reference tree
// (proj/include/lumi/renderer.h).  It adds a NON-TEMPLATE overload of render_rows for
// RadianceField<float>; overload resolution prefers it over the template at
// renderer.h:252-256, so every existing call site -- the run_frame worker lambdas
// (scheduler.cpp:126-135), evaluate() (trainer.cpp:205) -- renders on the GPU through the C
// ABI (include/lumi_cuda.h) without source changes.  Contract kept from the reference:
//   * out is caller-allocated at full image size; only rows [row_begin,row_end) are written;
//   * depth_out / opacity_out / stats are optional; stats gets one RowStats per row appended;
//   * a bad row range (or any device failure) throws lumi::Error via lumi::fail;
//   * re-entrant: concurrent calls on disjoint rows from run_frame workers are safe; each
//     worker thread may pick its GPU with lumi::cuda::set_thread_device().
// The field/grid are uploaded once per (object, device) and re-uploaded when their contents
// change, matching the reference's "read-only during a frame" rule (SPEC.md volume_renderer).
// The fingerprint checked on every call covers the whole occupancy grid and both MLPs, and
// samples the hash-grid table (every ~n/4096-th float): after an edit that touches only table
// entries (e.g. an optimizer step on the grid), call lumi::cuda::invalidate() -- it drops the
// cached device copies so the next call re-uploads.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "lumi/renderer.h"
#include "lumi_cuda.h"

namespace lumi {
namespace cuda {

inline void check(int rc, const char* what) {
  if (rc != LUMI_OK) fail(std::string(what) + ": " + lumi_last_error());
}

inline int& thread_device() {
  thread_local int dev = 0;
  return dev;
}
inline void set_thread_device(int device) { thread_device() = device; }

inline LumiFieldDesc to_desc(const FieldConfig& c) {
  LumiFieldDesc d{};
  d.levels = c.grid.levels;
  d.features_per_level = c.grid.features_per_level;
  d.base_resolution = c.grid.base_resolution;
  d.hidden_width = c.hidden_width;
  d.per_level_scale = c.grid.per_level_scale;
  d.table_size = c.grid.table_size;
  d.bottleneck = c.bottleneck;
  d.color_space = c.color_space == ColorSpaceMode::kPq ? 0 : 1;
  return d;
}

inline LumiCameraDesc to_desc(const CameraModel& c) {
  LumiCameraDesc d{};
  for (int i = 0; i < 9; ++i) d.rot[i] = c.pose.rot[i];
  d.origin[0] = c.pose.origin.x;
  d.origin[1] = c.pose.origin.y;
  d.origin[2] = c.pose.origin.z;
  d.fx = c.fx;
  d.fy = c.fy;
  d.cx = c.cx;
  d.cy = c.cy;
  d.width = c.width;
  d.height = c.height;
  d.t_near = c.t_near;
  d.t_far = c.t_far;
  return d;
}

inline LumiRenderOptions to_desc(const RenderOptions& o) {
  LumiRenderOptions d{};
  d.samples_per_ray = o.samples_per_ray;
  d.lod_enabled = o.lod_enabled ? 1 : 0;
  d.lod_bias = o.lod_bias;
  d.termination_transmittance = o.termination_transmittance;
  for (int c = 0; c < 3; ++c) d.background[c] = o.background[c];
  d.contraction = o.contraction.mode == ContractionMode::kNone ? 0 : 1;
  d.chunk_size = o.chunk_size;
  return d;
}

// Device-resident copy of one (field, grid) pair.
class DeviceField {
 public:
  DeviceField(const RadianceField<float>& field, const OccupancyGrid& grid, int device)
      : device_(device) {
    upload(field, grid);
  }
  ~DeviceField() { lumi_model_destroy(model_); }
  DeviceField(const DeviceField&) = delete;
  DeviceField& operator=(const DeviceField&) = delete;

  static uint64_t fingerprint(const RadianceField<float>& field, const OccupancyGrid& grid) {
    uint64_t h = 1469598103934665603ULL;
    auto mix = [&](const void* p, size_t n) {
      const auto* b = static_cast<const uint8_t*>(p);
      for (size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 1099511628211ULL;
    };
    const float* t = field.grid().parameters();
    const size_t n = field.grid().parameter_count();
    for (size_t i = 0; i < n; i += 1 + n / 4096) mix(t + i, sizeof(float));
    std::vector<float> p(field.density_net().parameter_count());
    field.density_net().copy_params(p.data());
    mix(p.data(), p.size() * sizeof(float));
    p.resize(field.color_net().parameter_count());
    field.color_net().copy_params(p.data());
    mix(p.data(), p.size() * sizeof(float));
    // every occupancy bit, 64 voxels per mixing step
    const int res = grid.resolution();
    mix(&res, sizeof(res));
    const size_t nv = grid.voxel_count();
    for (size_t i = 0; i < nv; i += 64) {
      uint64_t w = 0;
      const size_t hi = std::min<size_t>(64, nv - i);
      for (size_t b = 0; b < hi; ++b) w |= static_cast<uint64_t>(grid.occupied_bit(i + b)) << b;
      h = (h ^ w) * 0x9E3779B97F4A7C15ULL;
      h ^= h >> 29;
    }
    return h;
  }

  void upload(const RadianceField<float>& field, const OccupancyGrid& grid) {
    if (model_) lumi_model_destroy(model_);
    model_ = nullptr;
    const LumiFieldDesc d = to_desc(field.config());
    std::vector<float> dp(field.density_net().parameter_count()),
        cp(field.color_net().parameter_count());
    field.density_net().copy_params(dp.data());  // weights then bias (network.h:144-151)
    field.color_net().copy_params(cp.data());
    std::vector<uint8_t> occ(grid.voxel_count());
    for (size_t i = 0; i < occ.size(); ++i) occ[i] = grid.occupied_bit(i) ? 1 : 0;
    check(lumi_model_create(device_, &d, field.grid().parameters(), dp.data(), cp.data(),
                            occ.data(), grid.resolution(), &model_),
          "lumi_model_create");
    fp_ = fingerprint(field, grid);
  }

  LumiModel* model() const { return model_; }
  uint64_t fp() const { return fp_; }

 private:
  int device_;
  LumiModel* model_ = nullptr;
  uint64_t fp_ = 0;
};

inline std::mutex& cache_mutex() {
  static std::mutex m;
  return m;
}

inline std::map<std::tuple<const void*, const void*, int>, std::shared_ptr<DeviceField>>&
cache() {
  static std::map<std::tuple<const void*, const void*, int>, std::shared_ptr<DeviceField>> c;
  return c;
}

inline std::shared_ptr<DeviceField> device_field(const RadianceField<float>& field,
                                                 const OccupancyGrid& grid, int device) {
  const uint64_t fp = DeviceField::fingerprint(field, grid);
  std::lock_guard<std::mutex> lk(cache_mutex());
  auto key = std::make_tuple(static_cast<const void*>(&field), static_cast<const void*>(&grid),
                             device);
  auto& slot = cache()[key];
  if (!slot || slot->fp() != fp) slot = std::make_shared<DeviceField>(field, grid, device);
  return slot;
}

// Drops every cached device copy (e.g. before destroying the field).  In-flight renders keep
// their copy alive through the shared_ptr they hold.
inline void release_all() {
  std::lock_guard<std::mutex> lk(cache_mutex());
  cache().clear();
}

// Forces a re-upload of every cached copy of `field` on its next render (needed after edits the
// sampled table fingerprint cannot see, see the header comment).
template <class FieldT>
inline void invalidate(const FieldT& field) {
  std::lock_guard<std::mutex> lk(cache_mutex());
  for (auto it = cache().begin(); it != cache().end();)
    it = std::get<0>(it->first) == static_cast<const void*>(&field) ? cache().erase(it) : std::next(it);
}

}  // namespace cuda

// The drop-in (see header comment).  Chosen over the template render_rows<FieldT> of
// renderer.h:252 for RadianceField<float> arguments.
inline void render_rows(const RadianceField<float>& field, const OccupancyGrid& grid,
                        const CameraModel& cam, const RenderOptions& opts, int row_begin,
                        int row_end, Image<float>* out, Image<float>* depth_out,
                        Image<float>* opacity_out, std::vector<RowStats>* stats) {
  require(row_begin >= 0 && row_end <= cam.height && row_begin <= row_end,
          "render_rows: row range outside image");
  require(out && out->width == cam.width && out->height == cam.height && out->channels == 3,
          "render_rows: output image must be the camera's full size with 3 channels");
  if (depth_out)
    require(depth_out->width == cam.width && depth_out->height == cam.height,
            "render_rows: depth image size mismatch");
  if (opacity_out)
    require(opacity_out->width == cam.width && opacity_out->height == cam.height,
            "render_rows: opacity image size mismatch");
  auto dev = cuda::device_field(field, grid, cuda::thread_device());
  const LumiCameraDesc c = cuda::to_desc(cam);
  const LumiRenderOptions o = cuda::to_desc(opts);
  std::vector<LumiRowStats> st(stats ? static_cast<size_t>(row_end - row_begin) : 0);
  cuda::check(lumi_render_rows(dev->model(), &c, &o, row_begin, row_end, out->data.data(),
                               depth_out ? depth_out->data.data() : nullptr,
                               opacity_out ? opacity_out->data.data() : nullptr,
                               stats ? st.data() : nullptr),
              "lumi_render_rows");
  if (stats)
    for (const auto& s : st) stats->push_back({s.row, s.ms, s.rays, s.evals});
}

}  // namespace lumi
