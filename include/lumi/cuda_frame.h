// lumi/cuda_frame.h -- the reference's multi-worker frame (run_frame + next_assignment,
// proj/include/lumi/scheduler.h:60-73, proj/src/scheduler.cpp:114-162) with B200s as the
// workers, for C++ callers of the drop-in.
//
//   lumi::cuda::GpuFrameDriver drv(field, grid, {0, 1, 2, 3}, 2048, 2048, /*eyes=*/2);
//   Image<float> frame(2048, 2 * 2048, 3);             // both eyes stacked
//   FrameStats st = drv.render({left, right}, opts, &frame);
//
// One host thread per GPU inside liblumi_cuda.so renders its band of the stacked eyes; the
// bands land in one device frame on the first GPU over NVLink peer access (the render
// kernels store there directly), which is then copied into `frame`.  The next frame's bands
// follow next_assignment on the per-GPU CUDA-event times.  The same device may be listed
// several times (several workers sharing one GPU, one stream each).
#pragma once

#include <cstdint>
#include <memory>
#include <vector>

#include "lumi/cuda_renderer.h"
#include "lumi/scheduler.h"
#include "lumi_cuda.h"

namespace lumi {
namespace cuda {

class GpuFrameDriver {
 public:
  GpuFrameDriver(const RadianceField<float>& field, const OccupancyGrid& grid,
                 const std::vector<int>& devices, int width, int eye_height, int eyes = 2,
                 double dampening = 0.5)
      : width_(width), height_(eye_height * eyes), eyes_(eyes) {
    require(!devices.empty(), "GpuFrameDriver: need at least one device");
    std::vector<LumiModel*> models;
    for (int dev : devices) {
      replicas_.push_back(device_field(field, grid, dev));  // one upload per device
      models.push_back(replicas_.back()->model());
    }
    check(lumi_frame_driver_create(models.data(), static_cast<int>(models.size()), width,
                                   eye_height, eyes, dampening, &drv_),
          "lumi_frame_driver_create");
  }
  ~GpuFrameDriver() { lumi_frame_driver_destroy(drv_); }
  GpuFrameDriver(const GpuFrameDriver&) = delete;
  GpuFrameDriver& operator=(const GpuFrameDriver&) = delete;

  // The assignment the next render() uses (scheduler.h:22-35).
  WorkerAssignment assignment() const {
    const size_t n = replicas_.size();
    std::vector<int32_t> rows(n);
    WorkerAssignment a;
    a.shares.resize(n);
    check(lumi_frame_driver_assignment(drv_, rows.data(), a.shares.data()), "lumi_frame_driver_assignment");
    a.height = height_;
    int at = 0;
    for (size_t i = 0; i < n; ++i) {
      a.ranges.push_back({at, at + rows[i]});
      at += rows[i];
    }
    return a;
  }

  // One frame: out is (width x eyes*eye_height x 3), eye e's rows stacked at e * eye_height.
  FrameStats render(const std::vector<CameraModel>& eyes, const RenderOptions& opts, Image<float>* out) {
    require(static_cast<int>(eyes.size()) == eyes_, "GpuFrameDriver: one camera per eye");
    require(out && out->width == width_ && out->height == height_ && out->channels == 3,
            "GpuFrameDriver: output must hold the stacked eyes");
    std::vector<LumiCameraDesc> c;
    for (const auto& e : eyes) c.push_back(to_desc(e));
    const LumiRenderOptions o = to_desc(opts);
    FrameStats st;
    st.worker_ms.resize(replicas_.size());
    st.worker_rays.resize(replicas_.size());
    check(lumi_frame_driver_render_host(drv_, c.data(), &o, out->data.data(), &st.wall_ms,
                                        st.worker_ms.data(), st.worker_rays.data()),
          "lumi_frame_driver_render");
    st.rays = static_cast<int64_t>(height_) * width_;
    return st;
  }

 private:
  std::vector<std::shared_ptr<DeviceField>> replicas_;
  LumiFrameDriver* drv_ = nullptr;
  int width_, height_, eyes_;
};

}  // namespace cuda
}  // namespace lumi
