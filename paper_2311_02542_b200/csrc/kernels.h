// kernels.h -- host-visible launchers of the sm_100a kernels and their parameter blocks.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>

#include "render_common.cuh"

// Kernel attributes (cudaFuncSetAttribute: dynamic shared memory, carveout) belong to the
// device context, and the drop-in drives several GPUs from one process (run_frame workers, one
// per device, scheduler.cpp:114-152): every launcher keeps its one-time setup PER DEVICE, and
// the first calls of concurrent workers serialise on the mutex instead of racing.
struct PerDeviceInit {
  static constexpr int kMaxDevices = 64;
  std::mutex mu;
  int value[kMaxDevices];
  PerDeviceInit() {
    for (int& v : value) v = -1;
  }
  // init(int* out) runs once per device (the current one); *out is cached and returned
  template <class F>
  cudaError_t get(F&& init, int* out) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= kMaxDevices) return cudaErrorInvalidDevice;
    std::lock_guard<std::mutex> lk(mu);
    if (value[dev] < 0) {
      int v = 0;
      if ((e = init(&v)) != cudaSuccess) return e;
      value[dev] = v < 0 ? 0 : v;
    }
    *out = value[dev];
    return cudaSuccess;
  }
};

namespace lumi_dev {

struct BakeParams {
  GridDev grid;
  MlpDev mlp;
  int res, k, ncams;
  float alpha;
  const double* cam_origin;  // [ncams][3]
  const double* cam_tnear;   // [ncams]
  const double* cam_ratio;   // [ncams] host pow(t_far/t_near, 1/(spp-1))
  float* probe_max;
  uint8_t* occ;
};

// ---- training reverse path (train.cu) ----------------------------------------------------
// LumiTrainRay (include/lumi_cuda.h), TrainRay (trainer.h:90-97)
struct LumiTrainRayDev {
  double origin[3], dir[3];
  double norigin[3], ndir[3];
  float gt[3];
  int32_t camera;
  double gt_depth;
  double vignette_r;
};
static_assert(sizeof(LumiTrainRayDev) == 128, "LumiTrainRay layout");

// One occupancy-kept sample of a training ray (RayMarchRecord t/delta/inner + FieldChunk
// pos/lodw, renderer.h:34-50, field.h:30-35)
struct TrainSample {
  double c[3];  // contracted position
  double t, delta;
  int32_t ray;
  int32_t lod_full;
  float lod_frac;
  uint8_t floor_only, inner, _pad[2];
};

struct TrainParams {
  GridDev grid;
  MlpDev mlp;
  const uint8_t* occ;
  int occ_res;
  int n;  // samples_per_ray
  int lod_enabled;
  double lod_bias;
  double t_cut;
  double bg[3];
  int contraction;
  int chunk;
  // batch
  const LumiTrainRayDev* rays;
  int nrays;
  int ncams;
  const double* cam_ts;     // [ncams][n] host-computed exponential distances
  const double* cam_ratio;  // [ncams]
  const double* alpha_v;    // [ncams]
  // loss (TrainConfig, trainer.h:18-60)
  double lambda_depth, lambda_dvar, lambda_dist, inv_batch;
  int depth_active;
  int total;  // kept samples (set by the launcher)
  // outputs (device, accumulated)
  float* g_grid;
  float* g_density;
  float* g_color;
  double* alpha_grad;
  double* loss;  // [total, image, depth, dvar, dist]
  int32_t* ray_evals;
  int32_t* ray_contrib;
};

}  // namespace lumi_dev

cudaError_t launch_render_simt(const lumi_dev::RenderParams& p, cudaStream_t s);
cudaError_t launch_march_kept(const lumi_dev::RenderParams& p, uint32_t* mask, int32_t* counts,
                              cudaStream_t s);
cudaError_t launch_march_mask(const lumi_dev::RenderParams& p, cudaStream_t s);
uint32_t march_occ_bias(int res);  // RenderParams::occ_bias
// public [pixel][word] kept mask through the production (filtered) march pass
cudaError_t launch_march_public(lumi_dev::RenderParams p, uint32_t* mask, int32_t* counts,
                                cudaStream_t s);
cudaError_t launch_encode(const lumi_dev::GridDev& g, int n, const float* pos, const float* fl,
                          float* out, cudaStream_t s);
cudaError_t launch_gather_bench(const lumi_dev::GridDev& g, int n, int coherent, float* out,
                                cudaStream_t s);
cudaError_t launch_mlp_batch(const lumi_dev::MlpDev& mlp, const void* feat, const float* dirs, int n,
                             float* out, int num_sms, cudaStream_t s);
// the packed fp16 weight-tile image k_render_ws stages by TMA (bytes; build with the launcher)
size_t render_ws_weight_tile_bytes();
cudaError_t launch_pack_weight_tiles(const lumi_dev::MlpDev& mlp, void* img, cudaStream_t s);
// ev (optional): 3 events recorded before the march pass, between march and render, after render
cudaError_t launch_render_ws(lumi_dev::RenderParams p, cudaStream_t s, int num_sms,
                             cudaEvent_t* ev = nullptr);
cudaError_t launch_to_half(const float* src, void* dst_half, uint64_t n, cudaStream_t s);
cudaError_t launch_bake(const lumi_dev::BakeParams& p, cudaStream_t s);
cudaError_t launch_train_backward(lumi_dev::TrainParams p, cudaStream_t s, int num_sms,
                                  long long* kept_total, long long* eval_total);
size_t train_backward_smem_bytes();
