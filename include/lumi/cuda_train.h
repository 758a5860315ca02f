// lumi/cuda_train.h -- drop-in B200 backend for the training loop's per-ray body.
//
// The reference trains ray by ray (proj/src/trainer.cpp:549-562):
//
//   for (const auto& ray : batch) {
//     march_ray(field, occupancy, ray.ray, ray.neighbor, cam.t_near, cam.t_far, march_opts,
//               true, rec);
//     LossTerms lt = ray_loss(rec, ray, alpha_v[ray.camera], contraction, cfg, depth_active,
//                             inv_batch, &rg);
//     losses.image += lt.image; ... losses.dist += lt.dist;
//     backward_ray(field, rec, rg, march_opts.background, grads, scratch, dcol_scratch);
//     alpha_grad[ray.camera] += rg.d_alpha_v;
//   }
//
// lumi::cuda::train_rays_backward() runs that whole loop on the GPU through the C ABI
// (lumi_train_backward, include/lumi_cuda.h) and accumulates into the same FieldGradients
// and alpha_grad, returning the summed loss terms.  The occupancy-history recording of the
// pruning schedule (trainer.cpp:563-570) stays on the host and is not covered.
#pragma once

#include <cstring>
#include <vector>

#include "lumi/cuda_renderer.h"
#include "lumi/trainer.h"

namespace lumi {
namespace cuda {

inline LossTerms train_rays_backward(const RadianceField<float>& field, const OccupancyGrid& grid,
                                     const std::vector<CameraModel>& cameras,
                                     const std::vector<TrainRay>& batch,
                                     const std::vector<double>& alpha_v,
                                     const RenderOptions& march_opts, const TrainConfig& cfg,
                                     bool depth_active, double inv_batch,
                                     FieldGradients<float>& grads, std::vector<double>& alpha_grad) {
  require(alpha_v.size() == cameras.size() && alpha_grad.size() == cameras.size(),
          "train_rays_backward: one alpha_v / alpha_grad entry per camera");
  auto dev = device_field(field, grid, thread_device());
  std::vector<LumiTrainRay> rays(batch.size());
  for (size_t i = 0; i < batch.size(); ++i) {
    const TrainRay& r = batch[i];
    LumiTrainRay& d = rays[i];
    std::memset(&d, 0, sizeof(d));
    const Vec3* v[4] = {&r.ray.origin, &r.ray.dir, &r.neighbor.origin, &r.neighbor.dir};
    double* o[4] = {d.origin, d.dir, d.norigin, d.ndir};
    for (int k = 0; k < 4; ++k) {
      o[k][0] = v[k]->x;
      o[k][1] = v[k]->y;
      o[k][2] = v[k]->z;
    }
    for (int c = 0; c < 3; ++c) d.gt[c] = r.gt[c];
    d.camera = r.camera;
    d.gt_depth = r.gt_depth;
    d.vignette_r = r.vignette_r;
  }
  std::vector<double> tnf(2 * cameras.size());
  for (size_t c = 0; c < cameras.size(); ++c) {
    tnf[2 * c] = cameras[c].t_near;
    tnf[2 * c + 1] = cameras[c].t_far;
  }
  LumiLossConfig lc{};
  lc.lambda_depth = cfg.lambda_depth;
  lc.lambda_dvar = cfg.lambda_dvar;
  lc.lambda_dist = cfg.lambda_dist;
  lc.inv_batch = inv_batch;
  lc.depth_active = depth_active ? 1 : 0;
  LumiLossTerms lt{};
  LumiTrainGrads g{grads.grid.data(), grads.density.data(), grads.color.data(), alpha_grad.data(),
                   &lt};
  const LumiRenderOptions o = to_desc(march_opts);
  check(lumi_train_backward(dev->model(), rays.data(), static_cast<int>(rays.size()), tnf.data(),
                            alpha_v.data(), static_cast<int>(cameras.size()), &o, &lc, &g,
                            nullptr, nullptr),
        "lumi_train_backward");
  LossTerms out;
  out.image = lt.image;
  out.depth = lt.depth;
  out.dvar = lt.dvar;
  out.dist = lt.dist;
  out.total = lt.total;
  return out;
}

}  // namespace cuda
}  // namespace lumi
