// kernels.h -- host-visible launchers of the sm_100a kernels and their parameter blocks.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "render_common.cuh"

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

}  // namespace lumi_dev

cudaError_t launch_render_simt(const lumi_dev::RenderParams& p, cudaStream_t s);
cudaError_t launch_march_kept(const lumi_dev::RenderParams& p, uint32_t* mask, int32_t* counts,
                              cudaStream_t s);
// ev (optional): 3 events recorded before the march pass, between march and render, after render
cudaError_t launch_render_tc(lumi_dev::RenderParams p, cudaStream_t s, int num_sms,
                             cudaEvent_t* ev = nullptr);
size_t render_tc_smem_bytes();
cudaError_t launch_march_mask(const lumi_dev::RenderParams& p, cudaStream_t s);
// public [pixel][word] kept mask through the production (filtered) march pass
cudaError_t launch_march_public(lumi_dev::RenderParams p, uint32_t* mask, int32_t* counts,
                                cudaStream_t s);
cudaError_t launch_render_pk(lumi_dev::RenderParams p, cudaStream_t s, int num_sms,
                             cudaEvent_t* ev = nullptr);
cudaError_t launch_to_half(const float* src, void* dst_half, uint64_t n, cudaStream_t s);
cudaError_t launch_bake(const lumi_dev::BakeParams& p, cudaStream_t s);
