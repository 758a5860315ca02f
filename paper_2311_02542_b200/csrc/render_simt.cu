// render_simt.cu -- reference-structured kernels: thread-per-ray fused march with the MLP
// on CUDA cores (fp32 FFMA), and the occupancy-kept bitmask kernel.
//
// The SIMT renderer is the numerical baseline the tensor-core path (render_ws.cu) is
// checked against on the GPU; the march-kept kernel produces the bit-exact, MLP-independent
// sample index set of renderer.h:205-208.
#include <cuda_runtime.h>

#include "kernels.h"
#include "mlp_simt.cuh"
#include "render_common.cuh"

namespace lumi_dev {

__device__ __forceinline__ bool occupied(const RenderParams& p, d3 c) {
  const int64_t vi = voxel_index(c, p.occ_res);
  return vi >= 0 && __ldg(p.occ + vi) != 0;
}

// march_ray + render_rows (renderer.h:126-237, 252-278), one thread per ray.
__global__ void __launch_bounds__(128) k_render_simt(RenderParams p) {
  __shared__ double s_ts[kMaxSamples];
  for (int i = threadIdx.x; i < p.n; i += blockDim.x) s_ts[i] = p.ts[i];
  __syncthreads();
  const int W = p.cam.width;
  const long long lin = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (lin >= (long long)(p.row_end - p.row_begin) * W) return;
  const int y = p.row_begin + (int)(lin / W), x = (int)(lin % W);

  const d3 o{p.cam.origin[0], p.cam.origin[1], p.cam.origin[2]};
  const d3 d = ray_dir(p.cam, (double)x + 0.5, (double)y + 0.5);
  const d3 nd = ray_dir(p.cam, (double)x + 1.5, (double)y + 0.5);
  float sh[16];
  sh_encode(d, sh);

  RayResult r{0, 0, 0, 0, 0, 0, 0};
  double trans = 1.0;
  int kept = 0, cut_limit = 0x7fffffff, level_samples = 0, marched = 0;
  bool term = false;
  const int n = p.n;
  for (int i = 0; i < n; ++i) {
    ++marched;
    const double t = s_ts[i];
    const d3 c = contract(ray_at(o, d, t), p.contraction);
    if (!occupied(p, c)) continue;
    ++kept;
    if (term) {
      if (kept >= cut_limit) break;
      continue;
    }
    const double delta = (i + 1 < n) ? dsub(s_ts[i + 1], t) : dmul(t, dsub(p.ratio, 1.0));
    LodW lw{p.grid.levels, 0.f, false};
    if (p.lod_enabled) {
      const double rc = contracted_footprint(o, d, nd, t, p.contraction);
      lw = lod_weights(lod_level(dmax(rc, 1e-12), p.grid.two_base, p.grid.log_scale, p.grid.levels),
                       p.lod_bias, p.grid.levels);
    }
    level_samples += active_levels(lw, p.grid.levels);
    float feat[kFeat];
    encode(p.grid, c, lw, feat);
    float sigma, rgb[3];
    field_mlp(p.mlp, feat, sh, sigma, rgb);
    // flush compositing (renderer.h:170-190), double
    const double a = dsub(1.0, exp(dmul(-(double)sigma, delta)));
    const double w = dmul(trans, a);
    r.px = dadd(r.px, dmul(w, (double)rgb[0]));
    r.py = dadd(r.py, dmul(w, (double)rgb[1]));
    r.pz = dadd(r.pz, dmul(w, (double)rgb[2]));
    r.depth = dadd(r.depth, dmul(w, t));
    r.opacity = dadd(r.opacity, w);
    trans = dmul(trans, dsub(1.0, a));
    ++r.contributing;
    if (p.t_cut > 0 && trans < p.t_cut) {
      term = true;
      cut_limit = ((r.contributing + p.chunk - 1) / p.chunk) * p.chunk;
      if (kept >= cut_limit) break;
    }
  }
  r.evals = chunk_evals(term, r.contributing, kept, p.chunk);
  store_ray(p, x, y, r, trans);
  add_work_stats(p, r.contributing, level_samples, marched, 1);
}

// Occupancy-kept candidate indices (renderer.h:205-208) as a bitmask, no network.
__global__ void __launch_bounds__(128) k_march_kept(RenderParams p, uint32_t* mask, int32_t* counts) {
  __shared__ double s_ts[kMaxSamples];
  for (int i = threadIdx.x; i < p.n; i += blockDim.x) s_ts[i] = p.ts[i];
  __syncthreads();
  const int W = p.cam.width;
  const long long lin = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (lin >= (long long)(p.row_end - p.row_begin) * W) return;
  const int y = p.row_begin + (int)(lin / W), x = (int)(lin % W);
  const d3 o{p.cam.origin[0], p.cam.origin[1], p.cam.origin[2]};
  const d3 d = ray_dir(p.cam, (double)x + 0.5, (double)y + 0.5);
  const int words = (p.n + 31) / 32;
  const size_t pix = (size_t)y * W + x;
  int count = 0;
  for (int w0 = 0; w0 < words; ++w0) {
    uint32_t bits = 0;
    for (int b = 0; b < 32; ++b) {
      const int i = w0 * 32 + b;
      if (i >= p.n) break;
      if (occupied(p, contract(ray_at(o, d, s_ts[i]), p.contraction))) bits |= 1u << b;
    }
    count += __popc(bits);
    if (mask) mask[pix * words + w0] = bits;
  }
  if (counts) counts[pix] = count;
}

}  // namespace lumi_dev

using namespace lumi_dev;

cudaError_t launch_render_simt(const RenderParams& p, cudaStream_t s) {
  const long long rays = (long long)(p.row_end - p.row_begin) * p.cam.width;
  if (rays <= 0) return cudaSuccess;
  const unsigned blocks = (unsigned)((rays + 127) / 128);
  k_render_simt<<<blocks, 128, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_march_kept(const RenderParams& p, uint32_t* mask, int32_t* counts,
                              cudaStream_t s) {
  const long long rays = (long long)(p.row_end - p.row_begin) * p.cam.width;
  if (rays <= 0) return cudaSuccess;
  const unsigned blocks = (unsigned)((rays + 127) / 128);
  k_march_kept<<<blocks, 128, 0, s>>>(p, mask, counts);
  return cudaGetLastError();
}
