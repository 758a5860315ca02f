// bake.cu -- GPU occupancy bake: OccupancyGrid::probe (occupancy.cpp:97-142) with the
// density head (trainer.cpp:651-657: forward_chunk(with_color=false), all-ones LOD) and
// prune(alpha) (occupancy.cpp:144-154; no history, no carving).  One thread per voxel.
#include <cuda_runtime.h>

#include "kernels.h"
#include "mlp_simt.cuh"

namespace lumi_dev {


// uncontract (camera.cpp:51-66)
__device__ __forceinline__ d3 uncontract(d3 c) {
  const double m = dlinf(c);
  if (m <= 1.0) return c;
  const double mag = 1.0 / dsub(2.0, m);
  d3 out{dmul(c.x, mag), dmul(c.y, mag), dmul(c.z, mag)};
  if (fabs(c.x) == m)
    out.x = copysign(mag, c.x);
  else if (fabs(c.y) == m)
    out.y = copysign(mag, c.y);
  else
    out.z = copysign(mag, c.z);
  return out;
}

__global__ void __launch_bounds__(128) k_bake(BakeParams p) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long total = (long long)p.res * p.res * p.res;
  if (i >= total) return;
  const int res = p.res, k = p.k;
  const int ix = (int)(i % res), iy = (int)((i / res) % res), iz = (int)(i / ((long long)res * res));
  const double e = 4.0 / res;  // voxel_extent (occupancy.h:48)
  const d3 c{dadd(-2.0, dmul(ix + 0.5, e)), dadd(-2.0, dmul(iy + 0.5, e)),
             dadd(-2.0, dmul(iz + 0.5, e))};  // voxel_center (occupancy.cpp:31-37)
  const d3 world = dlinf(c) < 2.0 ? uncontract(c) : c;
  double dt = 1e30;
  for (int ci = 0; ci < p.ncams; ++ci) {
    const d3 dv{dsub(world.x, p.cam_origin[3 * ci]), dsub(world.y, p.cam_origin[3 * ci + 1]),
                dsub(world.z, p.cam_origin[3 * ci + 2])};
    const double dist = dmax(dnorm(dv), p.cam_tnear[ci]);
    dt = dmin(dt, dmul(dist, dsub(p.cam_ratio[ci], 1.0)));
  }
  if (!(dt < 1e29)) dt = e;
  const LodW ones{p.grid.levels, 0.f, false};
  float best = 0.f;
  for (int pz = 0; pz < k; ++pz)
    for (int py = 0; py < k; ++py)
      for (int px = 0; px < k; ++px) {
        const d3 pt{dadd(c.x, dmul(e, dsub((px + 1.0) / (k + 1), 0.5))),
                    dadd(c.y, dmul(e, dsub((py + 1.0) / (k + 1), 0.5))),
                    dadd(c.z, dmul(e, dsub((pz + 1.0) / (k + 1), 0.5)))};
        float feat[kFeat];
        encode(p.grid, pt, ones, feat);
        const float sigma = density_mlp(p.mlp, feat);
        const float conv = __double2float_rn(dsub(1.0, exp(dmul(-(double)sigma, dt))) / dt);
        best = best < conv ? conv : best;
      }
  p.probe_max[i] = best;
  p.occ[i] = (best < p.alpha) ? 0 : 1;  // prune with zero history (occupancy.cpp:150-152)
}

}  // namespace lumi_dev

cudaError_t launch_bake(const lumi_dev::BakeParams& p, cudaStream_t s) {
  const long long total = (long long)p.res * p.res * p.res;
  lumi_dev::k_bake<<<(unsigned)((total + 127) / 128), 128, 0, s>>>(p);
  return cudaGetLastError();
}

namespace lumi_dev {
// fp32 table -> fp16 pairs (round to nearest even), grid-stride.
__global__ void k_to_half(const float* __restrict__ src, __half* __restrict__ dst, uint64_t n) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    dst[i] = __float2half_rn(src[i]);
}
}  // namespace lumi_dev

cudaError_t launch_to_half(const float* src, void* dst, uint64_t n, cudaStream_t s) {
  lumi_dev::k_to_half<<<148 * 8, 256, 0, s>>>(src, static_cast<__half*>(dst), n);
  return cudaGetLastError();
}
