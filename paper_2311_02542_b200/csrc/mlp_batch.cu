// mlp_batch.cu -- the renderer's two stages in isolation: the tcgen05 MLP on a
// dense batch ("report tensor-pipe utilisation from ncu on an isolated dense batch, not only
// the fused kernel") and, at the end of the file, the hash-grid gather (the attainable gather
// rate, the denominator for the L2-resident tables of C1/C2).
//
// RadianceField::forward_chunk (field.h:106-137) minus the encoding: n samples of 32 fp16
// hash-grid features ([n][32], row-major) and a per-sample view direction go through exactly
// the production kernel's four layers (pk_parts.cuh: density L1 SS-form from shared memory,
// density L2 folded into colour L1 as one N=80 layer, colour L2, colour L3, activations in
// TMEM, biases as an extra K step) and out come sigma and the three colour channels.
// Persistent, 4 CTAs of 128 threads per SM (TMEM: 128 columns each); each 128-row tile is
// loaded with 16-byte vector loads into the chunk-major A tile.  Numerics are the renderer's,
// so it doubles as a parity check of the MLP stage alone (tests/test_gpu_parity.py).
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdlib>

#include "kernels.h"
#include "pk_parts.cuh"

namespace lumi_dev {
namespace mb {

using namespace pk;

struct __align__(16) Smem {
  uint8_t A[128 * (32 + kKb) * 2];
  uint8_t W1[64 * (32 + kKb) * 2];
  uint8_t F[80 * (80 + kKb) * 2];
  uint8_t C2[64 * (64 + kKb) * 2];
  uint8_t C3[16 * (64 + kKb) * 2];
  uint64_t mbar;
  uint32_t tmem_base;
};

__global__ void __launch_bounds__(128, 4) k_mlp_batch(MlpDev mlp, const __half* __restrict__ feat,
                                                      const float* __restrict__ dirs, int n,
                                                      float4* __restrict__ out) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  Smem& s = *reinterpret_cast<Smem*>(smem_raw);
  const int tid = threadIdx.x, warp = tid >> 5;
  const float* dp = mlp.dparams;
  const float* cp = mlp.cparams;
  const float* c2 = cp + 64 * 32 + 64;
  const float* c3 = c2 + 64 * 64 + 64;
  load_weight_tile(s.W1, dp, 64, 64, 32);
  load_weight_tile(s.F, mlp.fused, kHidden + 1, 80, 80);
  load_weight_tile(s.C2, c2, 64, 64, 64);
  load_weight_tile(s.C3, c3, 3, 16, 64);
  st16(s.A, a_off(tid, 4), make_uint4(0x3C00u, 0u, 0u, 0u));
  st16(s.A, a_off(tid, 5), make_uint4(0u, 0u, 0u, 0u));
  if (tid == 0) {
    ptx::mbar_init(&s.mbar, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 0) ptx::tmem_alloc<kTmemCols>(&s.tmem_base);
  ptx::fence_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = s.tmem_base;
  const uint32_t t_lane = tmem + ((uint32_t)(warp * 32) << 16);
  {
    const uint32_t ones[8] = {0x3C00u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
    ptx::tmem_st8(t_lane + kOnesCol, ones);
    ptx::tmem_st_wait();
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
  }
  const uint32_t a_tmem = tmem + kAcol, ones_tmem = tmem + kOnesCol, a_lane = t_lane + kAcol;
  uint32_t phase = 0;
  const int tiles = (n + 127) / 128;
  // a tile's 32 fp16 features per row (four 16-byte vectors) and its view direction, loaded one
  // tile ahead: the next tile's loads are in flight while this one runs through the layers
  uint4 nf[4];
  float ndx = 0.f, ndy = 0.f, ndz = 1.f;
  auto load_tile = [&](int tile) {
    const int row = tile * 128 + tid;
    const bool have = tile < tiles && row < n;
    const uint4* src = reinterpret_cast<const uint4*>(feat + (size_t)row * 32);
#pragma unroll
    for (int q = 0; q < 4; ++q) nf[q] = have ? __ldg(src + q) : make_uint4(0, 0, 0, 0);
    ndx = 0.f, ndy = 0.f, ndz = 1.f;
    if (have) {
      ndx = __ldg(dirs + 3 * (size_t)row);
      ndy = __ldg(dirs + 3 * (size_t)row + 1);
      ndz = __ldg(dirs + 3 * (size_t)row + 2);
    }
  };
  load_tile(blockIdx.x);
  for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const int row = tile * 128 + tid;
    const bool have = row < n;
#pragma unroll
    for (int q = 0; q < 4; ++q) st16(s.A, a_off(tid, q), nf[q]);
    const float dx = ndx, dy = ndy, dz = ndz;
    load_tile(tile + gridDim.x);
    ptx::fence_async_smem();
    ptx::tc_fence_before();
    __syncthreads();
    float v32[32];
    if (tid == 0) {
      ptx::tc_fence_after();
      issue_layer<64, 32>(s.A, s.W1, tmem);
      ptx::mma_commit(&s.mbar);
    }
    ptx::mbar_wait(&s.mbar, phase);
    phase ^= 1;
    ptx::tc_fence_after();
    relu64_to_tmem(t_lane, a_lane);
    {
      float sh[16];
      sh_encode(d3{(double)dx, (double)dy, (double)dz}, sh);
      uint32_t wv[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) wv[j] = pack2(sh[2 * j], sh[2 * j + 1]);
      ptx::tmem_st8(t_lane + kShCol, wv);
      ptx::tmem_st_wait();
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (tid == 0) {
      ptx::tc_fence_after();
      issue_layer_ts<80, 80>(a_tmem, ones_tmem, s.F, tmem);
      ptx::mma_commit(&s.mbar);
    }
    ptx::mbar_wait(&s.mbar, phase);
    phase ^= 1;
    ptx::tc_fence_after();
    ptx::tmem_ld16(t_lane + 64, v32);
    ptx::tmem_ld_wait();
    const float sigma = trunc_exp_fast(v32[0]);
    relu64_to_tmem(t_lane, a_lane);
    ptx::tc_fence_before();
    __syncthreads();
    if (tid == 0) {
      ptx::tc_fence_after();
      issue_layer_ts<64, 64>(a_tmem, ones_tmem, s.C2, tmem);
      ptx::mma_commit(&s.mbar);
    }
    ptx::mbar_wait(&s.mbar, phase);
    phase ^= 1;
    ptx::tc_fence_after();
    relu64_to_tmem(t_lane, a_lane);
    ptx::tc_fence_before();
    __syncthreads();
    if (tid == 0) {
      ptx::tc_fence_after();
      issue_layer_ts<16, 64>(a_tmem, ones_tmem, s.C3, tmem);
      ptx::mma_commit(&s.mbar);
    }
    ptx::mbar_wait(&s.mbar, phase);
    phase ^= 1;
    ptx::tc_fence_after();
    ptx::tmem_ld16(t_lane, v32);
    ptx::tmem_ld_wait();
    ptx::tc_fence_before();
    if (have) {
      float rgb[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) rgb[k] = mlp.color_space == 0 ? sigmoid_fast(v32[k]) : trunc_exp_fast(v32[k]);
      out[row] = make_float4(sigma, rgb[0], rgb[1], rgb[2]);
    }
    __syncthreads();  // the A tile and TMEM are rewritten by the next tile
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (warp == 0) ptx::tmem_dealloc<kTmemCols>(tmem);
}

}  // namespace mb
}  // namespace lumi_dev

using namespace lumi_dev;

cudaError_t launch_mlp_batch(const MlpDev& mlp, const void* feat, const float* dirs, int n, float* out,
                             int num_sms, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const size_t smem = sizeof(mb::Smem);
  static PerDeviceInit once;
  int ok = 0;
  cudaError_t e = once.get([&](int* v) {
    *v = 1;
    return cudaFuncSetAttribute(mb::k_mlp_batch, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  }, &ok);
  if (e != cudaSuccess) return e;
  const int tiles = (n + 127) / 128;
  mb::k_mlp_batch<<<std::min(tiles, 4 * num_sms), 128, smem, s>>>(
      mlp, static_cast<const __half*>(feat), dirs, n, reinterpret_cast<float4*>(out));
  return cudaGetLastError();
}

// ---- the hash-grid gather in isolation: the attainable gather rate ----------------------
// report the gather against a measured gather peak (the table of C1/C2 is
// L2-resident, so HBM is the wrong denominator there).  Every thread evaluates all levels of
// one point with the renderer's own gather_row (fp16 table, 8 corners, packed-fp16 lerps);
// points are either uniform random (no reuse between neighbouring threads) or coherent (the
// 32 lanes of a warp sample a small neighbourhood, like a packet of neighbouring rays).
namespace lumi_dev {
namespace mb {

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352du;
  x ^= x >> 15;
  x *= 0x846ca68bu;
  x ^= x >> 16;
  return x;
}
__device__ __forceinline__ float u01(uint32_t h) { return (h >> 8) * (1.f / 16777216.f); }

__global__ void __launch_bounds__(256) k_gather_bench(GridDev g, int n, int coherent, float* out) {
  __shared__ pk::LevelTab lt;
  pk::level_tab_init(lt, g, threadIdx.x, blockDim.x);
  __syncthreads();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float u, v, w;
  if (coherent) {  // warp = an 8x4 patch of rays at one distance: ~1e-3 apart in the unit cube
    const uint32_t wid = (uint32_t)i >> 5, lane = (uint32_t)i & 31u;
    u = 0.25f + 0.5f * u01(hash32(3u * wid + 1u)) + 1e-3f * (float)(lane & 7u);
    v = 0.25f + 0.5f * u01(hash32(3u * wid + 2u)) + 1e-3f * (float)(lane >> 3);
    w = 0.25f + 0.5f * u01(hash32(3u * wid + 3u));
  } else {
    u = u01(hash32(3u * i + 1u));
    v = u01(hash32(3u * i + 2u));
    w = u01(hash32(3u * i + 3u));
  }
  // the renderer's producer gather (pk::gather_row), every level at weight 1
  float acc = 0.f;
  pk::gather_row(lt, g.levels, u, v, w, (float)g.levels, [&](int, uint4 q) {
    const uint32_t qs[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&qs[k]));
      acc += f.x + f.y;
    }
  });
  out[i] = acc;
}

// The production encoding of n given samples (parity of the renderer's gather, grid.h:90-114):
// contracted positions [n][3] -> u = saturate((c + 2) / 4) as the render kernel computes it,
// LOD weights carried as fl (w_l = saturate(fl - l), the kernel's representation), every
// active level through pk::gather_row -> features [n][2 * levels] fp32 (zeros for w_l = 0).
__global__ void __launch_bounds__(256) k_encode(GridDev g, int n, const float* __restrict__ pos,
                                                const float* __restrict__ fl,
                                                float* __restrict__ out) {
  __shared__ pk::LevelTab lt;
  pk::level_tab_init(lt, g, threadIdx.x, blockDim.x);
  __syncthreads();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float u = pk::unit_below1((pos[3 * i] + 2.f) * 0.25f), v = pk::unit_below1((pos[3 * i + 1] + 2.f) * 0.25f),
              w = pk::unit_below1((pos[3 * i + 2] + 2.f) * 0.25f);
  const float f = fl[i];
  // the renderer's producer code (pk::gather_row): the levels past this sample's last active
  // one are not loaded (weight 0 either way) and come out zero
  int na = 0;
  for (int l = 0; l < g.levels; ++l)
    if (__saturatef(f - (float)l) > 0.f) na = l + 1;
  float* o = out + (size_t)i * 2 * g.levels;
  for (int l = 0; l < 2 * g.levels; ++l) o[l] = 0.f;
  pk::gather_row(lt, na, u, v, w, f, [&](int c, uint4 q4) {
    const uint32_t qs[4] = {q4.x, q4.y, q4.z, q4.w};
    for (int q = 0; q < 4; ++q) {
      const int l = 4 * c + q;
      if (l >= g.levels) break;
      const float2 r = __half22float2(*reinterpret_cast<const __half2*>(&qs[q]));
      o[2 * l] = r.x;
      o[2 * l + 1] = r.y;
    }
  });
}

}  // namespace mb
}  // namespace lumi_dev

cudaError_t launch_encode(const lumi_dev::GridDev& g, int n, const float* pos, const float* fl,
                          float* out, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  lumi_dev::mb::k_encode<<<(n + 255) / 256, 256, 0, s>>>(g, n, pos, fl, out);
  return cudaGetLastError();
}

cudaError_t launch_gather_bench(const lumi_dev::GridDev& g, int n, int coherent, float* out,
                                cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  // LUMI_GATHER_CARVEOUT=<0..100>: shared-memory carveout, i.e. how much of the 256 KB of L1 +
  // shared memory is left to the L1 data cache (the renderers run with ~20 KB of L1)
  if (const char* c = std::getenv("LUMI_GATHER_CARVEOUT"))
    cudaFuncSetAttribute(lumi_dev::mb::k_gather_bench, cudaFuncAttributePreferredSharedMemoryCarveout,
                         std::atoi(c));
  lumi_dev::mb::k_gather_bench<<<(n + 255) / 256, 256, 0, s>>>(g, n, coherent, out);
  return cudaGetLastError();
}
