// march.cu -- the march pass: every candidate sample of every ray through the occupancy test
// (renderer.h:205-208), one thread per ray, writing the kept-candidate bitmask [word][ray] and
// the kept count the frame kernel (render_ws.cu) streams.  Ray ids are packet-major (a warp of
// ids = one 8x4 pixel packet), so the frame kernel's warps read their packet's mask words with
// coalesced loads.
//
// Reference semantics: march_ray's exponential sample distances (renderer.h:135-142, computed on
// the host), contract (camera.cpp:34-49), OccupancyGrid::voxel_index / is_occupied
// (occupancy.cpp:22-29, occupancy.h:50-53).  The kept set is bit-exact: the production pass
// decides in fp32 with a certified error bound and re-tests undecided candidates in the exact
// double geometry (render_common.cuh).
#include <cuda_runtime.h>

#include <cstdlib>

#include "kernels.h"
#include "render_common.cuh"

namespace lumi_dev {
namespace march {
__device__ __forceinline__ bool occupied(const RenderParams& p, d3 c) {
  const int64_t vi = voxel_index(c, p.occ_res);
  return vi >= 0 && __ldg(p.occ + vi) != 0;
}

// ray id (tile-major: 16x8 tiles, row-major inside a tile) -> pixel; false for the padding
// ids of partial edge tiles
__device__ __forceinline__ bool ray_pixel(const RenderParams& p, long long idx, int& x, int& y) {
  const int tw = p.tile_w, th = p.tile_h;
  const long long tile = idx / (tw * th);
  const int w = (int)(idx % (tw * th));
  x = (int)(tile % p.tiles_x) * tw + (w % tw);
  y = p.row_begin + (int)(tile / p.tiles_x) * th + w / tw;
  return x < p.cam.width && y < p.row_end;
}

// March pass: every candidate of every ray through the exact occupancy test
// (renderer.h:205-208), one thread per ray in tile-major id order; writes the kept bitmask
// [word][ray] and the kept count.  Uniform 256-iteration loops, no divergence on ray length.
// RenderParams::ray_dirs for the packet renderer: the ray's fp32 direction and its right
// neighbour's (renderer.h:264-265), from the same double ray generation
__device__ __forceinline__ void store_ray_dirs(const RenderParams& p, long long idx, bool valid, int x, int y,
                                               const d3& d) {
  const d3 nn = valid ? ray_dir(p.cam, (double)x + 1.5, (double)y + 0.5) : d3{0, 0, 1};
  const size_t T = (size_t)p.total_rays;
  p.ray_dirs[idx] = (float)d.x;
  p.ray_dirs[T + idx] = (float)d.y;
  p.ray_dirs[2 * T + idx] = (float)d.z;
  p.ray_dirs[3 * T + idx] = (float)nn.x;
  p.ray_dirs[4 * T + idx] = (float)nn.y;
  p.ray_dirs[5 * T + idx] = (float)nn.z;
}

__global__ void __launch_bounds__(128) k_march_mask(RenderParams p) {
  __shared__ double s_ts[kMaxSamples];
  for (int i = threadIdx.x; i < p.n; i += blockDim.x) s_ts[i] = p.ts[i];
  __syncthreads();
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= p.total_rays) return;
  int x, y;
  const bool valid = ray_pixel(p, idx, x, y);
  const d3 o{p.cam.origin[0], p.cam.origin[1], p.cam.origin[2]};
  const d3 d = valid ? ray_dir(p.cam, (double)x + 0.5, (double)y + 0.5) : d3{0, 0, 1};
  if (p.ray_dirs && idx < p.total_rays) store_ray_dirs(p, idx, valid, x, y, d);
  int count = 0;
  for (int w0 = 0; w0 < p.mask_words; ++w0) {
    uint32_t bits = 0;
    if (valid) {
      const int hi = min(32, p.n - w0 * 32);
      for (int b = 0; b < hi; ++b)
        if (occupied(p, contract(ray_at(o, d, s_ts[w0 * 32 + b]), p.contraction))) bits |= 1u << b;
    }
    count += __popc(bits);
    p.kept_mask[(size_t)w0 * p.total_rays + idx] = p.mask_transposed ? warp_transpose32(bits) : bits;
  }
  p.kept_count[idx] = (uint16_t)count;
  add_work_stats(p, 0, 0, valid ? (unsigned long long)p.n : 0ull, 0);
}

// Filtered march pass: the same kept bitmask, decided in fp32 with a certified error bound
// (occupied_filtered, render_common.cuh) and the exact double test only where fp32 cannot decide.
#ifndef LUMI_MARCH_UNROLL
#define LUMI_MARCH_UNROLL 8
#endif
constexpr int kMarchUnroll = LUMI_MARCH_UNROLL;
#ifndef LUMI_MARCH_EXIT
#define LUMI_MARCH_EXIT 1
#endif
__global__ void __launch_bounds__(128) k_march_mask_fast(RenderParams p) {
  __shared__ double s_ts[kMaxSamples];
  __shared__ float s_tf[kMaxSamples];
  __shared__ double s_dir[4][32][3];        // per lane: exact direction (undecided re-tests)
  __shared__ uint16_t s_queue[4][32 * 32];  // per warp: undecided (lane, bit) of one word
  __shared__ uint32_t s_add[4][32];         // per lane: bits confirmed by the re-test
  for (int i = threadIdx.x; i < p.n; i += blockDim.x) {
    s_ts[i] = p.ts[i];
    s_tf[i] = (float)p.ts[i];
  }
  __syncthreads();
  const unsigned FULL = 0xffffffffu;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  int x = 0, y = 0;
  const bool valid = idx < p.total_rays && ray_pixel(p, idx, x, y);
  const d3 o{p.cam.origin[0], p.cam.origin[1], p.cam.origin[2]};
  const d3 d = valid ? ray_dir(p.cam, (double)x + 0.5, (double)y + 0.5) : d3{0, 0, 1};
  if (p.ray_dirs && idx < p.total_rays) store_ray_dirs(p, idx, valid, x, y, d);
  s_dir[warp][lane][0] = d.x;
  s_dir[warp][lane][1] = d.y;
  s_dir[warp][lane][2] = d.z;
  const float3 of = make_float3((float)o.x, (float)o.y, (float)o.z);
  const float3 df = make_float3((float)d.x, (float)d.y, (float)d.z);
  const float onorm = fabsf(of.x) + fabsf(of.y) + fabsf(of.z);
  const InsideMarch im = inside_march_setup(p, of, df);
#if LUMI_MARCH_EXIT
  // beyond the ray's exit from the unit cube (slab test in fp32, 1e-3 slack) the inside fast
  // path can only answer "undecided": go straight to the general test there
  float t_exit = 3.4e38f;
  {
    const float dd[3] = {df.x, df.y, df.z}, oo[3] = {of.x, of.y, of.z};
#pragma unroll
    for (int a = 0; a < 3; ++a)
      if (dd[a] != 0.f) t_exit = fminf(t_exit, ((dd[a] > 0.f ? 1.f : -1.f) - oo[a]) / dd[a]);
    t_exit = t_exit * 1.001f + 1e-3f;
  }
#endif
  int count = 0;
  for (int w0 = 0; w0 < p.mask_words; ++w0) {
    uint32_t bits = 0, unsure = 0;
    if (valid) {
      const int hi = min(32, p.n - w0 * 32);
#pragma unroll kMarchUnroll
      for (int b = 0; b < hi; ++b) {
        const float tf = s_tf[w0 * 32 + b];
#if LUMI_MARCH_EXIT
        int r = tf < t_exit ? occupied_inside(p, im, tf) : -1;
#else
        int r = occupied_inside(p, im, tf);  // -1: not certified inside the unit cube
#endif
        if (r < 0) r = occupied_filtered(p, of, df, onorm, tf);
        bits |= (uint32_t)(r & 1) << b;
        unsure |= (uint32_t)(r >> 1) << b;
      }
    }
    // undecided candidates of the whole warp, re-tested exactly one per lane
    if (__any_sync(FULL, unsure != 0)) {
      const int mine = __popc(unsure);
      int incl = mine;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int v = __shfl_up_sync(FULL, incl, off);
        if (lane >= off) incl += v;
      }
      const int total = __shfl_sync(FULL, incl, 31);
      int at = incl - mine;
      for (uint32_t u = unsure; u; u &= u - 1) s_queue[warp][at++] = (uint16_t)(lane << 5 | (__ffs(u) - 1));
      s_add[warp][lane] = 0;
      __syncwarp();
      for (int j = lane; j < total; j += 32) {
        const int e = s_queue[warp][j], ol = e >> 5, b = e & 31;
        const d3 od{s_dir[warp][ol][0], s_dir[warp][ol][1], s_dir[warp][ol][2]};
        if (occupied(p, contract(ray_at(o, od, s_ts[w0 * 32 + b]), p.contraction)))
          atomicOr(&s_add[warp][ol], 1u << b);
      }
      __syncwarp();
      bits |= s_add[warp][lane];
      __syncwarp();
    }
    count += __popc(bits);
    const uint32_t out = p.mask_transposed ? warp_transpose32(bits) : bits;  // warp-uniform
    if (idx < p.total_rays) p.kept_mask[(size_t)w0 * p.total_rays + idx] = out;
  }
  if (idx < p.total_rays) p.kept_count[idx] = (uint16_t)count;
  add_work_stats(p, 0, 0, valid ? (unsigned long long)p.n : 0ull, 0);
}

// ---- voxel runs ------------------------------------------------------------------------------
// The production march pass.  Inside the unit cube the contraction is the identity and the
// voxel coordinate is linear in t, g(t) = G0 + G1 t (fp32 certified: |g_f - g| <= eps(t) =
// E0 + E1 t, render_common.cuh).  When candidate i is certified in voxel k, every later
// candidate whose fp32 t keeps g(t) +- eps(t) strictly inside voxel k (and inside the cube) on
// every axis would pass the same certified test with the same voxel -- its exact point is in
// voxel k -- so the whole run of candidates up to the voxel's exit gets voxel k's occupancy bit
// from ONE test.  Per axis with G1 > E1 the run ends where g + eps reaches the upper face:
//   t < (min(k + 1, 3q) - G0 - E0) / (G1 + E1)     (the lower face recedes: G1 - E1 > 0),
// mirrored for G1 < -E1; an axis with |G1| <= E1 gets no run.  The bound is shrunk by a relative
// 1e-5 (approximate division).  At the reference's 256 samples a C3 ray holds ~138 candidates
// inside the cube in ~35 voxel runs.  Outside the cube every candidate is tested on its own (the
// contraction's max-axis switch is discontinuous, so runs there would need per-pyramid exits).
// Undecided candidates are re-tested in exact double, cooperatively per warp.
__global__ void __launch_bounds__(128) k_march_runs(RenderParams p) {
  extern __shared__ uint32_t s_bits[];  // [mask_words][128]: this CTA's kept bits
  __shared__ double s_ts[kMaxSamples];
  __shared__ float s_tf[kMaxSamples];
  __shared__ double s_dir[4][32][3];  // per lane: exact direction (undecided re-tests)
  constexpr int kQueue = 256;
  __shared__ uint16_t s_queue[4][kQueue];  // per warp: undecided (lane, candidate)
  __shared__ int s_qn[4];
  for (int i = threadIdx.x; i < p.n; i += blockDim.x) {
    s_ts[i] = p.ts[i];
    s_tf[i] = (float)p.ts[i];
  }
  for (int i = threadIdx.x; i < p.mask_words * 128; i += blockDim.x) s_bits[i] = 0u;
  if (threadIdx.x < 4) s_qn[threadIdx.x] = 0;
  __syncthreads();
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const long long idx = (long long)blockIdx.x * blockDim.x + tid;
  int x = 0, y = 0;
  const bool valid = idx < p.total_rays && ray_pixel(p, idx, x, y);
  const d3 o{p.cam.origin[0], p.cam.origin[1], p.cam.origin[2]};
  const d3 d = valid ? ray_dir(p.cam, (double)x + 0.5, (double)y + 0.5) : d3{0, 0, 1};
  if (p.ray_dirs && idx < p.total_rays) store_ray_dirs(p, idx, valid, x, y, d);
  s_dir[warp][lane][0] = d.x;
  s_dir[warp][lane][1] = d.y;
  s_dir[warp][lane][2] = d.z;
  const float3 of = make_float3((float)o.x, (float)o.y, (float)o.z);
  const float3 df = make_float3((float)d.x, (float)d.y, (float)d.z);
  const float onorm = fabsf(of.x) + fabsf(of.y) + fabsf(of.z);
  const InsideMarch im = inside_march_setup(p, of, df);
  // beyond the ray's exit from the unit cube (slab test in fp32, with slack) the inside test can
  // only answer "undecided": go straight to the general test there
  float t_exit = 3.4e38f;
  {
    const float dd[3] = {df.x, df.y, df.z}, oo[3] = {of.x, of.y, of.z};
#pragma unroll
    for (int a = 0; a < 3; ++a)
      if (dd[a] != 0.f) t_exit = fminf(t_exit, ((dd[a] > 0.f ? 1.f : -1.f) - oo[a]) / dd[a]);
    t_exit = t_exit * 1.001f + 1e-3f;
  }
  // candidate index of a distance: k = (n - 1) log(t / t_near) / log(t_far / t_near)
  const float k_scale = (float)(p.n - 1) / __logf(s_tf[p.n - 1] / s_tf[0]);
  const float inv_tn = 1.f / s_tf[0];
  const uint32_t r = (uint32_t)p.occ_res;
  constexpr float kMagic = 12582912.f;  // 1.5 * 2^23: rint on the FMA pipe
  uint32_t tested = 0;
  int i = 0;
  while (valid && i < p.n) {
    const float tf = s_tf[i];
    int j = i;  // the last candidate decided together with i
    int vi = -2;
    if (tf < t_exit) {
      const float gx = fmaf(im.g1.x, tf, im.g0.x), gy = fmaf(im.g1.y, tf, im.g0.y),
                  gz = fmaf(im.g1.z, tf, im.g0.z);
      const float eps = fmaf(im.e1, tf, im.e0);
      const float rx = __fsub_rn(__fadd_rn(gx, kMagic), kMagic), ry = __fsub_rn(__fadd_rn(gy, kMagic), kMagic),
                  rz = __fsub_rn(__fadd_rn(gz, kMagic), kMagic);
      const float dmin = fminf(fabsf(gx - rx), fminf(fabsf(gy - ry), fabsf(gz - rz)));
      const float gmin = fminf(gx, fminf(gy, gz)), gmax = fmaxf(gx, fmaxf(gy, gz));
      if (dmin > eps && gmin - eps > im.qlo && gmax + eps < im.qhi) {
        // floor(g) as a float integer and as an index
        const float bx = __fadd_rn(gx - 0.5f, kMagic), by = __fadd_rn(gy - 0.5f, kMagic),
                    bz = __fadd_rn(gz - 0.5f, kMagic);
        const uint32_t ix = (uint32_t)(__float_as_int(bx) - 0x4B400000),
                       iy = (uint32_t)(__float_as_int(by) - 0x4B400000),
                       iz = (uint32_t)(__float_as_int(bz) - 0x4B400000);
        vi = (int)((iz * r + iy) * r + ix);
        const float kx = bx - kMagic, ky = by - kMagic, kz = bz - kMagic;
        auto axis_exit = [&](float k, float g0, float g1) {
          if (g1 > im.e1) return __fdividef(fminf(k + 1.f, im.qhi) - g0 - im.e0, g1 + im.e1);
          if (g1 < -im.e1) return __fdividef(g0 - im.e0 - fmaxf(k, im.qlo), im.e1 - g1);
          return 0.f;
        };
        const float t_lim = fminf(axis_exit(kx, im.g0.x, im.g1.x),
                                  fminf(axis_exit(ky, im.g0.y, im.g1.y), axis_exit(kz, im.g0.z, im.g1.z))) *
                            0.99999f;
        if (i + 1 < p.n && s_tf[i + 1] < t_lim) {
          int jj = min((int)(__logf(t_lim * inv_tn) * k_scale), p.n - 1);
          while (jj > i && !(s_tf[jj] < t_lim)) --jj;
          while (jj + 1 < p.n && s_tf[jj + 1] < t_lim) ++jj;
          j = max(jj, i);
        }
      }
    }
    if (vi == -2) vi = voxel_filtered(p, of, df, onorm, tf);
    ++tested;
    if (vi == -2) {  // undecided: the warp re-tests it exactly below
      const int at = atomicAdd(&s_qn[warp], 1);
      if (at < kQueue) {
        s_queue[warp][at] = (uint16_t)(lane << 10 | i);
      } else if (occupied(p, contract(ray_at(o, d, s_ts[i]), p.contraction))) {
        s_bits[(i >> 5) * 128 + tid] |= 1u << (i & 31);
      }
    } else if (vi >= 0 && __ldg(p.occ + vi) != 0) {
      // set candidates i..j
      for (int w = i >> 5; w <= (j >> 5); ++w) {
        const int lo = max(i - 32 * w, 0), hi = min(j - 32 * w, 31);
        const uint32_t upto = hi == 31 ? 0xffffffffu : ((1u << (hi + 1)) - 1u);
        s_bits[w * 128 + tid] |= upto & ~((1u << lo) - 1u);
      }
    }
    i = j + 1;
  }
  __syncwarp();
  // undecided candidates of the whole warp, re-tested in exact double one per lane
  const int qn = min(s_qn[warp], kQueue);
  for (int k = lane; k < qn; k += 32) {
    const int e = s_queue[warp][k], ol = e >> 10, c = e & 1023;
    const d3 od{s_dir[warp][ol][0], s_dir[warp][ol][1], s_dir[warp][ol][2]};
    if (occupied(p, contract(ray_at(o, od, s_ts[c]), p.contraction)))
      atomicOr(&s_bits[(c >> 5) * 128 + warp * 32 + ol], 1u << (c & 31));
  }
  __syncwarp();
  if (idx < p.total_rays) {
    int count = 0;
    for (int w0 = 0; w0 < p.mask_words; ++w0) {
      const uint32_t bits = s_bits[w0 * 128 + tid];
      count += __popc(bits);
      p.kept_mask[(size_t)w0 * p.total_rays + idx] = p.mask_transposed ? warp_transpose32(bits) : bits;
    }
    p.kept_count[idx] = (uint16_t)count;
  }
  add_work_stats(p, 0, 0, valid ? (unsigned long long)tested : 0ull, 0);
}

}  // namespace march
}  // namespace lumi_dev

using namespace lumi_dev;

// The exact march pass (k_march_mask) over p.total_rays tile-ordered ray ids
// (p.tile_w x p.tile_h tiles) into p.kept_mask / p.kept_count.
cudaError_t launch_march_mask(const RenderParams& p, cudaStream_t s) {
  // LUMI_MARCH_EXACT=1: the double-precision pass; LUMI_MARCH_RUNS=1: the voxel-run pass
  // (A/B and tests; default: the certified fp32 pass candidate by candidate)
  static const bool exact = std::getenv("LUMI_MARCH_EXACT") != nullptr;
  static const bool runs = std::getenv("LUMI_MARCH_RUNS") != nullptr;
  const unsigned blocks = (unsigned)((p.total_rays + 127) / 128);
  if (exact)
    march::k_march_mask<<<blocks, 128, 0, s>>>(p);
  else if (runs)
    march::k_march_runs<<<blocks, 128, (size_t)p.mask_words * 128 * sizeof(uint32_t), s>>>(p);
  else
    march::k_march_mask_fast<<<blocks, 128, 0, s>>>(p);
  return cudaGetLastError();
}

namespace lumi_dev {
namespace march {
// [word][ray] production mask (row-major ray ids) -> the public [pixel][word] layout
__global__ void k_unpack_kept(RenderParams p, uint32_t* mask, int32_t* counts) {
  const long long ray = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (ray >= p.total_rays) return;
  const size_t pix = (size_t)p.row_begin * p.cam.width + ray;
  if (mask)
    for (int w = 0; w < p.mask_words; ++w)
      mask[pix * p.mask_words + w] = p.kept_mask[(size_t)w * p.total_rays + ray];
  if (counts) counts[pix] = p.kept_count[ray];
}
}  // namespace march
}  // namespace lumi_dev

// lumi_march_kept_async through the production march pass (the one the renderers consume)
cudaError_t launch_march_public(RenderParams p, uint32_t* mask, int32_t* counts, cudaStream_t s) {
  const long long rays = (long long)(p.row_end - p.row_begin) * p.cam.width;
  if (rays <= 0) return cudaSuccess;
  p.tile_w = p.cam.width;
  p.tile_h = 1;
  p.tiles_x = 1;
  p.total_rays = rays;
  p.mask_words = (p.n + 31) / 32;
  p.work_stats = nullptr;
  p.mask_transposed = 0;
  cudaError_t e;
  if ((e = cudaMallocAsync(&p.kept_mask, (size_t)rays * p.mask_words * 4, s)) != cudaSuccess) return e;
  if ((e = cudaMallocAsync(&p.kept_count, (size_t)rays * 2, s)) != cudaSuccess) return e;
  if ((e = launch_march_mask(p, s)) != cudaSuccess) return e;
  march::k_unpack_kept<<<(unsigned)((rays + 127) / 128), 128, 0, s>>>(p, mask, counts);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  cudaFreeAsync(p.kept_mask, s);
  cudaFreeAsync(p.kept_count, s);
  return cudaGetLastError();
}

