// render_tc.cu -- the B200 frame renderer: a persistent kernel in which every CTA owns 128
// live rays (one per thread), marches each to its next occupancy-kept sample, gathers the
// mip hash-grid features for that sample, runs the five 64-wide MLP layers of the whole
// 128-sample batch on the 5th-generation tensor cores (tcgen05.mma, fp16 operands staged in
// shared memory, fp32 accumulators in TMEM) and composites front to back in registers.
//
// Thread t  <->  ray slot t  <->  batch row t  <->  TMEM lane t.  Rays that terminate or run
// out of samples are replaced from a tile queue (16x8-pixel tiles handed out by a global
// atomic), so the batch stays full and spatially coherent (neighbouring rays at similar
// depths gather neighbouring hash-grid cells).
//
// Reference semantics: renderer.h:126-237 (march / flush / composite), field.h:106-137
// (forward_chunk), grid.h:90-167 (encode).  Geometry and the occupancy test are bit-exact
// (geometry.cuh); features are bit-exact (field.cuh); the MLP runs in fp16 x fp16 -> fp32 on
// tensor cores (oracle-measured error 1.6e-4 max |dPQ| at C1 vs the 1e-3 bar).
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cmath>
#include <cstdlib>

#include "kernels.h"
#include "render_common.cuh"
#include "tc_ptx.cuh"

namespace lumi_dev {
namespace tc {

constexpr int kThreads = 128;  // UMMA M
constexpr int kTileW = 16, kTileH = 8;
constexpr uint32_t kTmemCols = 64;
#ifndef LUMI_PPP
#define LUMI_PPP 2
#endif
constexpr int kPPP = LUMI_PPP;  // gather pairs per lane per pass
#ifdef LUMI_PHASE_TIMING
// per-phase warp-cycles (instrumented builds only): advance, gather, CTA sync, MLP,
// composite, round barrier
__device__ unsigned long long g_phase_cycles[6];
#endif

// Every layer's K carries one extra 16-wide step whose first column is 1 in A and the bias
// in B, so the tensor core adds the bias (fp16 x 1 into the fp32 accumulator).
constexpr int kKb = 16;
struct __align__(16) Smem {  // used straight from the __shared__ array: LDS/STS, not LD/ST
  uint8_t A[128 * (64 + kKb) * 2];  // activations, K-major core-matrix tile (K <= 64+16)
  uint8_t W1[64 * (32 + kKb) * 2];  // density L1  N=64 K=32(+bias)
  uint8_t W2[32 * (64 + kKb) * 2];  // density L2  N=32 (17 used) K=64(+bias)
  uint8_t C1[64 * (32 + kKb) * 2];  // colour L1   N=64 K=32(+bias)
  uint8_t C2[64 * (64 + kKb) * 2];  // colour L2   N=64 K=64(+bias)
  uint8_t C3[16 * (64 + kKb) * 2];  // colour L3   N=16 (3 used) K=64(+bias)
  uint64_t mbar;
  uint32_t tmem_base;
  int q_next, q_end, q_done;
  uint8_t pair_src[kThreads / 32][32 * kMaxLevels];  // per-warp (sample lane, level) work list
  uint8_t pair_lvl[kThreads / 32][32 * kMaxLevels];
};

// byte offset of (row, 8-element K chunk) in a K-major SWIZZLE_NONE tile with kchunks chunks
__device__ __forceinline__ uint32_t core_off(int row, int chunk, int kchunks) {
  return (uint32_t)((row >> 3) * (kchunks * 128) + chunk * 128 + (row & 7) * 16);
}

__device__ __forceinline__ uint4 pack8(const float* v) {
  __half2 h0 = __floats2half2_rn(v[0], v[1]), h1 = __floats2half2_rn(v[2], v[3]),
          h2 = __floats2half2_rn(v[4], v[5]), h3 = __floats2half2_rn(v[6], v[7]);
  uint4 u;
  u.x = *reinterpret_cast<uint32_t*>(&h0);
  u.y = *reinterpret_cast<uint32_t*>(&h1);
  u.z = *reinterpret_cast<uint32_t*>(&h2);
  u.w = *reinterpret_cast<uint32_t*>(&h3);
  return u;
}

__device__ __forceinline__ void st_shared16(uint8_t* base, uint32_t off, uint4 v) {
  *reinterpret_cast<uint4*>(base + off) = v;
}

// weights [n_real x K] fp32 row-major (network.h:64) and bias [n_real] -> fp16 tile with
// n_pad rows and K + 16 columns: [W | b 0 ... 0]
__device__ void load_weight_tile(uint8_t* dst, const float* __restrict__ W,
                                 const float* __restrict__ b, int n_real, int n_pad, int K) {
  const int kch = (K + kKb) / 8;
  for (int it = threadIdx.x; it < n_pad * kch; it += blockDim.x) {
    const int n = it / kch, j = it % kch;
    float v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int k = 8 * j + q;
      v[q] = n >= n_real ? 0.f : k < K ? __ldg(W + (size_t)n * K + k) : k == K ? __ldg(b + n) : 0.f;
    }
    st_shared16(dst, core_off(n, j, kch), pack8(v));
  }
}

// the [1 0 ... 0 | 0 ... 0] bias step of this thread's A row for a layer with K data columns
__device__ __forceinline__ void write_bias_step(uint8_t* A, int row, int K) {
  const int kch = (K + kKb) / 8;
  st_shared16(A, core_off(row, K / 8, kch), make_uint4(0x3C00u, 0u, 0u, 0u));  // fp16 1.0
  st_shared16(A, core_off(row, K / 8 + 1, kch), make_uint4(0u, 0u, 0u, 0u));
}

// fp32 x 8 -> fp16 x 8 with ReLU applied on the packed halves (max(h(x), 0) == h(max(x, 0)))
__device__ __forceinline__ uint4 pack8_relu(const float* v) {
  const __half2 z = __float2half2_rn(0.f);
  __half2 h0 = __hmax2(__floats2half2_rn(v[0], v[1]), z), h1 = __hmax2(__floats2half2_rn(v[2], v[3]), z),
          h2 = __hmax2(__floats2half2_rn(v[4], v[5]), z), h3 = __hmax2(__floats2half2_rn(v[6], v[7]), z);
  uint4 u;
  u.x = *reinterpret_cast<uint32_t*>(&h0);
  u.y = *reinterpret_cast<uint32_t*>(&h1);
  u.z = *reinterpret_cast<uint32_t*>(&h2);
  u.w = *reinterpret_cast<uint32_t*>(&h3);
  return u;
}

template <int N, int K>
__device__ __forceinline__ void issue_layer(const Smem& s, const uint8_t* B, uint32_t d_tmem) {
  constexpr uint32_t idesc = ptx::idesc_f16_f32<128, N>();
  const uint32_t a = ptx::smem_addr(s.A), b = ptx::smem_addr(B);
#pragma unroll
  for (int kk = 0; kk < K / 16; ++kk) {
    const uint64_t ad = ptx::make_smem_desc(a + kk * 256, 128, (K / 8) * 128);
    const uint64_t bd = ptx::make_smem_desc(b + kk * 256, 128, (K / 8) * 128);
    ptx::mma_f16(d_tmem, ad, bd, idesc, kk > 0 ? 1u : 0u);
  }
}

// Hidden-layer epilogue: TMEM row (64 fp32 accumulators of this thread's sample) + bias,
// ReLU, fp16 -> this thread's row of the next layer's A tile (K = 64).  Two halves of 32
// columns keep the live register count down.
__device__ __forceinline__ void relu64_to_A(uint32_t t_lane, uint8_t* A, int row) {
  constexpr int kch = (64 + kKb) / 8;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    float v[32];
    ptx::tmem_ld16(t_lane + 32 * h, v);
    ptx::tmem_ld16(t_lane + 32 * h + 16, v + 16);
    ptx::tmem_ld_wait();
#pragma unroll
    for (int j = 0; j < 4; ++j) st_shared16(A, core_off(row, 4 * h + j, kch), pack8_relu(v + 8 * j));
  }
  write_bias_step(A, row, 64);
}

struct Ray {
  int id, x, y;
  d3 d, nd;
  int wi, kept_total, contributing, cut_limit;
  uint32_t word;  // unvisited kept candidates of mask word wi
  bool term;
  double trans, px, py, pz, depth, opac;
};

struct Sample {
  d3 c;
  double t, delta;
  LodW lw;
};

struct Counters {
  unsigned evals, level_samples, marched, rays;
};

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

__device__ __forceinline__ bool take_ray(const RenderParams& p, Smem& s, Ray& r) {
  for (;;) {
    const int idx = atomicAdd(&s.q_next, 1);
    if (idx >= s.q_end) return false;
    int x, y;
    if (!ray_pixel(p, idx, x, y)) continue;
    r.id = idx;
    r.x = x;
    r.y = y;
    r.d = ray_dir(p.cam, (double)x + 0.5, (double)y + 0.5);
    r.nd = ray_dir(p.cam, (double)x + 1.5, (double)y + 0.5);
    r.wi = 0;
    r.word = __ldg(p.kept_mask + idx);
    r.kept_total = __ldg(p.kept_count + idx);
    r.contributing = 0;
    r.cut_limit = 0x7fffffff;
    r.term = false;
    r.trans = 1.0;
    r.px = r.py = r.pz = r.depth = r.opac = 0.0;
    return true;
  }
}

// Next occupancy-kept candidate of the ray (renderer.h:205-224), read from the march-pass
// bitmask.  Returns false when the ray is finished (no kept candidate left, or cut).
__device__ __forceinline__ bool advance(const RenderParams& p, const double* ts, Ray& r,
                                        Sample& smp, Counters& cnt) {
  if (r.term) return false;
  while (r.word == 0) {
    if (++r.wi >= p.mask_words) return false;
    r.word = __ldg(p.kept_mask + (size_t)r.wi * p.total_rays + r.id);
  }
  const int i = r.wi * 32 + __ffs(r.word) - 1;
  r.word &= r.word - 1;
  const d3 o{p.cam.origin[0], p.cam.origin[1], p.cam.origin[2]};
  const double t = __ldg(ts + i);
  smp.c = contract_fast(ray_at(o, r.d, t), p.contraction);
  smp.t = t;
  smp.delta = (i + 1 < p.n) ? dsub(__ldg(ts + i + 1), t) : dmul(t, dsub(p.ratio, 1.0));
  if (p.lod_enabled) {
    smp.lw = lod_weights_f(lod_eff_fast(o, r.d, r.nd, t, p.contraction, (float)p.grid.two_base,
                                        (float)(1.0 / p.grid.log_scale), p.grid.levels,
                                        (float)p.lod_bias),
                           p.grid.levels);
  } else {
    smp.lw = LodW{p.grid.levels, 0.f, false};
  }
  cnt.level_samples += active_levels(smp.lw, p.grid.levels);
  return true;
}

__device__ __forceinline__ void finish(const RenderParams& p, Ray& r, Counters& cnt) {
  RayResult res{r.px, r.py, r.pz, r.depth, r.opac,
                chunk_evals(r.term, r.contributing, r.kept_total, p.chunk), r.contributing};
  store_ray(p, r.x, r.y, res, r.trans);
  ++cnt.rays;
  r.id = -1;
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
    p.kept_mask[(size_t)w0 * p.total_rays + idx] = bits;
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
    if (idx < p.total_rays) p.kept_mask[(size_t)w0 * p.total_rays + idx] = bits;
  }
  if (idx < p.total_rays) p.kept_count[idx] = (uint16_t)count;
  add_work_stats(p, 0, 0, valid ? (unsigned long long)p.n : 0ull, 0);
}

__device__ void refill(const RenderParams& p, Smem& s, int total) {
  if (s.q_next < s.q_end || s.q_done) return;
  const int base = (int)atomicAdd(p.work_counter, (unsigned)(kTileW * kTileH));
  if (base >= total) {
    s.q_done = 1;
    s.q_next = s.q_end = 0;
  } else {
    s.q_next = base;
    s.q_end = min(base + kTileW * kTileH, total);
  }
}

__global__ void __launch_bounds__(kThreads, 4) k_render_tc(RenderParams p) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  Smem& s = *reinterpret_cast<Smem*>(smem_raw);
  const int tid = threadIdx.x, warp = tid >> 5;

  // ---- one-time setup: weights -> fp16 core-matrix tiles, biases, distances, TMEM --------
  const float* dp = p.mlp.dparams;
  const float* cp = p.mlp.cparams;
  // flattened weights-then-bias per layer (network.h:144-151)
  const float* d2 = dp + 64 * 32 + 64;
  const float* c2 = cp + 64 * 32 + 64;
  const float* c3 = c2 + 64 * 64 + 64;
  load_weight_tile(s.W1, dp, dp + 64 * 32, 64, 64, 32);
  load_weight_tile(s.W2, d2, d2 + 17 * 64, 1 + kBottleneck, 32, 64);
  load_weight_tile(s.C1, cp, cp + 64 * 32, 64, 64, 32);
  load_weight_tile(s.C2, c2, c2 + 64 * 64, 64, 64, 64);
  load_weight_tile(s.C3, c3, c3 + 3 * 64, 3, 16, 64);
  const int total = (int)p.total_rays;
  if (tid == 0) {
    ptx::mbar_init(&s.mbar, 1);
    ptx::fence_mbar_init();
    s.q_next = s.q_end = 0;
    s.q_done = 0;
    refill(p, s, total);
  }
  if (warp == 0) ptx::tmem_alloc<kTmemCols>(&s.tmem_base);
  ptx::fence_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = s.tmem_base;
  const uint32_t t_lane = tmem + ((uint32_t)(warp * 32) << 16);  // this warp's 32 TMEM lanes

  Counters cnt{0, 0, 0, 0};
  Ray r;
  r.id = -1;
  uint32_t phase = 0;
  const bool issuer = (tid == 0);
#ifdef LUMI_PHASE_TIMING
  long long pt[6] = {0, 0, 0, 0, 0, 0}, pt_last = clock64();
#define PT_MARK(k)                          \
  do {                                      \
    const long long _t = clock64();         \
    pt[k] += _t - pt_last;                  \
    pt_last = _t;                           \
  } while (0)
#else
#define PT_MARK(k) \
  do {             \
  } while (0)
#endif

  for (;;) {
    // ---- A: every thread brings one kept sample (refilling finished rays) ------------------
    Sample smp;
    bool have = false;
    for (;;) {
      if (r.id < 0 && !take_ray(p, s, r)) break;
      if (advance(p, p.ts, r, smp, cnt)) {  // distances via L1 (one load per sample)
        have = true;
        break;
      }
      finish(p, r, cnt);
    }
    __syncwarp();
    PT_MARK(0);
    // ---- B: warp-cooperative hash-grid gather (grid.h:90-167) ------------------------------
    // The warp's 32 samples have different numbers of active LOD levels; their (sample,
    // level) pairs are listed level-major and dealt round-robin to the 32 lanes, so every
    // lane gathers in every pass and neighbouring rays hit neighbouring cells of the same
    // level in one warp-wide load.  Features land as fp16 straight in this sample's A row.
    {
      const int lane = tid & 31;
      constexpr int kch = (32 + kKb) / 8;  // density L1 A layout: 32 features + bias step
      const uint4 zero = make_uint4(0, 0, 0, 0);
#pragma unroll
      for (int j = 0; j < 4; ++j) st_shared16(s.A, core_off(tid, j, kch), zero);
      write_bias_step(s.A, tid, 32);
      const int na = have ? active_levels(smp.lw, p.grid.levels) : 0;
      uint8_t* psrc = s.pair_src[warp];
      uint8_t* plvl = s.pair_lvl[warp];
      const unsigned lt = (1u << lane) - 1u;
      int npairs = 0;
      for (int l = 0; l < p.grid.levels; ++l) {
        const unsigned m = __ballot_sync(0xffffffffu, na > l);
        if (na > l) {
          const int at = npairs + __popc(m & lt);
          psrc[at] = (uint8_t)lane;
          plvl[at] = (uint8_t)l;
        }
        npairs += __popc(m);
      }
      __syncwarp();
      // unit-cube coordinates (grid.h:93-95), clamped once per sample (grid.h:146-148) and
      // split into float pairs for the fp32 cell arithmetic of encode_level_hf
      const double u = clamp01(have ? dmul(dadd(smp.c.x, 2.0), 0.25) : 0.0);
      const double v = clamp01(have ? dmul(dadd(smp.c.y, 2.0), 0.25) : 0.0);
      const double w = clamp01(have ? dmul(dadd(smp.c.z, 2.0), 0.25) : 0.0);
      const uint8_t* Abase = s.A + (warp * 32 / 8) * (kch * 128);
#pragma unroll 1
      // kPPP (sample, level) pairs per lane per pass: 8 * kPPP independent gathers in flight
      for (int base = 0; base < npairs; base += 32 * kPPP) {
        int src[kPPP], lv[kPPP];
        bool ok[kPPP];
        double su[kPPP], sv[kPPP], sw[kPPP];
        float wl[kPPP];
#pragma unroll
        for (int q = 0; q < kPPP; ++q) {
          const int pi = base + 32 * q + lane;
          ok[q] = pi < npairs;
          src[q] = ok[q] ? psrc[pi] : lane;
          lv[q] = ok[q] ? plvl[pi] : 0;
          su[q] = __shfl_sync(0xffffffffu, u, src[q]);
          sv[q] = __shfl_sync(0xffffffffu, v, src[q]);
          sw[q] = __shfl_sync(0xffffffffu, w, src[q]);
          LodW lw;
          lw.full = __shfl_sync(0xffffffffu, smp.lw.full, src[q]);
          lw.frac = __shfl_sync(0xffffffffu, smp.lw.frac, src[q]);
          lw.floor_only = __shfl_sync(0xffffffffu, (int)smp.lw.floor_only, src[q]) != 0;
          wl[q] = lod_weight_at(lw, lv[q]);
        }
        float2 f[kPPP];
#pragma unroll
        for (int q = 0; q < kPPP; ++q)
          f[q] = ok[q] && !(p.debug_flags & 1) ? encode_level_h(p.grid, p.grid.table16, lv[q], su[q], sv[q], sw[q], wl[q])
                       : make_float2(0.f, 0.f);
#pragma unroll
        for (int q = 0; q < kPPP; ++q)
          if (ok[q])
            *reinterpret_cast<__half2*>(const_cast<uint8_t*>(Abase) + core_off(src[q], lv[q] >> 2, kch) +
                                        (lv[q] & 3) * 4) = __floats2half2_rn(f[q].x, f[q].y);
      }
    }
    ptx::fence_async_smem();
    __syncwarp();
    PT_MARK(1);
    if (!__syncthreads_or(have)) {
      if (tid == 0) refill(p, s, total);
      __syncthreads();
      if (s.q_done && s.q_next >= s.q_end) break;
      continue;
    }
    PT_MARK(2);

    float v[32];
    float sigma = 1.f;
    if (!(p.debug_flags & 2)) {
    // ---- density L1: [128x32] x [32x64] -> relu -------------------------------------------
    if (issuer) {
      ptx::tc_fence_after();
      issue_layer<64, 32 + kKb>(s, s.W1, tmem);
      ptx::mma_commit(&s.mbar);
    }
    ptx::mbar_wait(&s.mbar, phase);
    phase ^= 1;
    ptx::tc_fence_after();
    relu64_to_A(t_lane, s.A, tid);
    ptx::fence_async_smem();
    ptx::tc_fence_before();
    __syncthreads();

    // ---- density L2: [128x64] x [64x32(17)] -> sigma, bottleneck ++ SH ---------------------
    if (issuer) {
      ptx::tc_fence_after();
      issue_layer<32, 64 + kKb>(s, s.W2, tmem);
      ptx::mma_commit(&s.mbar);
    }
    ptx::mbar_wait(&s.mbar, phase);
    phase ^= 1;
    ptx::tc_fence_after();
    ptx::tmem_ld16(t_lane, v);
    ptx::tmem_ld16(t_lane + 16, v + 16);
    ptx::tmem_ld_wait();
    sigma = trunc_exp(v[0]);
    {
      constexpr int kch = (32 + kKb) / 8;
      float cin[32];
#pragma unroll
      for (int j = 0; j < 16; ++j) cin[j] = v[1 + j];
      sh_encode(r.d, cin + 16);
#pragma unroll
      for (int j = 0; j < 4; ++j) st_shared16(s.A, core_off(tid, j, kch), pack8(cin + 8 * j));
      write_bias_step(s.A, tid, 32);
    }
    ptx::fence_async_smem();
    ptx::tc_fence_before();
    __syncthreads();

    // ---- colour L1: [128x32] x [32x64] -> relu -------------------------------------------
    if (issuer) {
      ptx::tc_fence_after();
      issue_layer<64, 32 + kKb>(s, s.C1, tmem);
      ptx::mma_commit(&s.mbar);
    }
    ptx::mbar_wait(&s.mbar, phase);
    phase ^= 1;
    ptx::tc_fence_after();
    relu64_to_A(t_lane, s.A, tid);
    ptx::fence_async_smem();
    ptx::tc_fence_before();
    __syncthreads();

    // ---- colour L2: [128x64] x [64x64] -> relu -------------------------------------------
    if (issuer) {
      ptx::tc_fence_after();
      issue_layer<64, 64 + kKb>(s, s.C2, tmem);
      ptx::mma_commit(&s.mbar);
    }
    ptx::mbar_wait(&s.mbar, phase);
    phase ^= 1;
    ptx::tc_fence_after();
    relu64_to_A(t_lane, s.A, tid);
    ptx::fence_async_smem();
    ptx::tc_fence_before();
    __syncthreads();

    // ---- colour L3: [128x64] x [64x16(3)] -> sigmoid (PQ head) ---------------------------
    if (issuer) {
      ptx::tc_fence_after();
      issue_layer<16, 64 + kKb>(s, s.C3, tmem);
      ptx::mma_commit(&s.mbar);
    }
    ptx::mbar_wait(&s.mbar, phase);
    phase ^= 1;
    ptx::tc_fence_after();
    ptx::tmem_ld16(t_lane, v);
    ptx::tmem_ld_wait();
    ptx::tc_fence_before();
    } else {
      v[0] = v[1] = v[2] = 0.f;
    }
    PT_MARK(3);

    // ---- C: front-to-back compositing (renderer.h:170-190), double ----------------------
    if (have) {
      float rgb[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const float raw = v[k];
        rgb[k] = p.mlp.color_space == 0 ? sigmoid(raw) : trunc_exp(raw);
      }
      const double a = dsub(1.0, exp(dmul(-(double)sigma, smp.delta)));
      const double w = dmul(r.trans, a);
      r.px = dadd(r.px, dmul(w, (double)rgb[0]));
      r.py = dadd(r.py, dmul(w, (double)rgb[1]));
      r.pz = dadd(r.pz, dmul(w, (double)rgb[2]));
      r.depth = dadd(r.depth, dmul(w, smp.t));
      r.opac = dadd(r.opac, w);
      r.trans = dmul(r.trans, dsub(1.0, a));
      ++r.contributing;
      ++cnt.evals;
      if (p.t_cut > 0 && r.trans < p.t_cut) {
        r.term = true;
        r.cut_limit = ((r.contributing + p.chunk - 1) / p.chunk) * p.chunk;
      }
    }
    __syncwarp();
    PT_MARK(4);
    if (tid == 0) refill(p, s, total);
    __syncthreads();
    PT_MARK(5);
  }

  // ---- teardown --------------------------------------------------------------------------
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (warp == 0) ptx::tmem_dealloc<kTmemCols>(tmem);
  add_work_stats(p, cnt.evals, cnt.level_samples, cnt.marched, cnt.rays);
#ifdef LUMI_PHASE_TIMING
  if ((tid & 31) == 0)
    for (int k = 0; k < 6; ++k) atomicAdd(&g_phase_cycles[k], (unsigned long long)pt[k]);
#endif
#undef PT_MARK
}

}  // namespace tc
}  // namespace lumi_dev

using namespace lumi_dev;

size_t render_tc_smem_bytes() { return sizeof(tc::Smem); }

cudaError_t launch_render_tc(RenderParams p, cudaStream_t s, int num_sms, cudaEvent_t* ev) {
  const long long rays = (long long)(p.row_end - p.row_begin) * p.cam.width;
  if (rays <= 0) return cudaSuccess;
  static int blocks_per_sm = -1;
  const size_t smem = render_tc_smem_bytes();
  if (blocks_per_sm < 0) {
    cudaError_t e = cudaFuncSetAttribute(tc::k_render_tc, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(tc::k_render_tc, cudaFuncAttributePreferredSharedMemoryCarveout,
                             cudaSharedmemCarveoutMaxShared);
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, tc::k_render_tc, tc::kThreads,
                                                      smem);
    if (e != cudaSuccess) return e;
    // The runtime's estimate has been seen to under-report for this kernel on sm_100 (1 vs the
    // 3 CTAs/SM ncu reports from registers/smem); take the register/smem bound directly.
    cudaFuncAttributes fa;
    if ((e = cudaFuncGetAttributes(&fa, tc::k_render_tc)) != cudaSuccess) return e;
    const int regs_per_warp = ((fa.numRegs * 32 + 255) / 256) * 256;
    const int by_regs = 65536 / (regs_per_warp * (tc::kThreads / 32));
    const int by_smem = (228 * 1024) / (int)(smem + 1024);
    blocks_per_sm = std::max(blocks_per_sm, std::max(1, std::min(by_regs, by_smem)));
    // Shared memory and L1 share one 256 KB array: reserve only what the resident CTAs need
    // so the rest stays L1 for the hash-table gathers (LUMI_MAX_CTAS caps residency).
    if (const char* cap = std::getenv("LUMI_MAX_CTAS"))
      blocks_per_sm = std::max(1, std::min(blocks_per_sm, std::atoi(cap)));
    const int carve = (int)std::ceil(100.0 * blocks_per_sm * (double)(smem + 1024) / (228.0 * 1024));
    if ((e = cudaFuncSetAttribute(tc::k_render_tc, cudaFuncAttributePreferredSharedMemoryCarveout,
                                  std::min(100, carve))) != cudaSuccess)
      return e;
    if (std::getenv("LUMI_DEBUG")) {
      cudaFuncAttributes fa;
      cudaFuncGetAttributes(&fa, tc::k_render_tc);
      int b0 = -1, b1 = -1;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b0, tc::k_render_tc, tc::kThreads, 0);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b1, tc::k_render_tc, tc::kThreads, 32768);
      std::fprintf(stderr,
                   "[lumi] k_render_tc: %zu B smem, %d CTAs/SM x %d SMs (regs %d, static smem %zu, "
                   "local %zu, maxdyn %d, occ@0=%d occ@32K=%d)\n",
                   smem, blocks_per_sm, num_sms, fa.numRegs, fa.sharedSizeBytes, fa.localSizeBytes,
                   fa.maxDynamicSharedSizeBytes, b0, b1);
    }
  }
  p.tile_w = tc::kTileW;
  p.tile_h = tc::kTileH;
  p.tiles_x = (p.cam.width + tc::kTileW - 1) / tc::kTileW;
  const long long tiles =
      (long long)p.tiles_x * ((p.row_end - p.row_begin + tc::kTileH - 1) / tc::kTileH);
  p.total_rays = tiles * tc::kTileW * tc::kTileH;
  if (p.total_rays >= (1ll << 31)) return cudaErrorInvalidValue;
  p.mask_words = (p.n + 31) / 32;
  cudaError_t e;
  if ((e = cudaMallocAsync(&p.kept_mask, (size_t)p.total_rays * p.mask_words * 4, s)) != cudaSuccess)
    return e;
  if ((e = cudaMallocAsync(&p.kept_count, (size_t)p.total_rays * 2, s)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(p.work_counter, 0, sizeof(unsigned int), s)) != cudaSuccess) return e;
  if (ev) cudaEventRecord(ev[0], s);
  if ((e = launch_march_mask(p, s)) != cudaSuccess) return e;
  if (ev) cudaEventRecord(ev[1], s);
  const long long grid = std::min<long long>((long long)blocks_per_sm * num_sms, tiles);
#ifdef LUMI_PHASE_TIMING
  unsigned long long zero6[6] = {0, 0, 0, 0, 0, 0};
  cudaMemcpyToSymbolAsync(tc::g_phase_cycles, zero6, sizeof(zero6), 0, cudaMemcpyHostToDevice, s);
#endif
  tc::k_render_tc<<<(unsigned)grid, tc::kThreads, smem, s>>>(p);
  if (ev) cudaEventRecord(ev[2], s);
#ifdef LUMI_PHASE_TIMING
  {
    unsigned long long pc[6];
    cudaMemcpyFromSymbolAsync(pc, tc::g_phase_cycles, sizeof(pc), 0, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    double tot = 0;
    for (int k = 0; k < 6; ++k) tot += (double)pc[k];
    std::fprintf(stderr, "[lumi] phase warp-cycles %%: advance %.1f gather %.1f ctasync %.1f mlp %.1f "
                 "composite %.1f roundbar %.1f\n", 100 * pc[0] / tot, 100 * pc[1] / tot,
                 100 * pc[2] / tot, 100 * pc[3] / tot, 100 * pc[4] / tot, 100 * pc[5] / tot);
  }
#endif
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  cudaFreeAsync(p.kept_mask, s);
  cudaFreeAsync(p.kept_count, s);
  return cudaGetLastError();
}

// The exact march pass (k_march_mask) over p.total_rays tile-ordered ray ids
// (p.tile_w x p.tile_h tiles) into p.kept_mask / p.kept_count.
cudaError_t launch_march_mask(const RenderParams& p, cudaStream_t s) {
  static const bool exact = std::getenv("LUMI_MARCH_EXACT") != nullptr;  // A/B and tests
  if (exact)
    tc::k_march_mask<<<(unsigned)((p.total_rays + 127) / 128), 128, 0, s>>>(p);
  else
    tc::k_march_mask_fast<<<(unsigned)((p.total_rays + 127) / 128), 128, 0, s>>>(p);
  return cudaGetLastError();
}

namespace lumi_dev {
namespace tc {
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
}  // namespace tc
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
  cudaError_t e;
  if ((e = cudaMallocAsync(&p.kept_mask, (size_t)rays * p.mask_words * 4, s)) != cudaSuccess) return e;
  if ((e = cudaMallocAsync(&p.kept_count, (size_t)rays * 2, s)) != cudaSuccess) return e;
  if ((e = launch_march_mask(p, s)) != cudaSuccess) return e;
  tc::k_unpack_kept<<<(unsigned)((rays + 127) / 128), 128, 0, s>>>(p, mask, counts);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  cudaFreeAsync(p.kept_mask, s);
  cudaFreeAsync(p.kept_count, s);
  return cudaGetLastError();
}
