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
    const uint32_t out = bits;
    if (idx < p.total_rays) p.kept_mask[(size_t)w0 * p.total_rays + idx] = out;
  }
  if (idx < p.total_rays) p.kept_count[idx] = (uint16_t)count;
  add_work_stats(p, 0, 0, valid ? (unsigned long long)p.n : 0ull, 0);
}

// ---- segment march (production) -------------------------------------------------------------
// Along one ray the voxel coordinate g = (contract(o + d t) + 2) q (q = res / 4) is, piece by
// piece, an AFFINE function of one scalar v:
//   * inside the unit cube (|x|_inf < 1, contraction = identity):   g_k = q (o_k + 2) + q d_k t,
//     v = t;
//   * in the final contraction pyramid -- axis a the unique max |x_a| > 1 with sign s, which
//     holds for every t past t_pyr when |d_a| > |d_b| -- with w = 1 / |x_a| = 1 / (s o_a + |d_a| t):
//       g_a = q (2 + 2 s) - q s w,
//       g_b = q (2 + d_b / |d_a|) + q K_b w,   K_b = o_b - d_b o_a / d_a   (camera.cpp:34-49),
//     v = w.
// Per ray the segment bounds are solved in double with margins (the reference's double m and
// max axis are certain inside them), converted to candidate-index ranges, and the per-axis
// constants A = g-intercept - 1/2, B rounded to fp32.  Per candidate the kernel then computes
// h = A + B v (g - 1/2), its nearest integer (the floor of g) and its distance to it with
// packed-f32x2 FFMA2 / FADD2 on TWO candidates at once, and certifies the floor when every
// axis is more than eps(v) = E0 + E1 v (a rigorous bound on |h_f32 - h_reference|, below) from a
// rounding tie -- ~18 thread-instructions per candidate instead of the certified contraction's
// ~80.  Candidates in neither segment (a max-axis switch after leaving the cube, a camera
// outside the cube) and the ~1e-4 undecided ones take the general certified test, then the
// warp's exact double re-test: the kept set stays bit-exact.
//
// Error bounds (fp32 unit roundoff u = 2^-24; A_f, B_f, P_f are the double constants rounded
// to fp32, t_f = fl(t)):
//   inside:  |h_f - h| <= u (|A| + res) + 2 u |B| t  (constants, t rounding, the FFMA rounding)
//   pyramid: x_f = fl(|d_a| t_f + s o_a) is within u (3 + 3 |o_a|) m of m = |x_a| (m >= 1), and
//            rcp.approx adds <= 2^-23 relative, so |w_f - w| <= eps_w w; then
//            |h_f - h| <= u (|A| + res) + |B| w (u + eps_w)
// plus the reference's own double roundings (< 1e-12 in g).  E0 / E1 take twice these.
struct SegC {
  float ax, ay, az, bx, by, bz;  // h_k = A_k + B_k v
  float pq, pc;                  // v = rcp(|pq t + pc|) in the pyramid (pq = 1, pc = 0 inside)
  float th0, th1;                // certified when max_k |h_k - rint(h_k)| < th0 + th1 v (= 1/2 - eps)
};

__device__ __forceinline__ uint64_t f2_pack(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void f2_unpack(uint64_t r, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
}
__device__ __forceinline__ uint64_t f2_fma(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t f2_add(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t f2_sub(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

constexpr float kRint = 12582912.f;  // 1.5 * 2^23: x + kRint rounds x to an integer (|x| < 2^22)
constexpr uint32_t kRintBits = 0x4B400000u;

// One pair of candidates through one segment's affine test: the biased voxel index of each,
// vb = (bz r + by) r + bx with b_k = kRintBits + floor(g_k) (the occupancy byte of the voxel sits
// at occ_adj + vb, occ_adj = occ - kRintBits (r^2 + r + 1)); valid only where ok is set.
template <bool kPyr>
__device__ __forceinline__ void seg_pair(const SegC& c, float2 t, uint32_t r, uint32_t& vb0, uint32_t& vb1,
                                         bool& ok0, bool& ok1) {
  uint64_t v;
  if (kPyr) {
    float x0, x1;
    f2_unpack(f2_fma(f2_pack(c.pq, c.pq), f2_pack(t.x, t.y), f2_pack(c.pc, c.pc)), x0, x1);
    v = f2_pack(rcp_approx(fabsf(x0)), rcp_approx(fabsf(x1)));
  } else {
    v = f2_pack(t.x, t.y);
  }
  const uint64_t M = f2_pack(kRint, kRint), nM = f2_pack(-kRint, -kRint);
  const uint64_t hx = f2_fma(f2_pack(c.bx, c.bx), v, f2_pack(c.ax, c.ax));
  const uint64_t hy = f2_fma(f2_pack(c.by, c.by), v, f2_pack(c.ay, c.ay));
  const uint64_t hz = f2_fma(f2_pack(c.bz, c.bz), v, f2_pack(c.az, c.az));
  const uint64_t rx = f2_add(hx, M), ry = f2_add(hy, M), rz = f2_add(hz, M);
  const uint64_t ex = f2_sub(hx, f2_add(rx, nM)), ey = f2_sub(hy, f2_add(ry, nM)), ez = f2_sub(hz, f2_add(rz, nM));
  const uint64_t th = f2_fma(f2_pack(c.th1, c.th1), v, f2_pack(c.th0, c.th0));
  float ex0, ex1, ey0, ey1, ez0, ez1, th0, th1, bx0, bx1, by0, by1, bz0, bz1;
  f2_unpack(ex, ex0, ex1);
  f2_unpack(ey, ey0, ey1);
  f2_unpack(ez, ez0, ez1);
  f2_unpack(th, th0, th1);
  f2_unpack(rx, bx0, bx1);
  f2_unpack(ry, by0, by1);
  f2_unpack(rz, bz0, bz1);
  ok0 = fmaxf(fabsf(ex0), fmaxf(fabsf(ey0), fabsf(ez0))) < th0;
  ok1 = fmaxf(fabsf(ex1), fmaxf(fabsf(ey1), fabsf(ez1))) < th1;
  vb0 = (__float_as_uint(bz0) * r + __float_as_uint(by0)) * r + __float_as_uint(bx0);
  vb1 = (__float_as_uint(bz1) * r + __float_as_uint(by1)) * r + __float_as_uint(bx1);
}

__device__ __forceinline__ uint32_t mad_u32(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

// occ_adj + vb in one IMAD.WIDE.U32 (vb < 2^32 - occ bias never wraps: checked on the host)
__device__ __forceinline__ const uint8_t* occ_at(uint64_t occ_adj, uint32_t vb) {
  uint64_t a;
  asm("mad.wide.u32 %0, %1, 1, %2;" : "=l"(a) : "r"(vb), "l"(occ_adj));
  return reinterpret_cast<const uint8_t*>(a);
}

// One 32-candidate word through one segment: candidates whose bit is set in `range` and that
// certify add their occupancy bit (bytes are 0 / 1) to `bits`; the others of `range` are
// flagged in `unsure`.  Eight candidates per loop step with compile-time bit offsets inside a
// step -- a small code footprint: the instruction cache, not the ALUs, bounded a fully unrolled
// word.  Each candidate's byte slot starts at 256 and a certified candidate's load overwrites
// it with 0 / 1, so one multiply-add per candidate packs the occupancy bits (bits 0-7) and the
// undecided flags (bits 8-15) of the step together.  kMasked: lanes whose word is not entirely
// in the segment (the range test gates the load so no out-of-segment index is dereferenced).
template <bool kPyr, bool kMasked>
__device__ __forceinline__ void seg_word(const SegC& c, const float* __restrict__ tw, uint32_t range,
                                         uint64_t occ_adj, uint32_t r, uint32_t& bits, uint32_t& unsure) {
#pragma unroll 1
  for (int g = 0; g < 32; g += 8) {
    const uint32_t rg = (range >> g) & 0xffu;
    if (!kMasked || rg) {
      const float4 ta = *reinterpret_cast<const float4*>(tw + g);
      const float4 tb = *reinterpret_cast<const float4*>(tw + g + 4);
      const float2 tp[4] = {make_float2(ta.x, ta.y), make_float2(ta.z, ta.w), make_float2(tb.x, tb.y),
                            make_float2(tb.z, tb.w)};
      uint32_t ob = 0;
#pragma unroll
      for (int k = 0; k < 8; k += 2) {
        uint32_t vb0, vb1;
        bool ok0, ok1;
        seg_pair<kPyr>(c, tp[k >> 1], r, vb0, vb1, ok0, ok1);
        if (kMasked) {
          ok0 = ok0 && (rg & (1u << k));
          ok1 = ok1 && (rg & (2u << k));
        }
        uint32_t o0 = 256u, o1 = 256u;
#ifdef LUMI_MARCH_BITS
        // occ_adj addresses the bitfield's words: word vb >> 5, bit vb & 31 (the bias is a
        // multiple of 2^22, so the low bits are the voxel's own)
        if (ok0) o0 = (__ldg(reinterpret_cast<const uint32_t*>(occ_at(occ_adj, (vb0 >> 5) * 4u))) >> (vb0 & 31u)) & 1u;
        if (ok1) o1 = (__ldg(reinterpret_cast<const uint32_t*>(occ_at(occ_adj, (vb1 >> 5) * 4u))) >> (vb1 & 31u)) & 1u;
#else
        if (ok0) o0 = __ldg(occ_at(occ_adj, vb0));
        if (ok1) o1 = __ldg(occ_at(occ_adj, vb1));
#endif
        ob = mad_u32(o0, 1u << k, ob);
        ob = mad_u32(o1, 2u << k, ob);
      }
      bits |= (ob & 0xffu) << g;
      unsure |= (kMasked ? (ob >> 8) & rg : ob >> 8) << g;
    }
  }
}

// bits [lo, hi) of a word (lo < 32 when lo < hi)
__device__ __forceinline__ uint32_t bits_range(int lo, int hi) {
  if (lo >= hi) return 0u;
  return (hi >= 32 ? 0xffffffffu : (1u << hi) - 1u) & ~((1u << lo) - 1u);
}

// first index i in [0, n) with ts[i] >= t (n if none); ts ascending
__device__ __forceinline__ int lower_index(const double* ts, int n, double t) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (ts[mid] < t) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// Per-ray segments (double): candidates [0, n_in) inside, [i_pyr, n) in the final pyramid.
// (Written without dynamic indexing of per-axis arrays, so nothing lands on the stack.)
__device__ __forceinline__ double sel3(int k, double x, double y, double z) { return k == 0 ? x : (k == 1 ? y : z); }

__device__ void seg_setup(const RenderParams& p, const double* ts, d3 o, d3 d, SegC& cin, SegC& cpy,
                          int& n_in, int& i_pyr) {
  const double q = 0.25 * p.occ_res, res = (double)p.occ_res, u = 5.9604644775390625e-08;  // 2^-24
  n_in = 0;
  i_pyr = p.n;
  // inside: every |x_k| <= L - delta (L = 1 with contraction: identity; L = 2 without: the
  // grid's domain), so the reference's double point is strictly inside too
  const double L = p.contraction ? 1.0 : 2.0, delta = 1e-6;
  if (fabs(o.x) < L - delta && fabs(o.y) < L - delta && fabs(o.z) < L - delta) {
    double t_in = 1e300;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const double ok = sel3(k, o.x, o.y, o.z), dk = sel3(k, d.x, d.y, d.z);
      if (dk > 0.0) t_in = fmin(t_in, (L - delta - ok) / dk);
      if (dk < 0.0) t_in = fmin(t_in, (-(L - delta) - ok) / dk);
    }
    n_in = lower_index(ts, p.n, t_in * (1.0 - 1e-12));
    const double Ax = q * (o.x + 2.0) - 0.5, Ay = q * (o.y + 2.0) - 0.5, Az = q * (o.z + 2.0) - 0.5;
    const double Bx = q * d.x, By = q * d.y, Bz = q * d.z;
    const double amax = fmax(fabs(Ax), fmax(fabs(Ay), fabs(Az))), bmax = fmax(fabs(Bx), fmax(fabs(By), fabs(Bz)));
    const double E0 = 2.0 * u * (amax + res) + 1e-9, E1 = 2.0 * 2.01 * u * bmax;
    cin = SegC{(float)Ax, (float)Ay, (float)Az, (float)Bx, (float)By, (float)Bz, 1.f, 0.f,
               (float)(0.5 - E0), (float)(-E1)};
  }
  if (!p.contraction) return;
  // the final pyramid: axis a with the strictly largest |d_a|, b and c the other two
  const double adx = fabs(d.x), ady = fabs(d.y), adz = fabs(d.z);
  const int a = (adx >= ady && adx >= adz) ? 0 : (ady >= adz ? 1 : 2);
  const int b = a == 0 ? 1 : 0, c = a == 2 ? 1 : 2;
  const double pq = sel3(a, adx, ady, adz), oa = sel3(a, o.x, o.y, o.z), da = sel3(a, d.x, d.y, d.z);
  const double ob = sel3(b, o.x, o.y, o.z), db = sel3(b, d.x, d.y, d.z);
  const double oc = sel3(c, o.x, o.y, o.z), dc = sel3(c, d.x, d.y, d.z);
  if (!(pq - fabs(db) >= 1e-6) || !(pq - fabs(dc) >= 1e-6)) return;  // near-tie: no certain final axis
  const double s = da > 0.0 ? 1.0 : -1.0, pc = s * oa;
  // m = pc + pq t >= 1 + delta, and |x_a| - |x_b| >= delta for both signs of x_b (and of x_c)
  double t_pyr = (1.0 + delta - pc) / pq;
  t_pyr = fmax(t_pyr, (delta - pc + ob) / (pq - db));
  t_pyr = fmax(t_pyr, (delta - pc - ob) / (pq + db));
  t_pyr = fmax(t_pyr, (delta - pc + oc) / (pq - dc));
  t_pyr = fmax(t_pyr, (delta - pc - oc) / (pq + dc));
  i_pyr = lower_index(ts, p.n, t_pyr * (1.0 + 1e-12) + 1e-12);
  const double Aa = q * (2.0 + 2.0 * s) - 0.5, Ba = -q * s;
  const double Ab = q * (2.0 + db / pq) - 0.5, Bb = q * (ob - db * oa / da);
  const double Ac = q * (2.0 + dc / pq) - 0.5, Bc = q * (oc - dc * oa / da);
  // (a, b, c) back to (x, y, z)
  const double Ax = a == 0 ? Aa : (b == 0 ? Ab : Ac), Bx = a == 0 ? Ba : (b == 0 ? Bb : Bc);
  const double Ay = a == 1 ? Aa : (b == 1 ? Ab : Ac), By = a == 1 ? Ba : (b == 1 ? Bb : Bc);
  const double Az = a == 2 ? Aa : (b == 2 ? Ab : Ac), Bz = a == 2 ? Ba : (b == 2 ? Bb : Bc);
  const double amax = fmax(fabs(Aa), fmax(fabs(Ab), fabs(Ac))), bmax = fmax(fabs(Ba), fmax(fabs(Bb), fabs(Bc)));
  const double eps_w = 2.0 * (u * (3.0 + 3.0 * fabs(oa)) + 2.0 * u);
  const double E0 = 2.0 * u * (amax + res) + 1e-9, E1 = 2.0 * bmax * (u + eps_w);
  cpy = SegC{(float)Ax, (float)Ay, (float)Az, (float)Bx, (float)By, (float)Bz, (float)pq, (float)pc,
             (float)(0.5 - E0), (float)(-E1)};
}

#ifndef LUMI_MARCH_SEG_CTAS
#define LUMI_MARCH_SEG_CTAS 7
#endif
__global__ void __launch_bounds__(128, LUMI_MARCH_SEG_CTAS) k_march_seg(RenderParams p) {
  __shared__ double s_ts[kMaxSamples];
  __shared__ __align__(16) float s_tf[kMaxSamples + 32];
  __shared__ double s_dir[4][32][3];        // per lane: exact direction (undecided re-tests)
  __shared__ uint16_t s_queue[4][32 * 32];  // per warp: undecided (lane, bit) of one word
  __shared__ uint32_t s_add[4][32];         // per lane: bits confirmed by the re-test
  for (int i = threadIdx.x; i < p.n + 32; i += blockDim.x) {
    if (i < p.n) s_ts[i] = p.ts[i];
    s_tf[i] = i < p.n ? (float)p.ts[i] : 0.f;
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
  SegC cin{}, cpy{};
  int n_in = 0, i_pyr = p.n;
  if (valid) seg_setup(p, s_ts, o, d, cin, cpy, n_in, i_pyr);
  const uint32_t r = (uint32_t)p.occ_res;
  // the occupancy bytes off the biased index (p.occ_bias = kRintBits (r^2 + r + 1) mod 2^32)
  // (held in a per-thread register pair -- the lane term is zero -- so every candidate's
  // address is one IMAD.WIDE.U32 instead of a uniform-operand IADD3 pair)
#ifdef LUMI_MARCH_BITS
  const uint64_t occ_adj = reinterpret_cast<uint64_t>(p.occ_bits) - (uint64_t)(p.occ_bias >> 5) * 4u +
                           (uint64_t)(p.zero & (uint32_t)lane);
#else
  const uint64_t occ_adj = reinterpret_cast<uint64_t>(p.occ) - (uint64_t)p.occ_bias +
                           (uint64_t)(p.zero & (uint32_t)lane);
#endif
  int count = 0;
  for (int w0 = 0; w0 < p.mask_words; ++w0) {
    const int base = w0 * 32, hi = min(32, p.n - base);
    uint32_t bits = 0, unsure = 0;
    if (valid) {
      const int in_hi = min(max(n_in - base, 0), hi), py_lo = min(max(i_pyr - base, 0), hi);
      const uint32_t all = hi == 32 ? 0xffffffffu : ((1u << hi) - 1u);
      const float* tw = s_tf + base;
      // each segment's pass over the word (skipped when no lane has a candidate in it); a
      // candidate in neither segment, or undecided in its own, takes the general test
      const unsigned act = __activemask();
      const uint32_t r_in = bits_range(0, in_hi), r_py = bits_range(py_lo, hi);
      // candidates of neither segment
      unsure = all & ~r_in & ~r_py;
      if (__all_sync(act, r_in == 0xffffffffu)) {
        seg_word<false, false>(cin, tw, r_in, occ_adj, r, bits, unsure);
      } else if (__all_sync(act, r_py == 0xffffffffu)) {
        seg_word<true, false>(cpy, tw, r_py, occ_adj, r, bits, unsure);
      } else {
        if (__any_sync(act, r_in != 0u)) seg_word<false, true>(cin, tw, r_in, occ_adj, r, bits, unsure);
        if (__any_sync(act, r_py != 0u)) seg_word<true, true>(cpy, tw, r_py, occ_adj, r, bits, unsure);
      }
      // the rest through the general certified test (lane-local; rare on the segments)
      const uint32_t todo = unsure & all;
      unsure = 0;
      for (uint32_t m = todo; m; m &= m - 1u) {
        const int b = __ffs(m) - 1;
        const int rr = occupied_filtered(p, of, df, onorm, tw[b]);
        if (rr == 2) unsure |= 1u << b;  // still undecided: exact re-test below
        else bits |= (uint32_t)rr << b;
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
    const uint32_t out = bits;
    if (idx < p.total_rays) p.kept_mask[(size_t)w0 * p.total_rays + idx] = out;
  }
  if (idx < p.total_rays) p.kept_count[idx] = (uint16_t)count;
  add_work_stats(p, 0, 0, valid ? (unsigned long long)p.n : 0ull, 0);
}

}  // namespace march
}  // namespace lumi_dev

using namespace lumi_dev;

// The segment pass addresses the occupancy bytes off a biased index (k_march_seg); the bias
// plus every voxel index must stay below 2^32 (true for res 128 and most others).
static bool march_seg_supported(int res) {
  const uint64_t r = (uint64_t)res;
  const uint64_t bias = (uint64_t)march::kRintBits * (r * r + r + 1) % (1ull << 32);
  return bias + r * r * r <= (1ull << 32);
}
uint32_t march_occ_bias(int res) {
  const uint32_t r = (uint32_t)res;
  return march::kRintBits * (r * r + r + 1u);
}

// The exact march pass (k_march_mask) over p.total_rays tile-ordered ray ids
// (p.tile_w x p.tile_h tiles) into p.kept_mask / p.kept_count.
cudaError_t launch_march_mask(const RenderParams& p, cudaStream_t s) {
  // LUMI_MARCH_EXACT=1: the double-precision pass; LUMI_MARCH_CERT=1: the certified contraction candidate by candidate (A/B and tests;
  // default: the segment pass)
  static const bool exact = std::getenv("LUMI_MARCH_EXACT") != nullptr;
  static const bool cert = std::getenv("LUMI_MARCH_CERT") != nullptr;
  const unsigned blocks = (unsigned)((p.total_rays + 127) / 128);
  if (exact)
    march::k_march_mask<<<blocks, 128, 0, s>>>(p);
  else if (cert || !march_seg_supported(p.occ_res))
    march::k_march_mask_fast<<<blocks, 128, 0, s>>>(p);
  else
    march::k_march_seg<<<blocks, 128, 0, s>>>(p);
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

