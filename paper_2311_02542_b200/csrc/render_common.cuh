// render_common.cuh -- kernel parameter block and shared per-ray epilogue.
#pragma once
#include <cstdint>

#include "field.cuh"
#include "geometry.cuh"

namespace lumi_dev {

constexpr int kMaxSamples = 1024;

struct RenderParams {
  CamDev cam;
  GridDev grid;
  MlpDev mlp;
  const uint8_t* occ;  // occ_res^3 bytes
  const uint32_t* occ_bits;  // the same grid as a bitfield: voxel i is bit i & 31 of word i >> 5
  int occ_res;
  uint32_t occ_bias;   // march_occ_bias(occ_res): the segment march pass's biased voxel index
  uint32_t zero;       // always 0 (a value the compiler cannot prove uniform: keeps per-thread
                       // copies of uniform 64-bit bases in registers)
  const double* ts;    // host-computed exponential distances (renderer.h:135-141)
  double ratio;        // host-computed pow(t_far/t_near, 1/(n-1)) (renderer.h:142)
  const float2* tdf;   // [n] host-computed {(float)t_i, (float)delta_i} (packet kernel compositing)
  int n;               // samples_per_ray
  int lod_enabled;
  double lod_bias;
  double t_cut;
  double bg[3];
  int contraction;
  int debug_flags;  // profiling ablations only (LUMI_DEBUG_SKIP): 1 = no gather, 2 = no MLP
  int chunk;
  int row_begin, row_end;
  // target (LumiFrameTarget)
  float* rgb;
  float* depth;
  float* opacity;
  int32_t* counts;
  int64_t* row_evals;
  int64_t* row_cycles;  // optional: per camera row, SM cycles of the packets covering it
  uint8_t* srgb8;
  unsigned long long* work_stats;  // [evals, active level-samples, candidates, rays]
  double exposure_gain;  // 2^bias
  int tw, th, row_offset;
  // persistent scheduling
  unsigned int* work_counter;
  int tile_w, tile_h, tiles_x, tiles_total;
  // occupancy-kept candidates per ray id (tile-major ids), from the march pass:
  // kept_mask[word * total_rays + id], kept_count[id]
  uint32_t* kept_mask;
  uint16_t* kept_count;
  // optional, written by the march pass for the packet renderer: fp32 direction of each ray id
  // and of its right neighbour (x + 1.5), SoA [6][total_rays], so a warp starting a packet
  // loads its rays instead of running the double-precision ray generation on its critical path
  float* ray_dirs;
  int mask_words;
  long long total_rays;
};

// 32x32 bit-matrix transpose across a warp (lane = row, bit = column in; lane = column, bit =
// row out): five butterfly stages swapping the off-diagonal blocks.  All 32 lanes must call it.
__device__ __forceinline__ uint32_t warp_transpose32(uint32_t x) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) {
    const uint32_t m = s == 16 ? 0x0000FFFFu : s == 8 ? 0x00FF00FFu : s == 4 ? 0x0F0F0F0Fu
                     : s == 2 ? 0x33333333u : 0x55555555u;
    const uint32_t y = __shfl_xor_sync(0xffffffffu, x, s);
    x = (lane & s) ? ((x & ~m) | ((y >> s) & m)) : ((x & m) | ((y << s) & ~m));
  }
  return x;
}

// color.cpp:17-44 constants (scene-linear 1.0 = 100 cd/m^2)
__device__ __forceinline__ double pq_decode_dev(double v) {
  const double m1 = 1305.0 / 8192.0, m2 = 2523.0 / 32.0, c1 = 107.0 / 128.0,
               c2 = 2413.0 / 128.0, c3 = 2392.0 / 128.0;
  const double p = pow(v, 1.0 / m2);
  double num = p - c1;
  if (num < 0.0) num = 0.0;
  const double den = c2 - c3 * p;
  return pow(num / den, 1.0 / m1) / (100.0 / 10000.0);
}

__device__ __forceinline__ double srgb_oetf_dev(double v) {
  v = clamp01(v);
  return v <= 0.0031308 ? 12.92 * v : 1.055 * pow(v, 1.0 / 2.4) - 0.055;
}

// Display epilogue: PQ -> scene linear (pq_to_srgb_float, trainer.cpp:175-182) scaled by
// 2^bias and mapped to sRGB8 as tonemap_srgb does (color.cpp:104-115).
__device__ __forceinline__ uint8_t display_srgb8(double v, int color_space, double gain) {
  const double lin = color_space == 0 ? pq_decode_dev(clamp01(v)) : (v > 0.0 ? v : 0.0);
  const double s = srgb_oetf_dev(clamp01(lin * gain));
  return (uint8_t)llround(s * 255.0);
}

struct RayResult {
  double px, py, pz, depth, opacity;
  int evals, contributing;
};

// Final per-ray bookkeeping (renderer.h:233-236) and output stores.
__device__ __forceinline__ void store_ray(const RenderParams& p, int x, int y, RayResult r,
                                          double trans) {
  r.px = dadd(r.px, dmul(trans, p.bg[0]));
  r.py = dadd(r.py, dmul(trans, p.bg[1]));
  r.pz = dadd(r.pz, dmul(trans, p.bg[2]));
  const double depth = r.depth / dadd(r.opacity, 1e-10);
  const size_t plane = (size_t)p.tw * p.th;
  const size_t pix = (size_t)(p.row_offset + y) * p.tw + x;
  p.rgb[pix] = __double2float_rn(r.px);
  p.rgb[plane + pix] = __double2float_rn(r.py);
  p.rgb[2 * plane + pix] = __double2float_rn(r.pz);
  if (p.depth) p.depth[pix] = __double2float_rn(depth);
  if (p.opacity) p.opacity[pix] = __double2float_rn(r.opacity);
  if (p.counts) {
    p.counts[2 * pix] = r.evals;
    p.counts[2 * pix + 1] = r.contributing;
  }
  if (p.srgb8) {
    p.srgb8[3 * pix + 0] = display_srgb8(r.px, p.mlp.color_space, p.exposure_gain);
    p.srgb8[3 * pix + 1] = display_srgb8(r.py, p.mlp.color_space, p.exposure_gain);
    p.srgb8[3 * pix + 2] = display_srgb8(r.pz, p.mlp.color_space, p.exposure_gain);
  }
  if (p.row_evals) atomicAdd((unsigned long long*)&p.row_evals[y], (unsigned long long)r.evals);
}

// RayMarchRecord::evals (renderer.h:168, 225-230): evaluated samples come in whole chunks;
// after a cut at `contributing`, the partially used chunk still counts in full unless it
// is the final one.
__device__ __forceinline__ int chunk_evals(bool terminated, int contributing, int kept_total_seen,
                                           int chunk) {
  if (!terminated) return kept_total_seen;
  const int lim = ((contributing + chunk - 1) / chunk) * chunk;
  return min(kept_total_seen, lim);
}

// Warp-aggregated work counters (one atomic per warp per counter).
__device__ __forceinline__ void add_work_stats(const RenderParams& p, unsigned long long evals,
                                               unsigned long long level_samples,
                                               unsigned long long candidates,
                                               unsigned long long rays) {
  if (!p.work_stats) return;
  // per-thread values stay far below 2^27, so 32-bit warp sums cannot overflow
  const unsigned mask = __activemask();
  const unsigned e = __reduce_add_sync(mask, (unsigned)evals);
  const unsigned l = __reduce_add_sync(mask, (unsigned)level_samples);
  const unsigned c = __reduce_add_sync(mask, (unsigned)candidates);
  const unsigned r = __reduce_add_sync(mask, (unsigned)rays);
  if ((threadIdx.x & 31) == (__ffs(mask) - 1)) {
    atomicAdd(p.work_stats + 0, (unsigned long long)e);
    atomicAdd(p.work_stats + 1, (unsigned long long)l);
    atomicAdd(p.work_stats + 2, (unsigned long long)c);
    atomicAdd(p.work_stats + 3, (unsigned long long)r);
  }
}

// The occupancy test of one candidate decided in fp32 with a certified error bound:
//
// x = o + d t in fp32 differs from the exact value by at most ex = 8 * 2^-24 * (|o| + t)
// (o, d, t rounded to fp32 plus one FMA rounding, 2x slack).  The contraction
// (camera.cpp:34-49) is 1-Lipschitz up to 2/max(1, m), so the contracted point is off by at
// most ec = 2 ex / max(1, m) + 2^-21 (reciprocal and product roundings), and the voxel
// coordinate g = (c + 2) * res / 4 by eg = res/4 * ec + res * 2^-23.  If every axis of g is
// further than 4 eg from an integer, floor(g) -- hence the voxel and its occupancy bit, and
// the domain test for the uncontracted mode -- equals the double computation's.  The
// contraction's max-axis choice is discontinuous at ties (|x_i| == |x_j| == m), so a second
// axis within 4 ex of the max is also undecided.  ~1e-3 of candidates are undecided; the
// warp re-tests them cooperatively in double (below), so a rare fallback never serialises
// a whole warp behind one lane.
// Returns 0 (empty), 1 (occupied) or 2 (undecided in fp32).
__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// The certified fp32 voxel of one candidate (see above): its voxel index (>= 0), -1 when it is
// certainly outside the grid's domain (free), -2 when fp32 cannot decide.  *m_out gets |x|_inf.
__device__ __forceinline__ int voxel_filtered(const RenderParams& p, float3 of, float3 df, float onorm,
                                              float tf, float* m_out = nullptr) {
  const float x = fmaf(df.x, tf, of.x), y = fmaf(df.y, tf, of.y), z = fmaf(df.z, tf, of.z);
  const float ax = fabsf(x), ay = fabsf(y), az = fabsf(z);
  const float m = fmaxf(ax, fmaxf(ay, az));
  if (m_out) *m_out = m;
  const float ex = 4.76837158e-07f * (onorm + tf);  // 8 * 2^-24 * (|o| + t)
  const bool contract = p.contraction != 0 && m > 1.f;
  const float inv = contract ? rcp_approx(m) : 1.f;  // ~1 ulp, inside the 2^-21 term
  const float mapped = 2.f - inv;
  // the reference maps the FIRST axis with |x_i| == m (camera.cpp:42-47)
  const bool isx = ax == m, isy = !isx && ay == m, isz = !isx && !isy;
  const float cx = contract && isx ? copysignf(mapped, x) : x * inv;
  const float cy = contract && isy ? copysignf(mapped, y) : y * inv;
  const float cz = contract && isz ? copysignf(mapped, z) : z * inv;
  const float m2 = isx ? fmaxf(ay, az) : (isy ? fmaxf(ax, az) : fmaxf(ax, ay));
  const float res = (float)p.occ_res, q = 0.25f * res;
  const float ec = 2.f * ex * inv + 4.76837158e-07f;
  const float eps = 4.f * (q * ec + res * 1.1920929e-07f);
  const float gx = fmaf(cx, q, 2.f * q), gy = fmaf(cy, q, 2.f * q), gz = fmaf(cz, q, 2.f * q);
  // Rounding by the 1.5 * 2^23 magic constant keeps the whole test on the FMA/ALU pipes
  // (no FRND/F2I on the narrow XU pipe): |g - rint(g)| is the distance to the nearest voxel
  // boundary, and rint(g - 1/2) = floor(g) for every certified g.
  constexpr float kMagic = 12582912.f;
  const float rx = __fsub_rn(__fadd_rn(gx, kMagic), kMagic), ry = __fsub_rn(__fadd_rn(gy, kMagic), kMagic),
              rz = __fsub_rn(__fadd_rn(gz, kMagic), kMagic);
  const float dmin = fminf(fabsf(gx - rx), fminf(fabsf(gy - ry), fabsf(gz - rz)));
  if (dmin <= eps || (contract && m - m2 <= 4.f * ex)) return -2;
  if (fminf(gx, fminf(gy, gz)) < 0.f || fmaxf(gx, fmaxf(gy, gz)) > res) return -1;
  const uint32_t r = (uint32_t)p.occ_res;  // res^3 < 2^32 (checked on the host)
  const uint32_t ix = (uint32_t)(__float_as_int(__fadd_rn(gx - 0.5f, kMagic)) - 0x4B400000),
                 iy = (uint32_t)(__float_as_int(__fadd_rn(gy - 0.5f, kMagic)) - 0x4B400000),
                 iz = (uint32_t)(__float_as_int(__fadd_rn(gz - 0.5f, kMagic)) - 0x4B400000);
  return (int)((iz * r + iy) * r + ix);
}

// Returns 0 (empty), 1 (occupied) or 2 (undecided in fp32).
__device__ __forceinline__ int occupied_filtered(const RenderParams& p, float3 of, float3 df,
                                                 float onorm, float tf) {
  const int vi = voxel_filtered(p, of, df, onorm, tf);
  if (vi == -2) return 2;
  return vi >= 0 && __ldg(p.occ + vi) != 0 ? 1 : 0;
}


// Fast path of the certified test for candidates strictly inside the unit cube, where the
// contraction is the identity: the voxel coordinate is one FMA in t per axis,
//   g = (o + d t + 2) q = G0 + G1 t,  G1 = fl(d_f q), G0 = fl(fl(o_f q) + 2q),  q = res / 4.
// Against the exact g (double o, d, t): |o_f - o| <= 2^-24 |o|, |d_f - d| <= 2^-24 |d|
// (|d| <= 1), |t_f - t| <= 2^-24 t; G1 and G0 add one rounding each and the FMA one more, so
// |g_f - g| <= 2^-24 (3 q t + 2 q |o|_inf + |G0| + |g_f|) <= 2^-24 q (3 t + 3 |o|_inf + 5)
// inside the cube (|G0|, |g| <= 3q + q|o|).  eps = E0 + E1 t takes 4x that.  The candidate is
// decided here only if every axis is more than eps inside (q, 3q) -- so the exact point is
// strictly inside too and contract() is the identity for both -- and more than eps from a
// voxel boundary; anything else returns -1 for the general test.
struct InsideMarch {
  float3 g0, g1;
  float e0, e1, qlo, qhi;
};

__device__ __forceinline__ InsideMarch inside_march_setup(const RenderParams& p, float3 of, float3 df) {
  const float q = 0.25f * (float)p.occ_res;
  InsideMarch m;
  m.g1 = make_float3(df.x * q, df.y * q, df.z * q);
  m.g0 = make_float3(of.x * q + 2.f * q, of.y * q + 2.f * q, of.z * q + 2.f * q);
  const float om = fmaxf(fabsf(of.x), fmaxf(fabsf(of.y), fabsf(of.z)));
  m.e0 = 2.384185791e-07f * q * (3.f * om + 5.f);  // 4 * 2^-24 * q * (3|o| + 5)
  m.e1 = 2.384185791e-07f * q * 3.f;
  m.qlo = q;
  m.qhi = 3.f * q;
  return m;
}

// voxel index (>= 0) when certified strictly inside the unit cube; -2: use voxel_filtered
__device__ __forceinline__ int voxel_inside(const RenderParams& p, const InsideMarch& m, float tf) {
  const float gx = fmaf(m.g1.x, tf, m.g0.x), gy = fmaf(m.g1.y, tf, m.g0.y), gz = fmaf(m.g1.z, tf, m.g0.z);
  const float eps = fmaf(m.e1, tf, m.e0);
  constexpr float kMagic = 12582912.f;  // 1.5 * 2^23: rint on the FMA pipe
  const float rx = __fsub_rn(__fadd_rn(gx, kMagic), kMagic), ry = __fsub_rn(__fadd_rn(gy, kMagic), kMagic),
              rz = __fsub_rn(__fadd_rn(gz, kMagic), kMagic);
  const float dmin = fminf(fabsf(gx - rx), fminf(fabsf(gy - ry), fabsf(gz - rz)));
  const float gmin = fminf(gx, fminf(gy, gz)), gmax = fmaxf(gx, fmaxf(gy, gz));
  if (!(dmin > eps && gmin - eps > m.qlo && gmax + eps < m.qhi)) return -2;
  const uint32_t r = (uint32_t)p.occ_res;
  const uint32_t ix = (uint32_t)(__float_as_int(__fadd_rn(gx - 0.5f, kMagic)) - 0x4B400000),
                 iy = (uint32_t)(__float_as_int(__fadd_rn(gy - 0.5f, kMagic)) - 0x4B400000),
                 iz = (uint32_t)(__float_as_int(__fadd_rn(gz - 0.5f, kMagic)) - 0x4B400000);
  return (int)((iz * r + iy) * r + ix);
}

// 0 / 1: decided (empty / occupied); -1: use occupied_filtered
__device__ __forceinline__ int occupied_inside(const RenderParams& p, const InsideMarch& m, float tf) {
  const int vi = voxel_inside(p, m, tf);
  return vi < 0 ? -1 : (__ldg(p.occ + vi) != 0 ? 1 : 0);
}

}  // namespace lumi_dev
