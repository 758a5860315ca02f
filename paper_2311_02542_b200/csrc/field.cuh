// field.cuh -- device-side radiance field: mip hash-grid gather and the fp32 MLPs.
#pragma once
#include <cuda_fp16.h>

#include <cstdint>

#include "geometry.cuh"

namespace lumi_dev {

constexpr int kMaxLevels = 16;
constexpr int kHidden = 64;
constexpr int kBottleneck = 16;
constexpr int kFeat = 2 * kMaxLevels;

// MultiResHashGrid layout (grid.h:58-74) as seen by the kernels.
struct GridDev {
  const float2* table;     // float pairs; level l starts at pair offset2[l]
  const __half2* table16;  // the same table in fp16 pairs (the production gather, render_ws.cu)
  int levels;
  int res[kMaxLevels];
  uint32_t hash_mask[kMaxLevels];  // entries-1 for hashed levels
  uint32_t dense_mask;             // bit l set: level l is dense
  uint64_t offset2[kMaxLevels];    // in float2 units
  double two_base;                 // 2.0 * base_resolution (grid.cpp:10)
  double log_scale;                // std::log(per_level_scale), host libm
};

// spatial_hash (grid.h:50-52)
__device__ __forceinline__ uint32_t spatial_hash(uint32_t x, uint32_t y, uint32_t z,
                                                 uint32_t mask) {
  return (x * 1u ^ y * 2654435761u ^ z * 805459861u) & mask;
}

__device__ __forceinline__ double clamp01(double v) { return v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v); }

// One level of MultiResHashGrid::encode/corners (grid.h:96-113, 144-167), bit-exact:
// double corner weights cast to float, float accumulation in corner order, times w_l.
__device__ __forceinline__ float2 encode_level(const GridDev& g, int l, double u, double v,
                                               double s, float wl) {
  const int res = g.res[l];
  const double r = (double)res;
  const double pu = dmul(clamp01(u), r), pv = dmul(clamp01(v), r), ps = dmul(clamp01(s), r);
  const int iu = min(__double2int_rz(pu), res - 1), iv = min(__double2int_rz(pv), res - 1),
            is = min(__double2int_rz(ps), res - 1);
  const double fu = dsub(pu, (double)iu), fv = dsub(pv, (double)iv), fs = dsub(ps, (double)is);
  const uint32_t verts = (uint32_t)res + 1u;
  const bool dense = (g.dense_mask >> l) & 1u;
  const float2* base = g.table + g.offset2[l];
  float2 e[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const uint32_t x = (uint32_t)iu + (k & 1), y = (uint32_t)iv + ((k >> 1) & 1),
                   z = (uint32_t)is + ((k >> 2) & 1);
    const uint32_t idx = dense ? (z * verts + y) * verts + x : spatial_hash(x, y, z, g.hash_mask[l]);
    e[k] = __ldg(base + idx);
  }
  float a0 = 0.f, a1 = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const double wu = (k & 1) ? fu : dsub(1.0, fu);
    const double wv = ((k >> 1) & 1) ? fv : dsub(1.0, fv);
    const double ws = ((k >> 2) & 1) ? fs : dsub(1.0, fs);
    const float tri = __double2float_rn(dmul(dmul(wu, wv), ws));
    a0 = __fadd_rn(a0, __fmul_rn(tri, e[k].x));
    a1 = __fadd_rn(a1, __fmul_rn(tri, e[k].y));
  }
  return make_float2(__fmul_rn(a0, wl), __fmul_rn(a1, wl));
}

// The 8 corner indices of one cell (grid.h:154-161) with the per-axis products hoisted:
// dense  (z*V + y)*V + x            = base + {0,1,V,V+1,V^2,...}   (all uint32, wraps as ref)
// hashed x ^ y*2654435761 ^ z*805459861, & mask                     (grid.h:50-52)
__device__ __forceinline__ void corner_indices(bool dense, int iu, int iv, int is, uint32_t verts,
                                               uint32_t mask, uint32_t* idx) {
  const uint32_t x0 = (uint32_t)iu, y0 = (uint32_t)iv, z0 = (uint32_t)is;
  if (dense) {
    const uint32_t vv = verts * verts;
    const uint32_t b = (z0 * verts + y0) * verts + x0;
    idx[0] = b;
    idx[1] = b + 1u;
    idx[2] = b + verts;
    idx[3] = b + verts + 1u;
    idx[4] = b + vv;
    idx[5] = b + vv + 1u;
    idx[6] = b + vv + verts;
    idx[7] = b + vv + verts + 1u;
  } else {
    // (x ^ hy ^ hz) & mask == (x & mask) ^ (hy & mask) ^ (hz & mask): mask the six terms once,
    // then one three-input LOP3 per corner
    const uint32_t hy0 = y0 * 2654435761u, hy1 = hy0 + 2654435761u;
    const uint32_t hz0 = z0 * 805459861u, hz1 = hz0 + 805459861u;
    const uint32_t xa = x0 & mask, xb = (x0 + 1u) & mask, ya = hy0 & mask, yb = hy1 & mask,
                   za = hz0 & mask, zb = hz1 & mask;
    idx[0] = xa ^ ya ^ za;
    idx[1] = xb ^ ya ^ za;
    idx[2] = xa ^ yb ^ za;
    idx[3] = xb ^ yb ^ za;
    idx[4] = xa ^ ya ^ zb;
    idx[5] = xb ^ ya ^ zb;
    idx[6] = xa ^ yb ^ zb;
    idx[7] = xb ^ yb ^ zb;
  }
}

// d = a * b + c with a, b fp16 and c, d fp32 (sm_100 FHFMA)
__device__ __forceinline__ float fma_f32_f16(__half a, __half b, float c) {
  float d;
  asm("fma.rn.f32.f16 %0, %1, %2, %3;"
      : "=f"(d)
      : "h"(__half_as_ushort(a)), "h"(__half_as_ushort(b)), "f"(c));
  return d;
}

// Full encode of one contracted point into 2*levels features (zero for masked levels,
// which touch no memory -- grid.h:98-101).
__device__ __forceinline__ void encode(const GridDev& g, d3 c, const LodW& lw, float* feat) {
  const double u = dmul(dadd(c.x, 2.0), 0.25), v = dmul(dadd(c.y, 2.0), 0.25),
               s = dmul(dadd(c.z, 2.0), 0.25);
#pragma unroll
  for (int l = 0; l < kMaxLevels; ++l) {
    float2 f = make_float2(0.f, 0.f);
    if (l < g.levels) {
      const float wl = lod_weight_at(lw, l);
      if (wl > 0.f) f = encode_level(g, l, u, v, s, wl);
    }
    feat[2 * l] = f.x;
    feat[2 * l + 1] = f.y;
  }
}

// fp32 MLP parameters (flattened weights-then-bias per layer, network.h:144-151),
// row-major [out x in] weights.
struct MlpDev {
  const float* dparams;
  const float* cparams;
  const float* fused;  // [65 x 80] + [65]: density L2 folded into colour L1 (lumi_api.cu)
  int color_space;
  // the packed-renderer's fp16 UMMA weight tiles (W1 | fused | C2 | C3), the exact shared-memory
  // image k_render_ws stages with one TMA bulk copy per CTA; built by launch_pack_weight_tiles
  const void* wtiles;
};

}  // namespace lumi_dev
