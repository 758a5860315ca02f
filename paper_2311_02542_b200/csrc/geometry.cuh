// geometry.cuh -- exact-double ray geometry for sm_100a.
//
// Every operation replays the reference's double-precision op order with explicit
// round-to-nearest intrinsics, so nvcc cannot contract a*b+c into an FMA.  That makes the
// occupancy test -- and therefore the set of marched sample indices -- bit-identical to
// the reference CPU renderer (whose non-SIMD translation units are built without FMA,
// proj/CMakeLists.txt:39-47).  Division and sqrt are IEEE correctly rounded by default
// (no -use_fast_math, no -prec-div=false) in double precision.
#pragma once
#include <cstdint>

namespace lumi_dev {

struct d3 {
  double x, y, z;
};

__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmax(double a, double b) { return a < b ? b : a; }  // std::max
__device__ __forceinline__ double dmin(double a, double b) { return b < a ? b : a; }  // std::min

// Vec3::norm (common.h:36-37): sqrt((x*x + y*y) + z*z)
__device__ __forceinline__ double dnorm(d3 v) {
  return sqrt(dadd(dadd(dmul(v.x, v.x), dmul(v.y, v.y)), dmul(v.z, v.z)));
}

// Vec3::linf (common.h:38)
__device__ __forceinline__ double dlinf(d3 v) {
  return dmax(fabs(v.x), dmax(fabs(v.y), fabs(v.z)));
}

struct CamDev {
  double rot[9];
  double origin[3];
  double fx, fy, cx, cy;
  int32_t width, height;
  double t_near, t_far;
};

// generate_ray_unchecked (camera.cpp:10-17) with Pose::rotate (common.h:49-53) and
// Vec3::normalized (common.h:39).
__device__ __forceinline__ d3 ray_dir(const CamDev& c, double px, double py) {
  const double vx = dsub(px, c.cx) / c.fx, vy = dsub(py, c.cy) / c.fy, vz = 1.0;
  d3 d;
  d.x = dadd(dadd(dmul(c.rot[0], vx), dmul(c.rot[1], vy)), dmul(c.rot[2], vz));
  d.y = dadd(dadd(dmul(c.rot[3], vx), dmul(c.rot[4], vy)), dmul(c.rot[5], vz));
  d.z = dadd(dadd(dmul(c.rot[6], vx), dmul(c.rot[7], vy)), dmul(c.rot[8], vz));
  const double n = dnorm(d);
  return d3{d.x / n, d.y / n, d.z / n};
}

// Ray::at (camera.h:29): origin + dir * t
__device__ __forceinline__ d3 ray_at(d3 o, d3 d, double t) {
  return d3{dadd(o.x, dmul(d.x, t)), dadd(o.y, dmul(d.y, t)), dadd(o.z, dmul(d.z, t))};
}

// contract (camera.cpp:34-49), L-inf cubic.  The reference's require(finite) cannot
// fire for finite cameras; non-finite input maps to an out-of-domain point here.
__device__ __forceinline__ d3 contract(d3 x, int mode) {
  if (mode == 0) return x;
  const double m = dlinf(x);
  if (!(m <= 1.0)) {
    d3 out{x.x / m, x.y / m, x.z / m};
    const double mapped = dsub(2.0, 1.0 / m);
    if (fabs(x.x) == m)
      out.x = copysign(mapped, x.x);
    else if (fabs(x.y) == m)
      out.y = copysign(mapped, x.y);
    else
      out.z = copysign(mapped, x.z);
    return out;
  }
  return x;
}

// OccupancyGrid::voxel_index (occupancy.cpp:22-29); -1 outside the domain.
__device__ __forceinline__ int64_t voxel_index(d3 c, int res) {
  const double u = dmul(dadd(c.x, 2.0), 0.25), v = dmul(dadd(c.y, 2.0), 0.25),
               w = dmul(dadd(c.z, 2.0), 0.25);
  if (u < 0 || u > 1 || v < 0 || v > 1 || w < 0 || w > 1) return -1;
  const double r = (double)res;
  int ix = __double2int_rz(dmul(u, r)), iy = __double2int_rz(dmul(v, r)),
      iz = __double2int_rz(dmul(w, r));
  ix = min(ix, res - 1);
  iy = min(iy, res - 1);
  iz = min(iz, res - 1);
  return ((int64_t)iz * res + iy) * res + ix;
}

// contracted_footprint (camera.cpp:68-73)
__device__ __forceinline__ double contracted_footprint(d3 o, d3 d, d3 nd, double t, int mode) {
  const d3 a = contract(ray_at(o, d, t), mode);
  const d3 b = contract(ray_at(o, nd, t), mode);
  return dmul(0.5, dnorm(d3{dsub(a.x, b.x), dsub(a.y, b.y), dsub(a.z, b.z)}));
}

// contract (camera.cpp:34-49) in fp32 with one reciprocal: the producers' sample geometry
__device__ __forceinline__ float3 contract_f(float3 x, int mode) {
  if (mode == 0) return x;
  const float m = fmaxf(fabsf(x.x), fmaxf(fabsf(x.y), fabsf(x.z)));
  if (!(m <= 1.f)) {
    const float inv = __frcp_rn(m);
    float3 out = make_float3(x.x * inv, x.y * inv, x.z * inv);
    const float mapped = 2.f - inv;
    if (fabsf(x.x) == m)
      out.x = copysignf(mapped, x.x);
    else if (fabsf(x.y) == m)
      out.y = copysignf(mapped, x.y);
    else
      out.z = copysignf(mapped, x.z);
    return out;
  }
  return x;
}

// lod_level (grid.cpp:8-13); log_scale = std::log(per_level_scale) precomputed on the host
// with the same libm the reference uses.
__device__ __forceinline__ double lod_level(double r, double two_base, double log_scale,
                                            int levels) {
  const double l = -log(dmul(two_base, r)) / log_scale;
  return dmin(l, (double)(levels - 1));
}

// lod_weights (grid.cpp:15-37), written as a per-level function of (fl, frac).
struct LodW {
  int full;     // levels [0, full) weight 1 (or level 0 = 1e-4 when floor_only)
  float frac;   // weight of level `full` when > 0
  bool floor_only;
};

__device__ __forceinline__ LodW lod_weights(double l_star, double bias, int levels) {
  const double eff = dadd(l_star, bias);
  LodW w;
  if (eff >= levels - 1) {
    w.full = levels;
    w.frac = 0.f;
    w.floor_only = false;
  } else if (eff < 0.0) {
    w.full = 0;
    w.frac = 0.f;
    w.floor_only = true;
  } else {
    const double fl = floor(eff);
    const double fr = dsub(eff, fl);
    w.full = (int)fl + 1;
    w.frac = fr > 0.0 ? __double2float_rn(fr) : 0.f;
    w.floor_only = false;
  }
  return w;
}

// Number of levels with w_l > 0 (grid.h:41-46).
__device__ __forceinline__ int active_levels(const LodW& w, int levels) {
  if (w.floor_only) return 1;
  return min(levels, w.full + (w.frac > 0.f ? 1 : 0));
}

// lod_weights (grid.cpp:15-37) on an fp32 effective level.
__device__ __forceinline__ LodW lod_weights_f(float eff, int levels) {
  LodW w;
  if (eff >= (float)(levels - 1)) {
    w.full = levels;
    w.frac = 0.f;
    w.floor_only = false;
  } else if (eff < 0.f) {
    w.full = 0;
    w.frac = 0.f;
    w.floor_only = true;
  } else {
    const float fl = floorf(eff);
    w.full = (int)fl + 1;
    w.frac = eff - fl;
    w.floor_only = false;
  }
  return w;
}

__device__ __forceinline__ float lod_weight_at(const LodW& w, int l) {
  if (w.floor_only) return l == 0 ? 1e-4f : 0.f;
  if (l < w.full) return 1.f;
  if (l == w.full) return w.frac;
  return 0.f;
}

// sh_encode_deg3 (network.h:17-37) for T = float, reference op order.
__device__ __forceinline__ void sh_encode(d3 d, float* out) {
  const float x = __double2float_rn(d.x), y = __double2float_rn(d.y), z = __double2float_rn(d.z);
  const float xx = __fmul_rn(x, x), yy = __fmul_rn(y, y), zz = __fmul_rn(z, z);
  out[0] = (float)0.28209479177387814;
  out[1] = __fmul_rn((float)-0.48860251190291987, y);
  out[2] = __fmul_rn((float)0.48860251190291987, z);
  out[3] = __fmul_rn((float)-0.48860251190291987, x);
  out[4] = __fmul_rn(__fmul_rn((float)1.0925484305920792, x), y);
  out[5] = __fmul_rn(__fmul_rn((float)-1.0925484305920792, y), z);
  out[6] = __fmul_rn((float)0.31539156525252005, __fsub_rn(__fmul_rn(3.f, zz), 1.f));
  out[7] = __fmul_rn(__fmul_rn((float)-1.0925484305920792, x), z);
  out[8] = __fmul_rn((float)0.5462742152960396, __fsub_rn(xx, yy));
  out[9] = __fmul_rn(__fmul_rn((float)-0.5900435899266435, y), __fsub_rn(__fmul_rn(3.f, xx), yy));
  out[10] = __fmul_rn(__fmul_rn(__fmul_rn((float)2.890611442640554, x), y), z);
  out[11] = __fmul_rn(__fmul_rn((float)-0.4570457994644658, y), __fsub_rn(__fmul_rn(5.f, zz), 1.f));
  out[12] = __fmul_rn(__fmul_rn((float)0.3731763325901154, z), __fsub_rn(__fmul_rn(5.f, zz), 3.f));
  out[13] = __fmul_rn(__fmul_rn((float)-0.4570457994644658, x), __fsub_rn(__fmul_rn(5.f, zz), 1.f));
  out[14] = __fmul_rn(__fmul_rn((float)1.445305721320277, z), __fsub_rn(xx, yy));
  out[15] = __fmul_rn(__fmul_rn((float)-0.5900435899266435, x), __fsub_rn(xx, __fmul_rn(3.f, yy)));
}

// trunc_exp / sigmoid (network.h:41-57), float.
__device__ __forceinline__ float trunc_exp(float x) {
  if (x <= 10.f) return expf(x);
  return __fmul_rn(expf(10.f), __fadd_rn(1.f, __fsub_rn(x, 10.f)));
}
__device__ __forceinline__ float sigmoid(float x) { return 1.f / __fadd_rn(1.f, expf(-x)); }

}  // namespace lumi_dev
