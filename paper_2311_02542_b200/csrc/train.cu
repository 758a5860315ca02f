// train.cu -- the training-side reverse of the rendering path on sm_100a.
//
// The reference trains ray by ray (proj/src/trainer.cpp:549-561): march_ray(record = true)
// (renderer.h:126-237) -> ray_loss (train_step.h:16-123) -> backward_ray (train_step.h:127-154)
// -> composite_backward_sigma (renderer.h:110-120) -> RadianceField::backward_chunk
// (field.h:141-179: Mlp::backward network.h:115-136, encode_backward grid.h:118-137), all
// accumulated into one FieldGradients (field.h:48-62).  On the GPU the batch is flattened
// into SAMPLE-major passes so every pass is wide:
//
//   k_train_count     thread per ray: occupancy-kept candidates (exact double march)
//   (scan)            per-ray sample offsets
//   k_train_samples   thread per ray: one record per kept sample (contracted position, t,
//                     delta, LOD weights, inner flag)
//   k_train_tiles<0>  the forward of every kept sample in 128-sample tiles (the backward's
//                     own forward, below): bit-exact fp32 encode + fp32 MLP -> sigma, colour
//   k_train_loss      thread per ray: front-to-back compositing with the early cut, the
//                     chunk-rounded evaluated count, ray_loss, composite_backward_sigma
//                     -> dL/dsigma and dL/dcolour per evaluated sample
//   (scan + compact)  the evaluated samples of every ray
//   k_train_tiles<1>  persistent, 128-sample tiles: recompute the activations into shared
//                     memory, back-propagate through the colour and density MLPs, weight
//                     gradients accumulated per CTA in shared memory (one owner thread per
//                     entry, register-blocked over the tile), hash-grid scatter-add with
//                     vector fp32 atomics (red.global.add.v2.f32)
//   k_train_reduce    deterministic sums of the per-ray loss terms and vignetting gradients
//
// Compiled with -fmad=false: double compositing/loss arithmetic and float expressions round
// like the reference's non-FMA translation units; the MLP uses explicit fmaf in the same
// four-chain order as the SIMT renderer (mlp_simt.cuh, the reference's AVX-512 order), and the
// forward pass and the backward's recomputation are the same code, so their activations (and
// ReLU masks) are bit-identical.
#include <cub/device/device_scan.cuh>
#include <cuda_runtime.h>

#include "kernels.h"
#include "mlp_simt.cuh"

namespace lumi_dev {
namespace tr {

constexpr int kTile = 128;              // samples per backward tile
#ifndef LUMI_TRAIN_SPLIT
#define LUMI_TRAIN_SPLIT 4
#endif
constexpr int kSplit = LUMI_TRAIN_SPLIT;  // threads per sample (they split rows / levels)
constexpr int kThreads = kTile * kSplit;
constexpr int kS = kTile + 4;           // activation row stride (floats): 16-B aligned rows
constexpr int kIn = kBottleneck + 16;   // colour-network input width
// activation rows in shared memory
constexpr int rFEAT = 0, rH = rFEAT + kFeat, rDOUT = rH + kHidden, rCIN = rDOUT + 1 + kBottleneck,
              rC1 = rCIN + kIn, rC2 = rC1 + kHidden, rCRAW = rC2 + kHidden, kRows = rCRAW + 3;
// parameter offsets (weights then bias per layer, network.h:144-151)
constexpr int oD1 = 0, oD2 = oD1 + kHidden * kFeat + kHidden,
              kDensityParams = oD2 + (1 + kBottleneck) * kHidden + 1 + kBottleneck;
constexpr int oC1 = 0, oC2 = oC1 + kHidden * kIn + kHidden, oC3 = oC2 + kHidden * kHidden + kHidden,
              kColorParams = oC3 + 3 * kHidden + 3;

constexpr int kDensityPad = (kDensityParams + 3) & ~3;  // colour weights start 16-B aligned
constexpr int kColorPad = (kColorParams + 3) & ~3;

struct Smem {
  float act[kRows * kS];
  float wts[kDensityPad + kColorPad];  // fp32 parameters, density then colour (network.h:144-151)
  float dW[kDensityParams + kColorParams];  // density then colour
  float dsig[kTile];
  float dcol[3][kTile];
  int sample[kTile];
};

__device__ __forceinline__ bool occupied(const TrainParams& p, d3 c) {
  const int64_t vi = voxel_index(c, p.occ_res);
  return vi >= 0 && __ldg(p.occ + vi) != 0;
}

__device__ __forceinline__ d3 ld3(const double* v) { return d3{v[0], v[1], v[2]}; }

// ---- march: counts and sample records (renderer.h:205-222) ---------------------------------
// One warp per (ray, 32-candidate word): each lane tests one candidate in the exact double
// geometry, the ballot is the word's kept mask.  A training batch has only ~10^4 rays, so a
// thread per ray would leave most SMs idle.
__device__ __forceinline__ uint32_t kept_word(const TrainParams& p, const LumiTrainRayDev& ray,
                                              const double* ts, int word, int lane) {
  const int i = word * 32 + lane;
  bool keep = false;
  if (i < p.n) keep = occupied(p, contract(ray_at(ld3(ray.origin), ld3(ray.dir), ts[i]), p.contraction));
  return __ballot_sync(0xffffffffu, keep);
}

__global__ void __launch_bounds__(128) k_train_count(TrainParams p, int words, uint32_t* masks, int* cnt) {
  const long long gw = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (gw >= (long long)p.nrays * words) return;
  const int r = (int)(gw / words), word = (int)(gw % words);
  const LumiTrainRayDev& ray = p.rays[r];
  const uint32_t m = kept_word(p, ray, p.cam_ts + (size_t)ray.camera * p.n, word, lane);
  if (lane == 0) {
    masks[gw] = m;
    if (m) atomicAdd(cnt + r, __popc(m));
  }
}

// one warp per (ray, word): the word's kept candidates get consecutive records after the
// popcounts of the ray's earlier words
__global__ void __launch_bounds__(128) k_train_samples(TrainParams p, int words, const uint32_t* masks,
                                                       const int* off, TrainSample* out) {
  const long long gw = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (gw >= (long long)p.nrays * words) return;
  const int r = (int)(gw / words), word = (int)(gw % words);
  const uint32_t m = masks[gw];
  if (!((m >> lane) & 1u)) return;
  int k = off[r] + __popc(m & ((1u << lane) - 1u));
  for (int w = 0; w < word; ++w) k += __popc(masks[(long long)r * words + w]);
  const LumiTrainRayDev& ray = p.rays[r];
  const double* ts = p.cam_ts + (size_t)ray.camera * p.n;
  const double ratio = p.cam_ratio[ray.camera];
  const d3 o = ld3(ray.origin), d = ld3(ray.dir), no = ld3(ray.norigin), nd = ld3(ray.ndir);
  const int i = word * 32 + lane;
  const double t = ts[i];
  const d3 c = contract(ray_at(o, d, t), p.contraction);
  TrainSample s;
  s.c[0] = c.x;
  s.c[1] = c.y;
  s.c[2] = c.z;
  s.t = t;
  s.delta = (i + 1 < p.n) ? dsub(ts[i + 1], t) : dmul(t, dsub(ratio, 1.0));
  LodW lw{p.grid.levels, 0.f, false};
  if (p.lod_enabled) {
    // contracted_footprint (camera.cpp:68-73) with the neighbour's own origin
    const d3 b = contract(ray_at(no, nd, t), p.contraction);
    const double rc = dmul(0.5, dnorm(d3{dsub(c.x, b.x), dsub(c.y, b.y), dsub(c.z, b.z)}));
    lw = lod_weights(lod_level(dmax(rc, 1e-12), p.grid.two_base, p.grid.log_scale, p.grid.levels),
                     p.lod_bias, p.grid.levels);
  }
  s.ray = r;
  s.lod_full = lw.full;
  s.lod_frac = lw.frac;
  s.floor_only = lw.floor_only ? 1 : 0;
  s.inner = dlinf(c) <= 1.0 ? 1 : 0;  // renderer.h:224
  out[k] = s;
}

__device__ __forceinline__ LodW lodw_of(const TrainSample& s) {
  return LodW{s.lod_full, s.lod_frac, s.floor_only != 0};
}

__device__ __forceinline__ d3 ray_dir_of(const TrainParams& p, int r) { return ld3(p.rays[r].dir); }

__device__ __forceinline__ double sgn(double x) { return x > 0 ? 1.0 : (x < 0 ? -1.0 : 0.0); }

// ---- per ray: compositing, ray_loss, composite_backward_sigma ---------------------------
// renderer.h:165-202 + 233-236, train_step.h:16-123, train_step.h:127-140, renderer.h:110-120
__global__ void __launch_bounds__(128) k_train_loss(TrainParams p, const int* off, const int* cnt,
                                                    const TrainSample* smp, const float* sig,
                                                    const float* col, double* wbuf, int* evals,
                                                    float* dsig, float* dcol, double* ray_terms) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= p.nrays) return;
  const LumiTrainRayDev& ray = p.rays[r];
  const int base = off[r], kept = cnt[r];
  double* A = wbuf;                        // alpha
  double* Tr = wbuf + (size_t)p.total;     // transmittance before the sample
  double* Wt = wbuf + 2 * (size_t)p.total; // weight
  double* G = wbuf + 3 * (size_t)p.total;  // dL/dw
  double trans = 1.0, px[3] = {0, 0, 0}, depth = 0, opac = 0;
  int contributing = 0;
  bool term = false;
  for (int i = 0; i < kept; ++i) {
    const int s = base + i;
    const double sigma = (double)sig[s];
    const double a = 1.0 - exp(-sigma * smp[s].delta);
    const double w = trans * a;
    A[s] = a;
    Tr[s] = trans;
    Wt[s] = w;
    for (int c = 0; c < 3; ++c) px[c] += w * (double)col[3 * s + c];
    depth += w * smp[s].t;
    opac += w;
    trans *= 1.0 - a;
    ++contributing;
    if (p.t_cut > 0 && trans < p.t_cut) {
      term = true;
      break;
    }
  }
  const int n = chunk_evals(term, contributing, kept, p.chunk);  // rec.t.size()
  for (int i = contributing; i < n; ++i) {                         // the cut chunk's tail
    A[base + i] = 0.0;
    Tr[base + i] = 0.0;
    Wt[base + i] = 0.0;
  }
  const double final_trans = trans;
  for (int c = 0; c < 3; ++c) px[c] += trans * p.bg[c];
  depth = depth / (opac + 1e-10);
  evals[r] = n;
  if (p.ray_evals) p.ray_evals[r] = n;
  if (p.ray_contrib) p.ray_contrib[r] = contributing;

  // ray_loss (train_step.h:16-123)
  const double inv_batch = p.inv_batch;
  const double v_raw = 1.0 - p.alpha_v[ray.camera] * ray.vignette_r;
  const double v = dmax(v_raw, 1e-3);
  double l_image = 0, l_depth = 0, l_dvar = 0, l_dist = 0;
  double dpix[3], dv_total = 0, d_alpha_v = 0;
  for (int c = 0; c < 3; ++c) {
    const double pred = v * px[c];
    const double diff = pred - (double)ray.gt[c];
    l_image += fabs(diff) / 3.0 * inv_batch;
    const double dpred = inv_batch * sgn(diff) / 3.0;
    dpix[c] = dpred * v;
    dv_total += dpred * px[c];
  }
  if (v_raw > 1e-3) d_alpha_v += dv_total * (-ray.vignette_r);
  for (int i = 0; i < n; ++i) {
    const int s = base + i;
    double gw = 0;
    for (int c = 0; c < 3; ++c) {
      gw += dpix[c] * (double)col[3 * s + c];
      dcol[3 * s + c] = (float)(dpix[c] * Wt[s]);  // backward_ray's cast (train_step.h:146-149)
    }
    G[s] = gw;
  }
  const double W = opac, D = depth, denom = W + 1e-10;
  double ddepth = 0;
  if (p.depth_active && p.lambda_depth > 0 && ray.gt_depth >= 0) {
    const double diff = D - ray.gt_depth;
    l_depth = p.lambda_depth * fabs(diff) * inv_batch;
    ddepth = p.lambda_depth * inv_batch * sgn(diff);
  }
  double dvar_dD = 0;
  if (p.lambda_dvar > 0) {
    double Wi = 0, S2 = 0;
    for (int i = 0; i < n; ++i) {
      const int s = base + i;
      if (!smp[s].inner) continue;
      const double tt = smp[s].t;
      Wi += Wt[s];
      S2 += Wt[s] * (tt - D) * (tt - D);
    }
    if (Wi > 1e-10) {
      const double V = S2 / Wi;
      l_dvar = p.lambda_dvar * V * inv_batch;
      for (int i = 0; i < n; ++i) {
        const int s = base + i;
        if (!smp[s].inner) continue;
        const double tt = smp[s].t;
        G[s] += p.lambda_dvar * inv_batch * ((tt - D) * (tt - D) - V) / Wi;
        dvar_dD += -2.0 * Wt[s] * (tt - D) / Wi;
      }
      dvar_dD *= p.lambda_dvar * inv_batch;
    }
  }
  if (p.lambda_dist > 0) {
    double Aa = 0, Bb = 0, val = 0;
    for (int i = 0; i < n; ++i) {
      const int s = base + i;
      const double tt = smp[s].t;
      val += Wt[s] * (tt * Aa - Bb);
      Aa += Wt[s];
      Bb += Wt[s] * tt;
    }
    val *= 2.0;
    l_dist = p.lambda_dist * val * inv_batch;
    double A_pre = 0, B_pre = 0;
    for (int i = 0; i < n; ++i) {
      const int s = base + i;
      const double tt = smp[s].t;
      const double A_suf = Aa - A_pre - Wt[s];
      const double B_suf = Bb - B_pre - Wt[s] * tt;
      const double d = 2.0 * (tt * A_pre - B_pre + B_suf - tt * A_suf);
      G[s] += p.lambda_dist * inv_batch * d;
      A_pre += Wt[s];
      B_pre += Wt[s] * tt;
    }
  }
  if (ddepth != 0 || dvar_dD != 0) {
    const double dD_total = ddepth + dvar_dD;
    for (int i = 0; i < n; ++i) G[base + i] += dD_total * (smp[base + i].t - D) / denom;
  }
  // composite_backward_sigma (renderer.h:110-120), background through final_trans
  double d_final_trans = 0;
  for (int c = 0; c < 3; ++c) d_final_trans += dpix[c] * p.bg[c];
  double suffix = d_final_trans * final_trans;
  for (int i = n - 1; i >= 0; --i) {
    const int s = base + i;
    const double d = smp[s].delta * ((1.0 - A[s]) * G[s] * Tr[s] - suffix);
    dsig[s] = (float)d;
    suffix += G[s] * Wt[s];
  }
  double* rt = ray_terms + 5 * (size_t)r;
  rt[0] = l_image;
  rt[1] = l_depth;
  rt[2] = l_dvar;
  rt[3] = l_dist;
  rt[4] = d_alpha_v;
}

__global__ void __launch_bounds__(128) k_train_compact(TrainParams p, const int* off, const int* aoff,
                                                       const int* evals, int* act) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= p.nrays) return;
  const int b = off[r], a = aoff[r], n = evals[r];
  for (int i = 0; i < n; ++i) act[a + i] = b + i;
}

// ---- backward over 128-sample tiles ------------------------------------------------------

// y[o][s] for the output blocks o = 4b .. 4b+3, b = h, h + kSplit, ... (the kSplit threads of sample s
// splits the rows): per output the same four-chain fmaf order as mlp_simt.cuh dense(), so
// activations are the same in both passes; four outputs share every activation load.
// W: the layer's weights [OUT x IN] then bias [OUT], in shared memory (16-B aligned rows).
template <int OUT, int IN, bool RELU>
__device__ __forceinline__ void fwd_layer(const float* W, const float* x, float* y, int s, int h) {
  const float* bias = W + OUT * IN;
  constexpr int NB = (OUT + 3) / 4;
#pragma unroll 1
  for (int b = h; b < NB; b += kSplit) {
    float a[4][4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      a[q][0] = (4 * b + q < OUT) ? bias[4 * b + q] : 0.f;
      a[q][1] = a[q][2] = a[q][3] = 0.f;
    }
#pragma unroll 4
    for (int c = 0; c < IN / 4; ++c) {
      const float x0 = x[(4 * c + 0) * kS + s], x1 = x[(4 * c + 1) * kS + s],
                  x2 = x[(4 * c + 2) * kS + s], x3 = x[(4 * c + 3) * kS + s];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (4 * b + q < OUT) {
          const float4 w = *reinterpret_cast<const float4*>(W + (4 * b + q) * IN + 4 * c);
          a[q][0] = fmaf(w.x, x0, a[q][0]);
          a[q][1] = fmaf(w.y, x1, a[q][1]);
          a[q][2] = fmaf(w.z, x2, a[q][2]);
          a[q][3] = fmaf(w.w, x3, a[q][3]);
        }
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (4 * b + q < OUT) {
        const float v = (a[q][0] + a[q][1]) + (a[q][2] + a[q][3]);
        y[(4 * b + q) * kS + s] = RELU ? fmaxf(v, 0.f) : v;
      }
    }
  }
}

// dx[i][s] = sum_o W[o][i] dy[o][s] (dense_backward_data, simd.h:53-64) for the input blocks
// i = 4b .. 4b+3 < NI, b = h, h + 2, ..., optionally masked by the ReLU of the layer below
// (relu_backward, simd.h:85-90: dy = 0 where y <= 0), written over x (each thread owns its
// sample's column).  One dy load and one 16-B weight load feed four FMAs.
template <int OUT, int IN, int NI, bool MASK>
__device__ __forceinline__ void bwd_data(const float* W, const float* dy, const float* x, float* dx,
                                         int s, int h) {
#pragma unroll 1
  for (int b = h; b < NI / 4; b += kSplit) {
    float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
#pragma unroll 8
    for (int o = 0; o < OUT; ++o) {
      const float d = dy[o * kS + s];
      const float4 w = *reinterpret_cast<const float4*>(W + o * IN + 4 * b);
      a0 = fmaf(w.x, d, a0);
      a1 = fmaf(w.y, d, a1);
      a2 = fmaf(w.z, d, a2);
      a3 = fmaf(w.w, d, a3);
    }
    float r[4] = {a0, a1, a2, a3};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int i = 4 * b + q;
      if (MASK && !(x[i * kS + s] > 0.f)) r[q] = 0.f;
      dx[i * kS + s] = r[q];
    }
  }
}

// dW[o][i] += sum_s dy[o][s] x[i][s], db[o] += sum_s dy[o][s] (dense_backward_weights,
// simd.h:66-83).  Thread t owns column i = t % IN of rows o = t / IN + j * (256 / IN): one
// 16-B load of x per 4 samples feeds all its rows (dy rows are warp-uniform broadcasts).
template <int OUT, int IN>
__device__ __forceinline__ void bwd_weights(float* dW, const float* dy, const float* x, int tid,
                                            int nvalid) {
  constexpr int G = kThreads / IN;            // row groups
  constexpr int J = (OUT + G - 1) / G;        // rows per thread
  const int i = tid % IN, o0 = tid / IN;
  float acc[J];
#pragma unroll
  for (int j = 0; j < J; ++j) acc[j] = 0.f;
  const int n4 = (nvalid + 3) >> 2;
#pragma unroll 1
  for (int q = 0; q < n4; ++q) {
    const float4 xv = *reinterpret_cast<const float4*>(x + i * kS + 4 * q);
#pragma unroll
    for (int j = 0; j < J; ++j) {
      const int o = o0 + j * G;
      if (o < OUT) {
        const float4 d = *reinterpret_cast<const float4*>(dy + o * kS + 4 * q);
        acc[j] = fmaf(d.x, xv.x, fmaf(d.y, xv.y, fmaf(d.z, xv.z, fmaf(d.w, xv.w, acc[j]))));
      }
    }
  }
#pragma unroll
  for (int j = 0; j < J; ++j) {
    const int o = o0 + j * G;
    if (o < OUT) dW[o * IN + i] += acc[j];
  }
  for (int o = tid; o < OUT; o += kThreads) {  // bias
    float b = 0.f;
    for (int q = 0; q < n4; ++q) {
      const float4 d = *reinterpret_cast<const float4*>(dy + o * kS + 4 * q);
      b += (d.x + d.y) + (d.z + d.w);
    }
    dW[OUT * IN + o] += b;
  }
}

// encode_backward (grid.h:118-137) of one level: the reference's corner weights (double
// product cast to float) times w_l, scattered with vector fp32 atomics.
__device__ __forceinline__ void scatter_level(const TrainParams& p, int l, double u, double v,
                                              double s, float wl, float g0, float g1) {
  const GridDev& g = p.grid;
  const int res = g.res[l];
  const double r = (double)res;
  const double pu = dmul(clamp01(u), r), pv = dmul(clamp01(v), r), ps = dmul(clamp01(s), r);
  const int iu = min(__double2int_rz(pu), res - 1), iv = min(__double2int_rz(pv), res - 1),
            is = min(__double2int_rz(ps), res - 1);
  const double fu = dsub(pu, (double)iu), fv = dsub(pv, (double)iv), fs = dsub(ps, (double)is);
  uint32_t idx[8];
  corner_indices((g.dense_mask >> l) & 1u, iu, iv, is, (uint32_t)res + 1u, g.hash_mask[l], idx);
  float2* base = reinterpret_cast<float2*>(p.g_grid) + g.offset2[l];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const double wu = (k & 1) ? fu : dsub(1.0, fu);
    const double wv = ((k >> 1) & 1) ? fv : dsub(1.0, fv);
    const double ws = ((k >> 2) & 1) ? fs : dsub(1.0, fs);
    const float coeff = __fmul_rn(__double2float_rn(dmul(dmul(wu, wv), ws)), wl);
    atomicAdd(base + idx[k], make_float2(__fmul_rn(coeff, g0), __fmul_rn(coeff, g1)));
  }
}

// BWD = false: the forward only, over every kept sample (act == nullptr), writing sigma and
// colour for the compositing pass -- the same arithmetic the backward recomputes.
template <bool BWD>
__global__ void __launch_bounds__(kThreads, 1) k_train_tiles(TrainParams p, const TrainSample* smp,
                                                             const int* act, int nact,
                                                             const float* dsig_g, const float* dcol_g,
                                                             float* sig_out, float* col_out) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  Smem& S = *reinterpret_cast<Smem*>(smem_raw);
  const int tid = threadIdx.x, s = tid & (kTile - 1), h = tid >> 7;
  float* X = S.act;
  float* dWd = S.dW;
  float* dWc = S.dW + kDensityParams;
  if (BWD)
    for (int e = tid; e < kDensityParams + kColorParams; e += kThreads) S.dW[e] = 0.f;
  for (int e = tid; e < kDensityParams; e += kThreads) S.wts[e] = __ldg(p.mlp.dparams + e);
  for (int e = tid; e < kColorParams; e += kThreads) S.wts[kDensityPad + e] = __ldg(p.mlp.cparams + e);
  const float* dp = S.wts;
  const float* cp = S.wts + kDensityPad;
  const int ntiles = (nact + kTile - 1) / kTile;

  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int nvalid = min(kTile, nact - tile * kTile);
    __syncthreads();  // previous tile's scatter reads FEAT; dW updates are owner-only
    // ---- 1. inputs: features (levels split over the sample's threads), SH and the output
    //      gradients (pair thread 1) ----
    {
      const int si = s < nvalid ? (BWD ? act[tile * kTile + s] : tile * kTile + s) : -1;
      if (h == 0) S.sample[s] = si;
      if (si >= 0) {
        const TrainSample q = smp[si];
        const LodW lw = lodw_of(q);
        const double u = dmul(dadd(q.c[0], 2.0), 0.25), v = dmul(dadd(q.c[1], 2.0), 0.25),
                     w = dmul(dadd(q.c[2], 2.0), 0.25);
        for (int l = h; l < kMaxLevels; l += kSplit) {  // encode (grid.h:90-114), bit-exact
          float2 f = make_float2(0.f, 0.f);
          if (l < p.grid.levels) {
            const float wl = lod_weight_at(lw, l);
            if (wl > 0.f) f = encode_level(p.grid, l, u, v, w, wl);
          }
          X[(rFEAT + 2 * l) * kS + s] = f.x;
          X[(rFEAT + 2 * l + 1) * kS + s] = f.y;
        }
      } else {
        for (int l = h; l < kMaxLevels; l += kSplit) {
          X[(rFEAT + 2 * l) * kS + s] = 0.f;
          X[(rFEAT + 2 * l + 1) * kS + s] = 0.f;
        }
      }
      if (h == 1) {
        float sh[16];
        float ds = 0.f, dc[3] = {0.f, 0.f, 0.f};
        if (si >= 0) {
          sh_encode(ray_dir_of(p, smp[si].ray), sh);
          if (BWD) {
            ds = dsig_g[si];
            dc[0] = dcol_g[3 * si + 0];
            dc[1] = dcol_g[3 * si + 1];
            dc[2] = dcol_g[3 * si + 2];
          }
        } else {
#pragma unroll
          for (int k = 0; k < 16; ++k) sh[k] = 0.f;
        }
#pragma unroll
        for (int k = 0; k < 16; ++k) X[(rCIN + kBottleneck + k) * kS + s] = sh[k];
        S.dsig[s] = ds;
        S.dcol[0][s] = dc[0];
        S.dcol[1][s] = dc[1];
        S.dcol[2][s] = dc[2];
      }
    }
    __syncthreads();
    // ---- 2. forward, activations kept (field.h:106-137) ---------------------------------
    fwd_layer<kHidden, kFeat, true>(dp + oD1, X + rFEAT * kS, X + rH * kS, s, h);
    __syncthreads();
    fwd_layer<1 + kBottleneck, kHidden, false>(dp + oD2, X + rH * kS, X + rDOUT * kS, s, h);
    __syncthreads();
    for (int b = h; b < kBottleneck; b += kSplit) X[(rCIN + b) * kS + s] = X[(rDOUT + 1 + b) * kS + s];
    __syncthreads();
    fwd_layer<kHidden, kIn, true>(cp + oC1, X + rCIN * kS, X + rC1 * kS, s, h);
    __syncthreads();
    fwd_layer<kHidden, kHidden, true>(cp + oC2, X + rC1 * kS, X + rC2 * kS, s, h);
    __syncthreads();
    fwd_layer<3, kHidden, false>(cp + oC3, X + rC2 * kS, X + rCRAW * kS, s, h);
    __syncthreads();
    if (!BWD) {  // sigma = trunc_exp(raw0), colour head (field.h:116-118, 131-136)
      if (h == 0 && s < nvalid) {
        const int si = tile * kTile + s;
        sig_out[si] = trunc_exp(X[rDOUT * kS + s]);
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          const float raw = X[(rCRAW + k) * kS + s];
          col_out[3 * si + k] = p.mlp.color_space == 0 ? sigmoid(raw) : trunc_exp(raw);
        }
      }
      continue;
    }
    // ---- 3. backward (field.h:141-179) -----------------------------------------------------
    if (h == 0) {  // colour head: dL/draw (field.h:148-160); padded rows get zero gradients
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const float raw = X[(rCRAW + k) * kS + s];
        float g;
        if (p.mlp.color_space == 0) {
          const float c = sigmoid(raw);
          g = c * (1.f - c);
        } else {
          g = expf(fminf(raw, 10.f));  // trunc_exp_grad (network.h:48-52)
        }
        X[(rCRAW + k) * kS + s] = S.dcol[k][s] * g;
      }
    }
    __syncthreads();
    bwd_weights<3, kHidden>(dWc + oC3, X + rCRAW * kS, X + rC2 * kS, tid, nvalid);
    __syncthreads();
    bwd_data<3, kHidden, kHidden, true>(cp + oC3, X + rCRAW * kS, X + rC2 * kS, X + rC2 * kS, s, h);
    __syncthreads();
    bwd_weights<kHidden, kHidden>(dWc + oC2, X + rC2 * kS, X + rC1 * kS, tid, nvalid);
    __syncthreads();
    bwd_data<kHidden, kHidden, kHidden, true>(cp + oC2, X + rC2 * kS, X + rC1 * kS, X + rC1 * kS, s, h);
    __syncthreads();
    bwd_weights<kHidden, kIn>(dWc + oC1, X + rC1 * kS, X + rCIN * kS, tid, nvalid);
    __syncthreads();
    // colour-input gradient of the bottleneck rows -> density output rows 1..16
    bwd_data<kHidden, kIn, kBottleneck, false>(cp + oC1, X + rC1 * kS, nullptr, X + (rDOUT + 1) * kS, s, h);
    if (h == 1) {  // row 0: dsigma * trunc_exp_grad(sigma_raw) (field.h:165-166)
      const float raw = X[rDOUT * kS + s];
      X[rDOUT * kS + s] = S.dsig[s] * expf(fminf(raw, 10.f));
    }
    __syncthreads();
    bwd_weights<1 + kBottleneck, kHidden>(dWd + oD2, X + rDOUT * kS, X + rH * kS, tid, nvalid);
    __syncthreads();
    bwd_data<1 + kBottleneck, kHidden, kHidden, true>(dp + oD2, X + rDOUT * kS, X + rH * kS, X + rH * kS, s, h);
    __syncthreads();
    bwd_weights<kHidden, kFeat>(dWd + oD1, X + rH * kS, X + rFEAT * kS, tid, nvalid);
    __syncthreads();
    bwd_data<kHidden, kFeat, kFeat, false>(dp + oD1, X + rH * kS, nullptr, X + rFEAT * kS, s, h);
    __syncthreads();
    // ---- 4. hash-grid scatter-add (grid.h:118-137), levels split over the sample's threads ----
    if (s < nvalid) {
      const TrainSample q = smp[S.sample[s]];
      const LodW lw = lodw_of(q);
      const double u = dmul(dadd(q.c[0], 2.0), 0.25), v = dmul(dadd(q.c[1], 2.0), 0.25),
                   w = dmul(dadd(q.c[2], 2.0), 0.25);
      for (int l = h; l < p.grid.levels; l += kSplit) {
        const float wl = lod_weight_at(lw, l);
        if (!(wl > 0.f)) continue;
        scatter_level(p, l, u, v, w, wl, X[(rFEAT + 2 * l) * kS + s], X[(rFEAT + 2 * l + 1) * kS + s]);
      }
    }
  }
  if (BWD) {
    __syncthreads();
    for (int e = tid; e < kDensityParams; e += kThreads) atomicAdd(p.g_density + e, dWd[e]);
    for (int e = tid; e < kColorParams; e += kThreads) atomicAdd(p.g_color + e, dWc[e]);
  }
}

// Deterministic sums over rays: block 0 the loss terms (trainer.cpp:556-559), block 1 + c the
// vignetting gradient of camera c (trainer.cpp:562).  Fixed-shape tree reductions.
__device__ __forceinline__ double block_sum(double v, double* red) {
  red[threadIdx.x] = v;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  const double r = red[0];
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(256) k_train_reduce(TrainParams p, const double* ray_terms) {
  __shared__ double red[256];
  if (blockIdx.x == 0) {
    double sums[4];
    for (int k = 0; k < 4; ++k) {
      double acc = 0;
      for (int r = threadIdx.x; r < p.nrays; r += 256) acc += ray_terms[5 * (size_t)r + k];
      sums[k] = block_sum(acc, red);
    }
    if (threadIdx.x == 0) {
      for (int k = 0; k < 4; ++k) p.loss[1 + k] += sums[k];
      p.loss[0] = ((p.loss[1] + p.loss[2]) + p.loss[3]) + p.loss[4];
    }
    return;
  }
  const int c = blockIdx.x - 1;
  double acc = 0;
  for (int r = threadIdx.x; r < p.nrays; r += 256)
    if (p.rays[r].camera == c) acc += ray_terms[5 * (size_t)r + 4];
  const double tot = block_sum(acc, red);
  if (threadIdx.x == 0) p.alpha_grad[c] += tot;
}

}  // namespace tr
}  // namespace lumi_dev

using namespace lumi_dev;

size_t train_backward_smem_bytes() { return sizeof(tr::Smem); }

namespace {
template <typename T>
struct Scratch {
  T* p = nullptr;
  cudaStream_t s;
  explicit Scratch(cudaStream_t st) : s(st) {}
  cudaError_t alloc(size_t n) { return cudaMallocAsync(&p, n * sizeof(T), s); }
  ~Scratch() {
    if (p) cudaFreeAsync(p, s);
  }
};
}  // namespace

// The whole reverse pass for one batch of rays (see the file comment).  Synchronises once
// on `s` to learn the number of kept samples (the size of every per-sample buffer).
cudaError_t launch_train_backward(TrainParams p, cudaStream_t s, int num_sms, long long* kept_total,
                                  long long* eval_total) {
  cudaError_t e;
  if (p.nrays <= 0) return cudaSuccess;
  const unsigned rb = (unsigned)((p.nrays + 127) / 128);
  Scratch<int> cnt(s), off(s), evals(s), aoff(s);
  Scratch<uint32_t> masks(s);
  const int words = (p.n + 31) / 32;
  const long long march_threads = (long long)p.nrays * words * 32;
  const unsigned mb = (unsigned)((march_threads + 127) / 128);
  Scratch<uint8_t> tmp(s);
  if ((e = cnt.alloc(p.nrays + 1)) || (e = off.alloc(p.nrays + 1)) || (e = evals.alloc(p.nrays + 1)) ||
      (e = aoff.alloc(p.nrays + 1)) || (e = masks.alloc((size_t)p.nrays * words)))
    return e;
  size_t tmp_bytes = 0;
  if ((e = cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, cnt.p, off.p, p.nrays + 1, s))) return e;
  if ((e = tmp.alloc(tmp_bytes))) return e;
  if ((e = cudaMemsetAsync(cnt.p, 0, sizeof(int) * (p.nrays + 1), s))) return e;
  tr::k_train_count<<<mb, 128, 0, s>>>(p, words, masks.p, cnt.p);
  if ((e = cub::DeviceScan::ExclusiveSum(tmp.p, tmp_bytes, cnt.p, off.p, p.nrays + 1, s))) return e;
  int total = 0;
  if ((e = cudaMemcpyAsync(&total, off.p + p.nrays, sizeof(int), cudaMemcpyDeviceToHost, s)) ||
      (e = cudaStreamSynchronize(s)))
    return e;
  if (kept_total) *kept_total = total;
  p.total = total;
  Scratch<TrainSample> smp(s);
  Scratch<float> sig(s), col(s), dsig(s), dcol(s);
  Scratch<double> wbuf(s), terms(s);
  Scratch<int> act(s);
  const size_t T = (size_t)std::max(total, 1);
  if ((e = smp.alloc(T)) || (e = sig.alloc(T)) || (e = col.alloc(3 * T)) || (e = dsig.alloc(T)) ||
      (e = dcol.alloc(3 * T)) || (e = wbuf.alloc(4 * T)) || (e = terms.alloc(5 * (size_t)p.nrays)) ||
      (e = act.alloc(T)))
    return e;
  tr::k_train_samples<<<mb, 128, 0, s>>>(p, words, masks.p, off.p, smp.p);
  static PerDeviceInit once;
  const size_t smem = sizeof(tr::Smem);
  int ok = 0;
  if ((e = once.get([&](int* v) {
         *v = 1;
         cudaError_t x = cudaFuncSetAttribute(tr::k_train_tiles<true>,
                                              cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
         if (x == cudaSuccess)
           x = cudaFuncSetAttribute(tr::k_train_tiles<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem);
         return x;
       }, &ok)))
    return e;
  if (total > 0) {
    const int ftiles = (total + tr::kTile - 1) / tr::kTile;
    tr::k_train_tiles<false><<<std::min(ftiles, num_sms), tr::kThreads, smem, s>>>(
        p, smp.p, nullptr, total, nullptr, nullptr, sig.p, col.p);
  }
  if ((e = cudaMemsetAsync(evals.p + p.nrays, 0, sizeof(int), s))) return e;
  tr::k_train_loss<<<rb, 128, 0, s>>>(p, off.p, cnt.p, smp.p, sig.p, col.p, wbuf.p, evals.p, dsig.p,
                                      dcol.p, terms.p);
  if ((e = cub::DeviceScan::ExclusiveSum(tmp.p, tmp_bytes, evals.p, aoff.p, p.nrays + 1, s))) return e;
  int nact = 0;
  if ((e = cudaMemcpyAsync(&nact, aoff.p + p.nrays, sizeof(int), cudaMemcpyDeviceToHost, s)) ||
      (e = cudaStreamSynchronize(s)))
    return e;
  if (eval_total) *eval_total = nact;
  tr::k_train_compact<<<rb, 128, 0, s>>>(p, off.p, aoff.p, evals.p, act.p);
  if (nact > 0) {
    const int tiles = (nact + tr::kTile - 1) / tr::kTile;
    tr::k_train_tiles<true><<<std::min(tiles, num_sms), tr::kThreads, smem, s>>>(
        p, smp.p, act.p, nact, dsig.p, dcol.p, nullptr, nullptr);
  }
  tr::k_train_reduce<<<1 + p.ncams, 256, 0, s>>>(p, terms.p);
  return cudaGetLastError();
}

