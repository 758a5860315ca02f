// mlp_simt.cuh -- the density/colour MLPs on CUDA cores (fp32 FMA), one sample per thread.
#pragma once
#include "field.cuh"

namespace lumi_dev {

// One dense layer on one sample: y = W x + b (row-major W [OUT x IN]), fp32 FMA.
template <int OUT, int IN, bool RELU>
__device__ __forceinline__ void dense(const float* __restrict__ W, const float* __restrict__ b,
                                      const float* x, float* y) {
#pragma unroll 4
  for (int r = 0; r < OUT; ++r) {
    const float4* w4 = reinterpret_cast<const float4*>(W + r * IN);
    float a0 = __ldg(b + r), a1 = 0.f, a2 = 0.f, a3 = 0.f;
#pragma unroll
    for (int c = 0; c < IN / 4; ++c) {
      const float4 w = __ldg(w4 + c);
      a0 = fmaf(w.x, x[4 * c + 0], a0);
      a1 = fmaf(w.y, x[4 * c + 1], a1);
      a2 = fmaf(w.z, x[4 * c + 2], a2);
      a3 = fmaf(w.w, x[4 * c + 3], a3);
    }
    float v = (a0 + a1) + (a2 + a3);
    y[r] = RELU ? fmaxf(v, 0.f) : v;
  }
}

// RadianceField::forward_chunk for one sample (field.h:106-137).
// Density head only (field.h:114-120, with_color = false).
__device__ __forceinline__ float density_mlp(const MlpDev& m, const float* feat) {
  float h[kHidden], dout[1 + kBottleneck];
  const float* dp = m.dparams;
  dense<kHidden, kFeat, true>(dp, dp + kHidden * kFeat, feat, h);
  dp += kHidden * kFeat + kHidden;
  dense<1 + kBottleneck, kHidden, false>(dp, dp + (1 + kBottleneck) * kHidden, h, dout);
  return trunc_exp(dout[0]);
}

__device__ __forceinline__ void field_mlp(const MlpDev& m, const float* feat, const float* sh,
                                          float& sigma, float* rgb) {
  float h[kHidden], h2[kHidden], dout[1 + kBottleneck];
  const float* dp = m.dparams;
  dense<kHidden, kFeat, true>(dp, dp + kHidden * kFeat, feat, h);
  dp += kHidden * kFeat + kHidden;
  dense<1 + kBottleneck, kHidden, false>(dp, dp + (1 + kBottleneck) * kHidden, h, dout);
  sigma = trunc_exp(dout[0]);
  float cin[kBottleneck + 16];
#pragma unroll
  for (int i = 0; i < kBottleneck; ++i) cin[i] = dout[1 + i];
#pragma unroll
  for (int i = 0; i < 16; ++i) cin[kBottleneck + i] = sh[i];
  const float* cp = m.cparams;
  dense<kHidden, kBottleneck + 16, true>(cp, cp + kHidden * (kBottleneck + 16), cin, h);
  cp += kHidden * (kBottleneck + 16) + kHidden;
  dense<kHidden, kHidden, true>(cp, cp + kHidden * kHidden, h, h2);
  cp += kHidden * kHidden + kHidden;
  float raw[3];
  dense<3, kHidden, false>(cp, cp + 3 * kHidden, h2, raw);
#pragma unroll
  for (int k = 0; k < 3; ++k) rgb[k] = m.color_space == 0 ? sigmoid(raw[k]) : trunc_exp(raw[k]);
}

}  // namespace lumi_dev
