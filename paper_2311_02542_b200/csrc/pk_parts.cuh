// pk_parts.cuh -- pieces of the packet renderer (render_ws.cu) and the isolated MLP / gather
// benchmarks (mlp_batch.cu): the
// TMEM / A-tile layout, the tcgen05 layer issue and epilogue helpers, the hash-grid gather of
// one (sample, level) pair, and the per-ray compositing state.
#pragma once
#include <cuda_fp16.h>

#include "render_common.cuh"
#include "tc_ptx.cuh"

namespace lumi_dev {
namespace pk {

constexpr int kThreads = 128;  // UMMA M: 4 warps x 32 rows
constexpr int kWarps = kThreads / 32;
constexpr int kPW = 8, kPH = 4;  // packet: 8 x 4 pixels = one warp of rays
// TMEM columns: [0,80) fp32 accumulators (N <= 80), [80,112) hidden activations h (fp16 pairs,
// the TS-form A operand), [112,120) the SH encoding (fused layer only), [120,128) the
// constant [1 0 ... 0] bias block
constexpr uint32_t kTmemCols = 128;
constexpr uint32_t kAcol = 80;
constexpr uint32_t kShCol = 112;
constexpr uint32_t kOnesCol = 120;
constexpr int kKb = 16;              // every layer's bias is one extra K = 16 step
constexpr int kAch = (32 + kKb) / 8; // 8-element K chunks of the layer-1 A tile


__device__ __forceinline__ uint32_t core_off(int row, int chunk, int kchunks) {
  return (uint32_t)((row >> 3) * (kchunks * 128) + chunk * 128 + (row & 7) * 16);
}

// The layer-1 A tile is chunk-major (all 128 rows of an 8-element K chunk contiguous; core
// matrices LBO = 2048 B along K, SBO = 128 B along M), so row r, chunk c starts at c*2048 + r*16.
constexpr uint32_t kALbo = 2048;
__device__ __forceinline__ uint32_t a_off(int row, int chunk) { return (uint32_t)(chunk * kALbo + row * 16); }

__device__ __forceinline__ uint32_t h2u(__half2 h) { return *reinterpret_cast<uint32_t*>(&h); }

__device__ __forceinline__ void st16(uint8_t* base, uint32_t off, uint4 v) {
  *reinterpret_cast<uint4*>(base + off) = v;
}

__device__ __forceinline__ uint4 pack8(const float* v) {
  return make_uint4(h2u(__floats2half2_rn(v[0], v[1])), h2u(__floats2half2_rn(v[2], v[3])),
                    h2u(__floats2half2_rn(v[4], v[5])), h2u(__floats2half2_rn(v[6], v[7])));
}

// weights [n_real x K] fp32 row-major + bias [n_real] (network.h:64, 144-151) -> fp16 UMMA
// tile [n_pad][K + 16] with the bias in column K
static __device__ void load_weight_tile(uint8_t* dst, const float* __restrict__ W, int n_real, int n_pad,
                                 int K) {
  const float* bias = W + (size_t)n_real * K;
  const int kch = (K + kKb) / 8;
  for (int it = threadIdx.x; it < n_pad * kch; it += blockDim.x) {
    const int n = it / kch, j = it % kch;
    float v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int k = 8 * j + q;
      v[q] = n >= n_real ? 0.f : k < K ? __ldg(W + (size_t)n * K + k) : k == K ? __ldg(bias + n) : 0.f;
    }
    st16(dst, core_off(n, j, kch), pack8(v));
  }
}

// layer 1 (SS form): A = features + ones block in shared memory (chunk-major, a_off), B the
// row-group-major weight tile
template <int N, int K>
__device__ __forceinline__ void issue_layer(const uint8_t* A, const uint8_t* B, uint32_t d_tmem) {
  constexpr uint32_t idesc = ptx::idesc_f16_f32<128, N>();
  constexpr uint32_t sbo = ((K + kKb) / 8) * 128;
  const uint32_t a = ptx::smem_addr(A), b = ptx::smem_addr(B);
#pragma unroll
  for (int kk = 0; kk < (K + kKb) / 16; ++kk)
    ptx::mma_f16(d_tmem, ptx::make_smem_desc(a + kk * 2 * kALbo, kALbo, 128),
                 ptx::make_smem_desc(b + kk * 256, 128, sbo), idesc, kk > 0 ? 1u : 0u);
}

// hidden layers (TS form): A = activations in TMEM columns [a_tmem, a_tmem + K/2), then the
// TMEM ones block against the bias column of B
template <int N, int K>
__device__ __forceinline__ void issue_layer_ts(uint32_t a_tmem, uint32_t ones_tmem, const uint8_t* B,
                                               uint32_t d_tmem) {
  constexpr uint32_t idesc = ptx::idesc_f16_f32<128, N>();
  constexpr uint32_t sbo = ((K + kKb) / 8) * 128;
  const uint32_t b = ptx::smem_addr(B);
#pragma unroll
  for (int kk = 0; kk < K / 16; ++kk)  // 16 fp16 of K = 8 TMEM columns per step
    ptx::mma_f16_ts(d_tmem, a_tmem + kk * 8, ptx::make_smem_desc(b + kk * 256, 128, sbo), idesc,
                    kk > 0 ? 1u : 0u);
  ptx::mma_f16_ts(d_tmem, ones_tmem, ptx::make_smem_desc(b + (K / 16) * 256, 128, sbo), idesc, 1u);
}

// two fp32 -> packed fp16 (lo, hi), optionally clamped at 0, in one F2FP
__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
  uint32_t d;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(hi), "f"(lo));
  return d;
}
__device__ __forceinline__ uint32_t pack2_relu(float lo, float hi) {
  uint32_t d;
  asm("cvt.rn.relu.f16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(hi), "f"(lo));
  return d;
}

// hidden-layer epilogue into TMEM: D row (64 fp32, bias included), ReLU, fp16 pairs -> the A
// columns of this thread's lane for the next layer
__device__ __forceinline__ void relu64_to_tmem(uint32_t t_lane, uint32_t a_lane) {
#pragma unroll
  for (int h = 0; h < 4; ++h) {
    float v[16];
    ptx::tmem_ld16(t_lane + 16 * h, v);
    ptx::tmem_ld_wait();
    uint32_t w[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) w[j] = pack2_relu(v[2 * j], v[2 * j + 1]);
    ptx::tmem_st8(a_lane + 8 * h, w);
  }
  ptx::tmem_st_wait();
}

// ---- the production gather ------------------------------------------------------------------
// MultiResHashGrid::corners + encode (grid.h:96-113, 144-167) restated for the fp16 table:
//  * cell and fractions of TWO levels at once in packed f32x2: p = u r rounded to nearest (half
//    the fraction error of rounding down), b = p + 2^23 rounded down holds floor(p) in its low
//    mantissa bits (b = 0x4B000000 + floor(p) as an integer), f = p - (b - 2^23).  No clamp to
//    res - 1: when p rounds up onto an integer k (at most r, as u < 1), the cell is k with
//    fraction 0, which interpolates to the value of cell k - 1 at fraction 1 (the shared face's
//    corners are the same entries; the k + 1 corners get weight exactly 0 -- hashed indices are
//    masked into the level, a dense one at most one entry past it, inside the padded table);
//  * corner indices straight off those biased bits: the bias is folded into per-level addends
//    (dense: idx = x + y V + z V^2; hashed: (x ^ y P1 ^ z P2) & mask, where the mask < 2^24
//    strips the bias bits of x), dense corners x+1 as a +4-byte load offset;
//  * the trilinear value as seven packed-fp16 lerps, the fractions of two levels packed per
//    axis (operand swizzles select the halves);
//  * software-pipelined over level pairs (gather_row, below).
struct LevelTab {
  float res[kMaxLevels];       // resolution as float
  uint32_t mask[kMaxLevels];   // hashed: table entries - 1; dense: 0
  uint32_t m1[kMaxLevels];     // y multiplier: dense V = res + 1, hashed 2654435761
  uint32_t m2[kMaxLevels];     // z multiplier: dense V^2, hashed 805459861
  uint32_t k1[kMaxLevels];     // y addend folding the bias (and, dense, x's bias)
  uint32_t k2[kMaxLevels];     // z addend folding the bias
  unsigned long long base[kMaxLevels];  // the level's first fp16 entry pair (byte address)
  uint32_t dense_mask;         // bit l: level l is dense
};

constexpr uint32_t kFloorBias = 0x4B000000u;  // bits of 2^23

// fill one CTA's table (any thread count; call before a barrier)
__device__ __forceinline__ void level_tab_init(LevelTab& t, const GridDev& g, int tid, int nthreads) {
  for (int l = tid; l < kMaxLevels; l += nthreads) {
    const bool live = l < g.levels;
    const uint32_t res = live ? (uint32_t)g.res[l] : 1u;
    const bool dense = live && ((g.dense_mask >> l) & 1u);
    const uint32_t V = res + 1u;
    t.res[l] = (float)res;
    t.mask[l] = dense ? 0u : (live ? g.hash_mask[l] : 0u);
    t.m1[l] = dense ? V : 2654435761u;
    t.m2[l] = dense ? V * V : 805459861u;
    // dense: y_b V + k1 = y V - C (y_b = C + y, so k1 = -C (V + 1)): x's bias cancels in the sum
    t.k1[l] = dense ? 0u - kFloorBias * (V + 1u) : 0u - kFloorBias * 2654435761u;
    t.k2[l] = dense ? 0u - kFloorBias * (V * V) : 0u - kFloorBias * 805459861u;
    t.base[l] = reinterpret_cast<unsigned long long>(g.table16 + (live ? g.offset2[l] : 0));
  }
  if (tid == 0) t.dense_mask = g.dense_mask & ((1u << g.levels) - 1u);
}

__device__ __forceinline__ uint64_t f2pk(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float2 f2upk(uint64_t r) {
  float2 v;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(v.x), "=f"(v.y) : "l"(r));
  return v;
}

// floor bits and fractions of coordinate a at the two resolutions r2 (levels l, l + 1)
__device__ __forceinline__ void cell2(float a, uint64_t r2, uint32_t& b0, uint32_t& b1, float& f0, float& f1) {
  uint64_t p, b, fl, f;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(p) : "l"(f2pk(a, a)), "l"(r2));
  asm("add.rm.f32x2 %0, %1, %2;" : "=l"(b) : "l"(p), "l"(f2pk(8388608.f, 8388608.f)));
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(fl) : "l"(b), "l"(f2pk(-8388608.f, -8388608.f)));
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(f) : "l"(p), "l"(fl));
  const float2 bb = f2upk(b), ff = f2upk(f);
  b0 = __float_as_uint(bb.x);
  b1 = __float_as_uint(bb.y);
  f0 = ff.x;
  f1 = ff.y;
}


// (a ^ b) & c in one LOP3 (immediate 0x28: (0xF0 ^ 0xCC) & 0xAA)
__device__ __forceinline__ uint32_t xor_and(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, 0x28;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

// the 8 corner entries of one level (biased cell bits xb, yb, zb)
__device__ __forceinline__ void corners8(const LevelTab& t, int l, uint32_t xb, uint32_t yb, uint32_t zb,
                                         __half2* e) {
  const uint32_t m1 = t.m1[l], m2 = t.m2[l], mask = t.mask[l];
  const uint32_t hy0 = yb * m1 + t.k1[l], hy1 = hy0 + m1;
  const uint32_t hz0 = zb * m2 + t.k2[l], hz1 = hz0 + m2;
  const __half2* base = reinterpret_cast<const __half2*>(t.base[l]);
  if (mask == 0u) {  // dense: x + y V + z V^2, x + 1 one entry on
    const uint32_t i0 = xb + hy0 + hz0, i2 = xb + hy1 + hz0, i4 = xb + hy0 + hz1, i6 = xb + hy1 + hz1;
    const __half2 *p0 = base + i0, *p2 = base + i2, *p4 = base + i4, *p6 = base + i6;
    e[0] = __ldg(p0);
    e[1] = __ldg(p0 + 1);
    e[2] = __ldg(p2);
    e[3] = __ldg(p2 + 1);
    e[4] = __ldg(p4);
    e[5] = __ldg(p4 + 1);
    e[6] = __ldg(p6);
    e[7] = __ldg(p6 + 1);
  } else {  // hashed (grid.h:50-52): (x ^ yz) & mask as ONE three-input LOP3 per corner
    const uint32_t xb1 = xb + 1u;
    const uint32_t yz00 = hy0 ^ hz0, yz10 = hy1 ^ hz0, yz01 = hy0 ^ hz1, yz11 = hy1 ^ hz1;
    e[0] = __ldg(base + xor_and(xb, yz00, mask));
    e[1] = __ldg(base + xor_and(xb1, yz00, mask));
    e[2] = __ldg(base + xor_and(xb, yz10, mask));
    e[3] = __ldg(base + xor_and(xb1, yz10, mask));
    e[4] = __ldg(base + xor_and(xb, yz01, mask));
    e[5] = __ldg(base + xor_and(xb1, yz01, mask));
    e[6] = __ldg(base + xor_and(xb, yz11, mask));
    e[7] = __ldg(base + xor_and(xb1, yz11, mask));
  }
}

// a hashed level's corners with the multipliers and bias addends as immediates (only the mask
// and the base come from the table)
__device__ __forceinline__ void corners8_hashed(const LevelTab& t, int l, uint32_t xb, uint32_t yb, uint32_t zb,
                                                __half2* e) {
  constexpr uint32_t P1 = 2654435761u, P2 = 805459861u;
  constexpr uint32_t K1 = 0u - kFloorBias * P1, K2 = 0u - kFloorBias * P2;
  const uint32_t mask = t.mask[l];
  const uint32_t hy0 = yb * P1 + K1, hy1 = hy0 + P1;
  const uint32_t hz0 = zb * P2 + K2, hz1 = hz0 + P2;
  const __half2* base = reinterpret_cast<const __half2*>(t.base[l]);
  const uint32_t xb1 = xb + 1u;
  const uint32_t yz00 = hy0 ^ hz0, yz10 = hy1 ^ hz0, yz01 = hy0 ^ hz1, yz11 = hy1 ^ hz1;
  e[0] = __ldg(base + xor_and(xb, yz00, mask));
  e[1] = __ldg(base + xor_and(xb1, yz00, mask));
  e[2] = __ldg(base + xor_and(xb, yz10, mask));
  e[3] = __ldg(base + xor_and(xb1, yz10, mask));
  e[4] = __ldg(base + xor_and(xb, yz01, mask));
  e[5] = __ldg(base + xor_and(xb1, yz01, mask));
  e[6] = __ldg(base + xor_and(xb, yz11, mask));
  e[7] = __ldg(base + xor_and(xb1, yz11, mask));
}

// ---- the production gather, software-pipelined over level pairs ------------------------------
// Every level of one sample, two levels (one cell2) at a time, with the corner loads of the next
// two pairs in flight while a pair is combined: the loads of pair k + 2 are issued right after
// pair k is combined, so ~100 instructions (the next pair's combine and the following pair's
// cells, indices and loads) separate a load from its use instead of none (+1.2 % frame rate
// over four levels at a time with one full load wait per four).
struct LvlPair {
  __half2 e[2][8];
  __half2 hu, hv, hs;  // the fractions of the pair's two levels (low half: level l, high: l + 1)
};

// cells and corner loads of levels l (even) and l + 1 (the second only if `two`, warp-uniform;
// otherwise q.e[1] keeps what it holds -- zeros or an earlier pair's finite entries -- and the
// level's weight 0 makes its feature 0)
__device__ __forceinline__ void pair_issue(const LevelTab& t, uint32_t dense_mask, int l, bool two, float u,
                                           float v, float w, LvlPair& q) {
  const uint64_t r2 = *reinterpret_cast<const uint64_t*>(&t.res[l]);
  uint32_t xb0, xb1, yb0, yb1, zb0, zb1;
  float f0, f1;
  cell2(u, r2, xb0, xb1, f0, f1);
  q.hu = __floats2half2_rn(f0, f1);
  cell2(v, r2, yb0, yb1, f0, f1);
  q.hv = __floats2half2_rn(f0, f1);
  cell2(w, r2, zb0, zb1, f0, f1);
  q.hs = __floats2half2_rn(f0, f1);
  if (((dense_mask >> l) & 3u) == 0u) {
    corners8_hashed(t, l, xb0, yb0, zb0, q.e[0]);
    if (two) corners8_hashed(t, l + 1, xb1, yb1, zb1, q.e[1]);
  } else {
    corners8(t, l, xb0, yb0, zb0, q.e[0]);
    if (two) corners8(t, l + 1, xb1, yb1, zb1, q.e[1]);
  }
}

// level l + i of the pair, weighted by w_l = saturate(flc) (flc = fl - (l + i)): seven packed
// lerps a + (b - a) f (HADD2 + HFMA2 each, both features at once) with the pair's packed
// fractions selected by half, times w_l
__device__ __forceinline__ uint32_t pair_combine(const LvlPair& q, int i, float flc) {
  const __half2 hu = i ? __high2half2(q.hu) : __low2half2(q.hu);
  const __half2 hv = i ? __high2half2(q.hv) : __low2half2(q.hv);
  const __half2 hs = i ? __high2half2(q.hs) : __low2half2(q.hs);
  const __half2* e = q.e[i];
  const __half2 x00 = __hfma2(__hsub2(e[1], e[0]), hu, e[0]), x10 = __hfma2(__hsub2(e[3], e[2]), hu, e[2]),
                x01 = __hfma2(__hsub2(e[5], e[4]), hu, e[4]), x11 = __hfma2(__hsub2(e[7], e[6]), hu, e[6]);
  const __half2 y0 = __hfma2(__hsub2(x10, x00), hv, x00), y1 = __hfma2(__hsub2(x11, x01), hv, x01);
  return h2u(__hmul2(__hfma2(__hsub2(y1, y0), hs, y0), __float2half2_rn(__saturatef(flc))));
}

// Levels [0, na_max) of one sample (na_max warp-uniform: the longest level count of the warp's
// rows; a lane with fewer levels gathers the others with weight 0) -> store(c, chunk) for every
// A chunk c = levels 4c .. 4c + 3 that holds a level; chunks past them are not stored.
template <class Store>
__device__ __forceinline__ void gather_row(const LevelTab& t, int na_max, float u, float v, float w, float fl,
                                           Store&& store) {
  const int np = (na_max + 1) >> 1;  // level pairs
  const uint32_t dm = t.dense_mask;  // read once per row (the pair issues test it per pair)
  LvlPair qa, qb;
#pragma unroll
  for (int k = 0; k < 8; ++k) qa.e[1][k] = qb.e[1][k] = __half2{};  // never NaN (see pair_issue)
  if (np > 0) pair_issue(t, dm, 0, na_max > 1, u, v, w, qa);
  if (np > 1) pair_issue(t, dm, 2, na_max > 3, u, v, w, qb);
#pragma unroll 1
  for (int c = 0; 2 * c < np; ++c) {  // chunk c: pair 2c in qa, pair 2c + 1 in qb
    const float flc = fl - (float)(4 * c);
    const uint32_t o0 = pair_combine(qa, 0, flc), o1 = pair_combine(qa, 1, flc - 1.f);
    if (2 * c + 2 < np) pair_issue(t, dm, 4 * c + 4, na_max > 4 * c + 5, u, v, w, qa);
    uint32_t o2 = 0u, o3 = 0u;
    if (2 * c + 1 < np) {
      o2 = pair_combine(qb, 0, flc - 2.f);
      o3 = pair_combine(qb, 1, flc - 3.f);
      if (2 * c + 3 < np) pair_issue(t, dm, 4 * c + 6, na_max > 4 * c + 7, u, v, w, qb);
    }
    store(c, make_uint4(o0, o1, o2, o3));
  }
}

// the clamp every caller of gather_row applies: [0, 1] -> [0, 1 - 2^-24]
__device__ __forceinline__ float unit_below1(float x) { return fminf(__saturatef(x), 0.99999994f); }

// trunc_exp / sigmoid (network.h:41-57) with the MUFU exp2 / reciprocal: ~2 ulp, far below the
// fp16 MLP operands' 1.6e-4 (oracle-measured)
__device__ __forceinline__ float trunc_exp_fast(float x) {
  return x <= 10.f ? __expf(x) : 22026.4657948f * (1.f + (x - 10.f));
}
__device__ __forceinline__ float sigmoid_fast(float x) { return __fdividef(1.f, 1.f + __expf(-x)); }

// position of the (k+1)-th set bit of m (k < popc(m))
__device__ __forceinline__ int nth_set_bit(uint32_t m, int k) {
  int pos = 0;
#pragma unroll
  for (int w = 16; w > 0; w >>= 1) {
    const int c = __popc(m & ((1u << w) - 1u));
    if (k >= c) {
      k -= c;
      m >>= w;
      pos += w;
    }
  }
  return pos;
}

using accum_t = float;

// The owner-lane state of one ray of the packet.
struct Ray {
  bool valid, alive;  // pixel inside the range / still compositing
  int x, y, id;
  float3 d, nd;       // fp32 directions for the network-input geometry
  int kept_total, contributing;
  bool term;
  double trans;
  // the running colour / depth / opacity sums in fp32 (5 registers fewer in the row-owning
  // warps than double); the transmittance, which decides the termination cut, stays double
  accum_t px, py, pz, depth, opac;
};

struct Counters {
  unsigned evals, level_samples, marched, rays;
};

}  // namespace pk
}  // namespace lumi_dev
