// render_ws.cu -- warp-specialised packet renderer (the production frame kernel).
//
// The round-1 packet kernel (render_pk.cu, retired) was latency bound with 16 warps per SM, and every resource
// that would admit more row-owning warps is full (TMEM 4 x 128 columns, 128 registers x 512
// threads, 57 KB of shared memory x 4).  Here each CTA pairs a CONSUMER warpgroup -- the four
// row-owning warps: packet streams, geometry, the tcgen05 MLP and compositing -- with a
// PRODUCER warpgroup of four warps that clears the A rows, builds the gather list and runs the
// hash-grid gather (half the instructions).  The two are pipelined one round apart through
// double-buffered layer-1 A tiles and row inputs, synchronised with named barriers (one pair
// per buffer), so a CTA of 8 warps fits 3 times per SM: 24 warps instead of 16.  The math of
// every stage is the packet kernel's (pk_parts.cuh); only the schedule differs:
//
//   consumers, iteration j:  fill + geometry of round j into buffer j&1 (per row: grid
//                            coordinates, LOD, active levels; per warp: its pair count)
//                            -> arrive LIST_READY[j&1]
//                            -> wait GATHER_DONE[(j-1)&1] -> MLP + composite of round j-1
//   producers, iteration j:  wait LIST_READY[j&1] -> clear A rows, write ONE concatenated
//                            level-major list whose codes are the features' A offsets ->
//                            gather it over 128 threads -> arrive GATHER_DONE[j&1]
//
// Because round j is filled before round j-1 is composited, a packet whose stream ends is
// stored only after the last round holding its rows is composited (one idle round per packet
// for that warp), and rows of rays that terminate in round j-1 may still be evaluated in round
// j (they are skipped by the compositing, exactly as in the packet kernel).
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstddef>
#include <cstdio>
#include <cstdlib>
#include <algorithm>

#include "kernels.h"
#include "pk_parts.cuh"

namespace lumi_dev {
namespace ws {

using namespace pk;

#ifndef WS_SHARED_ONES
#define WS_SHARED_ONES 1
#endif
#ifndef WS_PREFETCH
#define WS_PREFETCH 1
#endif
#ifndef WS_MARCH_DIRS
#define WS_MARCH_DIRS 1
#endif
#ifndef WS_PROD_WARPS
#define WS_PROD_WARPS 4
#endif
constexpr int kProdWarps = WS_PROD_WARPS;              // producer warps (4 or 8)
constexpr int kProdThreads = 32 * kProdWarps;
constexpr int kCtaThreads = 128 + kProdThreads;        // consumers [0, 128), producers after
// WS_REGSPLIT: the warpgroups trade registers with setmaxnreg after the launch allocation
// (80 per thread at 3 CTAs x 256 threads): the consumers, whose MLP epilogues and compositing
// state are the register-bound side, get WS_CONS_REGS, the producers keep WS_PROD_REGS
// (128 * C + kProdThreads * P <= kCtaThreads * launch).  With 8 producer warps (3 CTAs x 384
// threads, 56 per thread at launch) the split is 88 / 40.
#ifndef WS_REGSPLIT
#define WS_REGSPLIT 1
#endif
#ifndef WS_CONS_REGS
#define WS_CONS_REGS 88
#endif
#ifndef WS_PROD_REGS
#define WS_PROD_REGS (WS_PROD_WARPS == 4 ? 72 : 40)
#endif
constexpr int kCtasPerSm = (kProdWarps == 4 || WS_REGSPLIT) ? 3 : 2;  // (registers: <= 85 per thread)
#ifndef WS_PROD_PAIRS
#define WS_PROD_PAIRS 3
#endif
constexpr int kProdPairs = WS_PROD_PAIRS;  // pairs per producer thread per gather step
// WS_PAIRS: producer warp w gathers exactly consumer warp w's 32 rows, so the list handoff is a
// per-warp-pair barrier (64 threads): a producer warp starts as soon as ITS consumer warp has
// filled its rows instead of waiting for the slowest of the four.  The round's MMA still waits
// for all four producer warps (GATHER_DONE).  Stop: producers cannot see the consumers' stop
// decision before they start, so they gather the final (empty) round too; the consumers then
// drain its GATHER_DONE, raise `halt` and wake each producer warp one last time.
#ifndef WS_PAIRS
#define WS_PAIRS 0
#endif
// named barriers: 0 = __syncthreads (setup / teardown), LIST_READY 1 + b, GATHER_DONE 4 + b
// (b < kStages), 7 = consumer warpgroup only, 8 = producer warpgroup only
#if WS_PAIRS
// LIST_READY of (warp w, stage b) = kBarPair + 2 w + b (1 .. 8), GATHER_DONE 9 + b
constexpr int kBarPair = 1, kBarList = 0, kBarGather = 9, kBarCons = 11, kBarProd = 12;
#else
constexpr int kBarList = 1, kBarGather = 4, kBarCons = 7, kBarProd = 8, kBarPair = 0;
#endif
#ifndef WS_CONS_LEVELS
#define WS_CONS_LEVELS 0
#endif
constexpr int kConsLevels = WS_CONS_LEVELS;  // LOD levels gathered by the consumers (<= 4)
// WS_ROWMAJOR (default): producer thread t gathers ALL active levels of row t, four levels (one
// 16-byte A chunk) at a time, straight from the row's (u, v, w, fl) -- no shared (row, level)
// list to build or decode.  The 32 rows of a warp are neighbouring rays of one packet at nearly
// the same distance, so their LOD (hence their level count) is nearly uniform and the lanes of a
// warp walk the same level together (coherent hash cells, warp-uniform dense/hashed branch).
#ifndef WS_ROWMAJOR
#define WS_ROWMAJOR 1
#endif
// WS_GATHER2: the producers run pk::gather_chunk4 (packed-f32x2 cells off biased float bits,
// bias-folded corner indices, dense x+1 as a load offset); 0 = the round-1/2 gather_prep path
#ifndef WS_GATHER2
#define WS_GATHER2 1
#endif
// WS_PROD_GEOM: the producers compute each row's sample geometry (position, contraction, LOD
// footprint and weights) from the row's ray directions and candidate, which the consumers pass
// through shared memory -- the consumers' fill phase loses its heaviest part
#ifndef WS_PROD_GEOM
#define WS_PROD_GEOM 1
#endif
// WS_FILL_TRANSPOSE: a new mask word's per-candidate ray sets by one 32x32 bit transpose across
// the warp (5 shuffle stages) and a scan, instead of 32 ballots with a serial running count
#ifndef WS_FILL_TRANSPOSE
#define WS_FILL_TRANSPOSE 1
#endif
// WS_PROD_DIRS: the producers also load each row's ray directions (march-pass SoA planes, by the
// packet id and ray lane the consumers pass) and hand the direction back for the SH encoding;
// the consumers keep no directions and a new packet costs them no loads but its first mask
// word, which is prefetched one packet ahead
#ifndef WS_PROD_DIRS
#define WS_PROD_DIRS 0  // measured -6 %: the direction loads lengthen the producers' critical path
#endif
// WS_NEXT_FIRST: the next packet's first mask word is loaded one round after the next packet id
// (so a new packet's first word switch does not wait on a load)
#ifndef WS_NEXT_FIRST
#define WS_NEXT_FIRST 1
#endif
#ifndef WS_F32_ALPHA
#define WS_F32_ALPHA 1
#endif
// WS_STAGES: rounds in flight between the two warpgroups (2 = double-buffered, 3 = the
// consumers fill two rounds ahead of the MLP, so a slow round on either side is absorbed)
#ifndef WS_STAGES
#define WS_STAGES 2
#endif
constexpr int kStages = WS_STAGES;
#if WS_PAIRS
static_assert(kStages == 2 && WS_ROWMAJOR, "the per-pair handoff is built for the 2-stage row-major kernel");
#endif

static_assert(kStages == 2 || kStages == 3, "2 or 3 pipeline stages");
// WS_TMASK: the march pass stores each packet's mask words transposed (candidate-major), so a
// warp starting a word scans 32 counts instead of transposing the word with 32 ballots, and
// expands it once into a (candidate, ray) sample stream its rows index directly
#ifndef WS_TMASK
#define WS_TMASK 0
#endif
#if WS_ROWMAJOR
static_assert(kConsLevels == 0, "the row-major producers gather every level");
static_assert(WS_PROD_WARPS == 4, "row-major producers: one thread per row");
#endif

#ifdef LUMI_PHASE_TIMING
// warp-cycles: producers [wait list, gather], consumers [fill+geometry+list, wait gather, MLP,
// composite]
__device__ unsigned long long g_ws_cycles[8];
#define WS_T(k)                                                    \
  do {                                                             \
    const long long _t = clock64();                                \
    if (lane == 0) atomicAdd(&g_ws_cycles[k], (unsigned long long)(_t - t_last)); \
    t_last = _t;                                                   \
  } while (0)
#else
#define WS_T(k) \
  do {          \
  } while (0)
#endif

struct __align__(16) Smem {
#if WS_SHARED_ONES
  // double-buffered layer-1 A tiles, features only (chunk-major, a_off); the bias step's
  // [1 0 ... 0] block is one shared pair of core matrices read with SBO = 0 by every row group
  uint8_t A[kStages][128 * 32 * 2];
  uint8_t ones[2 * 128];
#else
  uint8_t A[kStages][128 * (32 + kKb) * 2];  // layer-1 A tiles per stage (chunk-major, a_off)
#endif
  uint8_t W1[64 * (32 + kKb) * 2];
  uint8_t F[80 * (80 + kKb) * 2];
  uint8_t C2[64 * (64 + kKb) * 2];
  uint8_t C3[16 * (64 + kKb) * 2];
  float4 res[128];
#if WS_TMASK
  uint16_t stream[kWarps][32 * 32];  // per warp: the current mask word's (candidate, ray) samples
#else
  uint32_t ballot[kWarps][32];
  uint16_t prefix[kWarps][33];
#endif
  uint32_t own[kStages][kWarps][32];
  uint16_t rowcand[kStages][kWarps][32];
  uint8_t rowlane[kStages][128];
  int rowpkt[kStages][kWarps];  // per warp: the packet of the round's rows
  uint64_t mbar;
  uint64_t wbar;  // the weight tiles' TMA bulk copy
  uint32_t tmem_base;
  int stop[kStages];
  int halt;  // WS_PAIRS: the consumers have stopped (no further round)
  uint4 lvl[kMaxLevels];
  LevelTab lt;
#if !WS_PROD_GEOM || !WS_ROWMAJOR
  float4 samp[kStages][128];  // per row: grid coordinates + LOD (fl), from the consumers
#endif
#if WS_PROD_GEOM
  float4 rdir[kStages][128];   // per row: ray direction xyz + neighbour direction x
#if !WS_PROD_DIRS
  float2 rdir2[kStages][128];  // neighbour direction yz
#endif
#endif
  uint8_t na[kStages][128];                  // per row: active LOD levels (0 = no sample)
#if !WS_ROWMAJOR
  uint16_t pairs[kWarps * 32 * kMaxLevels];  // the round's gather list, warp lists concatenated
  int cnt[2][kWarps];                        // per warp: pairs the producers will list
#endif
};

// the four weight tiles are consecutive in Smem: one contiguous image, one bulk copy
constexpr size_t kWeightTileBytes = sizeof(Smem::W1) + sizeof(Smem::F) + sizeof(Smem::C2) + sizeof(Smem::C3);
static_assert(offsetof(Smem, F) == offsetof(Smem, W1) + sizeof(Smem::W1) &&
                  offsetof(Smem, C2) == offsetof(Smem, F) + sizeof(Smem::F) &&
                  offsetof(Smem, C3) == offsetof(Smem, C2) + sizeof(Smem::C2),
              "weight tiles must be contiguous");
static_assert(kWeightTileBytes % 16 == 0 && offsetof(Smem, W1) % 16 == 0, "bulk copy alignment");

// the weight tiles' shared-memory image in global memory (the same load_weight_tile code,
// storing through a generic pointer), built once per model / parameter update
__global__ void k_pack_weight_tiles(MlpDev mlp, uint8_t* img) {
  const float* dp = mlp.dparams;
  const float* cp = mlp.cparams;
  const float* c2 = cp + 64 * 32 + 64;
  const float* c3 = c2 + 64 * 64 + 64;
  uint8_t* W1 = img;
  uint8_t* F = W1 + sizeof(Smem::W1);
  uint8_t* C2 = F + sizeof(Smem::F);
  uint8_t* C3 = C2 + sizeof(Smem::C2);
  load_weight_tile(W1, dp, 64, 64, 32);
  load_weight_tile(F, mlp.fused, kHidden + 1, 80, 80);
  load_weight_tile(C2, c2, 64, 64, 64);
  load_weight_tile(C3, c3, 3, 16, 64);
}

// layer 1 with the bias step's A from the shared ones block (LBO 128 B between its two core
// matrices, SBO 0: every 8-row group reads the same [1 0 ... 0] rows)
__device__ __forceinline__ void issue_layer1_shared_ones(const uint8_t* A, const uint8_t* ones,
                                                         const uint8_t* B, uint32_t d_tmem) {
  constexpr uint32_t idesc = ptx::idesc_f16_f32<128, 64>();
  constexpr uint32_t sbo = ((32 + kKb) / 8) * 128;
  const uint32_t a = ptx::smem_addr(A), o = ptx::smem_addr(ones), b = ptx::smem_addr(B);
#pragma unroll
  for (int kk = 0; kk < 2; ++kk)
    ptx::mma_f16(d_tmem, ptx::make_smem_desc(a + kk * 2 * kALbo, kALbo, 128),
                 ptx::make_smem_desc(b + kk * 256, 128, sbo), idesc, kk > 0 ? 1u : 0u);
  ptx::mma_f16(d_tmem, ptx::make_smem_desc(o, 128, 0), ptx::make_smem_desc(b + 2 * 256, 128, sbo), idesc, 1u);
}

// named barriers with immediate ids, so ptxas reserves only the barriers used (a register id
// would reserve all 16, which caps residency at one CTA per SM)
template <int ID, int N>
__device__ __forceinline__ void bar_sync() {
  asm volatile("bar.sync %0, %1;" ::"n"(ID), "n"(N) : "memory");
}
template <int ID, int N>
__device__ __forceinline__ void bar_arrive() {
  asm volatile("bar.arrive %0, %1;" ::"n"(ID), "n"(N) : "memory");
}
template <int ID, int N>
__device__ __forceinline__ bool bar_and(bool v) {
  uint32_t r;
  asm volatile(
      "{\n .reg .pred p, q;\n setp.ne.u32 p, %1, 0;\n bar.red.and.pred q, %2, %3, p;\n"
      " selp.u32 %0, 1, 0, q;\n}"
      : "=r"(r)
      : "r"((uint32_t)v), "n"(ID), "n"(N)
      : "memory");
  return r != 0;
}
// per-warp-pair list handoff (WS_PAIRS): 64 threads, consumer warp w + producer warp w
template <int ID>
__device__ __forceinline__ void pair_bar(bool arrive) {
  if (arrive) bar_arrive<ID, 64>(); else bar_sync<ID, 64>();
}
__device__ __forceinline__ void pair_ready(int w, int b, bool arrive) {
  switch (2 * w + b) {
    case 0: pair_bar<kBarPair + 0>(arrive); break;
    case 1: pair_bar<kBarPair + 1>(arrive); break;
    case 2: pair_bar<kBarPair + 2>(arrive); break;
    case 3: pair_bar<kBarPair + 3>(arrive); break;
    case 4: pair_bar<kBarPair + 4>(arrive); break;
    case 5: pair_bar<kBarPair + 5>(arrive); break;
    case 6: pair_bar<kBarPair + 6>(arrive); break;
    default: pair_bar<kBarPair + 7>(arrive); break;
  }
}

// stage-indexed barriers: b < kStages
__device__ __forceinline__ void list_ready_sync(int b) {
  if (b == 0) bar_sync<kBarList, kCtaThreads>();
  else if (b == 1) bar_sync<kBarList + 1, kCtaThreads>();
  else bar_sync<kBarList + 2, kCtaThreads>();
}
__device__ __forceinline__ void list_ready_arrive(int b) {
  if (b == 0) bar_arrive<kBarList, kCtaThreads>();
  else if (b == 1) bar_arrive<kBarList + 1, kCtaThreads>();
  else bar_arrive<kBarList + 2, kCtaThreads>();
}
__device__ __forceinline__ void gather_done_sync(int b) {
  if (b == 0) bar_sync<kBarGather, kCtaThreads>();
  else if (b == 1) bar_sync<kBarGather + 1, kCtaThreads>();
  else bar_sync<kBarGather + 2, kCtaThreads>();
}
__device__ __forceinline__ void gather_done_arrive(int b) {
  if (b == 0) bar_arrive<kBarGather, kCtaThreads>();
  else if (b == 1) bar_arrive<kBarGather + 1, kCtaThreads>();
  else bar_arrive<kBarGather + 2, kCtaThreads>();
}

// One row's sample geometry (renderer.h:205-222 in fp32): position o + d t, contraction, the
// grid coordinates (u, v, w) in [0, 1), the LOD footprint against the neighbour ray and the
// weights as fl (w_l = saturate(fl - l)); returns the active level count (0: no sample).
struct GeomConst {
  float3 o;
  float two_base, inv_log, bias;
  int levels;
};
__device__ __forceinline__ int row_geometry(const RenderParams& p, const GeomConst& gc, float3 d, float3 nd,
                                            int cand, float4& out) {
  const float t = (float)__ldg(p.ts + cand);
  const float3 c = contract_f(make_float3(gc.o.x + d.x * t, gc.o.y + d.y * t, gc.o.z + d.z * t), p.contraction);
  const float u = unit_below1((c.x + 2.f) * 0.25f);  // [0, 1): the gather's cells need no clamp
  const float v = unit_below1((c.y + 2.f) * 0.25f);
  const float w = unit_below1((c.z + 2.f) * 0.25f);
  LodW lw;
  if (p.lod_enabled) {
    const float3 bq = contract_f(make_float3(gc.o.x + nd.x * t, gc.o.y + nd.y * t, gc.o.z + nd.z * t), p.contraction);
    const float ex = c.x - bq.x, ey = c.y - bq.y, ez = c.z - bq.z;
    const float rc = fmaxf(0.5f * sqrtf(ex * ex + ey * ey + ez * ez), 1e-12f);
    const float l = fminf(-__logf(gc.two_base * rc) * gc.inv_log, (float)(gc.levels - 1));
    lw = lod_weights_f(l + gc.bias, gc.levels);
  } else {
    lw = LodW{gc.levels, 0.f, false};
  }
  out = make_float4(u, v, w, lw.floor_only ? 1e-4f : (float)lw.full + lw.frac);
  return active_levels(lw, gc.levels);
}

__global__ void __launch_bounds__(kCtaThreads, kCtasPerSm) k_render_ws(RenderParams p) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  Smem& s = *reinterpret_cast<Smem*>(smem_raw);
  const int tid = threadIdx.x, wg = tid >= 128 ? 1 : 0, ctid = wg ? tid - 128 : tid, warp = ctid >> 5,
            lane = tid & 31;
  const unsigned FULL = 0xffffffffu;

  // ---- setup (all 256 threads) -------------------------------------------------------------
  // the four fp16 UMMA weight tiles: one TMA bulk copy of their packed image (built once per
  // model, launch_pack_weight_tiles), or converted from the fp32 parameters here
  const bool tma_weights = p.mlp.wtiles != nullptr;
  if (tma_weights) {
    if (tid == 0) {
      ptx::mbar_init(&s.wbar, 1);
      ptx::fence_mbar_init();
      ptx::mbar_arrive_expect_tx(&s.wbar, (uint32_t)kWeightTileBytes);
      ptx::tma_bulk_g2s(s.W1, p.mlp.wtiles, (uint32_t)kWeightTileBytes, &s.wbar);
    }
  } else {
    const float* dp = p.mlp.dparams;
    const float* cp = p.mlp.cparams;
    const float* c2 = cp + 64 * 32 + 64;
    const float* c3 = c2 + 64 * 64 + 64;
    load_weight_tile(s.W1, dp, 64, 64, 32);
    load_weight_tile(s.F, p.mlp.fused, kHidden + 1, 80, 80);
    load_weight_tile(s.C2, c2, 64, 64, 64);
    load_weight_tile(s.C3, c3, 3, 16, 64);
  }
#if WS_SHARED_ONES
  if (tid < 16) st16(s.ones, (uint32_t)tid * 16u, make_uint4(tid < 8 ? 0x3C00u : 0u, 0u, 0u, 0u));
#else
  // constant ones block of both A buffers (never overwritten)
  if (ctid < 128) {
    st16(s.A[wg], a_off(ctid, 4), make_uint4(0x3C00u, 0u, 0u, 0u));
    st16(s.A[wg], a_off(ctid, 5), make_uint4(0u, 0u, 0u, 0u));
  }
#endif
  for (int l = tid; l < kMaxLevels; l += kCtaThreads) {
    const int res = l < p.grid.levels ? p.grid.res[l] : 1;
    const bool dense = (p.grid.dense_mask >> l) & 1u;
    const unsigned long long base =
        reinterpret_cast<unsigned long long>(p.grid.table16 + (l < p.grid.levels ? p.grid.offset2[l] : 0));
    s.lvl[l] = make_uint4((uint32_t)res, dense ? 0u : p.grid.hash_mask[l], (uint32_t)base,
                          (uint32_t)(base >> 32));
  }
  level_tab_init(s.lt, p.grid, tid, kCtaThreads);
  if (tid == 0) {
    s.halt = 0;
    ptx::mbar_init(&s.mbar, 1);
    ptx::fence_mbar_init();
  }
  if (tid < 32) ptx::tmem_alloc<kTmemCols>(&s.tmem_base);
  ptx::fence_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = s.tmem_base;
#if WS_REGSPLIT
  static_assert(128 * WS_CONS_REGS + kProdThreads * WS_PROD_REGS <= kCtaThreads * (65536 / (kCtaThreads * kCtasPerSm) / 8 * 8),
                "register split exceeds the launch allocation");
  // the warpgroup giving registers up decreases first, the other one increases
  if ((wg == 1) == (WS_PROD_REGS < WS_CONS_REGS)) {
    if (wg == 1)
      asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(WS_PROD_REGS));
    else
      asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(WS_CONS_REGS));
  } else {
    if (wg == 1)
      asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(WS_PROD_REGS));
    else
      asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(WS_CONS_REGS));
  }
#endif
#ifdef LUMI_PHASE_TIMING
  long long t_last = clock64();
#endif

  if (wg == 1) {
    // ================================ producers ==============================================
#if WS_PROD_GEOM
    const GeomConst gc{make_float3((float)p.cam.origin[0], (float)p.cam.origin[1], (float)p.cam.origin[2]),
                       (float)p.grid.two_base, (float)(1.0 / p.grid.log_scale), (float)p.lod_bias,
                       p.grid.levels};
    unsigned pcnt_levels = 0;
#endif
    int b = 0;  // j % kStages
#pragma unroll 1
    for (int j = 0;; ++j, b = b + 1 == kStages ? 0 : b + 1) {
#if WS_PAIRS
      pair_ready(warp, b, false);
      WS_T(0);
      if (s.halt) break;
#else
      list_ready_sync(b);
      WS_T(0);
      if (s.stop[b]) break;
#endif
#if WS_ROWMAJOR
      {
#if WS_PROD_GEOM
        // row ctid: its ray directions and candidate from the consumers -> grid coordinates,
        // LOD (fl) and active level count
        float4 P = make_float4(0.f, 0.f, 0.f, 0.f);
        int na = 0;
        if (s.na[b][ctid]) {
#if WS_PROD_DIRS
          const size_t T = (size_t)p.total_rays;
          const float* rd = p.ray_dirs + ((size_t)s.rowpkt[b][warp] * 32 + s.rowlane[b][ctid]);
          const float3 d = make_float3(__ldg(rd), __ldg(rd + T), __ldg(rd + 2 * T));
          const float3 nd = make_float3(__ldg(rd + 3 * T), __ldg(rd + 4 * T), __ldg(rd + 5 * T));
          s.rdir[b][ctid] = make_float4(d.x, d.y, d.z, 0.f);  // for the consumers' SH encoding
          na = row_geometry(p, gc, d, nd, s.rowcand[b][warp][lane], P);
#else
          const float4 d4 = s.rdir[b][ctid];
          const float2 d2 = s.rdir2[b][ctid];
          na = row_geometry(p, gc, make_float3(d4.x, d4.y, d4.z), make_float3(d4.w, d2.x, d2.y),
                            s.rowcand[b][warp][lane], P);
#endif
          pcnt_levels += (unsigned)na;
        }
#else
        // row ctid: grid coordinates + LOD (fl) and its active level count, from the consumers
        const float4 P = s.samp[b][ctid];
        const int na = s.na[b][ctid];
#endif
        const int na_max = __reduce_max_sync(FULL, (unsigned)na);
#pragma unroll 1
        for (int c = 0; c < kMaxLevels / 4; ++c) {  // A chunk c = levels 4c .. 4c + 3
          uint4 out = make_uint4(0u, 0u, 0u, 0u);
          const int nq = min(4, na_max - 4 * c);  // levels of the chunk active in some lane (uniform)
#if WS_GATHER2
          // a lane whose row has fewer levels than the warp's longest gathers the level anyway
          // (a valid cell next to its neighbours') with weight 0
          if (nq > 0) out = gather_chunk4(s.lt, 4 * c, nq, P.x, P.y, P.z, P.w);
          (void)na;
#else
          if (nq > 0) {
            const float fl0 = P.w - (float)(4 * c);
            GatherPrep gp[4];
            float wl[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              // a lane whose row has fewer levels than the warp's longest gathers the level
              // anyway (a valid cell next to its neighbours') with weight 0
              wl[q] = 4 * c + q < na ? __saturatef(fl0 - (float)q) : 0.f;
              gather_prep(s.lvl[4 * c + q], P.x, P.y, P.z, gp[q]);
            }
            // all corner loads of the chunk in flight before the first combine; levels no lane
            // of the warp needs (the last chunk) are not loaded
            __half2 e[4][8];
            if (nq == 4) {
#pragma unroll
              for (int q = 0; q < 4; ++q)
#pragma unroll
                for (int k = 0; k < 8; ++k) e[q][k] = __ldg(gp[q].base + gp[q].idx[k]);
            } else {
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                const bool act = q < nq;
#pragma unroll
                for (int k = 0; k < 8; ++k) e[q][k] = act ? __ldg(gp[q].base + gp[q].idx[k]) : __half2{};
              }
            }
            uint32_t f[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) f[q] = h2u(gather_combine_h(e[q], gp[q].fu, gp[q].fv, gp[q].fs, wl[q]));
            out = make_uint4(f[0], f[1], f[2], f[3]);
          }
#endif
          st16(s.A[b], a_off(ctid, c), out);
        }
      }
      ptx::fence_async_smem();
      gather_done_arrive(b);
      WS_T(1);
      continue;
#else
      if (ctid < 128) {  // producer thread ctid < 128: row ctid
        // clear this row's features (buffer b's last reader, the MMA of round j-2, is done)
        // and list the (row, level) pairs of producer warp w's 32 rows, level-major
        const uint4 zero = make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int q = 1; q < 4; ++q) st16(s.A[b], a_off(ctid, q), zero);  // chunk 0: consumers
        const int na = s.na[b][ctid];
        int npairs = 0, total = 0;  // this warp's list starts after the lower warps' (counted by the consumers)
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
          const int c = s.cnt[b][w];
          npairs += w < warp ? c : 0;
          total += c;
        }
        const unsigned lt = (1u << lane) - 1u;
        for (int l = kConsLevels; l < kMaxLevels; ++l) {
          const unsigned m = __ballot_sync(FULL, na > l);
          if (m == 0u) break;
          if (na > l) s.pairs[npairs + __popc(m & lt)] = (uint16_t)pair_code(ctid, l);
          npairs += __popc(m);
        }
        (void)total;
      }
      bar_sync<kBarProd, kProdThreads>();
      int total = 0;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) total += s.cnt[b][w];
      const uint8_t* Pb = reinterpret_cast<const uint8_t*>(s.samp[b]);
#pragma unroll 1
      for (int base = 0; base < total; base += kProdThreads * kProdPairs) {
        // branch-free over the pairs (past the end of the list a lane re-gathers the last pair
        // and does not store it), so all kProdPairs x 8 corner loads are in flight before the
        // first FHFMA; code = the feature's byte offset in A, row * 16 in samp
        uint32_t code[kProdPairs];
        bool ok[kProdPairs];
#pragma unroll
        for (int q = 0; q < kProdPairs; ++q) {
          const int pi = base + kProdThreads * q + ctid;
          ok[q] = pi < total;
          code[q] = s.pairs[ok[q] ? pi : total - 1];
        }
        GatherPrep gp[kProdPairs];
        float wl[kProdPairs];
#pragma unroll
        for (int q = 0; q < kProdPairs; ++q) {
          const float4 P = *reinterpret_cast<const float4*>(Pb + (code[q] & 0x7F0u));
          const int lv = pair_level(code[q]);
          wl[q] = __saturatef(P.w - (float)lv);
          gather_prep(s.lvl[lv], P.x, P.y, P.z, gp[q]);
        }
        __half2 e[kProdPairs][8];
#pragma unroll
        for (int q = 0; q < kProdPairs; ++q)
#pragma unroll
          for (int k = 0; k < 8; ++k) e[q][k] = __ldg(gp[q].base + gp[q].idx[k]);
#pragma unroll
        for (int q = 0; q < kProdPairs; ++q) {
          const float2 f = gather_combine(e[q], gp[q].fu, gp[q].fv, gp[q].fs, wl[q]);
          if (ok[q]) *reinterpret_cast<__half2*>(s.A[b] + code[q]) = __floats2half2_rn(f.x, f.y);
        }
      }
      ptx::fence_async_smem();
      bar_sync<kBarProd, kProdThreads>();  // every producer is done with this round's lists
      gather_done_arrive(b);
      WS_T(1);
#endif
    }
#if WS_PROD_GEOM
    add_work_stats(p, 0, pcnt_levels, 0, 0);
#endif
  } else {
    // ================================ consumers ==============================================
    if (tma_weights) ptx::mbar_wait(&s.wbar, 0);  // the weight tiles have landed
    const uint32_t t_lane = tmem + ((uint32_t)(warp * 32) << 16);
    {
      const uint32_t ones[8] = {0x3C00u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
      ptx::tmem_st8(t_lane + kOnesCol, ones);
      ptx::tmem_st_wait();
      ptx::tc_fence_before();
      bar_sync<kBarCons, 128>();
      ptx::tc_fence_after();
    }
    const float3 o = make_float3((float)p.cam.origin[0], (float)p.cam.origin[1], (float)p.cam.origin[2]);
    const float two_base = (float)p.grid.two_base, inv_log = (float)(1.0 / p.grid.log_scale);
    const int levels = p.grid.levels;
    const long long packets_x = p.tiles_x;
    const long long total_packets = p.total_rays / 32;
    const uint32_t a_tmem = tmem + kAcol, ones_tmem = tmem + kOnesCol;
    const uint32_t a_lane = t_lane + kAcol;
    const bool issuer = (ctid == 0);

    Counters cnt{0, 0, 0, 0};
    Ray r;
    r.valid = r.alive = false;
    bool packet_live = false, no_more = false, pending = false;
    int last_round = -1;  // the last round holding rows of the pending packet
    int word = 0, g_next = 0, word_total = 0;
#if WS_PREFETCH
    // one packet id and one mask word ahead: the atomic and the word load are off the fill's
    // dependency chain
    long long next_pkt = 0;
    if (lane == 0) next_pkt = (long long)atomicAdd(p.work_counter, 1u);
    uint32_t next_bits = 0;
#endif
#if WS_NEXT_FIRST
    // the next packet's first mask word, loaded once its id has arrived (the round after the
    // atomic was issued)
    uint32_t next_first = 0;
    bool nf_ready = false;
#endif
    uint32_t phase = 0;
    long long pkt_cycles = 0;  // this warp's cycles on its current packet (RowStats.ms diagnostic)

    int b = 0, stop_round = -1;  // b = j % kStages; stop_round: the first round with no rows
#pragma unroll 1
    for (int j = 0;; ++j, b = b + 1 == kStages ? 0 : b + 1) {
      const long long t_iter = clock64();
      if (stop_round < 0) {
      // ---- F(j): this warp's rows of round j from its packet stream -----------------------
      int take = 0, rl = lane, cand = 0;
#if WS_NEXT_FIRST
      if (!nf_ready) {
        const long long np = __shfl_sync(FULL, next_pkt, 0);
        next_first = np < total_packets ? __ldg(p.kept_mask + np * 32 + lane) : 0u;
        nf_ready = true;
      }
#endif
      while (take < 32 && !no_more && !pending) {
        if (!packet_live) {
          long long pkt = 0;
#if WS_PREFETCH
          if (lane == 0) {
            pkt = next_pkt;
            next_pkt = (long long)atomicAdd(p.work_counter, 1u);
          }
#else
          if (lane == 0) pkt = (long long)atomicAdd(p.work_counter, 1u);
#endif
          pkt = __shfl_sync(FULL, pkt, 0);
          if (pkt >= total_packets) {
            no_more = true;
            break;
          }
          const long long rid = pkt * 32 + lane;
          // the pixel and the kept count are re-derived when the packet is stored: fewer
          // registers live across the rounds
          const int px_ = (int)(pkt % packets_x) * kPW + (lane % kPW);
          const int py_ = p.row_begin + (int)(pkt / packets_x) * kPH + lane / kPW;
          r.id = (int)rid;
          r.valid = px_ < p.cam.width && py_ < p.row_end;
          r.alive = r.valid;
          if (r.valid) {
#if WS_PROD_DIRS
#elif WS_MARCH_DIRS
            const size_t T = (size_t)p.total_rays;
            const float* rd = p.ray_dirs + rid;
            r.d = make_float3(__ldg(rd), __ldg(rd + T), __ldg(rd + 2 * T));
            r.nd = make_float3(__ldg(rd + 3 * T), __ldg(rd + 4 * T), __ldg(rd + 5 * T));
#else
            const d3 dd = ray_dir(p.cam, (double)px_ + 0.5, (double)py_ + 0.5);
            const d3 nn = ray_dir(p.cam, (double)px_ + 1.5, (double)py_ + 0.5);
            r.d = make_float3((float)dd.x, (float)dd.y, (float)dd.z);
            r.nd = make_float3((float)nn.x, (float)nn.y, (float)nn.z);
#endif
            ++cnt.rays;
          }
          r.contributing = 0;
          r.term = false;
          r.trans = 1.0;
          r.px = r.py = r.pz = r.depth = r.opac = 0.0;
          packet_live = true;
          word = -1;
          g_next = word_total = 0;
#if WS_TMASK
          next_bits = __ldg(p.kept_mask + r.id);  // lane = candidate of word 0: its rays
#elif WS_NEXT_FIRST
          next_bits = next_first;  // (bits of invalid rays are masked by r.alive)
          nf_ready = false;
#elif WS_PREFETCH
          next_bits = r.valid ? __ldg(p.kept_mask + r.id) : 0u;
#endif
        }
        if (g_next < word_total) {
          const int n = min(32 - take, word_total - g_next);
          if (lane >= take && lane < take + n) {
            const int g = g_next + (lane - take);
#if WS_TMASK
            const uint32_t e = s.stream[warp][g];
            rl = (int)(e & 31u);
            cand = word * 32 + (int)(e >> 5);
#else
            int lo = 0;
#pragma unroll
            for (int st = 16; st > 0; st >>= 1)
              if (s.prefix[warp][lo + st] <= g) lo += st;
            rl = nth_set_bit(s.ballot[warp][lo], g - s.prefix[warp][lo]);
            cand = word * 32 + lo;
#endif
          }
          take += n;
          g_next += n;
          continue;
        }
        if (word + 1 >= p.mask_words) {
          // stream exhausted: store the pixels once the last round with its rows is composited
          pending = true;
          last_round = take > 0 ? j : j - 1;
          break;
        }
        ++word;
#if WS_TMASK
        {
          // the march pass stored the packet's words transposed: lane c holds the rays keeping
          // candidate word * 32 + c.  Drop terminated rays, scan the per-candidate counts and
          // expand the word into the candidate-major sample stream (candidate, ray) of the warp
          const uint32_t alive_m = __ballot_sync(FULL, r.alive);
          const uint32_t col = next_bits & alive_m;
          if (word + 1 < p.mask_words && alive_m != 0u)
            next_bits = __ldg(p.kept_mask + (size_t)(word + 1) * p.total_rays + r.id);
          const int c = __popc(col);
          int incl = c;
#pragma unroll
          for (int off = 1; off < 32; off <<= 1) {
            const int v = __shfl_up_sync(FULL, incl, off);
            if (lane >= off) incl += v;
          }
          int pos = incl - c;
          for (uint32_t m = col; m; m &= m - 1u) s.stream[warp][pos++] = (uint16_t)((lane << 5) | (__ffs(m) - 1));
          __syncwarp();
          g_next = 0;
          word_total = __shfl_sync(FULL, incl, 31);
        }
#else
#if WS_PREFETCH
        const uint32_t bits = r.alive ? next_bits : 0u;
        if (word + 1 < p.mask_words && r.alive)
          next_bits = __ldg(p.kept_mask + (size_t)(word + 1) * p.total_rays + r.id);
#else
        const uint32_t bits = r.alive ? __ldg(p.kept_mask + (size_t)word * p.total_rays + r.id) : 0u;
#endif
#if WS_FILL_TRANSPOSE
        // lane i: the rays keeping candidate word * 32 + i (a 32x32 bit transpose instead of 32
        // ballots), then an exclusive scan of the per-candidate counts
        {
          const uint32_t col = warp_transpose32(bits);
          const int cnt_c = __popc(col);
          int incl = cnt_c;
#pragma unroll
          for (int off = 1; off < 32; off <<= 1) {
            const int v = __shfl_up_sync(FULL, incl, off);
            if (lane >= off) incl += v;
          }
          s.ballot[warp][lane] = col;
          s.prefix[warp][lane] = (uint16_t)(incl - cnt_c);
          if (lane == 31) s.prefix[warp][32] = (uint16_t)incl;
          __syncwarp();
          g_next = 0;
          word_total = __shfl_sync(FULL, incl, 31);
        }
#else
        int run = 0;
        for (int i = 0; i < 32; ++i) {
          const uint32_t bb = __ballot_sync(FULL, (bits >> i) & 1u);
          if (lane == 0) {
            s.ballot[warp][i] = bb;
            s.prefix[warp][i] = (uint16_t)run;
          }
          run += __popc(bb);
        }
        if (lane == 0) s.prefix[warp][32] = (uint16_t)run;
        __syncwarp();
        g_next = 0;
        word_total = run;
#endif
#endif
      }
      WS_T(6);
      const bool have = lane < take;
      {
        s.own[b][warp][lane] = 0u;
        __syncwarp();
        const unsigned same = __match_any_sync(FULL, have ? rl : 32 + lane);
        if (have) {
          s.own[b][warp][rl] = same;
          s.rowcand[b][warp][lane] = (uint16_t)cand;
        }
        s.rowlane[b][ctid] = (uint8_t)rl;
        __syncwarp();
      }
#if WS_PROD_DIRS
      if (lane == 0) s.rowpkt[b][warp] = r.id >> 5;
#else
      const float dx = __shfl_sync(FULL, r.d.x, rl), dy = __shfl_sync(FULL, r.d.y, rl),
                  dz = __shfl_sync(FULL, r.d.z, rl);
      const float nx = __shfl_sync(FULL, r.nd.x, rl), ny = __shfl_sync(FULL, r.nd.y, rl),
                  nz = __shfl_sync(FULL, r.nd.z, rl);
#endif
#if WS_PROD_GEOM
      // the producers derive the row's geometry: pass its ray directions (the candidate is in
      // rowcand) and a has-sample flag
      if (have) {
#if !WS_PROD_DIRS
        s.rdir[b][ctid] = make_float4(dx, dy, dz, nx);
        s.rdir2[b][ctid] = make_float2(ny, nz);
#endif
        ++cnt.evals;
      }
      s.na[b][ctid] = have ? 1 : 0;
#else
      float u = 0.f, v = 0.f, w = 0.f;
      LodW lw{0, 0.f, false};
      int na = 0;
      if (have) {
        const float t = (float)__ldg(p.ts + cand);
        const float3 c = contract_f(make_float3(o.x + dx * t, o.y + dy * t, o.z + dz * t), p.contraction);
        u = unit_below1((c.x + 2.f) * 0.25f);  // [0, 1): the gather's cells need no clamp
        v = unit_below1((c.y + 2.f) * 0.25f);
        w = unit_below1((c.z + 2.f) * 0.25f);
        if (p.lod_enabled) {
          const float3 bq = contract_f(make_float3(o.x + nx * t, o.y + ny * t, o.z + nz * t), p.contraction);
          const float ex = c.x - bq.x, ey = c.y - bq.y, ez = c.z - bq.z;
          const float rc = fmaxf(0.5f * sqrtf(ex * ex + ey * ey + ez * ez), 1e-12f);
          const float l = fminf(-__logf(two_base * rc) * inv_log, (float)(levels - 1));
          lw = lod_weights_f(l + (float)p.lod_bias, levels);
        } else {
          lw = LodW{levels, 0.f, false};
        }
        na = active_levels(lw, levels);
        cnt.level_samples += na;
        ++cnt.evals;
      }
      {  // the row's gather input for the producers: grid coordinates, LOD, active levels
        const float fl = lw.floor_only ? 1e-4f : (float)lw.full + lw.frac;
#if !WS_ROWMAJOR
        // the consumers gather the first kConsLevels levels of their own rows themselves (it
        // balances the two warpgroups) into A chunk 0, which they also clear
        {
          uint32_t wds[4] = {0u, 0u, 0u, 0u};
#pragma unroll
          for (int l = 0; l < kConsLevels; ++l) {
            float2 f = make_float2(0.f, 0.f);
            if (na > l) f = gather_level(s.lvl[l], u, v, w, __saturatef(fl - (float)l));
            wds[l] = h2u(__floats2half2_rn(f.x, f.y));
          }
          st16(s.A[b], a_off(ctid, 0), make_uint4(wds[0], wds[1], wds[2], wds[3]));
        }
#endif
        if (have) s.samp[b][ctid] = make_float4(u, v, w, fl);
        s.na[b][ctid] = (uint8_t)na;
#if !WS_ROWMAJOR
        const int mine = na > kConsLevels ? na - kConsLevels : 0;  // the producers' pairs of this row
        const int wsum = __reduce_add_sync(FULL, (unsigned)mine);
        if (lane == 0) s.cnt[b][warp] = wsum;
#endif
      }
#endif  // WS_PROD_GEOM
#if !WS_ROWMAJOR
      ptx::fence_async_smem();  // A chunk 0 (the MMA's async proxy reads it)
#endif
      WS_T(7);
#if WS_PAIRS
      pair_ready(warp, b, true);  // this warp's rows are ready: its producer warp may start
      // all consumer warps finished (every packet stored) -> no round j
      const bool stop = bar_and<kBarCons, 128>(no_more && !packet_live);
#else
      // all consumer warps finished (every packet stored) -> the producers stop at round j
      const bool stop = bar_and<kBarCons, 128>(no_more && !packet_live);
      if (ctid == 0) s.stop[b] = stop ? 1 : 0;
      list_ready_arrive(b);
#endif
      if (stop) stop_round = j;
      WS_T(2);
      }

      // the round whose MLP and compositing run now: kStages - 1 rounds behind the fill
      const int jm = j - (kStages - 1);
      if (jm >= 0 && (stop_round < 0 || jm < stop_round)) {
        // ---- M(jm): the tcgen05 MLP over round jm's 128 rows (field.h:106-137) -------------
        const int bp = b + 1 == kStages ? 0 : b + 1;  // jm % kStages
        gather_done_sync(bp);
        WS_T(3);
        const int rlp = s.rowlane[bp][ctid];
#if WS_PROD_DIRS
        const float4 pd4 = s.rdir[bp][ctid];  // written by the producers (rows without a sample: stale, unused)
        const float pdx = pd4.x, pdy = pd4.y, pdz = pd4.z;
        (void)rlp;
#else
        const float pdx = __shfl_sync(FULL, r.d.x, rlp), pdy = __shfl_sync(FULL, r.d.y, rlp),
                    pdz = __shfl_sync(FULL, r.d.z, rlp);
#endif
        float v32[32];
        if (issuer) {
          ptx::tc_fence_after();
#if WS_SHARED_ONES
          issue_layer1_shared_ones(s.A[bp], s.ones, s.W1, tmem);
#else
          issue_layer<64, 32>(s.A[bp], s.W1, tmem);
#endif
          ptx::mma_commit(&s.mbar);
        }
        ptx::mbar_wait(&s.mbar, phase);
        phase ^= 1;
        ptx::tc_fence_after();
        relu64_to_tmem(t_lane, a_lane);
        {
          float sh[16];
          sh_encode(d3{(double)pdx, (double)pdy, (double)pdz}, sh);
          uint32_t wv[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) wv[q] = pack2(sh[2 * q], sh[2 * q + 1]);
          ptx::tmem_st8(t_lane + kShCol, wv);
          ptx::tmem_st_wait();
        }
        ptx::tc_fence_before();
        bar_sync<kBarCons, 128>();
        if (issuer) {
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
        bar_sync<kBarCons, 128>();
        if (issuer) {
          ptx::tc_fence_after();
          issue_layer_ts<64, 64>(a_tmem, ones_tmem, s.C2, tmem);
          ptx::mma_commit(&s.mbar);
        }
        ptx::mbar_wait(&s.mbar, phase);
        phase ^= 1;
        ptx::tc_fence_after();
        relu64_to_tmem(t_lane, a_lane);
        ptx::tc_fence_before();
        bar_sync<kBarCons, 128>();
        if (issuer) {
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
        {
          float rgb[3];
#pragma unroll
          for (int k = 0; k < 3; ++k) {
            const float raw = v32[k];
            rgb[k] = p.mlp.color_space == 0 ? sigmoid_fast(raw) : trunc_exp_fast(raw);
          }
          s.res[ctid] = make_float4(sigma, rgb[0], rgb[1], rgb[2]);
        }
        __syncwarp();
        WS_T(4);
        // ---- C(jm): owners composite their samples of round jm in order ------------------
        uint32_t mine = s.own[bp][warp][lane];
        while (mine && r.alive) {
          const int jj = __ffs(mine) - 1;
          mine &= mine - 1;
          const float4 e = s.res[warp * 32 + jj];
          const int cnd = s.rowcand[bp][warp][jj];
          const double t = __ldg(p.ts + cnd);
          const double delta = (cnd + 1 < p.n) ? dsub(__ldg(p.ts + cnd + 1), t) : dmul(t, dsub(p.ratio, 1.0));
#if WS_F32_ALPHA
          // alpha and the sample's weight in fp32 (the MUFU exp: ~2 ulp, far below the fp16 sigma's
          // error); the transmittance that decides the cut keeps accumulating in double
          const float ef = __expf(-e.x * (float)delta);
          const float wgt = (float)r.trans * (1.f - ef);
          r.px += wgt * e.y;
          r.py += wgt * e.z;
          r.pz += wgt * e.w;
          r.depth += wgt * (float)t;
          r.opac += wgt;
          r.trans = dmul(r.trans, (double)ef);
#else
          const double a = dsub(1.0, exp(dmul(-(double)e.x, delta)));
          const double wgt = dmul(r.trans, a);
          r.px = dadd(r.px, dmul(wgt, (double)e.y));
          r.py = dadd(r.py, dmul(wgt, (double)e.z));
          r.pz = dadd(r.pz, dmul(wgt, (double)e.w));
          r.depth = dadd(r.depth, dmul(wgt, t));
          r.opac = dadd(r.opac, wgt);
          r.trans = dmul(r.trans, dsub(1.0, a));
#endif
          ++r.contributing;
          if (p.t_cut > 0 && r.trans < p.t_cut) {
            r.term = true;
            r.alive = false;
          }
        }
      }
      WS_T(5);
      // a finished packet is stored once its last round is composited (renderer.h:233-236)
      if (packet_live) pkt_cycles += clock64() - t_iter;
      if (pending && jm >= last_round) {
        if (p.row_cycles && (lane & (kPW - 1)) == 0) {  // one lane per packet row
          const long long pk_ = r.id >> 5;
          const int py_ = p.row_begin + (int)(pk_ / packets_x) * kPH + lane / kPW;
          if (py_ < p.row_end) atomicAdd((unsigned long long*)&p.row_cycles[py_], (unsigned long long)(pkt_cycles / kPH));
        }
        pkt_cycles = 0;
        if (r.valid) {
          const long long pk_ = r.id >> 5;
          const int px_ = (int)(pk_ % packets_x) * kPW + (lane % kPW);
          const int py_ = p.row_begin + (int)(pk_ / packets_x) * kPH + lane / kPW;
          const int kept_total = __ldg(p.kept_count + r.id);
          RayResult res{r.px, r.py, r.pz, r.depth, r.opac,
                        chunk_evals(r.term, r.contributing, kept_total, p.chunk), r.contributing};
          store_ray(p, px_, py_, res, r.trans);
        }
        pending = false;
        packet_live = false;
      }
      if (stop_round >= 0 && jm + 1 >= stop_round) break;  // every round with rows composited
    }
#if WS_PAIRS
    // the producers gathered the (empty) stop round: drain it, then wake every producer warp
    // once more with `halt` raised (written by each consumer thread before its own arrive)
    gather_done_sync(b);
    s.halt = 1;
    pair_ready(warp, b + 1 == kStages ? 0 : b + 1, true);
#endif
    ptx::tc_fence_before();
    bar_sync<kBarCons, 128>();
    ptx::tc_fence_after();
    if (warp == 0) ptx::tmem_dealloc<kTmemCols>(tmem);
    add_work_stats(p, cnt.evals, cnt.level_samples, cnt.marched, cnt.rays);
  }
}

}  // namespace ws
}  // namespace lumi_dev

using namespace lumi_dev;

size_t render_ws_smem_bytes() { return sizeof(ws::Smem); }
size_t render_ws_weight_tile_bytes() { return ws::kWeightTileBytes; }

cudaError_t launch_pack_weight_tiles(const MlpDev& mlp, void* img, cudaStream_t s) {
  ws::k_pack_weight_tiles<<<1, 256, 0, s>>>(mlp, static_cast<uint8_t*>(img));
  return cudaGetLastError();
}

// march pass over packet-ordered ray ids + the warp-specialised kernel
cudaError_t launch_render_ws(RenderParams p, cudaStream_t s, int num_sms, cudaEvent_t* ev) {
  const long long rays = (long long)(p.row_end - p.row_begin) * p.cam.width;
  if (rays <= 0) return cudaSuccess;
  static PerDeviceInit once;
  const size_t smem = render_ws_smem_bytes();
  int blocks_per_sm = 0;
  cudaError_t e = once.get([&](int* out) {
    cudaError_t x;
    if ((x = cudaFuncSetAttribute(ws::k_render_ws, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem)) != cudaSuccess)
      return x;
    if ((x = cudaFuncSetAttribute(ws::k_render_ws, cudaFuncAttributePreferredSharedMemoryCarveout,
                                  100)) != cudaSuccess)
      return x;
    int n = 0;
    if ((x = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, ws::k_render_ws, ws::kCtaThreads, smem)) !=
        cudaSuccess)
      return x;
    cudaFuncAttributes fa;
    if ((x = cudaFuncGetAttributes(&fa, ws::k_render_ws)) != cudaSuccess) return x;
    int dev = 0, smem_sm = 0;
    if ((x = cudaGetDevice(&dev)) != cudaSuccess ||
        (x = cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev)) != cudaSuccess)
      return x;
    const int by_regs = 65536 / (((fa.numRegs * 32 + 255) / 256) * 256 * (ws::kCtaThreads / 32));
    const int by_smem = smem_sm / (int)(smem + 1024);
    int b = std::max(1, std::min({by_regs, by_smem, 4}));  // TMEM: 128 columns per CTA
    if (std::getenv("LUMI_MAX_CTAS")) b = std::max(1, std::min(b, std::atoi(std::getenv("LUMI_MAX_CTAS"))));
    // only the shared memory the resident CTAs need; the rest of the 256 KB stays L1 data cache,
    // which the irregular hash-grid gather depends on
    const int carve = (int)std::ceil(100.0 * b * (double)(smem + 1024) / smem_sm);
    if ((x = cudaFuncSetAttribute(ws::k_render_ws, cudaFuncAttributePreferredSharedMemoryCarveout,
                                  std::min(100, carve))) != cudaSuccess)
      return x;
    if (std::getenv("LUMI_DEBUG"))
      std::fprintf(stderr, "[lumi] k_render_ws on device %d: %zu B smem (SM %d), %d regs, occupancy API %d, "
                   "by regs %d, by smem %d -> %d CTAs/SM, carveout %d%%\n", dev, smem, smem_sm, fa.numRegs,
                   n, by_regs, by_smem, b, std::min(100, carve));
    *out = b;
    return cudaSuccess;
  }, &blocks_per_sm);
  if (e != cudaSuccess) return e;
  p.tile_w = pk::kPW;
  p.tile_h = pk::kPH;
  p.tiles_x = (p.cam.width + pk::kPW - 1) / pk::kPW;
  const long long packets =
      (long long)p.tiles_x * ((p.row_end - p.row_begin + pk::kPH - 1) / pk::kPH);
  p.total_rays = packets * 32;
  if (p.total_rays >= (1ll << 31)) return cudaErrorInvalidValue;
  p.mask_words = (p.n + 31) / 32;
  p.mask_transposed = WS_TMASK;
  if ((e = cudaMallocAsync(&p.kept_mask, (size_t)p.total_rays * p.mask_words * 4, s)) != cudaSuccess)
    return e;
  if ((e = cudaMallocAsync(&p.kept_count, (size_t)p.total_rays * 2, s)) != cudaSuccess) return e;
#if WS_MARCH_DIRS
  if ((e = cudaMallocAsync(&p.ray_dirs, (size_t)p.total_rays * 6 * sizeof(float), s)) != cudaSuccess)
    return e;
#endif
  // the packet counter of THIS launch (stream-ordered allocation: concurrent launches on other
  // streams never share it)
  if ((e = cudaMallocAsync(&p.work_counter, 256, s)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(p.work_counter, 0, sizeof(unsigned int), s)) != cudaSuccess) return e;
  RenderParams pm = p;  // the march pass counts the candidates it tests (work_stats[2])
  if (ev) cudaEventRecord(ev[0], s);
  if ((e = launch_march_mask(pm, s)) != cudaSuccess) return e;
  if (ev) cudaEventRecord(ev[1], s);
  const long long grid = std::min<long long>((long long)blocks_per_sm * num_sms, (packets + 3) / 4);
#ifdef LUMI_PHASE_TIMING
  unsigned long long z6[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  cudaMemcpyToSymbolAsync(ws::g_ws_cycles, z6, sizeof(z6), 0, cudaMemcpyHostToDevice, s);
#endif
  ws::k_render_ws<<<(unsigned)grid, ws::kCtaThreads, smem, s>>>(p);
#ifdef LUMI_PHASE_TIMING
  {
    unsigned long long c[8];
    cudaMemcpyFromSymbolAsync(c, ws::g_ws_cycles, sizeof(c), 0, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    const double tp = (double)(c[0] + c[1]), tc = (double)(c[2] + c[3] + c[4] + c[5] + c[6] + c[7]);
    std::fprintf(stderr, "[lumi] ws producers: wait list %.1f%% gather %.1f%% | consumers: stream fill %.1f%% "
                 "geometry %.1f%% fill barrier %.1f%% wait gather %.1f%% mlp %.1f%% composite %.1f%%\n",
                 100 * c[0] / tp, 100 * c[1] / tp, 100 * c[6] / tc, 100 * c[7] / tc, 100 * c[2] / tc,
                 100 * c[3] / tc, 100 * c[4] / tc, 100 * c[5] / tc);
  }
#endif
  if (ev) cudaEventRecord(ev[2], s);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  cudaFreeAsync(p.kept_mask, s);
  cudaFreeAsync(p.kept_count, s);
  cudaFreeAsync(p.work_counter, s);
  if (p.ray_dirs) cudaFreeAsync(p.ray_dirs, s);
  return cudaGetLastError();
}
