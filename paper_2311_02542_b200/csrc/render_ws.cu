// render_ws.cu -- warp-specialised packet renderer (the production frame kernel).
//
// A persistent kernel, 3 CTAs x 8 warps per SM.  Each CTA pairs a CONSUMER warpgroup -- four
// warps, each owning a stream of 8x4 ray packets: the sample stream fill, the tcgen05 MLP and
// the compositing -- with a PRODUCER warpgroup of four warps: each producer thread owns one of
// the round's 128 rows (samples), derives its geometry (position, contraction, LOD) and gathers
// every active hash-grid level of it into the layer-1 A tile.  The two are pipelined one round
// apart through double-buffered A tiles and row inputs, synchronised with named barriers (one
// pair per buffer):
//
//   consumers, iteration j:  fill round j into buffer j&1 (per row: ray lane, candidate; the
//                            packet's directions and SH sit in a shared-memory packet slot)
//                            -> post done flag, arrive LIST_READY[j&1] (no consumer barrier)
//                            -> wait GATHER_DONE[(j-1)&1] -> MLP + composite of round j-1
//   producers, iteration j:  wait LIST_READY[j&1] -> geometry + gather of round j's rows
//                            (software-pipelined over level pairs) -> arrive GATHER_DONE[j&1]
//
// Because round j is filled before round j-1 is composited, a packet whose stream ends is
// stored only after the last round holding its rows is composited (one idle round per packet
// for that warp), and rows of rays that terminate in round j-1 may still be evaluated in round
// j (they are skipped by the compositing, so the result is the reference's).
//
// Variants measured and rejected (DESIGN.md §4 and git history): a shared (row, level) gather
// list, consumers gathering the coarse levels or a row's last level pair, per-warp-pair or
// per-producer-warp list handoff, a third stage, transposed mask words or an expanded per-word
// sample list, producers loading the ray directions or encoding the SH, balanced gather units,
// two producer threads per row, the geometry on the consumers, other packet claim orders.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstddef>
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <vector>

#include "kernels.h"
#include "pk_parts.cuh"

namespace lumi_dev {
namespace ws {

using namespace pk;

constexpr int kProdWarps = 4;                     // producer thread t owns row t of a round
constexpr int kProdThreads = 32 * kProdWarps;
constexpr int kCtaThreads = 128 + kProdThreads;   // consumers [0, 128), producers after
constexpr int kCtasPerSm = 3;
constexpr int kStages = 2;                        // rounds in flight between the warpgroups
// register split (setmaxnreg after the launch allocation of 80 per thread at 3 CTAs x 256
// threads).  Even since the consumers keep no ray directions (packet slots) and the producer
// gather needs no per-pair zero fill: 88 / 72 measured 1.8 % slower (producers spill)
#ifndef WS_CONS_REGS
#define WS_CONS_REGS 80
#endif
#ifndef WS_PROD_REGS
#define WS_PROD_REGS 80
#endif
static_assert(128 * WS_CONS_REGS + kProdThreads * WS_PROD_REGS <=
                  kCtaThreads * (65536 / (kCtaThreads * kCtasPerSm) / 8 * 8),
              "register split exceeds the launch allocation");
// named barriers: 0 = __syncthreads (setup / teardown), LIST_READY 1 + b, GATHER_DONE 3 + b,
// 5 = consumer warpgroup only
constexpr int kBarList = 1, kBarGather = 3, kBarCons = 5;
// No consumer barrier after the fill: each consumer warp posts a done flag and arrives at
// LIST_READY on its own, so fast warps start waiting for the gather while a slow one still
// fills; the producers decide the stop from the four flags and pass it back with GATHER_DONE.
// Producer gather: pk::gather_row, the row's levels two at a time with the next two level pairs'
// corner loads in flight while a pair is combined.


#ifdef LUMI_PHASE_TIMING
// warp-cycles: producers [wait list, gather], consumers [fill barrier, wait gather, MLP,
// composite, stream fill, row handoff]
__device__ unsigned long long g_ws_cycles[8];
// [rounds with rows (per CTA), rows holding a sample, warp-rounds with no row, packets stored]
__device__ unsigned long long g_ws_rows[4];
// per consumer warp: globaltimer at its start and when it leaves the round loop
__device__ unsigned long long g_ws_t[2][4096];
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
  // double-buffered layer-1 A tiles, features only (chunk-major, a_off); the bias step's
  // [1 0 ... 0] block is one shared pair of core matrices read with SBO = 0 by every row group
  uint8_t A[kStages][128 * 32 * 2];
  uint8_t ones[2 * 128];
  // the four fp16 UMMA weight tiles, contiguous: one TMA bulk copy of the per-model image
  uint8_t W1[64 * (32 + kKb) * 2];
  uint8_t F[80 * (80 + kKb) * 2];
  uint8_t C2[64 * (64 + kKb) * 2];
  uint8_t C3[16 * (64 + kKb) * 2];
  uint32_t ballot[kWarps][32];        // per warp: the current mask word, candidate-major
  uint16_t prefix[kWarps][33];        //   and its exclusive per-candidate sample counts
  uint32_t own[kStages][kWarps][32];  // per ray lane: the rows of the round it owns
  uint16_t rowcand[kStages][kWarps][32];
  uint8_t rowlane[kStages][128];
  uint64_t mbar;  // MMA completion
  uint64_t wbar;  // the weight tiles' TMA bulk copy
  uint32_t tmem_base;
  int stop[kStages];
  uint8_t wdone[kStages][kWarps];  // per round: consumer warp w has stored its last packet
  alignas(16) LevelTab lt;
  // per consumer warp, two packet slots (current / next, prefetched by cp.async): the packet's
  // ray and neighbour directions [component][ray lane], from the march pass
  float pdir[2][kWarps][6][32];
  // per consumer warp: its current packet's rays' SH encodings (network.h:17-37) in fp16,
  // computed when the packet starts (the previous packet's rows are all composited by then); a
  // row's SH block is a copy into TMEM
  uint4 psh[kWarps][32][2];
  uint8_t rowslot[kStages][kWarps];  // per round and consumer warp: the slot of its rows' packet
  uint8_t na[kStages][128];    // per row: 1 = the row holds a sample
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

// The shared-memory matrix descriptors of the weight tiles, the A stages and the ones block,
// built from the CTA's layout; a K step only adds its offset to the start-address field
struct MmaDescs {
  uint64_t w1, f, c2, c3, ones, a[kStages];
};
__device__ __forceinline__ MmaDescs make_descs(const Smem& s) {
  MmaDescs d;
  d.w1 = ptx::make_smem_desc(ptx::smem_addr(s.W1), 128, ((32 + kKb) / 8) * 128);
  d.f = ptx::make_smem_desc(ptx::smem_addr(s.F), 128, ((80 + kKb) / 8) * 128);
  d.c2 = ptx::make_smem_desc(ptx::smem_addr(s.C2), 128, ((64 + kKb) / 8) * 128);
  d.c3 = ptx::make_smem_desc(ptx::smem_addr(s.C3), 128, ((64 + kKb) / 8) * 128);
  d.ones = ptx::make_smem_desc(ptx::smem_addr(s.ones), 128, 0);
  for (int b = 0; b < kStages; ++b) d.a[b] = ptx::make_smem_desc(ptx::smem_addr(s.A[b]), kALbo, 128);
  return d;
}
// the start-address field counts 16-byte units
__device__ __forceinline__ uint64_t desc_at(uint64_t d, uint32_t bytes) {
  // a 32-bit add on the low word: the 14-bit address field cannot carry out (smem < 256 KB)
  return ((d >> 32) << 32) | (uint32_t)((uint32_t)d + (bytes >> 4));
}
__device__ __forceinline__ void issue_l1_pre(uint64_t a, uint64_t ones, uint64_t w1, uint32_t d_tmem) {
  constexpr uint32_t idesc = ptx::idesc_f16_f32<128, 64>();
#pragma unroll
  for (int kk = 0; kk < 2; ++kk)
    ptx::mma_f16(d_tmem, desc_at(a, kk * 2 * kALbo), desc_at(w1, kk * 256), idesc, kk > 0 ? 1u : 0u);
  ptx::mma_f16(d_tmem, ones, desc_at(w1, 2 * 256), idesc, 1u);
}
template <int N, int K>
__device__ __forceinline__ void issue_ts_pre(uint32_t a_tmem, uint32_t ones_tmem, uint64_t b, uint32_t d_tmem) {
  constexpr uint32_t idesc = ptx::idesc_f16_f32<128, N>();
#pragma unroll
  for (int kk = 0; kk < K / 16; ++kk)
    ptx::mma_f16_ts(d_tmem, a_tmem + kk * 8, desc_at(b, kk * 256), idesc, kk > 0 ? 1u : 0u);
  ptx::mma_f16_ts(d_tmem, ones_tmem, desc_at(b, (K / 16) * 256), idesc, 1u);
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

// 4-byte cp.async (global -> shared, L1-allocating) and its group handling
__device__ __forceinline__ void cp_async4(float* dst, const float* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(ptx::smem_addr(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// stage-indexed barriers: b < kStages
__device__ __forceinline__ void list_ready_sync(int b) {
  if (b == 0) bar_sync<kBarList, kCtaThreads>();
  else bar_sync<kBarList + 1, kCtaThreads>();
}
__device__ __forceinline__ void list_ready_arrive(int b) {
  if (b == 0) bar_arrive<kBarList, kCtaThreads>();
  else bar_arrive<kBarList + 1, kCtaThreads>();
}
__device__ __forceinline__ void gather_done_sync(int b) {
  if (b == 0) bar_sync<kBarGather, kCtaThreads>();
  else bar_sync<kBarGather + 1, kCtaThreads>();
}
__device__ __forceinline__ void gather_done_arrive(int b) {
  if (b == 0) bar_arrive<kBarGather, kCtaThreads>();
  else bar_arrive<kBarGather + 1, kCtaThreads>();
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
  const float t = __ldg(p.tdf + cand).x;
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
  if (tid < 16) st16(s.ones, (uint32_t)tid * 16u, make_uint4(tid < 8 ? 0x3C00u : 0u, 0u, 0u, 0u));
  level_tab_init(s.lt, p.grid, tid, kCtaThreads);
  if (tid == 0) {
    ptx::mbar_init(&s.mbar, 1);
    ptx::fence_mbar_init();
  }
  if (tid < 32) ptx::tmem_alloc<kTmemCols>(&s.tmem_base);
  ptx::fence_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = s.tmem_base;
  // the warpgroup giving registers up decreases first, the other one increases (with an even
  // split both "increase" to the launch allocation: a no-op in hardware, but it lets ptxas
  // allocate each warpgroup's code on its own -- without it the kernel spills)
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
#ifdef LUMI_PHASE_TIMING
  long long t_last = clock64();
#endif

  if (wg == 1) {
    // ================================ producers ==============================================
    const GeomConst gc{make_float3((float)p.cam.origin[0], (float)p.cam.origin[1], (float)p.cam.origin[2]),
                       (float)p.grid.two_base, (float)(1.0 / p.grid.log_scale), (float)p.lod_bias,
                       p.grid.levels};
    unsigned pcnt_levels = 0;
    int b = 0;  // j % kStages
#pragma unroll 1
    for (int j = 0;; ++j, b ^= 1) {
      list_ready_sync(b);
      WS_T(0);
      {
        const bool stop = s.wdone[b][0] & s.wdone[b][1] & s.wdone[b][2] & s.wdone[b][3];
        if (ctid == 0) s.stop[b] = stop ? 1 : 0;
        if (stop) {  // round j holds no rows: tell the consumers through its GATHER_DONE
          gather_done_arrive(b);
          break;
        }
      }
      // row ctid: its ray directions and candidate from the consumers -> grid coordinates, LOD
      // (fl) and active level count.  The 32 rows of a warp are neighbouring rays of one packet
      // at nearly the same distance, so their LOD (hence their level count) is nearly uniform
      // and the lanes of a warp walk the same level together (coherent hash cells,
      // warp-uniform dense/hashed branch).
      float4 P = make_float4(0.f, 0.f, 0.f, 0.f);
      int na = 0;
      if (s.na[b][ctid]) {
        const float(*pd)[32] = s.pdir[s.rowslot[b][warp]][warp];
        const int rl = s.rowlane[b][ctid];
        na = row_geometry(p, gc, make_float3(pd[0][rl], pd[1][rl], pd[2][rl]),
                          make_float3(pd[3][rl], pd[4][rl], pd[5][rl]), s.rowcand[b][warp][lane], P);
        pcnt_levels += (unsigned)na;
      }
      const int na_max = __reduce_max_sync(FULL, (unsigned)na);
      {
        uint8_t* arow = s.A[b] + a_off(ctid, 0);
        int nst = 0;
        gather_row(s.lt, na_max, P.x, P.y, P.z, P.w, [&](int c, uint4 q) {
          st16(arow, (uint32_t)c * kALbo, q);
          nst = c + 1;
        });
        for (int c = nst; c < kMaxLevels / 4; ++c) st16(arow, (uint32_t)c * kALbo, make_uint4(0u, 0u, 0u, 0u));
      }
      ptx::fence_async_smem();
      gather_done_arrive(b);
      WS_T(1);
    }
    add_work_stats(p, 0, pcnt_levels, 0, 0);
  } else {
    // ================================ consumers ==============================================
    if (tma_weights) ptx::mbar_wait(&s.wbar, 0);  // the weight tiles have landed
#ifdef LUMI_PHASE_TIMING
    if (lane == 0 && blockIdx.x * 4 + warp < 4096) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      g_ws_t[0][blockIdx.x * 4 + warp] = t;
    }
#endif
    const uint32_t t_lane = tmem + ((uint32_t)(warp * 32) << 16);
    {
      const uint32_t ones[8] = {0x3C00u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
      ptx::tmem_st8(t_lane + kOnesCol, ones);
      ptx::tmem_st_wait();
      ptx::tc_fence_before();
      bar_sync<kBarCons, 128>();
      ptx::tc_fence_after();
    }
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
    // one packet id and one mask word ahead: the atomic and the word load are off the fill's
    // dependency chain
    long long next_pkt = 0;
    if (lane == 0) next_pkt = (long long)atomicAdd(p.work_counter, 1u);
    uint32_t next_bits = 0;
    // the next packet's first mask word, loaded once its id has arrived (the round after the
    // atomic was issued)
    uint32_t next_first = 0;
    bool nf_ready = false;
    int slot = 1;  // the current packet's direction slot (the first packet flips it to 0)
    uint32_t phase = 0;
    // the SM clock (low 32 bits) when the current packet started: its cycles at the store are the
    // RowStats.ms diagnostic (a packet lasts far less than 2^32 cycles)
    uint32_t pkt_t0 = 0;

    int b = 0;  // j % kStages
#pragma unroll 1
    for (int j = 0;; ++j, b ^= 1) {
      {
        // ---- F(j): this warp's rows of round j from its packet stream ---------------------
        int take = 0, rl = lane, cand = 0;
        if (!nf_ready) {
          const long long np = __shfl_sync(FULL, next_pkt, 0);
          next_first = np < total_packets ? __ldg(p.kept_mask + np * 32 + lane) : 0u;
          if (np < total_packets) {
            // the next packet's directions into the other slot (free: the packet that used it
            // had every round gathered before the current one could start)
            const size_t T = (size_t)p.total_rays;
            const float* rd = p.ray_dirs + np * 32 + lane;
#pragma unroll
            for (int k = 0; k < 6; ++k) cp_async4(&s.pdir[slot ^ 1][warp][k][lane], rd + k * T);
            cp_async_commit();
          }
          nf_ready = true;
        }
        while (take < 32 && !no_more && !pending) {
          if (!packet_live) {
            long long pkt = 0;
            if (lane == 0) {
              pkt = next_pkt;
              next_pkt = (long long)atomicAdd(p.work_counter, 1u);
            }
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
            if (r.valid) ++cnt.rays;
            cp_async_wait_all();  // its directions (prefetched a round or more ago)
            __syncwarp();
            slot ^= 1;
            {
              float sh[16];
              sh_encode(d3{(double)s.pdir[slot][warp][0][lane], (double)s.pdir[slot][warp][1][lane],
                           (double)s.pdir[slot][warp][2][lane]}, sh);
              s.psh[warp][lane][0] = make_uint4(pack2(sh[0], sh[1]), pack2(sh[2], sh[3]),
                                                      pack2(sh[4], sh[5]), pack2(sh[6], sh[7]));
              s.psh[warp][lane][1] = make_uint4(pack2(sh[8], sh[9]), pack2(sh[10], sh[11]),
                                                      pack2(sh[12], sh[13]), pack2(sh[14], sh[15]));
            }
            r.contributing = 0;
            r.term = false;
            r.trans = 1.0;
            r.px = r.py = r.pz = r.depth = r.opac = 0.0;
            packet_live = true;
            pkt_t0 = (uint32_t)clock();
            word = -1;
            g_next = word_total = 0;
            next_bits = next_first;  // (bits of invalid rays are masked by r.alive)
            nf_ready = false;
          }
          if (g_next < word_total) {
            // lanes [take, take + n): the next samples of the current word, candidate-major
            const int n = min(32 - take, word_total - g_next);
            if (lane >= take && lane < take + n) {
              const int g = g_next + (lane - take);
              int lo = 0;
#pragma unroll
              for (int st = 16; st > 0; st >>= 1)
                if (s.prefix[warp][lo + st] <= g) lo += st;
              rl = nth_set_bit(s.ballot[warp][lo], g - s.prefix[warp][lo]);
              cand = word * 32 + lo;
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
          const uint32_t bits = r.alive ? next_bits : 0u;
          if (word + 1 < p.mask_words && r.alive)
            next_bits = __ldg(p.kept_mask + (size_t)(word + 1) * p.total_rays + r.id);
          // lane i: the rays keeping candidate word * 32 + i (a 32x32 bit transpose across the
          // warp instead of 32 ballots), then an exclusive scan of the per-candidate counts
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
        // the producers find the row's directions by its packet slot and ray lane
        if (have) ++cnt.evals;
#ifdef LUMI_PHASE_TIMING
        {
          const unsigned nh = __popc(__ballot_sync(FULL, have));
          if (lane == 0) {
            atomicAdd(&g_ws_rows[1], (unsigned long long)nh);
            if (nh == 0) atomicAdd(&g_ws_rows[2], 1ull);
            if (warp == 0) atomicAdd(&g_ws_rows[0], 1ull);
          }
        }
#endif
        s.na[b][ctid] = have ? 1 : 0;
        if (lane == 0) s.rowslot[b][warp] = (uint8_t)slot;
        WS_T(7);
        if (lane == 0) s.wdone[b][warp] = (no_more && !packet_live) ? 1 : 0;
        list_ready_arrive(b);
        WS_T(2);
      }

      // the round whose MLP and compositing run now: one round behind the fill
      const int jm = j - 1;
      if (jm >= 0) {
        // ---- M(jm): the tcgen05 MLP over round jm's 128 rows (field.h:106-137) -------------
        const int bp = b ^ 1;  // jm % kStages
        gather_done_sync(bp);
        if (s.stop[bp]) break;  // round jm is the first with no rows anywhere: every packet stored
        WS_T(3);
        const int rlp = s.rowlane[bp][ctid];
        const uint4* shp = s.psh[warp][rlp];
        if (issuer) {
          ptx::tc_fence_after();
          {
            const MmaDescs dd = make_descs(s);
            issue_l1_pre(bp ? dd.a[1] : dd.a[0], dd.ones, dd.w1, tmem);
          }
          ptx::mma_commit(&s.mbar);
        }
        {
          // the row's SH block into its TMEM columns while layer 1 runs (the MMA writes columns
          // [0, 64); the previous round's fused layer, the last reader, has completed)
          const uint4 h0 = shp[0], h1 = shp[1];
          const uint32_t wv[8] = {h0.x, h0.y, h0.z, h0.w, h1.x, h1.y, h1.z, h1.w};
          ptx::tmem_st8(t_lane + kShCol, wv);
        }
        ptx::mbar_wait(&s.mbar, phase);
        phase ^= 1;
        ptx::tc_fence_after();
        relu64_to_tmem(t_lane, a_lane);  // (its store wait covers the SH block)
        ptx::tc_fence_before();
        bar_sync<kBarCons, 128>();
        if (issuer) {
          ptx::tc_fence_after();
          issue_ts_pre<80, 80>(a_tmem, ones_tmem, make_descs(s).f, tmem);
          ptx::mma_commit(&s.mbar);
        }
        ptx::mbar_wait(&s.mbar, phase);
        phase ^= 1;
        ptx::tc_fence_after();
        const float sigma_raw = ptx::tmem_ld1(t_lane + 64);  // (the epilogue's first load wait covers it)
        relu64_to_tmem(t_lane, a_lane);
        const float sigma = trunc_exp_fast(sigma_raw);
        ptx::tc_fence_before();
        bar_sync<kBarCons, 128>();
        if (issuer) {
          ptx::tc_fence_after();
          issue_ts_pre<64, 64>(a_tmem, ones_tmem, make_descs(s).c2, tmem);
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
          issue_ts_pre<16, 64>(a_tmem, ones_tmem, make_descs(s).c3, tmem);
          ptx::mma_commit(&s.mbar);
        }
        ptx::mbar_wait(&s.mbar, phase);
        phase ^= 1;
        ptx::tc_fence_after();
        float v4[4];
        ptx::tmem_ld4(t_lane, v4);
        ptx::tmem_ld_wait();
        ptx::tc_fence_before();
        {
          float rgb[3];
#pragma unroll
          for (int k = 0; k < 3; ++k) {
            const float raw = v4[k];
            rgb[k] = p.mlp.color_space == 0 ? sigmoid_fast(raw) : trunc_exp_fast(raw);
          }
          // per row (sigma, rgb) for the compositing, in the first 2 KB of the round's A tile:
          // its last reader (layer 1) has completed, and the producers refill it only after
          // the next list handoff
          reinterpret_cast<float4*>(s.A[bp])[ctid] = make_float4(sigma, rgb[0], rgb[1], rgb[2]);
        }
        __syncwarp();
        WS_T(4);
        // ---- C(jm): owners composite their samples of round jm in order ------------------
        uint32_t mine = s.own[bp][warp][lane];
        while (mine && r.alive) {
          const int jj = __ffs(mine) - 1;
          mine &= mine - 1;
          const float4 e = reinterpret_cast<const float4*>(s.A[bp])[warp * 32 + jj];
          const int cnd = s.rowcand[bp][warp][jj];
          const float2 td = __ldg(p.tdf + cnd);  // (float)t, (float)delta (host, renderer.h:209)
          // alpha and the sample's weight in fp32 (the MUFU exp: ~2 ulp, far below the fp16
          // sigma's error); the transmittance that decides the cut accumulates in double
          const float ef = __expf(-e.x * td.y);
          const float wgt = (float)r.trans * (1.f - ef);
          r.px += wgt * e.y;
          r.py += wgt * e.z;
          r.pz += wgt * e.w;
          r.depth += wgt * td.x;
          r.opac += wgt;
          r.trans = dmul(r.trans, (double)ef);
          ++r.contributing;
          if (p.t_cut > 0 && r.trans < p.t_cut) {
            r.term = true;
            r.alive = false;
          }
        }
      }
      WS_T(5);
      // a finished packet is stored once its last round is composited (renderer.h:233-236)
      if (pending && jm >= last_round) {
        if (p.row_cycles && (lane & (kPW - 1)) == 0) {  // one lane per packet row
          const long long pk_ = r.id >> 5;
          const int py_ = p.row_begin + (int)(pk_ / packets_x) * kPH + lane / kPW;
          const uint32_t pkt_cycles = (uint32_t)clock() - pkt_t0;
          if (py_ < p.row_end) atomicAdd((unsigned long long*)&p.row_cycles[py_], (unsigned long long)(pkt_cycles / kPH));
        }
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
#ifdef LUMI_PHASE_TIMING
        if (lane == 0) atomicAdd(&g_ws_rows[3], 1ull);
#endif
      }
    }
#ifdef LUMI_PHASE_TIMING
    if (lane == 0 && blockIdx.x * 4 + warp < 4096) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      g_ws_t[1][blockIdx.x * 4 + warp] = t;
    }
#endif
    ptx::tc_fence_before();
    bar_sync<kBarCons, 128>();
    ptx::tc_fence_after();
    if (warp == 0) ptx::tmem_dealloc<kTmemCols>(tmem);
    add_work_stats(p, cnt.evals, 0, cnt.marched, cnt.rays);
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
  if ((e = cudaMallocAsync(&p.kept_mask, (size_t)p.total_rays * p.mask_words * 4, s)) != cudaSuccess)
    return e;
  if ((e = cudaMallocAsync(&p.kept_count, (size_t)p.total_rays * 2, s)) != cudaSuccess) return e;
  if ((e = cudaMallocAsync(&p.ray_dirs, (size_t)p.total_rays * 6 * sizeof(float), s)) != cudaSuccess)
    return e;
  // the packet counter of THIS launch (stream-ordered allocation: concurrent launches on other
  // streams never share it)
  if ((e = cudaMallocAsync(&p.work_counter, 256, s)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(p.work_counter, 0, sizeof(unsigned int), s)) != cudaSuccess) return e;
  if (ev) cudaEventRecord(ev[0], s);
  if ((e = launch_march_mask(p, s)) != cudaSuccess) return e;  // counts its candidates (work_stats[2])
  if (ev) cudaEventRecord(ev[1], s);
  const long long grid = std::min<long long>((long long)blocks_per_sm * num_sms, (packets + 3) / 4);
#ifdef LUMI_PHASE_TIMING
  unsigned long long z6[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  cudaMemcpyToSymbolAsync(ws::g_ws_cycles, z6, sizeof(z6), 0, cudaMemcpyHostToDevice, s);
  cudaMemcpyToSymbolAsync(ws::g_ws_rows, z6, sizeof(ws::g_ws_rows), 0, cudaMemcpyHostToDevice, s);
#endif
  ws::k_render_ws<<<(unsigned)grid, ws::kCtaThreads, smem, s>>>(p);
#ifdef LUMI_PHASE_TIMING
  {
    unsigned long long c[8];
    cudaMemcpyFromSymbolAsync(c, ws::g_ws_cycles, sizeof(c), 0, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    const double tp = (double)(c[0] + c[1]), tc = (double)(c[2] + c[3] + c[4] + c[5] + c[6] + c[7]);
    std::fprintf(stderr, "[lumi] ws producers: wait list %.1f%% geometry+gather %.1f%% | consumers: stream fill %.1f%% "
                 "row handoff %.1f%% fill barrier %.1f%% wait gather %.1f%% mlp %.1f%% composite %.1f%%\n",
                 100 * c[0] / tp, 100 * c[1] / tp, 100 * c[6] / tc, 100 * c[7] / tc, 100 * c[2] / tc,
                 100 * c[3] / tc, 100 * c[4] / tc, 100 * c[5] / tc);
    unsigned long long rw[4];
    cudaMemcpyFromSymbol(rw, ws::g_ws_rows, sizeof(rw));
    std::fprintf(stderr, "[lumi] ws rounds %llu, rows with a sample %llu (%.1f%% of 128 per round), "
                 "warp-rounds with no row %llu (%.1f%%), packets %llu\n", rw[0], rw[1],
                 100.0 * rw[1] / (128.0 * rw[0]), rw[2], 100.0 * rw[2] / (4.0 * rw[0]), rw[3]);
    // the launch's tail: consumer warps that ran out of packets before the last one finished
    static unsigned long long tt[2][4096];
    cudaMemcpyFromSymbol(tt, ws::g_ws_t, sizeof(tt));
    const int nw = (int)std::min<long long>(4 * grid, 4096);
    unsigned long long t0 = ~0ull, t1 = 0;
    for (int i = 0; i < nw; ++i) { t0 = std::min(t0, tt[0][i]); t1 = std::max(t1, tt[1][i]); }
    double idle = 0.0;
    std::vector<double> ends(nw);
    for (int i = 0; i < nw; ++i) { idle += (double)(t1 - tt[1][i]); ends[i] = (double)(tt[1][i] - t0) * 1e-3; }
    std::sort(ends.begin(), ends.end());
    std::fprintf(stderr, "[lumi] ws tail: span %.1f us, warps done at p1 %.1f / p50 %.1f / max %.1f us, "
                 "idle warp-time after their last packet %.2f%%\n", (t1 - t0) * 1e-3, ends[nw / 100],
                 ends[nw / 2], ends[nw - 1], 100.0 * idle / ((double)nw * (double)(t1 - t0)));
  }
#endif
  if (ev) cudaEventRecord(ev[2], s);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  cudaFreeAsync(p.kept_mask, s);
  cudaFreeAsync(p.kept_count, s);
  cudaFreeAsync(p.work_counter, s);
  cudaFreeAsync(p.ray_dirs, s);
  return cudaGetLastError();
}
