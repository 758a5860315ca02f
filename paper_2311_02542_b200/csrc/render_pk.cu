// render_pk.cu -- packet-coherent B200 frame renderer.
//
// Each warp owns a PACKET of 32 neighbouring rays (an 8x4 pixel patch) and streams the
// packet's occupancy-kept samples in candidate-major order: all rays' samples at candidate i
// before those at i+1.  Every round a warp contributes 32 consecutive samples of its stream
// as its 32 rows of the CTA's 128-row MLP batch, so the rows of a warp are neighbouring rays
// at the same distance -- they gather neighbouring (often identical) hash-grid cells, which
// is what keeps the L1 wavefront count per gather low.  The batch then runs through four
// tcgen05 layers (density L2 folded into colour L1), and each ray's owner lane composites its
// samples of the round in order (renderer.h:170-190).  The production renderer, render_ws.cu,
// runs the same stages warp-specialised; this kernel stays as LUMI_KERNEL=packet.
//
// Per-sample geometry for the network input is fp32 (position, contraction, LOD footprint):
// the oracle measures no change against double coordinates (1.24e-4 vs 1.36e-4 max |dPQ| on
// a 2K band of the T=2^22 model, both dominated by the fp16 MLP operands).  The occupancy
// test that selects the samples stays the bit-exact double march pass.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "kernels.h"
#include "render_common.cuh"
#include "tc_ptx.cuh"
#include "pk_parts.cuh"

namespace lumi_dev {
namespace pk {

#ifdef LUMI_PHASE_TIMING
// per-phase warp-cycles (instrumented builds only): fill, geometry, gather, CTA sync, MLP,
// composite, round barrier
__device__ unsigned long long g_phase_cycles_pk[7];
__device__ unsigned long long g_counts_pk[4];  // warp-rounds, rows, gather passes, pairs
#endif

// UMMA no-swizzle operands need 16-byte alignment only; the struct is used straight from
// the dynamic __shared__ array so every access compiles to LDS/STS (not generic LD/ST).
struct __align__(16) Smem {
  // K-major core-matrix tiles; every layer carries its bias as one extra K = 16 block
  // (bias in column K of B, a constant [1 0 ... 0] block in A), so epilogues add nothing
  uint8_t A[128 * (32 + kKb) * 2];  // layer-1 input: hash-grid features + ones block
  uint8_t W1[64 * (32 + kKb) * 2];  // density L1  N=64 K=32
  uint8_t F[80 * (80 + kKb) * 2];   // density L2 folded into colour L1: N=80 (65 used) K=64+16
  uint8_t C2[64 * (64 + kKb) * 2];  // colour L2   N=64 K=64
  uint8_t C3[16 * (64 + kKb) * 2];  // colour L3   N=16 (3 used) K=64
  float4 res[kThreads];     // per row: sigma, r, g, b (row lane -> owner lane)
  uint32_t ballot[kWarps][32];   // per warp: lanes with candidate bit i of the current word
  uint16_t prefix[kWarps][33];   // exclusive prefix of popc(ballot[i])
  uint32_t own[kWarps][32];      // per ray lane: the rows of this round holding its samples
  uint16_t rowcand[kWarps][32];  // per row: its candidate index
  uint64_t mbar;
  uint32_t tmem_base;
  uint4 lvl[kMaxLevels];         // per level: res, hash mask (0 = dense), level base address (lo, hi)
  float4 samp[kWarps][32];       // per row: grid coordinates u, v, w and the LOD fraction
  uint16_t pairs[kWarps][32 * kMaxLevels];  // (sample, level) gather list: row | l<<5
};

__global__ void __launch_bounds__(kThreads, 4) k_render_pk(RenderParams p) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  Smem& s = *reinterpret_cast<Smem*>(smem_raw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const unsigned FULL = 0xffffffffu;

  // ---- setup: weights, biases, mbarrier, TMEM ------------------------------------------
  const float* dp = p.mlp.dparams;
  const float* cp = p.mlp.cparams;
  const float* c2 = cp + 64 * 32 + 64;
  const float* c3 = c2 + 64 * 64 + 64;
  load_weight_tile(s.W1, dp, 64, 64, 32);
  load_weight_tile(s.F, p.mlp.fused, kHidden + 1, 80, 80);
  load_weight_tile(s.C2, c2, 64, 64, 64);
  load_weight_tile(s.C3, c3, 3, 16, 64);
  // this row's constant ones block of the layer-1 A tile (never overwritten)
  st16(s.A, a_off(tid, 4), make_uint4(0x3C00u, 0u, 0u, 0u));  // fp16 1.0
  st16(s.A, a_off(tid, 5), make_uint4(0u, 0u, 0u, 0u));
  for (int l = tid; l < kMaxLevels; l += kThreads) {
    const int res = l < p.grid.levels ? p.grid.res[l] : 1;
    const bool dense = (p.grid.dense_mask >> l) & 1u;
    const unsigned long long base =
        reinterpret_cast<unsigned long long>(p.grid.table16 + (l < p.grid.levels ? p.grid.offset2[l] : 0));
    s.lvl[l] = make_uint4((uint32_t)res, dense ? 0u : p.grid.hash_mask[l], (uint32_t)base,
                          (uint32_t)(base >> 32));
  }
  if (tid == 0) {
    ptx::mbar_init(&s.mbar, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 0) ptx::tmem_alloc<kTmemCols>(&s.tmem_base);
  ptx::fence_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = s.tmem_base;
  const uint32_t t_lane = tmem + ((uint32_t)(warp * 32) << 16);
  {  // this lane's constant ones block of the hidden layers' TMEM A operand
    const uint32_t ones[8] = {0x3C00u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
    ptx::tmem_st8(t_lane + kOnesCol, ones);
    ptx::tmem_st_wait();
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
  }

  const float3 o = make_float3((float)p.cam.origin[0], (float)p.cam.origin[1], (float)p.cam.origin[2]);
  const float two_base = (float)p.grid.two_base, inv_log = (float)(1.0 / p.grid.log_scale);
  const int levels = p.grid.levels;
  const long long packets_x = p.tiles_x;
  const long long total_packets = p.total_rays / 32;

  Counters cnt{0, 0, 0, 0};
  Ray r;
  r.valid = r.alive = false;
  // warp-uniform packet stream state
  bool packet_live = false, no_more = false;
  int word = 0;        // current mask word of the packet
  int g_next = 0;      // next stream position inside the word
  int word_total = 0;  // samples in the word
  uint32_t phase = 0;
  const bool issuer = (tid == 0);
#ifdef LUMI_PHASE_TIMING
  long long pt[7] = {0, 0, 0, 0, 0, 0, 0}, pt_last = clock64();
#define PT_MARK(k)                  \
  do {                              \
    __syncwarp();                   \
    const long long _t = clock64(); \
    pt[k] += _t - pt_last;          \
    pt_last = _t;                   \
  } while (0)
#else
#define PT_MARK(k) \
  do {             \
  } while (0)
#endif

  for (;;) {
    // ---- A: this warp's 32 rows: the next samples of its packet stream, across as many
    //      mask words as it takes to fill the round (a round never mixes packets) ---------
    int take = 0;     // rows filled this round
    int ci = 0, rl = lane, cand = 0;  // this row lane's candidate slot / ray lane / candidate
    while (take < 32 && !no_more) {
      if (!packet_live) {
        if (take > 0) break;
        long long pkt = 0;
        if (lane == 0) pkt = (long long)atomicAdd(p.work_counter, 1u);
        pkt = __shfl_sync(FULL, pkt, 0);
        if (pkt >= total_packets) {
          no_more = true;
          break;
        }
        const long long rid = pkt * 32 + lane;
        r.x = (int)(pkt % packets_x) * kPW + (lane % kPW);
        r.y = p.row_begin + (int)(pkt / packets_x) * kPH + lane / kPW;
        r.id = (int)rid;
        r.valid = r.x < p.cam.width && r.y < p.row_end;
        r.alive = r.valid;
        if (r.valid) {
          const d3 dd = ray_dir(p.cam, (double)r.x + 0.5, (double)r.y + 0.5);
          const d3 nn = ray_dir(p.cam, (double)r.x + 1.5, (double)r.y + 0.5);
          r.d = make_float3((float)dd.x, (float)dd.y, (float)dd.z);
          r.nd = make_float3((float)nn.x, (float)nn.y, (float)nn.z);
          r.kept_total = __ldg(p.kept_count + rid);
          ++cnt.rays;
          cnt.marched += p.n;
        }
        r.contributing = 0;
        r.term = false;
        r.trans = 1.0;
        r.px = r.py = r.pz = r.depth = r.opac = 0.0;
        packet_live = true;
        word = -1;
        g_next = word_total = 0;
      }
      if (g_next < word_total) {
        // rows [take, take + n) <- stream positions [g_next, g_next + n) of the current word
        const int n = min(32 - take, word_total - g_next);
        if (lane >= take && lane < take + n) {
          const int g = g_next + (lane - take);
          int lo = 0;  // largest i with prefix[i] <= g
#pragma unroll
          for (int st = 16; st > 0; st >>= 1)
            if (s.prefix[warp][lo + st] <= g) lo += st;
          ci = lo;
          rl = nth_set_bit(s.ballot[warp][ci], g - s.prefix[warp][ci]);
          cand = word * 32 + ci;
        }
        take += n;
        g_next += n;
        continue;
      }
      if (word + 1 >= p.mask_words) {
        if (take > 0) break;  // composite this round first; the pixels are stored next round
        // packet exhausted: owners store their pixels (renderer.h:233-236, 267-276)
        if (r.valid) {
          RayResult res{r.px, r.py, r.pz, r.depth, r.opac,
                        chunk_evals(r.term, r.contributing, r.kept_total, p.chunk),
                        r.contributing};
          store_ray(p, r.x, r.y, res, r.trans);
        }
        packet_live = false;
        continue;
      }
      ++word;
      const uint32_t bits = r.alive ? __ldg(p.kept_mask + (size_t)word * p.total_rays + r.id) : 0u;
      int run = 0;
      for (int i = 0; i < 32; ++i) {
        const uint32_t b = __ballot_sync(FULL, (bits >> i) & 1u);
        if (lane == 0) {
          s.ballot[warp][i] = b;
          s.prefix[warp][i] = (uint16_t)run;
        }
        run += __popc(b);
      }
      if (lane == 0) s.prefix[warp][32] = (uint16_t)run;
      __syncwarp();
      g_next = 0;
      word_total = run;
    }
    PT_MARK(0);

    // row lane: its ray and network-input geometry
    const bool have = lane < take;
    {  // owner lanes learn which rows of the round hold their ray's samples
      s.own[warp][lane] = 0u;
      __syncwarp();
      const unsigned same = __match_any_sync(FULL, have ? rl : 32 + lane);
      if (have) {
        s.own[warp][rl] = same;
        s.rowcand[warp][lane] = (uint16_t)cand;
      }
      __syncwarp();
    }
    const float dx = __shfl_sync(FULL, r.d.x, rl), dy = __shfl_sync(FULL, r.d.y, rl),
                dz = __shfl_sync(FULL, r.d.z, rl);
    const float nx = __shfl_sync(FULL, r.nd.x, rl), ny = __shfl_sync(FULL, r.nd.y, rl),
                nz = __shfl_sync(FULL, r.nd.z, rl);
    float u = 0.f, v = 0.f, w = 0.f;
    LodW lw{0, 0.f, false};
    int na = 0;
    if (have) {
      const float t = (float)__ldg(p.ts + cand);
      const float3 c = contract_f(make_float3(o.x + dx * t, o.y + dy * t, o.z + dz * t), p.contraction);
      u = __saturatef((c.x + 2.f) * 0.25f);
      v = __saturatef((c.y + 2.f) * 0.25f);
      w = __saturatef((c.z + 2.f) * 0.25f);
      if (p.lod_enabled) {
        const float3 b = contract_f(make_float3(o.x + nx * t, o.y + ny * t, o.z + nz * t), p.contraction);
        const float ex = c.x - b.x, ey = c.y - b.y, ez = c.z - b.z;
        const float rc = fmaxf(0.5f * sqrtf(ex * ex + ey * ey + ez * ez), 1e-12f);
        const float l = fminf(-__logf(two_base * rc) * inv_log, (float)(levels - 1));
        lw = lod_weights_f(l + (float)p.lod_bias, levels);
      } else {
        lw = LodW{levels, 0.f, false};
      }
      na = active_levels(lw, levels);
      cnt.level_samples += na;
    }

    PT_MARK(1);
    // ---- B: warp-cooperative hash-grid gather, level-major (sample, level) pairs ----------
    {
      const uint4 zero = make_uint4(0, 0, 0, 0);
#pragma unroll
      for (int j = 0; j < 4; ++j) st16(s.A, a_off(tid, j), zero);
      // LOD weights as one number: w_l = saturate(fl - l) with fl = full + frac (grid.cpp:15-37;
      // 1e-4 for the floor-only case, levels for all-on)
      const float fl = lw.floor_only ? 1e-4f : (float)lw.full + lw.frac;
      if (have) s.samp[warp][lane] = make_float4(u, v, w, fl);
      uint16_t* pc = s.pairs[warp];
      const unsigned lt = (1u << lane) - 1u;
      int npairs = 0;
      for (int l = 0; l < levels; ++l) {
        const unsigned m = __ballot_sync(FULL, na > l);
        if (m == 0u) break;  // active levels are a prefix [0, na)
        if (na > l) {
          pc[npairs + __popc(m & lt)] = (uint16_t)pair_code(lane, l);
        }
        npairs += __popc(m);
      }
      __syncwarp();
      uint8_t* Abase = s.A + a_off(warp * 32, 0);
      const uint8_t* Pbase = reinterpret_cast<const uint8_t*>(s.samp[warp]);
#ifdef LUMI_PHASE_TIMING
      if (lane == 0) {
        atomicAdd(&g_counts_pk[2], (unsigned long long)((npairs + 32 * kPairs - 1) / (32 * kPairs)));
        atomicAdd(&g_counts_pk[3], (unsigned long long)npairs);
      }
#endif
#pragma unroll 1
      for (int base = 0; base < npairs; base += 32 * kPairs) {
        uint32_t code[kPairs];
        float2 f[kPairs];
#pragma unroll
        for (int q = 0; q < kPairs; ++q) {
          const int pi = base + 32 * q + lane;
          code[q] = pi < npairs ? (uint32_t)pc[pi] : 0xffffu;
        }
#pragma unroll
        for (int q = 0; q < kPairs; ++q) {
          f[q] = make_float2(0.f, 0.f);
          if (code[q] != 0xffffu) {
            const float4 P = *reinterpret_cast<const float4*>(Pbase + (code[q] & 0x1F0u));
            const int lv = pair_level(code[q]);
            const float wl = __saturatef(P.w - (float)lv);
            f[q] = gather_level(s.lvl[lv], P.x, P.y, P.z, wl);
          }
        }
#pragma unroll
        for (int q = 0; q < kPairs; ++q)
          if (code[q] != 0xffffu)
            *reinterpret_cast<__half2*>(Abase + code[q]) = __floats2half2_rn(f[q].x, f[q].y);
      }
    }
    ptx::fence_async_smem();
    PT_MARK(2);
#ifdef LUMI_PHASE_TIMING
    if (lane == 0) {
      atomicAdd(&g_counts_pk[0], 1ull);
      atomicAdd(&g_counts_pk[1], (unsigned long long)take);
    }
#endif
    if (!__syncthreads_or(have)) {
      if (__syncthreads_and(no_more)) break;  // every warp's stream is exhausted
      continue;
    }
    PT_MARK(3);

    // ---- MLP: four tcgen05 layers (density L2 folded into colour L1) over the 128-row batch (field.h:106-137) -------------
    float v32[32];
    // layer 1 reads the gathered features from shared memory (SS form); the hidden layers
    // keep their fp16 activations in TMEM columns [kAcol, kAcol + K/2) as the A operand
    // (TS form), so epilogues store with tcgen05.st and never touch shared memory.
    const uint32_t a_tmem = tmem + kAcol, ones_tmem = tmem + kOnesCol;
    const uint32_t a_lane = t_lane + kAcol;
    if (issuer) {
      ptx::tc_fence_after();
      issue_layer<64, 32>(s.A, s.W1, tmem);
      ptx::mma_commit(&s.mbar);
    }
    ptx::mbar_wait(&s.mbar, phase);
    phase ^= 1;
    ptx::tc_fence_after();
    relu64_to_tmem(t_lane, a_lane);
    {  // the colour network's direction input, SH degree 3 (network.h:17-37), next to h
      float sh[16];
      sh_encode(d3{(double)dx, (double)dy, (double)dz}, sh);
      uint32_t wv[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) wv[j] = pack2(sh[2 * j], sh[2 * j + 1]);
      ptx::tmem_st8(t_lane + kShCol, wv);
      ptx::tmem_st_wait();
    }
    ptx::tc_fence_before();
    __syncthreads();

    // density L2 + colour L1 as one layer on [h, sh] (lumi_api.cu fuse_l2_c1): outputs 0..63
    // are the colour hidden pre-activations, output 64 is sigma's
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
    __syncthreads();

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
    __syncthreads();

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
    if (have) {
      float rgb[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const float raw = v32[k];
        rgb[k] = p.mlp.color_space == 0 ? sigmoid_fast(raw) : trunc_exp_fast(raw);
      }
      s.res[tid] = make_float4(sigma, rgb[0], rgb[1], rgb[2]);
    }
    __syncwarp();

    PT_MARK(4);
    // ---- C: owners composite their samples of this round, in order (renderer.h:170-190) ---
    {
      uint32_t mine = s.own[warp][lane];
      while (mine && r.alive) {
        const int j = __ffs(mine) - 1;  // rows are in stream order: increasing candidate
        mine &= mine - 1;
        const float4 e = s.res[warp * 32 + j];
        const int cnd = s.rowcand[warp][j];
        const double t = __ldg(p.ts + cnd);
        const double delta = (cnd + 1 < p.n) ? dsub(__ldg(p.ts + cnd + 1), t) : dmul(t, dsub(p.ratio, 1.0));
        const double a = dsub(1.0, exp(dmul(-(double)e.x, delta)));
        const double wgt = dmul(r.trans, a);
        r.px = dadd(r.px, dmul(wgt, (double)e.y));
        r.py = dadd(r.py, dmul(wgt, (double)e.z));
        r.pz = dadd(r.pz, dmul(wgt, (double)e.w));
        r.depth = dadd(r.depth, dmul(wgt, t));
        r.opac = dadd(r.opac, wgt);
        r.trans = dmul(r.trans, dsub(1.0, a));
        ++r.contributing;
        if (p.t_cut > 0 && r.trans < p.t_cut) {
          r.term = true;
          r.alive = false;
        }
      }
    }
    cnt.evals += have ? 1u : 0u;
    PT_MARK(5);
    __syncthreads();  // res[] and the A tile are rewritten next round
    PT_MARK(6);
  }

  // ---- teardown --------------------------------------------------------------------------
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (warp == 0) ptx::tmem_dealloc<kTmemCols>(tmem);
  add_work_stats(p, cnt.evals, cnt.level_samples, cnt.marched, cnt.rays);
#ifdef LUMI_PHASE_TIMING
  if (lane == 0)
    for (int k = 0; k < 7; ++k) atomicAdd(&g_phase_cycles_pk[k], (unsigned long long)pt[k]);
#endif
#undef PT_MARK
}

}  // namespace pk
}  // namespace lumi_dev

using namespace lumi_dev;

size_t render_pk_smem_bytes() { return sizeof(pk::Smem); }

// march pass over packet-ordered ray ids + the packet kernel
cudaError_t launch_render_pk(RenderParams p, cudaStream_t s, int num_sms, cudaEvent_t* ev) {
  const long long rays = (long long)(p.row_end - p.row_begin) * p.cam.width;
  if (rays <= 0) return cudaSuccess;
  static int blocks_per_sm = -1;
  const size_t smem = render_pk_smem_bytes();
  cudaError_t e;
  if (blocks_per_sm < 0) {
    if ((e = cudaFuncSetAttribute(pk::k_render_pk, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem)) != cudaSuccess)
      return e;
    cudaFuncAttributes fa;
    if ((e = cudaFuncGetAttributes(&fa, pk::k_render_pk)) != cudaSuccess) return e;
    const int regs_per_warp = ((fa.numRegs * 32 + 255) / 256) * 256;
    const int by_regs = 65536 / (regs_per_warp * (pk::kThreads / 32));
    const int by_smem = (228 * 1024) / (int)(smem + 1024);
    blocks_per_sm = std::max(1, std::min(by_regs, by_smem));
    if (const char* cap = std::getenv("LUMI_MAX_CTAS"))
      blocks_per_sm = std::max(1, std::min(blocks_per_sm, std::atoi(cap)));
    const int carve = (int)std::ceil(100.0 * blocks_per_sm * (double)(smem + 1024) / (228.0 * 1024));
    if ((e = cudaFuncSetAttribute(pk::k_render_pk, cudaFuncAttributePreferredSharedMemoryCarveout,
                                  std::min(100, carve))) != cudaSuccess)
      return e;
    if (std::getenv("LUMI_DEBUG"))
      std::fprintf(stderr, "[lumi] k_render_pk: %zu B smem, %d regs, %d CTAs/SM\n", smem,
                   fa.numRegs, blocks_per_sm);
  }
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
  if ((e = cudaMemsetAsync(p.work_counter, 0, sizeof(unsigned int), s)) != cudaSuccess) return e;
  // the march pass's work counters are reported by the packet kernel (per ray), not here
  RenderParams pm = p;
  pm.work_stats = nullptr;
  if (ev) cudaEventRecord(ev[0], s);
  if ((e = launch_march_mask(pm, s)) != cudaSuccess) return e;
  if (ev) cudaEventRecord(ev[1], s);
  const long long grid = std::min<long long>((long long)blocks_per_sm * num_sms, (packets + 3) / 4);
#ifdef LUMI_PHASE_TIMING
  unsigned long long zero7[7] = {0, 0, 0, 0, 0, 0, 0};
  cudaMemcpyToSymbolAsync(pk::g_phase_cycles_pk, zero7, sizeof(zero7), 0, cudaMemcpyHostToDevice, s);
  cudaMemcpyToSymbolAsync(pk::g_counts_pk, zero7, 4 * sizeof(unsigned long long), 0, cudaMemcpyHostToDevice, s);
#endif
  pk::k_render_pk<<<(unsigned)grid, pk::kThreads, smem, s>>>(p);
  if (ev) cudaEventRecord(ev[2], s);
#ifdef LUMI_PHASE_TIMING
  {
    unsigned long long pc[7];
    cudaMemcpyFromSymbolAsync(pc, pk::g_phase_cycles_pk, sizeof(pc), 0, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    double tot = 0;
    for (int k = 0; k < 7; ++k) tot += (double)pc[k];
    std::fprintf(stderr, "[lumi] pk phase %%: fill %.1f geom %.1f gather %.1f ctasync %.1f mlp %.1f "
                 "composite %.1f roundbar %.1f\n", 100 * pc[0] / tot, 100 * pc[1] / tot,
                 100 * pc[2] / tot, 100 * pc[3] / tot, 100 * pc[4] / tot, 100 * pc[5] / tot,
                 100 * pc[6] / tot);
    unsigned long long cn[4];
    cudaMemcpyFromSymbolAsync(cn, pk::g_counts_pk, sizeof(cn), 0, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    std::fprintf(stderr, "[lumi] pk counts: warp-rounds %llu rows %llu (fill %.3f) gather passes %llu "
                 "pairs %llu (lane use %.3f)\n", cn[0], cn[1], cn[1] / (32.0 * cn[0]), cn[2], cn[3],
                 cn[3] / (64.0 * cn[2]));
  }
#endif
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  cudaFreeAsync(p.kept_mask, s);
  cudaFreeAsync(p.kept_count, s);
  return cudaGetLastError();
}
