// lumi_api.cpp -- the C ABI (include/lumi_cuda.h): model upload, render entry points, the
// GPU occupancy bake driver and the row scheduler.
//
// Host arithmetic that feeds bit-exact device geometry (sample distances, step ratio,
// per-level resolutions, log of the level scale) is computed here with the same libm as
// the reference, never on the device (renderer.h:135-142, grid.h:25-27, grid.cpp:10-11).
#include "lumi_cuda.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <map>
#include <memory>
#include <mutex>
#include <numeric>
#include <string>
#include <tuple>
#include <vector>

#include "kernels.h"
#include "render_common.cuh"

using lumi_dev::RenderParams;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define LUMI_CUDA_TRY(expr)                                                               \
  do {                                                                                    \
    cudaError_t _e = (expr);                                                              \
    if (_e != cudaSuccess)                                                                \
      return fail(LUMI_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e));     \
  } while (0)

// ---- pcg32, proj/include/lumi/common.h:78-114 ----------------------------------------
struct Pcg32 {
  static constexpr uint64_t kMult = 6364136223846793005ULL;
  uint64_t state = 0, inc = 0;
  explicit Pcg32(uint64_t seed, uint64_t stream = 0xda3e39cb94b95bdbULL) {
    inc = (stream << 1u) | 1u;
    next();
    state += seed;
    next();
  }
  uint32_t next() {
    uint64_t old = state;
    state = old * kMult + inc;
    uint32_t xs = static_cast<uint32_t>(((old >> 18u) ^ old) >> 27u);
    uint32_t rot = static_cast<uint32_t>(old >> 59u);
    return (xs >> rot) | (xs << ((32u - rot) & 31u));
  }
  void advance(uint64_t delta) {  // LCG jump-ahead
    uint64_t cm = kMult, cp = inc, am = 1, ap = 0;
    while (delta) {
      if (delta & 1) {
        am *= cm;
        ap = ap * cm + cp;
      }
      cp = (cm + 1) * cp;
      cm *= cm;
      delta >>= 1;
    }
    state = am * state + ap;
  }
  double uniform() { return next() * (1.0 / 4294967296.0); }
  double normal() {
    double u1 = std::max(uniform(), 1e-12);
    double u2 = uniform();
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2);
  }
};

int check_desc(const LumiFieldDesc* d) {
  if (!d) return fail(LUMI_ERR_INVALID, "null field descriptor");
  if (d->levels < 1 || d->levels > LUMI_MAX_LEVELS)
    return fail(LUMI_ERR_UNSUPPORTED, "levels must be in [1, 16]");
  if (d->features_per_level != 2)
    return fail(LUMI_ERR_UNSUPPORTED, "features_per_level must be 2");
  if (d->hidden_width != 64) return fail(LUMI_ERR_UNSUPPORTED, "hidden_width must be 64");
  if (d->bottleneck != 16) return fail(LUMI_ERR_UNSUPPORTED, "bottleneck must be 16");
  if (d->table_size == 0 || (d->table_size & (d->table_size - 1)))
    return fail(LUMI_ERR_INVALID, "table_size must be a power of two");
  if (d->color_space != 0 && d->color_space != 1) return fail(LUMI_ERR_INVALID, "bad color_space");
  if (!(d->per_level_scale > 1.0) || d->base_resolution < 1)
    return fail(LUMI_ERR_INVALID, "bad grid scale/base resolution");
  return LUMI_OK;
}

int layout_of(const LumiFieldDesc* d, LumiGridLayout* out) {
  std::memset(out, 0, sizeof(*out));
  out->levels = d->levels;
  out->features_per_level = d->features_per_level;
  uint64_t off = 0;
  for (int l = 0; l < d->levels; ++l) {
    // HashGridConfig::resolution (grid.h:25-27)
    int res = static_cast<int>(std::floor(d->base_resolution * std::pow(d->per_level_scale, l)));
    if (l > 0 && res <= out->resolution[l - 1])
      return fail(LUMI_ERR_INVALID, "hash grid: resolutions must be strictly increasing");
    if (res < 1 || res > (1 << 30)) return fail(LUMI_ERR_UNSUPPORTED, "resolution out of range");
    uint64_t v = static_cast<uint64_t>(res) + 1;
    uint64_t dense = v * v * v;
    out->resolution[l] = res;
    out->dense[l] = dense <= d->table_size;
    out->entries[l] = out->dense[l] ? static_cast<uint32_t>(dense) : d->table_size;
    out->offset[l] = off;
    off += static_cast<uint64_t>(out->entries[l]) * d->features_per_level;
  }
  out->total_floats = off;
  const uint64_t F = static_cast<uint64_t>(d->levels) * d->features_per_level, H = d->hidden_width,
                 B = d->bottleneck;
  out->density_params = F * H + H + H * (1 + B) + (1 + B);
  out->color_params = (B + 16) * H + H + H * H + H + H * 3 + 3;
  return LUMI_OK;
}

int check_cam(const LumiCameraDesc* c) {
  if (!c) return fail(LUMI_ERR_INVALID, "null camera");
  if (!(c->fx > 0 && c->fy > 0))
    return fail(LUMI_ERR_INVALID, "generate_ray: focal lengths must be positive");
  if (c->width < 1 || c->height < 1) return fail(LUMI_ERR_INVALID, "bad image size");
  for (int i = 0; i < 9; ++i)
    if (!std::isfinite(c->rot[i])) return fail(LUMI_ERR_INVALID, "non-finite pose");
  for (int i = 0; i < 3; ++i)
    if (!std::isfinite(c->origin[i])) return fail(LUMI_ERR_INVALID, "non-finite pose");
  if (!(c->t_near > 0 && c->t_far > c->t_near))
    return fail(LUMI_ERR_INVALID, "march_ray: bad sampling interval");
  return LUMI_OK;
}

int check_opts(const LumiRenderOptions* o) {
  if (!o) return fail(LUMI_ERR_INVALID, "null render options");
  if (o->samples_per_ray < 2) return fail(LUMI_ERR_INVALID, "march_ray: bad sampling interval");
  if (o->samples_per_ray > lumi_dev::kMaxSamples)
    return fail(LUMI_ERR_UNSUPPORTED, "samples_per_ray must be <= 1024");
  if (o->chunk_size < 1) return fail(LUMI_ERR_INVALID, "chunk_size must be positive");
  if (o->contraction != 0 && o->contraction != 1) return fail(LUMI_ERR_INVALID, "bad contraction");
  return LUMI_OK;
}

}  // namespace

// One host-buffer render_rows call's device resources (reused across calls).
struct Staging {
  cudaStream_t s = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  void* buf = nullptr;
  size_t bytes = 0;
  ~Staging() {
    if (s) cudaStreamSynchronize(s);
    cudaFree(buf);
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
    if (s) cudaStreamDestroy(s);
  }
};

struct LumiModel {
  int device = 0;
  LumiFieldDesc desc{};
  LumiGridLayout layout{};
  float* d_table = nullptr;   // reference fp32 layout (SIMT cross-check kernel)
  void* d_table16 = nullptr;  // half2 copy (the production gather; padded, pk::cell2)
  float* d_dparams = nullptr;
  float* d_cparams = nullptr;
  float* d_fused = nullptr;  // density L2 folded into colour L1 (packet kernel), see fuse_l2_c1
  void* d_wtiles = nullptr;  // the packet kernel's fp16 weight-tile image (TMA-staged per CTA)
  uint8_t* d_occ = nullptr;
  uint32_t* d_occ_bits = nullptr;  // the same grid, 1 bit per voxel (the march pass)
  int occ_res = 0;
  int kernel = LUMI_KERNEL_WS;
  int num_sms = 148;
  std::mutex mu;
  std::map<std::tuple<double, double, int>, std::pair<double*, double>> ts_cache;
  bool timing = false;
  std::vector<std::array<cudaEvent_t, 3>> ev_pool;  // [march start, render start, render end]
  size_t ev_used = 0;
  std::vector<std::unique_ptr<Staging>> staging;  // lumi_render_rows slots
};

namespace {

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

// The per-launch march masks come from the stream-ordered allocator; keep freed blocks in
// the device's default pool instead of returning them at every synchronisation.
cudaError_t keep_pool_memory(int device) {
  cudaMemPool_t pool;
  cudaError_t e = cudaDeviceGetDefaultMemPool(&pool, device);
  if (e != cudaSuccess) return e;
  uint64_t keep = UINT64_MAX;
  return cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
}

// Exponential sample distances and step ratio (renderer.h:135-142) on the host.
int get_ts(LumiModel* m, double tn, double tf, int n, const double** d_ts, double* ratio) {
  std::lock_guard<std::mutex> lk(m->mu);
  auto key = std::make_tuple(tn, tf, n);
  auto it = m->ts_cache.find(key);
  if (it == m->ts_cache.end()) {
    std::vector<double> ts(n);
    const double log_ratio = std::log(tf / tn);
    for (int i = 0; i < n; ++i) ts[i] = tn * std::exp(log_ratio * (static_cast<double>(i) / (n - 1)));
    ts[0] = tn;
    ts[n - 1] = tf;
    const double r = std::pow(tf / tn, 1.0 / (n - 1));
    // followed by the packet kernel's compositing inputs per candidate, {(float)t_i,
    // (float)delta_i}, delta as march_ray forms it (renderer.h:209: next t minus t, the last
    // one t (ratio - 1)) in IEEE double like the device's dsub / dmul
    std::vector<float2> tdf(n);
    for (int i = 0; i < n; ++i) {
      const double dl = i + 1 < n ? ts[i + 1] - ts[i] : ts[i] * (r - 1.0);
      tdf[i] = make_float2(static_cast<float>(ts[i]), static_cast<float>(dl));
    }
    double* d = nullptr;
    LUMI_CUDA_TRY(cudaMalloc(&d, (sizeof(double) + sizeof(float2)) * n));
    LUMI_CUDA_TRY(cudaMemcpy(d, ts.data(), sizeof(double) * n, cudaMemcpyHostToDevice));
    LUMI_CUDA_TRY(cudaMemcpy(d + n, tdf.data(), sizeof(float2) * n, cudaMemcpyHostToDevice));
    it = m->ts_cache.emplace(key, std::make_pair(d, r)).first;
  }
  *d_ts = it->second.first;
  *ratio = it->second.second;
  return LUMI_OK;
}

int make_params(LumiModel* m, const LumiCameraDesc* cam, const LumiRenderOptions* o, int b, int e,
                RenderParams* p) {
  int rc;
  if ((rc = check_cam(cam)) || (rc = check_opts(o))) return rc;
  if (!(b >= 0 && e <= cam->height && b <= e))
    return fail(LUMI_ERR_INVALID, "render_rows: row range outside image");
  std::memset(p, 0, sizeof(*p));
  std::memcpy(p->cam.rot, cam->rot, sizeof(cam->rot));
  std::memcpy(p->cam.origin, cam->origin, sizeof(cam->origin));
  p->cam.fx = cam->fx;
  p->cam.fy = cam->fy;
  p->cam.cx = cam->cx;
  p->cam.cy = cam->cy;
  p->cam.width = cam->width;
  p->cam.height = cam->height;
  p->cam.t_near = cam->t_near;
  p->cam.t_far = cam->t_far;
  auto& g = p->grid;
  g.table = reinterpret_cast<const float2*>(m->d_table);
  g.table16 = reinterpret_cast<const __half2*>(m->d_table16);
  g.levels = m->layout.levels;
  for (int l = 0; l < g.levels; ++l) {
    g.res[l] = m->layout.resolution[l];
    g.hash_mask[l] = m->layout.entries[l] - 1u;
    if (m->layout.dense[l]) g.dense_mask |= 1u << l;
    g.offset2[l] = m->layout.offset[l] / 2;
  }
  g.two_base = 2.0 * m->desc.base_resolution;  // grid.cpp:10 evaluates 2.0 * base first
  g.log_scale = std::log(m->desc.per_level_scale);
  p->mlp.dparams = m->d_dparams;
  p->mlp.cparams = m->d_cparams;
  p->mlp.fused = m->d_fused;
  // LUMI_WS_TMA=0 (A/B): each CTA converts the fp32 parameters itself instead of the TMA copy
  static const bool tma = [] {
    const char* e = std::getenv("LUMI_WS_TMA");
    return !(e && e[0] == '0');
  }();
  p->mlp.wtiles = tma ? m->d_wtiles : nullptr;
  p->mlp.color_space = m->desc.color_space;
  p->occ = m->d_occ;
  p->occ_bits = m->d_occ_bits;
  p->occ_res = m->occ_res;
  p->occ_bias = march_occ_bias(m->occ_res);
  if ((rc = get_ts(m, cam->t_near, cam->t_far, o->samples_per_ray, &p->ts, &p->ratio))) return rc;
  p->tdf = reinterpret_cast<const float2*>(p->ts + o->samples_per_ray);
  p->n = o->samples_per_ray;
  p->lod_enabled = o->lod_enabled ? 1 : 0;
  p->lod_bias = o->lod_bias;
  p->t_cut = o->termination_transmittance;
  for (int c = 0; c < 3; ++c) p->bg[c] = o->background[c];
  p->contraction = o->contraction;
  if (const char* dbg = std::getenv("LUMI_DEBUG_SKIP")) p->debug_flags = std::atoi(dbg);
  p->chunk = o->chunk_size;
  p->row_begin = b;
  p->row_end = e;
  p->work_counter = nullptr;  // allocated per launch by the launcher (stream-ordered)
  return LUMI_OK;
}

int set_target(RenderParams* p, const LumiFrameTarget* t, int b, int e) {
  if (!t || !t->rgb) return fail(LUMI_ERR_INVALID, "frame target needs an rgb plane");
  if (t->width != p->cam.width)
    return fail(LUMI_ERR_INVALID, "frame target width must equal the camera width");
  if (t->row_offset + b < 0 || t->row_offset + e > t->height)
    return fail(LUMI_ERR_INVALID, "frame target too small for the row range");
  p->rgb = t->rgb;
  p->depth = t->depth;
  p->opacity = t->opacity;
  p->counts = t->counts;
  p->row_evals = t->row_evals;
  p->row_cycles = t->row_cycles;
  p->srgb8 = t->srgb8;
  p->work_stats = reinterpret_cast<unsigned long long*>(t->work_stats);
  p->exposure_gain = std::exp2(t->exposure_bias_stops);
  p->tw = t->width;
  p->th = t->height;
  p->row_offset = t->row_offset;
  return LUMI_OK;
}

}  // namespace

extern "C" {

const char* lumi_last_error(void) { return g_err.c_str(); }
int lumi_set_error(int code, const char* msg) { return fail(code, msg); }
int lumi_abi_version(void) { return LUMI_ABI_VERSION; }

int lumi_device_info(int device, char* info, size_t len) {
  cudaDeviceProp prop;
  LUMI_CUDA_TRY(cudaGetDeviceProperties(&prop, device));
  if (info && len)
    std::snprintf(info, len, "%s sm_%d%d SMs=%d mem=%.1fGiB", prop.name, prop.major, prop.minor,
                  prop.multiProcessorCount, prop.totalGlobalMem / 1073741824.0);
  if (prop.major != 10)
    return fail(LUMI_ERR_UNSUPPORTED, std::string("need an sm_100 (B200) device, got ") + prop.name);
  return LUMI_OK;
}

int lumi_field_layout(const LumiFieldDesc* desc, LumiGridLayout* out) {
  int rc = check_desc(desc);
  if (rc) return rc;
  if (!out) return fail(LUMI_ERR_INVALID, "null layout");
  return layout_of(desc, out);
}

int lumi_synth_params(const LumiFieldDesc* desc, uint64_t seed, double amp, float* table,
                      float* dparams, float* cparams) {
  LumiGridLayout lay;
  int rc = lumi_field_layout(desc, &lay);
  if (rc) return rc;
  if (!table || !dparams || !cparams) return fail(LUMI_ERR_INVALID, "null output buffer");
  // RadianceField::init_random (field.h:88-93): grid uniform(+-1e-4) (grid.h:82-84), then the
  // density and colour nets (He-normal weights, zero bias, network.h:73-78).
  Pcg32 rng(seed);
  if (amp > 0) {
    rng.advance(lay.total_floats);  // the grid draws are overwritten below
  } else {
    for (uint64_t i = 0; i < lay.total_floats; ++i)
      table[i] = static_cast<float>(-1e-4 + (1e-4 - -1e-4) * rng.uniform());
  }
  auto layer = [&](int in, int out, float* p) {
    const double scale = std::sqrt(2.0 / in);
    for (int i = 0; i < in * out; ++i) p[i] = static_cast<float>(rng.normal() * scale);
    for (int i = 0; i < out; ++i) p[in * out + i] = 0.0f;
    return p + static_cast<size_t>(in) * out + out;
  };
  const int F = desc->levels * desc->features_per_level, H = desc->hidden_width,
            B = desc->bottleneck;
  float* p = layer(F, H, dparams);
  layer(H, 1 + B, p);
  p = layer(B + 16, H, cparams);
  p = layer(H, H, p);
  layer(H, 3, p);
  if (amp > 0) {  // grid overwrite, the pattern of trainer.cpp:257-259
    Pcg32 g(seed + 1);
    for (uint64_t i = 0; i < lay.total_floats; ++i)
      table[i] = static_cast<float>(-amp + (amp - -amp) * g.uniform());
  }
  return LUMI_OK;
}

namespace {
// The density network's output layer is linear (field.h:116-122: sigma = trunc_exp(out[0]),
// bottleneck = out[1..17) straight into the colour input), so colour layer 1 applied to
// [bottleneck, sh] equals one layer on [h1, sh]:
//   C1a (W2' h1 + b2') + C1b sh + cb1 = (C1a W2') h1 + C1b sh + (C1a b2' + cb1),
// with sigma's row W2[0] . h1 + b2[0] appended as output 64.  Returns [65 x 80] weights
// then [65] biases (products accumulated in double).  The packet kernel runs this as one
// tcgen05 layer (N = 80, K = 64 + 16), one MMA round trip fewer per batch.
std::vector<float> fuse_l2_c1(const float* dp, const float* cp) {
  constexpr int H = 64, B = 16, CIN = 32, K = H + 16;
  const float* W2 = dp + H * 32 + H;  // [17 x 64]
  const float* b2 = W2 + (1 + B) * H;
  const float* C1 = cp;               // [64 x 32]
  const float* cb1 = cp + H * CIN;
  std::vector<float> f((H + 1) * K + (H + 1), 0.f);
  float* bias = f.data() + (H + 1) * K;
  for (int n = 0; n < H; ++n) {
    for (int k = 0; k < H; ++k) {
      double acc = 0.0;
      for (int j = 0; j < B; ++j) acc += (double)C1[n * CIN + j] * (double)W2[(1 + j) * H + k];
      f[n * K + k] = (float)acc;
    }
    for (int k = 0; k < 16; ++k) f[n * K + H + k] = C1[n * CIN + B + k];
    double acc = cb1[n];
    for (int j = 0; j < B; ++j) acc += (double)C1[n * CIN + j] * (double)b2[1 + j];
    bias[n] = (float)acc;
  }
  for (int k = 0; k < H; ++k) f[H * K + k] = W2[k];
  bias[H] = b2[0];
  return f;
}
}  // namespace

int lumi_model_create(int device, const LumiFieldDesc* desc, const float* table,
                      const float* dparams, const float* cparams, const uint8_t* occ, int occ_res,
                      LumiModel** out) {
  if (!out) return fail(LUMI_ERR_INVALID, "null output handle");
  *out = nullptr;
  LumiGridLayout lay;
  int rc = lumi_field_layout(desc, &lay);
  if (rc) return rc;
  if (!table || !dparams || !cparams) return fail(LUMI_ERR_INVALID, "null parameter buffer");
  if (lay.total_floats / 2 >= (1ull << 32))  // the gather indexes table pairs with 32 bits
    return fail(LUMI_ERR_INVALID, "hash-grid table exceeds 2^32 feature pairs");
  int ndev = 0;
  LUMI_CUDA_TRY(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return fail(LUMI_ERR_CUDA, "no such CUDA device");
  if ((rc = lumi_device_info(device, nullptr, 0))) return rc;
  DeviceGuard dg(device);
  auto m = new LumiModel();
  m->device = device;
  m->desc = *desc;
  m->layout = lay;
  auto cleanup = [&](int code) {
    lumi_model_destroy(m);
    return code;
  };
  cudaError_t e;
  if ((e = cudaMalloc(&m->d_table, lay.total_floats * sizeof(float))) != cudaSuccess ||
      (e = cudaMalloc(&m->d_dparams, lay.density_params * sizeof(float))) != cudaSuccess ||
      (e = cudaMalloc(&m->d_cparams, lay.color_params * sizeof(float))) != cudaSuccess ||
      (e = cudaMemcpy(m->d_table, table, lay.total_floats * sizeof(float),
                      cudaMemcpyHostToDevice)) != cudaSuccess ||
      (e = cudaMemcpy(m->d_dparams, dparams, lay.density_params * sizeof(float),
                      cudaMemcpyHostToDevice)) != cudaSuccess ||
      (e = cudaMemcpy(m->d_cparams, cparams, lay.color_params * sizeof(float),
                      cudaMemcpyHostToDevice)) != cudaSuccess ||
      (e = cudaDeviceGetAttribute(&m->num_sms, cudaDevAttrMultiProcessorCount, device)) != cudaSuccess ||
      (e = keep_pool_memory(device)) != cudaSuccess ||
      // (+256 B: a dense level's top cell may address one corner past the level, pk::cell2)
      (e = cudaMalloc(&m->d_table16, lay.total_floats * 2 + 256)) != cudaSuccess ||
      (e = launch_to_half(m->d_table, m->d_table16, lay.total_floats, nullptr)) != cudaSuccess ||
      (e = cudaDeviceSynchronize()) != cudaSuccess)
    return cleanup(fail(LUMI_ERR_CUDA, std::string("model upload: ") + cudaGetErrorString(e)));
  {
    const std::vector<float> fused = fuse_l2_c1(dparams, cparams);
    if ((e = cudaMalloc(&m->d_fused, fused.size() * sizeof(float))) != cudaSuccess ||
        (e = cudaMemcpy(m->d_fused, fused.data(), fused.size() * sizeof(float),
                        cudaMemcpyHostToDevice)) != cudaSuccess)
      return cleanup(fail(LUMI_ERR_CUDA, std::string("model upload: ") + cudaGetErrorString(e)));
  }
  if ((e = cudaMalloc(&m->d_wtiles, render_ws_weight_tile_bytes())) != cudaSuccess ||
      (e = launch_pack_weight_tiles(lumi_dev::MlpDev{m->d_dparams, m->d_cparams, m->d_fused,
                                                      m->desc.color_space, nullptr},
                                    m->d_wtiles, nullptr)) != cudaSuccess ||
      (e = cudaDeviceSynchronize()) != cudaSuccess)
    return cleanup(fail(LUMI_ERR_CUDA, std::string("model upload: ") + cudaGetErrorString(e)));
  if ((rc = lumi_model_set_occupancy(m, occ, occ_res))) return cleanup(rc);
  if (const char* k = std::getenv("LUMI_KERNEL")) {
    const std::string ks(k);
    m->kernel = ks == "simt" ? LUMI_KERNEL_SIMT : LUMI_KERNEL_WS;
  }
  *out = m;
  return LUMI_OK;
}

int lumi_model_set_occupancy(LumiModel* m, const uint8_t* occ, int res) {
  if (!m) return fail(LUMI_ERR_INVALID, "null model");
  if (res < 1 || res > 1024) return fail(LUMI_ERR_INVALID, "occupancy: bad resolution");  // occupancy.cpp:14
  DeviceGuard dg(m->device);
  const size_t n = static_cast<size_t>(res) * res * res;
  std::vector<uint8_t> bits(n, 1);  // default all occupied (occupancy.cpp:15)
  if (occ)
    for (size_t i = 0; i < n; ++i) bits[i] = occ[i] ? 1 : 0;
  std::vector<uint32_t> words((n + 31) / 32, 0u);
  for (size_t i = 0; i < n; ++i) words[i >> 5] |= (uint32_t)bits[i] << (i & 31);
  if (m->d_occ) cudaFree(m->d_occ);
  if (m->d_occ_bits) cudaFree(m->d_occ_bits);
  m->d_occ = nullptr;
  m->d_occ_bits = nullptr;
  LUMI_CUDA_TRY(cudaMalloc(&m->d_occ, n));
  LUMI_CUDA_TRY(cudaMemcpy(m->d_occ, bits.data(), n, cudaMemcpyHostToDevice));
  LUMI_CUDA_TRY(cudaMalloc(&m->d_occ_bits, words.size() * 4));
  LUMI_CUDA_TRY(cudaMemcpy(m->d_occ_bits, words.data(), words.size() * 4, cudaMemcpyHostToDevice));
  m->occ_res = res;
  return LUMI_OK;
}

int lumi_model_destroy(LumiModel* m) {
  if (!m) return LUMI_OK;
  DeviceGuard dg(m->device);
  cudaFree(m->d_table);
  cudaFree(m->d_table16);
  cudaFree(m->d_dparams);
  cudaFree(m->d_cparams);
  cudaFree(m->d_fused);
  cudaFree(m->d_wtiles);
  cudaFree(m->d_occ);
  cudaFree(m->d_occ_bits);
  for (auto& kv : m->ts_cache) cudaFree(kv.second.first);
  for (auto& a : m->ev_pool)
    for (auto x : a) cudaEventDestroy(x);
  m->staging.clear();
  delete m;
  return LUMI_OK;
}

int lumi_model_set_kernel(LumiModel* m, int kernel) {
  if (!m) return fail(LUMI_ERR_INVALID, "null model");
  if (kernel == LUMI_KERNEL_TC || kernel == LUMI_KERNEL_PACKET)
    return fail(LUMI_ERR_UNSUPPORTED, "kernel variant retired (superseded by LUMI_KERNEL_WS)");
  if (kernel != LUMI_KERNEL_SIMT && kernel != LUMI_KERNEL_WS)
    return fail(LUMI_ERR_INVALID, "unknown kernel variant");
  m->kernel = kernel;
  return LUMI_OK;
}

int lumi_model_bytes(const LumiModel* m, uint64_t* bytes) {
  if (!m || !bytes) return fail(LUMI_ERR_INVALID, "null argument");
  *bytes = (m->layout.total_floats + m->layout.density_params + m->layout.color_params) * 4 +
           static_cast<uint64_t>(m->occ_res) * m->occ_res * m->occ_res;
  return LUMI_OK;
}

int lumi_model_device(const LumiModel* m, int* device) {
  if (!m || !device) return fail(LUMI_ERR_INVALID, "null argument");
  *device = m->device;
  return LUMI_OK;
}

int lumi_render_rows_async(LumiModel* m, const LumiCameraDesc* cam, const LumiRenderOptions* o,
                           int b, int e, const LumiFrameTarget* t, void* stream) {
  if (!m) return fail(LUMI_ERR_INVALID, "null model");
  DeviceGuard dg(m->device);
  RenderParams p;
  int rc = make_params(m, cam, o, b, e, &p);
  if (rc) return rc;
  if ((rc = set_target(&p, t, b, e))) return rc;
  cudaEvent_t* ev = nullptr;
  if (m->timing) {
    std::lock_guard<std::mutex> lk(m->mu);
    if (m->ev_used == m->ev_pool.size()) {
      std::array<cudaEvent_t, 3> a{};
      for (auto& x : a) LUMI_CUDA_TRY(cudaEventCreate(&x));
      m->ev_pool.push_back(a);
    }
    ev = m->ev_pool[m->ev_used++].data();
  }
  const auto st = static_cast<cudaStream_t>(stream);
  if (m->kernel == LUMI_KERNEL_SIMT) {
    if (ev) LUMI_CUDA_TRY(cudaEventRecord(ev[0], st));
    if (ev) LUMI_CUDA_TRY(cudaEventRecord(ev[1], st));
    LUMI_CUDA_TRY(launch_render_simt(p, st));
    if (ev) LUMI_CUDA_TRY(cudaEventRecord(ev[2], st));
  } else {
    LUMI_CUDA_TRY(launch_render_ws(p, st, m->num_sms, ev));
  }
  return LUMI_OK;
}

int lumi_model_set_timing(LumiModel* m, int enable) {
  if (!m) return fail(LUMI_ERR_INVALID, "null model");
  m->timing = enable != 0;
  return LUMI_OK;
}

int lumi_model_take_timing(LumiModel* m, double* march_ms, double* render_ms, int* launches) {
  if (!m) return fail(LUMI_ERR_INVALID, "null model");
  DeviceGuard dg(m->device);
  std::lock_guard<std::mutex> lk(m->mu);
  double a = 0.0, b = 0.0;
  for (size_t i = 0; i < m->ev_used; ++i) {
    auto& ev = m->ev_pool[i];
    LUMI_CUDA_TRY(cudaEventSynchronize(ev[2]));
    float x = 0.f, y = 0.f;
    LUMI_CUDA_TRY(cudaEventElapsedTime(&x, ev[0], ev[1]));
    LUMI_CUDA_TRY(cudaEventElapsedTime(&y, ev[1], ev[2]));
    a += x;
    b += y;
  }
  if (march_ms) *march_ms = a;
  if (render_ms) *render_ms = b;
  if (launches) *launches = (int)m->ev_used;
  m->ev_used = 0;
  return LUMI_OK;
}

int lumi_march_kept_async(LumiModel* m, const LumiCameraDesc* cam, const LumiRenderOptions* o,
                          int b, int e, uint32_t* mask, int32_t* counts, void* stream) {
  if (!m) return fail(LUMI_ERR_INVALID, "null model");
  DeviceGuard dg(m->device);
  RenderParams p;
  int rc = make_params(m, cam, o, b, e, &p);
  if (rc) return rc;
  // the SIMT cross-check model marches exactly per ray; the tensor-core renderers consume the
  // filtered mask pass, which is what this entry point then reports
  if (m->kernel == LUMI_KERNEL_SIMT)
    LUMI_CUDA_TRY(launch_march_kept(p, mask, counts, static_cast<cudaStream_t>(stream)));
  else
    LUMI_CUDA_TRY(launch_march_public(p, mask, counts, static_cast<cudaStream_t>(stream)));
  return LUMI_OK;
}

// Device address of page-locked host memory (nullptr for pageable memory, or when
// LUMI_ZERO_COPY=0 disables direct stores).
static float* zero_copy_ptr(float* host) {
  static const bool enabled = [] {
    const char* e = std::getenv("LUMI_ZERO_COPY");
    return !(e && e[0] == '0');
  }();
  if (!enabled || !host) return nullptr;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, host) != cudaSuccess) {
    cudaGetLastError();  // pageable memory on older runtimes reports an error: clear it
    return nullptr;
  }
  if (a.type != cudaMemoryTypeHost || !a.devicePointer) return nullptr;
  return static_cast<float*>(a.devicePointer);
}

int lumi_render_rows(LumiModel* m, const LumiCameraDesc* cam, const LumiRenderOptions* o, int b,
                     int e, float* out, float* depth, float* opacity, LumiRowStats* stats) {
  if (!m) return fail(LUMI_ERR_INVALID, "null model");
  if (!out) return fail(LUMI_ERR_INVALID, "null output image");
  int rc;
  if ((rc = check_cam(cam)) || (rc = check_opts(o))) return rc;
  if (!(b >= 0 && e <= cam->height && b <= e))
    return fail(LUMI_ERR_INVALID, "render_rows: row range outside image");
  if (b == e) return LUMI_OK;
  DeviceGuard dg(m->device);
  const int W = cam->width, rows = e - b;
  const size_t plane = static_cast<size_t>(W) * rows;
  const int nplanes = 3 + (depth ? 1 : 0) + (opacity ? 1 : 0);
  // a staging slot (stream, events, device planes) from the model's pool: concurrent
  // run_frame workers each take their own; slots are reused across calls
  std::unique_ptr<Staging> st;
  {
    std::lock_guard<std::mutex> lk(m->mu);
    if (!m->staging.empty()) {
      st = std::move(m->staging.back());
      m->staging.pop_back();
    }
  }
  if (!st) {
    st.reset(new Staging());
    LUMI_CUDA_TRY(cudaStreamCreateWithFlags(&st->s, cudaStreamNonBlocking));
    LUMI_CUDA_TRY(cudaEventCreate(&st->e0));
    LUMI_CUDA_TRY(cudaEventCreate(&st->e1));
  }
  auto done = [&](int code) {
    cudaStreamSynchronize(st->s);
    std::lock_guard<std::mutex> lk(m->mu);
    m->staging.push_back(std::move(st));
    return code;
  };
  const size_t need = plane * nplanes * sizeof(float) + 2 * rows * sizeof(int64_t) + 512;
  cudaError_t ce;
  if (st->bytes < need) {
    cudaFree(st->buf);
    st->buf = nullptr;
    st->bytes = 0;
    if ((ce = cudaMalloc(&st->buf, need)) != cudaSuccess)
      return done(fail(LUMI_ERR_CUDA, cudaGetErrorString(ce)));
    st->bytes = need;
  }
  cudaStream_t s = st->s;
  float* d_buf = static_cast<float*>(st->buf);
  // the per-row eval counters (64-bit atomics) start 256-byte aligned after the planes
  const size_t rows_off = (plane * nplanes * sizeof(float) + 255) & ~static_cast<size_t>(255);
  int64_t* d_rows = reinterpret_cast<int64_t*>(static_cast<char*>(st->buf) + rows_off);
  int64_t* d_cyc = d_rows + rows;
  if ((ce = cudaMemsetAsync(d_rows, 0, 2 * rows * sizeof(int64_t), s)) != cudaSuccess)
    return done(fail(LUMI_ERR_CUDA, cudaGetErrorString(ce)));
  // Zero-copy output: when the caller's planes are pinned (page-locked, hence mapped into the
  // device's address space under UVA), the kernel stores the pixels straight into them over
  // PCIe while it renders -- a packet's 8-pixel rows are 32-byte coalesced writes -- and no
  // device->host copy follows.  Pageable planes go through the device staging planes.
  float* z_rgb = zero_copy_ptr(out);
  float* z_depth = depth ? zero_copy_ptr(depth) : nullptr;
  float* z_opac = opacity ? zero_copy_ptr(opacity) : nullptr;
  const bool zero_copy = z_rgb && (!depth || z_depth) && (!opacity || z_opac);
  float* d_depth = depth ? d_buf + 3 * plane : nullptr;
  float* d_opac = opacity ? d_buf + (3 + (depth ? 1 : 0)) * plane : nullptr;
  LumiFrameTarget t{};
  t.rgb = d_buf;
  t.depth = d_depth;
  t.opacity = d_opac;
  t.row_evals = d_rows - b;  // indexed by camera row
  t.row_cycles = stats ? d_cyc - b : nullptr;
  t.width = W;
  t.height = rows;
  t.row_offset = -b;
  if (zero_copy) {
    t.rgb = z_rgb;
    t.depth = z_depth;
    t.opacity = z_opac;
    t.height = cam->height;
    t.row_offset = 0;
  }
  cudaEventRecord(st->e0, s);
  if ((rc = lumi_render_rows_async(m, cam, o, b, e, &t, s))) return done(rc);
  cudaEventRecord(st->e1, s);
  const size_t full = static_cast<size_t>(W) * cam->height;
  for (int c = 0; c < 3 && !zero_copy; ++c)
    if ((ce = cudaMemcpyAsync(out + c * full + static_cast<size_t>(b) * W, d_buf + c * plane,
                              plane * sizeof(float), cudaMemcpyDeviceToHost, s)) != cudaSuccess)
      return done(fail(LUMI_ERR_CUDA, cudaGetErrorString(ce)));
  if (depth && !zero_copy &&
      (ce = cudaMemcpyAsync(depth + static_cast<size_t>(b) * W, d_depth, plane * sizeof(float),
                            cudaMemcpyDeviceToHost, s)) != cudaSuccess)
    return done(fail(LUMI_ERR_CUDA, cudaGetErrorString(ce)));
  if (opacity && !zero_copy &&
      (ce = cudaMemcpyAsync(opacity + static_cast<size_t>(b) * W, d_opac, plane * sizeof(float),
                            cudaMemcpyDeviceToHost, s)) != cudaSuccess)
    return done(fail(LUMI_ERR_CUDA, cudaGetErrorString(ce)));
  std::vector<int64_t> row_ev(stats ? 2 * rows : 0);
  if (stats && (ce = cudaMemcpyAsync(row_ev.data(), d_rows, 2 * rows * sizeof(int64_t),
                                     cudaMemcpyDeviceToHost, s)) != cudaSuccess)
    return done(fail(LUMI_ERR_CUDA, cudaGetErrorString(ce)));
  if ((ce = cudaStreamSynchronize(s)) != cudaSuccess)
    return done(fail(LUMI_ERR_CUDA, cudaGetErrorString(ce)));
  if (stats) {
    float ms = 0;
    cudaEventElapsedTime(&ms, st->e0, st->e1);
    // The device renders all rows of the band in one launch: each row gets the share of the
    // launch time its packets took in SM cycles (the reference times each row on the CPU,
    // renderer.h:261, 272-276); kernels without the cycle counters split it evenly.
    double cyc_total = 0.0;
    for (int i = 0; i < rows; ++i) cyc_total += (double)row_ev[rows + i];
    for (int y = b; y < e; ++y) {
      stats[y - b].row = y;
      stats[y - b].ms = cyc_total > 0 ? ms * (double)row_ev[rows + y - b] / cyc_total : (double)ms / rows;
      stats[y - b].rays = W;
      stats[y - b].evals = row_ev[y - b];
    }
  }
  return done(LUMI_OK);
}

int lumi_bake_occupancy(LumiModel* m, const LumiCameraDesc* cams, int ncams, int spp, int k,
                        int res, float alpha, uint8_t* occ_out, float* probe_out) {
  if (!m) return fail(LUMI_ERR_INVALID, "null model");
  if (k < 1) return fail(LUMI_ERR_INVALID, "probe: need at least one point per axis");
  if (res < 1 || res > 1024) return fail(LUMI_ERR_INVALID, "occupancy: bad resolution");
  if (spp < 2 || ncams < 0 || (ncams > 0 && !cams)) return fail(LUMI_ERR_INVALID, "bad cameras");
  if (!occ_out) return fail(LUMI_ERR_INVALID, "null occupancy output");
  DeviceGuard dg(m->device);
  // Per-camera step ratios on the host libm (occupancy.cpp:106-108).
  std::vector<double> cam_buf(5 * static_cast<size_t>(std::max(ncams, 1)));
  for (int i = 0; i < ncams; ++i) {
    for (int j = 0; j < 3; ++j) cam_buf[3 * i + j] = cams[i].origin[j];
    cam_buf[3 * ncams + i] = cams[i].t_near;
    cam_buf[4 * ncams + i] = std::pow(cams[i].t_far / cams[i].t_near, 1.0 / (spp - 1));
  }
  const size_t n = static_cast<size_t>(res) * res * res;
  double* d_cam = nullptr;
  float* d_probe = nullptr;
  uint8_t* d_occ = nullptr;
  auto done = [&](int code) {
    cudaFree(d_cam);
    cudaFree(d_probe);
    cudaFree(d_occ);
    return code;
  };
  cudaError_t ce;
  if ((ce = cudaMalloc(&d_cam, cam_buf.size() * sizeof(double))) != cudaSuccess ||
      (ce = cudaMalloc(&d_probe, n * sizeof(float))) != cudaSuccess ||
      (ce = cudaMalloc(&d_occ, n)) != cudaSuccess ||
      (ce = cudaMemcpy(d_cam, cam_buf.data(), cam_buf.size() * sizeof(double),
                       cudaMemcpyHostToDevice)) != cudaSuccess)
    return done(fail(LUMI_ERR_CUDA, cudaGetErrorString(ce)));
  RenderParams rp;
  LumiCameraDesc dummy{};
  dummy.rot[0] = dummy.rot[4] = dummy.rot[8] = 1.0;
  dummy.fx = dummy.fy = 1.0;
  dummy.width = dummy.height = 1;
  dummy.t_near = 0.05;
  dummy.t_far = 10.0;
  LumiRenderOptions o{};
  o.samples_per_ray = spp;
  o.chunk_size = 32;
  o.contraction = 1;
  int rc = make_params(m, &dummy, &o, 0, 0, &rp);
  if (rc) return done(rc);
  lumi_dev::BakeParams bp;
  bp.grid = rp.grid;
  bp.mlp = rp.mlp;
  bp.res = res;
  bp.k = k;
  bp.ncams = ncams;
  bp.alpha = alpha;
  bp.cam_origin = d_cam;
  bp.cam_tnear = d_cam + 3 * ncams;
  bp.cam_ratio = d_cam + 4 * ncams;
  bp.probe_max = d_probe;
  bp.occ = d_occ;
  if ((ce = launch_bake(bp, nullptr)) != cudaSuccess ||
      (ce = cudaMemcpy(occ_out, d_occ, n, cudaMemcpyDeviceToHost)) != cudaSuccess ||
      (probe_out &&
       (ce = cudaMemcpy(probe_out, d_probe, n * sizeof(float), cudaMemcpyDeviceToHost)) != cudaSuccess))
    return done(fail(LUMI_ERR_CUDA, cudaGetErrorString(ce)));
  return done(LUMI_OK);
}

int lumi_gather_bench_async(LumiModel* m, int n, int coherent, float* out, void* stream) {
  if (!m) return fail(LUMI_ERR_INVALID, "null model");
  if (n < 0 || (n > 0 && !out)) return fail(LUMI_ERR_INVALID, "gather_bench: bad buffers");
  DeviceGuard dg(m->device);
  RenderParams rp;
  LumiCameraDesc dummy{};
  dummy.rot[0] = dummy.rot[4] = dummy.rot[8] = 1.0;
  dummy.fx = dummy.fy = 1.0;
  dummy.width = dummy.height = 1;
  dummy.t_near = 0.05;
  dummy.t_far = 10.0;
  LumiRenderOptions o{};
  o.samples_per_ray = 2;
  o.chunk_size = 32;
  int rc = make_params(m, &dummy, &o, 0, 0, &rp);
  if (rc) return rc;
  cudaError_t e = launch_gather_bench(rp.grid, n, coherent, out, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return fail(LUMI_ERR_CUDA, std::string("gather_bench: ") + cudaGetErrorString(e));
  return LUMI_OK;
}

int lumi_encode_async(LumiModel* m, int n, const float* pos, const float* lod, float* out,
                      void* stream) {
  if (!m) return fail(LUMI_ERR_INVALID, "null model");
  if (n < 0 || (n > 0 && (!pos || !lod || !out))) return fail(LUMI_ERR_INVALID, "encode: bad buffers");
  DeviceGuard dg(m->device);
  RenderParams rp;
  LumiCameraDesc dummy{};
  dummy.rot[0] = dummy.rot[4] = dummy.rot[8] = 1.0;
  dummy.fx = dummy.fy = 1.0;
  dummy.width = dummy.height = 1;
  dummy.t_near = 0.05;
  dummy.t_far = 10.0;
  LumiRenderOptions o{};
  o.samples_per_ray = 2;
  o.chunk_size = 32;
  int rc = make_params(m, &dummy, &o, 0, 0, &rp);
  if (rc) return rc;
  cudaError_t e = launch_encode(rp.grid, n, pos, lod, out, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return fail(LUMI_ERR_CUDA, std::string("encode: ") + cudaGetErrorString(e));
  return LUMI_OK;
}

int lumi_mlp_batch_async(LumiModel* m, const void* features, const float* dirs, int n, float* out,
                         void* stream) {
  if (!m) return fail(LUMI_ERR_INVALID, "null model");
  if (n < 0 || (n > 0 && (!features || !dirs || !out))) return fail(LUMI_ERR_INVALID, "mlp_batch: bad buffers");
  if ((reinterpret_cast<uintptr_t>(features) & 15) != 0)
    return fail(LUMI_ERR_INVALID, "mlp_batch: features must be 16-byte aligned");
  DeviceGuard dg(m->device);
  lumi_dev::MlpDev mlp{m->d_dparams, m->d_cparams, m->d_fused, m->desc.color_space, nullptr};
  cudaError_t e = launch_mlp_batch(mlp, features, dirs, n, out, m->num_sms, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return fail(LUMI_ERR_CUDA, std::string("mlp_batch: ") + cudaGetErrorString(e));
  return LUMI_OK;
}

// ---- training reverse path (trainer.cpp:549-561) ------------------------------------------

static_assert(sizeof(LumiTrainRay) == sizeof(lumi_dev::LumiTrainRayDev), "LumiTrainRay layout");

int lumi_train_backward_async(LumiModel* m, const LumiTrainRay* rays, int nrays,
                              const double* cam_tnf, const double* alpha_v, int ncams,
                              const LumiRenderOptions* o, const LumiLossConfig* lc,
                              const LumiTrainGrads* g, int32_t* ray_evals, int32_t* ray_contrib,
                              void* stream) {
  if (!m) return fail(LUMI_ERR_INVALID, "null model");
  if (!lc || !g || !g->grid || !g->density || !g->color || !g->alpha_v || !g->loss)
    return fail(LUMI_ERR_INVALID, "train_backward: null loss config or gradient buffer");
  if (nrays < 0 || (nrays > 0 && !rays)) return fail(LUMI_ERR_INVALID, "train_backward: bad rays");
  if (ncams < 1 || !cam_tnf || !alpha_v) return fail(LUMI_ERR_INVALID, "train_backward: bad cameras");
  int rc;
  if ((rc = check_opts(o))) return rc;
  for (int c = 0; c < ncams; ++c)  // renderer.h:134
    if (!(cam_tnf[2 * c] > 0 && cam_tnf[2 * c + 1] > cam_tnf[2 * c]))
      return fail(LUMI_ERR_INVALID, "march_ray: bad sampling interval");
  DeviceGuard dg(m->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // grid / MLP / occupancy descriptors through the render parameter block
  RenderParams rp;
  LumiCameraDesc dummy{};
  dummy.rot[0] = dummy.rot[4] = dummy.rot[8] = 1.0;
  dummy.fx = dummy.fy = 1.0;
  dummy.width = dummy.height = 1;
  dummy.t_near = cam_tnf[0];
  dummy.t_far = cam_tnf[1];
  if ((rc = make_params(m, &dummy, o, 0, 0, &rp))) return rc;
  // per-camera exponential distances and step ratios (renderer.h:135-142), host libm
  const int n = o->samples_per_ray;
  std::vector<double> host((size_t)ncams * n + 2 * (size_t)ncams);
  for (int c = 0; c < ncams; ++c) {
    const double tn = cam_tnf[2 * c], tf = cam_tnf[2 * c + 1];
    double* ts = host.data() + (size_t)c * n;
    const double log_ratio = std::log(tf / tn);
    for (int i = 0; i < n; ++i) ts[i] = tn * std::exp(log_ratio * (static_cast<double>(i) / (n - 1)));
    ts[0] = tn;
    ts[n - 1] = tf;
    host[(size_t)ncams * n + c] = std::pow(tf / tn, 1.0 / (n - 1));
    host[(size_t)ncams * n + ncams + c] = alpha_v[c];
  }
  double* d_cam = nullptr;
  LUMI_CUDA_TRY(cudaMallocAsync(&d_cam, host.size() * sizeof(double), s));
  cudaError_t e = cudaMemcpyAsync(d_cam, host.data(), host.size() * sizeof(double),
                                  cudaMemcpyHostToDevice, s);
  lumi_dev::TrainParams p;
  std::memset(&p, 0, sizeof(p));
  p.grid = rp.grid;
  p.mlp = rp.mlp;
  p.occ = rp.occ;
  p.occ_res = rp.occ_res;
  p.n = n;
  p.lod_enabled = rp.lod_enabled;
  p.lod_bias = rp.lod_bias;
  p.t_cut = rp.t_cut;
  for (int c = 0; c < 3; ++c) p.bg[c] = rp.bg[c];
  p.contraction = rp.contraction;
  p.chunk = rp.chunk;
  p.rays = reinterpret_cast<const lumi_dev::LumiTrainRayDev*>(rays);
  p.nrays = nrays;
  p.ncams = ncams;
  p.cam_ts = d_cam;
  p.cam_ratio = d_cam + (size_t)ncams * n;
  p.alpha_v = d_cam + (size_t)ncams * n + ncams;
  p.lambda_depth = lc->lambda_depth;
  p.lambda_dvar = lc->lambda_dvar;
  p.lambda_dist = lc->lambda_dist;
  p.inv_batch = lc->inv_batch;
  p.depth_active = lc->depth_active;
  p.g_grid = g->grid;
  p.g_density = g->density;
  p.g_color = g->color;
  p.alpha_grad = g->alpha_v;
  p.loss = reinterpret_cast<double*>(g->loss);
  p.ray_evals = ray_evals;
  p.ray_contrib = ray_contrib;
  if (e == cudaSuccess) e = launch_train_backward(p, s, m->num_sms, nullptr, nullptr);
  cudaFreeAsync(d_cam, s);
  if (e != cudaSuccess) return fail(LUMI_ERR_CUDA, std::string("train_backward: ") + cudaGetErrorString(e));
  return LUMI_OK;
}

int lumi_train_backward(LumiModel* m, const LumiTrainRay* rays, int nrays, const double* cam_tnf,
                        const double* alpha_v, int ncams, const LumiRenderOptions* o,
                        const LumiLossConfig* lc, const LumiTrainGrads* g, int32_t* ray_evals,
                        int32_t* ray_contrib) {
  if (!m) return fail(LUMI_ERR_INVALID, "null model");
  if (!g || !g->grid || !g->density || !g->color || !g->alpha_v || !g->loss)
    return fail(LUMI_ERR_INVALID, "train_backward: null gradient buffer");
  if (ncams < 1) return fail(LUMI_ERR_INVALID, "train_backward: bad cameras");
  DeviceGuard dg(m->device);
  const size_t ng = m->layout.total_floats, nd = m->layout.density_params,
               nc = m->layout.color_params, nr = (size_t)std::max(nrays, 0);
  char* buf = nullptr;
  const size_t bytes = nr * sizeof(LumiTrainRay) + (ng + nd + nc) * sizeof(float) +
                       ncams * sizeof(double) + sizeof(LumiLossTerms) + 2 * nr * sizeof(int32_t) + 256;
  LUMI_CUDA_TRY(cudaMalloc(&buf, bytes));
  auto done = [&](int code) {
    cudaFree(buf);
    return code;
  };
  LumiTrainRay* d_rays = reinterpret_cast<LumiTrainRay*>(buf);
  LumiTrainGrads dg_{};
  dg_.grid = reinterpret_cast<float*>(d_rays + nr);
  dg_.density = dg_.grid + ng;
  dg_.color = dg_.density + nd;
  dg_.alpha_v = reinterpret_cast<double*>(
      (reinterpret_cast<uintptr_t>(dg_.color + nc) + 7) & ~static_cast<uintptr_t>(7));
  dg_.loss = reinterpret_cast<LumiLossTerms*>(dg_.alpha_v + ncams);
  int32_t* d_ev = reinterpret_cast<int32_t*>(dg_.loss + 1);
  int32_t* d_co = d_ev + nr;
  cudaError_t e;
  if ((nr && (e = cudaMemcpy(d_rays, rays, nr * sizeof(LumiTrainRay), cudaMemcpyHostToDevice))) ||
      (e = cudaMemcpy(dg_.grid, g->grid, ng * sizeof(float), cudaMemcpyHostToDevice)) ||
      (e = cudaMemcpy(dg_.density, g->density, nd * sizeof(float), cudaMemcpyHostToDevice)) ||
      (e = cudaMemcpy(dg_.color, g->color, nc * sizeof(float), cudaMemcpyHostToDevice)) ||
      (e = cudaMemcpy(dg_.alpha_v, g->alpha_v, ncams * sizeof(double), cudaMemcpyHostToDevice)) ||
      (e = cudaMemcpy(dg_.loss, g->loss, sizeof(LumiLossTerms), cudaMemcpyHostToDevice)))
    return done(fail(LUMI_ERR_CUDA, cudaGetErrorString(e)));
  int rc = lumi_train_backward_async(m, d_rays, nrays, cam_tnf, alpha_v, ncams, o, lc, &dg_, d_ev,
                                     d_co, nullptr);
  if (rc) return done(rc);
  if ((e = cudaMemcpy(g->grid, dg_.grid, ng * sizeof(float), cudaMemcpyDeviceToHost)) ||
      (e = cudaMemcpy(g->density, dg_.density, nd * sizeof(float), cudaMemcpyDeviceToHost)) ||
      (e = cudaMemcpy(g->color, dg_.color, nc * sizeof(float), cudaMemcpyDeviceToHost)) ||
      (e = cudaMemcpy(g->alpha_v, dg_.alpha_v, ncams * sizeof(double), cudaMemcpyDeviceToHost)) ||
      (e = cudaMemcpy(g->loss, dg_.loss, sizeof(LumiLossTerms), cudaMemcpyDeviceToHost)) ||
      (ray_evals && nr && (e = cudaMemcpy(ray_evals, d_ev, nr * sizeof(int32_t), cudaMemcpyDeviceToHost))) ||
      (ray_contrib && nr && (e = cudaMemcpy(ray_contrib, d_co, nr * sizeof(int32_t), cudaMemcpyDeviceToHost))))
    return done(fail(LUMI_ERR_CUDA, cudaGetErrorString(e)));
  return done(LUMI_OK);
}

int lumi_model_device_params(LumiModel* m, float** table, float** density, float** color) {
  if (!m) return fail(LUMI_ERR_INVALID, "null model");
  if (table) *table = m->d_table;
  if (density) *density = m->d_dparams;
  if (color) *color = m->d_cparams;
  return LUMI_OK;
}

int lumi_model_params_updated(LumiModel* m) {
  if (!m) return fail(LUMI_ERR_INVALID, "null model");
  DeviceGuard dg(m->device);
  std::vector<float> dp(m->layout.density_params), cp(m->layout.color_params);
  LUMI_CUDA_TRY(cudaDeviceSynchronize());
  LUMI_CUDA_TRY(launch_to_half(m->d_table, m->d_table16, m->layout.total_floats, nullptr));
  LUMI_CUDA_TRY(cudaMemcpy(dp.data(), m->d_dparams, dp.size() * sizeof(float), cudaMemcpyDeviceToHost));
  LUMI_CUDA_TRY(cudaMemcpy(cp.data(), m->d_cparams, cp.size() * sizeof(float), cudaMemcpyDeviceToHost));
  const std::vector<float> fused = fuse_l2_c1(dp.data(), cp.data());
  LUMI_CUDA_TRY(cudaMemcpy(m->d_fused, fused.data(), fused.size() * sizeof(float), cudaMemcpyHostToDevice));
  LUMI_CUDA_TRY(launch_pack_weight_tiles(lumi_dev::MlpDev{m->d_dparams, m->d_cparams, m->d_fused,
                                                         m->desc.color_space, nullptr},
                                         m->d_wtiles, nullptr));
  LUMI_CUDA_TRY(cudaDeviceSynchronize());
  return LUMI_OK;
}

// ---- scheduler (scheduler.cpp:18-162) -----------------------------------------------------

static void round_rows(const double* shares, int n, int height, int32_t* rows) {
  std::vector<std::pair<double, int>> rem(n);
  int assigned = 0;
  for (int i = 0; i < n; ++i) {
    double exact = shares[i] * height;
    rows[i] = static_cast<int>(std::floor(exact));
    rem[i] = {exact - rows[i], i};
    assigned += rows[i];
  }
  std::sort(rem.begin(), rem.end(), [](const auto& a, const auto& b) {
    if (a.first != b.first) return a.first > b.first;
    return a.second < b.second;
  });
  for (int k = 0; k < height - assigned; ++k) rows[rem[k % n].second] += 1;
  if (height >= n) {
    for (int i = 0; i < n; ++i) {
      while (rows[i] == 0) {
        int big = static_cast<int>(std::max_element(rows, rows + n) - rows);
        rows[big] -= 1;
        rows[i] += 1;
      }
    }
  }
}

// ---- peer-memory frame gather ----------------------------------------------------------
// The reference's workers store their rows into one shared Image (scheduler.cpp:114-152); here
// a rank maps rank 0's frame buffer and its render kernel stores its band there over NVLink.
// The handle names the whole cudaMalloc allocation (a torch caching-allocator segment), so the
// pointer's offset inside it travels alongside; the allocation base comes from the driver's
// cuMemGetAddressRange, fetched through the runtime (no -lcuda link).
static std::mutex g_ipc_mu;
static std::map<void*, void*> g_ipc_maps;  // returned pointer -> mapped allocation base

int lumi_ipc_export(const void* ptr, void* handle, uint64_t* offset) {
  if (!ptr || !handle || !offset) return fail(LUMI_ERR_INVALID, "null argument");
  using GetRange = int (*)(unsigned long long*, size_t*, unsigned long long);
  static GetRange get_range = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuMemGetAddressRange", &fn, 12000, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      fn = nullptr;
    return reinterpret_cast<GetRange>(fn);
  }();
  if (!get_range) return fail(LUMI_ERR_CUDA, "cuMemGetAddressRange unavailable");
  unsigned long long base = 0;
  size_t size = 0;
  const auto p = reinterpret_cast<unsigned long long>(ptr);
  if (get_range(&base, &size, p) != 0) return fail(LUMI_ERR_INVALID, "ipc export: not a device allocation");
  cudaIpcMemHandle_t h;
  LUMI_CUDA_TRY(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
  static_assert(sizeof(h) == LUMI_IPC_HANDLE_BYTES, "handle size");
  std::memcpy(handle, &h, sizeof(h));
  *offset = p - base;
  return LUMI_OK;
}

int lumi_ipc_open(int device, const void* handle, uint64_t offset, void** out) {
  if (!handle || !out) return fail(LUMI_ERR_INVALID, "null argument");
  DeviceGuard dg(device);
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  void* base = nullptr;
  LUMI_CUDA_TRY(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
  void* p = static_cast<char*>(base) + offset;
  std::lock_guard<std::mutex> lk(g_ipc_mu);
  g_ipc_maps[p] = base;
  *out = p;
  return LUMI_OK;
}

int lumi_ipc_close(int device, void* ptr) {
  void* base = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_ipc_mu);
    auto it = g_ipc_maps.find(ptr);
    if (it == g_ipc_maps.end()) return fail(LUMI_ERR_INVALID, "ipc close: pointer was not opened here");
    base = it->second;
    g_ipc_maps.erase(it);
  }
  DeviceGuard dg(device);
  LUMI_CUDA_TRY(cudaIpcCloseMemHandle(base));
  return LUMI_OK;
}

int lumi_equal_assignment(int height, int workers, int32_t* rows, double* shares) {
  if (workers < 1) return fail(LUMI_ERR_INVALID, "assignment: need at least one worker");
  if (height < workers) return fail(LUMI_ERR_INVALID, "assignment: more workers than rows");
  if (!rows || !shares) return fail(LUMI_ERR_INVALID, "null output");
  std::vector<double> s(workers, 1.0 / workers);
  round_rows(s.data(), workers, height, rows);
  for (int i = 0; i < workers; ++i) shares[i] = static_cast<double>(rows[i]) / height;
  return LUMI_OK;
}

int lumi_assign_rows(int height, int n, const double* tp, const double* prev_shares, double damp,
                     int32_t* rows, double* shares) {
  if (!(n >= 1 && height >= n)) return fail(LUMI_ERR_INVALID, "assign_rows: more workers than rows");
  if (!tp || !prev_shares || !rows || !shares) return fail(LUMI_ERR_INVALID, "null argument");
  double total = 0;
  for (int i = 0; i < n; ++i) {
    if (!(tp[i] > 0)) return fail(LUMI_ERR_INVALID, "assign_rows: throughputs must be positive");
    total += tp[i];
  }
  std::vector<double> s(n);
  for (int i = 0; i < n; ++i) {
    double target = tp[i] / total;
    s[i] = prev_shares[i] + damp * (target - prev_shares[i]);
  }
  double sum = std::accumulate(s.begin(), s.end(), 0.0);
  for (auto& v : s) v /= sum;
  round_rows(s.data(), n, height, rows);
  int at = 0;
  for (int i = 0; i < n; ++i) {
    shares[i] = static_cast<double>(rows[i]) / height;
    at += rows[i];
  }
  if (at != height) return fail(LUMI_ERR_INVALID, "assign_rows: partition does not cover all rows");
  return LUMI_OK;
}

int lumi_next_assignment(int height, int n, const double* prev_shares, const int32_t* prev_rows,
                         const double* worker_ms, int width, double damp, int32_t* rows,
                         double* shares) {
  if (!prev_rows || !worker_ms) return fail(LUMI_ERR_INVALID, "null argument");
  std::vector<double> tp(n);
  for (int i = 0; i < n; ++i) {
    double ms = std::max(worker_ms[i], 1e-6);
    tp[i] = std::max(static_cast<double>(static_cast<int64_t>(prev_rows[i]) * width), 1.0) /
            (ms / 1000.0);
  }
  return lumi_assign_rows(height, n, tp.data(), prev_shares, damp, rows, shares);
}

int lumi_aggregate_stats(const double* ms, int n, double* mean_fps, double* std_fps,
                         double* p99_fps) {
  if (n <= 0 || !ms) return fail(LUMI_ERR_INVALID, "aggregate_stats: no frames");
  std::vector<double> times(ms, ms + n);
  auto fps = [](double w) { return w > 0 ? 1000.0 / w : 0.0; };
  double mean = 0;
  for (double w : times) mean += fps(w);
  mean /= n;
  double var = 0;
  for (double w : times) var += (fps(w) - mean) * (fps(w) - mean);
  var /= n;
  std::sort(times.begin(), times.end());
  double idx = 0.99 * (times.size() - 1);
  size_t lo = static_cast<size_t>(std::floor(idx));
  size_t hi = std::min(lo + 1, times.size() - 1);
  double frac = idx - lo;
  double p99 = times[lo] * (1 - frac) + times[hi] * frac;
  if (mean_fps) *mean_fps = mean;
  if (std_fps) *std_fps = std::sqrt(var);
  if (p99_fps) *p99_fps = p99 > 0 ? 1000.0 / p99 : 0.0;
  return LUMI_OK;
}

}  // extern "C"
