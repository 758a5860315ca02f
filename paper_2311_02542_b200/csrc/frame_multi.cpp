// frame_multi.cpp -- the native multi-GPU frame driver behind the C ABI (lumi_frame_driver_*).
//
// The reference's multi-worker frame (run_frame, proj/src/scheduler.cpp:114-152) starts one
// std::thread per worker, each renders its contiguous row range of one shared Image, the frame
// joins, per-worker times feed next_assignment (scheduler.cpp:154-162).  Here a worker is a GPU
// (or, for testing, one stream of a shared GPU): one persistent host thread per worker drives
// its own device model through lumi_render_rows_async on its own stream, and the render
// kernel's pixel stores go straight into the frame target on the target device -- over NVLink
// peer access when the worker's GPU is not the target's -- so the gather of the reference's
// shared Image is the kernels' epilogue, with no copy afterwards.  Per-worker CUDA-event
// milliseconds drive the native next_assignment for the following frame.  Worker failures
// abort the frame with the reference's message ("run_frame: worker i failed: ...").
//
// Layered on the public C ABI only (include/lumi_cuda.h), as run_frame is layered on
// render_rows.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <set>
#include <string>
#include <thread>
#include <utility>
#include <vector>

#include "lumi_cuda.h"

extern "C" int lumi_set_error(int code, const char* msg);

namespace {

int fail(int code, const std::string& msg) { return lumi_set_error(code, msg.c_str()); }

}  // namespace

struct LumiFrameDriver {
  struct Worker {
    LumiModel* model = nullptr;
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    std::thread th;
    // per frame
    int rc = LUMI_OK;
    std::string err;
    double ms = 0.0;
  };
  std::vector<Worker> w;
  int width = 0, eye_height = 0, eyes = 0, height = 0;
  double damp = 0.5;
  std::vector<int32_t> rows;
  std::vector<double> shares;
  std::set<std::pair<int, int>> peer_enabled;  // (worker device, target device)
  // the frame being rendered
  std::mutex mu;
  std::condition_variable go, done;
  uint64_t frame = 0;
  int pending = 0;
  bool quit = false;
  const LumiCameraDesc* cams = nullptr;
  LumiRenderOptions opts{};
  LumiFrameTarget target{};
  // the frame lumi_frame_driver_render_host renders into (worker 0's device, lazily allocated)
  float* d_frame = nullptr;

  void work(int i);
  int render_band(int i, int b, int e);
};

int LumiFrameDriver::render_band(int i, int b, int e) {
  // a band of the stacked image becomes one launch per eye it touches
  for (int eye = 0; eye < eyes; ++eye) {
    const int lo = std::max(b, eye * eye_height), hi = std::min(e, (eye + 1) * eye_height);
    if (lo >= hi) continue;
    LumiFrameTarget t = target;
    t.row_offset = target.row_offset + eye * eye_height;
    const int rc = lumi_render_rows_async(w[i].model, &cams[eye], &opts, lo - eye * eye_height,
                                          hi - eye * eye_height, &t, w[i].stream);
    if (rc) return rc;
  }
  return LUMI_OK;
}

void LumiFrameDriver::work(int i) {
  uint64_t seen = 0;
  for (;;) {
    int b = 0, e = 0;
    {
      std::unique_lock<std::mutex> lk(mu);
      go.wait(lk, [&] { return quit || frame != seen; });
      if (quit) return;
      seen = frame;
      for (int k = 0; k < i; ++k) b += rows[k];
      e = b + rows[i];
    }
    Worker& me = w[i];
    me.rc = LUMI_OK;
    me.err.clear();
    me.ms = 0.0;
    cudaError_t ce = cudaSetDevice(me.device);
    if (ce == cudaSuccess) ce = cudaEventRecord(me.e0, me.stream);
    if (ce != cudaSuccess) {
      me.rc = LUMI_ERR_CUDA;
      me.err = cudaGetErrorString(ce);
    } else {
      me.rc = render_band(i, b, e);
      if (me.rc) me.err = lumi_last_error();
      if ((ce = cudaEventRecord(me.e1, me.stream)) != cudaSuccess ||
          (ce = cudaEventSynchronize(me.e1)) != cudaSuccess) {
        if (!me.rc) me.err = cudaGetErrorString(ce);
        me.rc = me.rc ? me.rc : LUMI_ERR_CUDA;
      } else if (!me.rc) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, me.e0, me.e1);
        me.ms = ms;
      }
    }
    std::lock_guard<std::mutex> lk(mu);
    if (--pending == 0) done.notify_all();
  }
}

extern "C" {

int lumi_frame_driver_create(LumiModel* const* models, int workers, int width, int eye_height,
                             int eyes, double dampening, LumiFrameDriver** out) {
  if (!out) return fail(LUMI_ERR_INVALID, "null output handle");
  *out = nullptr;
  if (!models || workers < 1) return fail(LUMI_ERR_INVALID, "frame driver: need at least one worker");
  if (width < 1 || eye_height < 1 || eyes < 1 || eyes > 2)
    return fail(LUMI_ERR_INVALID, "frame driver: bad frame size");
  if (!(dampening > 0.0 && dampening <= 1.0)) return fail(LUMI_ERR_INVALID, "frame driver: bad dampening");
  auto d = new LumiFrameDriver();
  d->width = width;
  d->eye_height = eye_height;
  d->eyes = eyes;
  d->height = eyes * eye_height;
  d->damp = dampening;
  d->rows.resize(workers);
  d->shares.resize(workers);
  int rc = lumi_equal_assignment(d->height, workers, d->rows.data(), d->shares.data());
  if (rc) {
    delete d;
    return rc;
  }
  d->w.resize(workers);
  int prev = 0;
  cudaGetDevice(&prev);
  for (int i = 0; i < workers; ++i) {
    auto& wk = d->w[i];
    wk.model = models[i];
    if (!wk.model || (rc = lumi_model_device(wk.model, &wk.device))) {
      lumi_frame_driver_destroy(d);
      return rc ? rc : fail(LUMI_ERR_INVALID, "frame driver: null model");
    }
    cudaError_t ce;
    if ((ce = cudaSetDevice(wk.device)) != cudaSuccess ||
        (ce = cudaStreamCreateWithFlags(&wk.stream, cudaStreamNonBlocking)) != cudaSuccess ||
        (ce = cudaEventCreate(&wk.e0)) != cudaSuccess || (ce = cudaEventCreate(&wk.e1)) != cudaSuccess) {
      cudaSetDevice(prev);
      lumi_frame_driver_destroy(d);
      return fail(LUMI_ERR_CUDA, std::string("frame driver: ") + cudaGetErrorString(ce));
    }
  }
  cudaSetDevice(prev);
  for (int i = 0; i < workers; ++i) d->w[i].th = std::thread([d, i] { d->work(i); });
  *out = d;
  return LUMI_OK;
}

int lumi_frame_driver_destroy(LumiFrameDriver* d) {
  if (!d) return LUMI_OK;
  {
    std::lock_guard<std::mutex> lk(d->mu);
    d->quit = true;
  }
  d->go.notify_all();
  for (auto& wk : d->w)
    if (wk.th.joinable()) wk.th.join();
  if (d->d_frame) {
    cudaSetDevice(d->w[0].device);
    cudaFree(d->d_frame);
  }
  for (auto& wk : d->w) {
    if (!wk.stream) continue;
    cudaSetDevice(wk.device);
    cudaStreamSynchronize(wk.stream);
    cudaEventDestroy(wk.e0);
    cudaEventDestroy(wk.e1);
    cudaStreamDestroy(wk.stream);
  }
  delete d;
  return LUMI_OK;
}

int lumi_frame_driver_assignment(const LumiFrameDriver* d, int32_t* rows, double* shares) {
  if (!d) return fail(LUMI_ERR_INVALID, "null frame driver");
  const size_t n = d->rows.size();
  if (rows) std::memcpy(rows, d->rows.data(), n * sizeof(int32_t));
  if (shares) std::memcpy(shares, d->shares.data(), n * sizeof(double));
  return LUMI_OK;
}

int lumi_frame_driver_set_assignment(LumiFrameDriver* d, const int32_t* rows) {
  if (!d || !rows) return fail(LUMI_ERR_INVALID, "null argument");
  int total = 0;
  for (size_t i = 0; i < d->rows.size(); ++i) {
    if (rows[i] < 0) return fail(LUMI_ERR_INVALID, "run_frame: invalid assignment");
    total += rows[i];
  }
  if (total != d->height) return fail(LUMI_ERR_INVALID, "run_frame: invalid assignment");
  for (size_t i = 0; i < d->rows.size(); ++i) {
    d->rows[i] = rows[i];
    d->shares[i] = static_cast<double>(rows[i]) / d->height;
  }
  return LUMI_OK;
}

int lumi_frame_driver_render(LumiFrameDriver* d, const LumiCameraDesc* cams,
                             const LumiRenderOptions* opts, const LumiFrameTarget* target,
                             double* wall_ms, double* worker_ms, int64_t* worker_rays) {
  if (!d) return fail(LUMI_ERR_INVALID, "null frame driver");
  if (!cams || !opts || !target || !target->rgb) return fail(LUMI_ERR_INVALID, "null argument");
  if (target->width != d->width || target->row_offset < 0 ||
      target->row_offset + d->height > target->height)
    return fail(LUMI_ERR_INVALID, "frame driver: frame target does not hold the stacked eyes");
  for (int e = 0; e < d->eyes; ++e)
    if (cams[e].width != d->width || cams[e].height != d->eye_height)
      return fail(LUMI_ERR_INVALID, "frame driver: camera size differs from the eyebuffer size");
  // the workers' kernels store into the target's device: enable peer access once per pair
  cudaPointerAttributes pa;
  cudaError_t ce = cudaPointerGetAttributes(&pa, target->rgb);
  if (ce != cudaSuccess || pa.type != cudaMemoryTypeDevice) {
    cudaGetLastError();
    return fail(LUMI_ERR_INVALID, "frame driver: the frame target must be device memory");
  }
  int prev = 0;
  cudaGetDevice(&prev);
  for (auto& wk : d->w) {
    const auto key = std::make_pair(wk.device, pa.device);
    if (wk.device == pa.device || d->peer_enabled.count(key)) continue;
    int can = 0;
    cudaDeviceCanAccessPeer(&can, wk.device, pa.device);
    if (!can) {
      cudaSetDevice(prev);
      return fail(LUMI_ERR_UNSUPPORTED, "frame driver: GPU " + std::to_string(wk.device) +
                                            " cannot access GPU " + std::to_string(pa.device));
    }
    cudaSetDevice(wk.device);
    ce = cudaDeviceEnablePeerAccess(pa.device, 0);
    if (ce != cudaSuccess && ce != cudaErrorPeerAccessAlreadyEnabled) {
      cudaSetDevice(prev);
      return fail(LUMI_ERR_CUDA, std::string("frame driver: peer access: ") + cudaGetErrorString(ce));
    }
    cudaGetLastError();
    d->peer_enabled.insert(key);
  }
  cudaSetDevice(prev);
  const auto t0 = std::chrono::steady_clock::now();
  {
    std::unique_lock<std::mutex> lk(d->mu);
    d->cams = cams;
    d->opts = *opts;
    d->target = *target;
    d->pending = static_cast<int>(d->w.size());
    ++d->frame;
    d->go.notify_all();
    d->done.wait(lk, [&] { return d->pending == 0; });
  }
  const double wall =
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  const int n = static_cast<int>(d->w.size());
  for (int i = 0; i < n; ++i)
    if (d->w[i].rc)
      return fail(d->w[i].rc, "run_frame: worker " + std::to_string(i) + " failed: " + d->w[i].err);
  std::vector<double> ms(n);
  for (int i = 0; i < n; ++i) {
    ms[i] = d->w[i].ms;
    if (worker_ms) worker_ms[i] = ms[i];
    if (worker_rays) worker_rays[i] = static_cast<int64_t>(d->rows[i]) * d->width;
  }
  if (wall_ms) *wall_ms = wall;
  // next frame's partition from this frame's per-GPU throughput (scheduler.cpp:154-162)
  if (n > 1) {
    std::vector<int32_t> rows(n);
    std::vector<double> shares(n);
    const int rc = lumi_next_assignment(d->height, n, d->shares.data(), d->rows.data(), ms.data(),
                                        d->width, d->damp, rows.data(), shares.data());
    if (rc) return rc;
    d->rows = rows;
    d->shares = shares;
  }
  return LUMI_OK;
}

int lumi_frame_driver_render_host(LumiFrameDriver* d, const LumiCameraDesc* cams,
                                  const LumiRenderOptions* opts, float* out, double* wall_ms,
                                  double* worker_ms, int64_t* worker_rays) {
  if (!d) return fail(LUMI_ERR_INVALID, "null frame driver");
  if (!out) return fail(LUMI_ERR_INVALID, "null output image");
  const size_t n = static_cast<size_t>(3) * d->height * d->width;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaError_t ce = cudaSetDevice(d->w[0].device);
  if (ce == cudaSuccess && !d->d_frame) ce = cudaMalloc(&d->d_frame, n * sizeof(float));
  cudaSetDevice(prev);
  if (ce != cudaSuccess) return fail(LUMI_ERR_CUDA, std::string("frame driver: ") + cudaGetErrorString(ce));
  LumiFrameTarget t{};
  t.rgb = d->d_frame;
  t.width = d->width;
  t.height = d->height;
  const auto t0 = std::chrono::steady_clock::now();
  int rc = lumi_frame_driver_render(d, cams, opts, &t, nullptr, worker_ms, worker_rays);
  if (rc) return rc;
  cudaSetDevice(d->w[0].device);
  ce = cudaMemcpy(out, d->d_frame, n * sizeof(float), cudaMemcpyDeviceToHost);
  cudaSetDevice(prev);
  if (ce != cudaSuccess) return fail(LUMI_ERR_CUDA, std::string("frame driver: ") + cudaGetErrorString(ce));
  if (wall_ms)
    *wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  return LUMI_OK;
}

}  // extern "C"
