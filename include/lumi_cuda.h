/*
 * lumi_cuda.h -- C ABI of the B200-native VR-NeRF frame renderer.
 *
 * This is the drop-in boundary for the reference's rendering path: every entry point
 * takes plain pointers, sizes and POD descriptors (no CUDA, C++ or torch types; CUDA
 * streams are passed as `void*`), returns a LUMI_* status and leaves a thread-local
 * message in lumi_last_error().  The C++ shim in include/lumi/cuda_renderer.h binds the
 * reference API (proj/include/lumi/renderer.h) onto it; INTEGRATION.md shows the binding.
 *
 * Reference interfaces replaced (paths relative to the reference checkout):
 *   lumi_render_rows            render_rows<FieldT>          proj/include/lumi/renderer.h:252-278
 *   lumi_render_rows_async      (device-resident form of the same, one stream per worker)
 *   lumi_march_kept_async       march_ray occupancy skip     proj/include/lumi/renderer.h:205-208
 *   lumi_model_create           RadianceField<float> + OccupancyGrid state
 *                               proj/include/lumi/field.h:65-93, grid.h:58-74,
 *                               network.h:144-159, occupancy.h:32-100
 *   lumi_field_layout           MultiResHashGrid layout      proj/include/lumi/grid.h:58-74
 *   lumi_synth_params           RadianceField::init_random   proj/include/lumi/field.h:88-93
 *   lumi_bake_occupancy         OccupancyGrid::probe + prune proj/src/occupancy.cpp:97-154
 *   lumi_equal_assignment, lumi_assign_rows, lumi_next_assignment, lumi_aggregate_stats
 *                               the row scheduler            proj/src/scheduler.cpp:18-162
 *   lumi_train_backward[_async] the training loop's per-ray body: march_ray(record) +
 *                               ray_loss + backward_ray      proj/src/trainer.cpp:549-561,
 *                               proj/include/lumi/train_step.h:16-154, renderer.h:110-120,
 *                               field.h:141-179, network.h:115-136, grid.h:118-137
 *   lumi_model_device_params, lumi_model_params_updated
 *                               in-place parameter access for a device-side optimizer
 *   lumi_frame_driver_create / _render[_host] / _assignment / _set_assignment / _destroy
 *                               run_frame + next_assignment with GPUs as the workers: one
 *                               host thread per GPU, bands stored into one device frame
 *                               over NVLink peer access  proj/src/scheduler.cpp:114-162
 *   lumi_checkpoint_read, lumi_checkpoint_write
 *                               load_checkpoint / save_checkpoint   proj/src/scene.cpp:320-394
 *   lumi_ipc_export, lumi_ipc_open, lumi_ipc_close
 *                               the frame gather of run_frame (results gathered by row
 *                               index into one shared Image, proj/src/scheduler.cpp:114-152)
 *                               as peer memory: a rank maps rank 0's frame buffer and its
 *                               render kernel stores its band there over NVLink
 *
 * All device work is sm_100a CUDA (paper_2311_02542_b200/csrc); there is no CPU
 * fallback -- without a usable B200 the calls fail with LUMI_ERR_CUDA.
 */
#ifndef LUMI_CUDA_H
#define LUMI_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LUMI_ABI_VERSION 1
#define LUMI_MAX_LEVELS 16

enum {
  LUMI_OK = 0,
  LUMI_ERR_INVALID = 1,     /* bad argument; the reference raises lumi::Error */
  LUMI_ERR_CUDA = 2,        /* CUDA runtime failure / no device */
  LUMI_ERR_UNSUPPORTED = 3, /* configuration outside what the kernels implement */
};

/* proj/include/lumi/grid.h:18-29 + proj/include/lumi/field.h:22-27 */
typedef struct LumiFieldDesc {
  int32_t levels;             /* <= LUMI_MAX_LEVELS */
  int32_t features_per_level; /* must be 2 */
  int32_t base_resolution;
  int32_t hidden_width; /* must be 64 */
  double per_level_scale;
  uint32_t table_size; /* power of two */
  int32_t bottleneck;  /* must be 16 */
  int32_t color_space; /* 0 = kPq (sigmoid head), 1 = kLinear (trunc_exp head) */
  int32_t _pad;
} LumiFieldDesc;

/* MultiResHashGrid storage layout (grid.h:58-74): one float array, level l at
   offset[l] floats, entry e at +e*features_per_level. */
typedef struct LumiGridLayout {
  int32_t levels;
  int32_t features_per_level;
  int32_t resolution[LUMI_MAX_LEVELS];
  uint32_t entries[LUMI_MAX_LEVELS];
  uint8_t dense[LUMI_MAX_LEVELS];
  uint64_t offset[LUMI_MAX_LEVELS];
  uint64_t total_floats;
  uint64_t density_params; /* floats, weights then bias per layer (network.h:144-151) */
  uint64_t color_params;
} LumiGridLayout;

/* proj/include/lumi/camera.h:15-23 (pose row-major world <- camera) */
typedef struct LumiCameraDesc {
  double rot[9];
  double origin[3];
  double fx, fy, cx, cy;
  int32_t width, height;
  double t_near, t_far;
} LumiCameraDesc;

/* proj/include/lumi/renderer.h:22-30 */
typedef struct LumiRenderOptions {
  int32_t samples_per_ray; /* 2..1024 */
  int32_t lod_enabled;
  double lod_bias;
  double termination_transmittance; /* 0 disables the early cut */
  double background[3];             /* model-space (PQ) background */
  int32_t contraction;              /* 0 = kNone, 1 = kLInfCubic */
  int32_t chunk_size;               /* only shapes RowStats.evals, as in the reference */
} LumiRenderOptions;

/* proj/include/lumi/renderer.h:241-246 */
typedef struct LumiRowStats {
  int32_t row;
  int32_t _pad;
  double ms;
  int64_t rays;
  int64_t evals;
} LumiRowStats;

/* Device-resident frame target for the async entry points.  Planar channel-major
   images (image.h:16-35) of `width` x `height`; camera row y lands in target row
   `row_offset + y` (so both eyes of a stereo pair stack into one buffer).  Optional
   planes may be NULL.  `counts` receives per pixel {evals, contributing} (int32 x2);
   `row_evals` receives per camera row the sum of evals (indexed by camera row); `row_cycles`
   (optional, appended for the per-row cost diagnostic of RowStats.ms, renderer.h:261-276)
   receives per camera row the SM cycles the render kernel's packet streams spent on it (each
   packet's cycles split evenly over its 4 rows), accumulated. */
typedef struct LumiFrameTarget {
  float* rgb;
  float* depth;
  float* opacity;
  int32_t* counts;
  int64_t* row_evals;
  uint8_t* srgb8; /* optional interleaved RGB8 display buffer (PQ -> sRGB epilogue) */
  /* optional device counters, accumulated (not reset): [0] network evaluations actually
     executed, [1] active (w_l > 0) level-samples gathered, [2] candidates the march pass
     tested (empty-space skipping jumps the rest),
     [3] rays.  Used for the algorithmic-bytes roofline. */
  uint64_t* work_stats;
  double exposure_bias_stops;
  int32_t width;
  int32_t height;
  int32_t row_offset;
  int32_t _pad;
  int64_t* row_cycles;
} LumiFrameTarget;

typedef struct LumiModel LumiModel;

const char* lumi_last_error(void);
int lumi_abi_version(void);
/* Fills `info` (>= 256 bytes) with the device name / SM count; LUMI_ERR_CUDA without one. */
int lumi_device_info(int device, char* info, size_t info_len);

/* ---- model ---------------------------------------------------------------------- */
int lumi_field_layout(const LumiFieldDesc* desc, LumiGridLayout* out);
/* Seeded synthetic parameters, bit-identical to RadianceField<float>::init_random(seed)
   followed (amp > 0) by the grid overwrite Rng(seed+1).uniform(-amp, amp). Host memory. */
int lumi_synth_params(const LumiFieldDesc* desc, uint64_t seed, double amp, float* table,
                      float* density_params, float* color_params);
/* Uploads a field + occupancy (host pointers) to `device`.  occupancy: occ_res^3 bytes,
   nonzero = occupied, index (iz*res+iy)*res+ix (occupancy.cpp:22-29). */
int lumi_model_create(int device, const LumiFieldDesc* desc, const float* table,
                      const float* density_params, const float* color_params,
                      const uint8_t* occupancy, int occ_res, LumiModel** out);
int lumi_model_set_occupancy(LumiModel* m, const uint8_t* occupancy, int occ_res);
/* Frame-renderer variant: LUMI_KERNEL_WS (the production kernel: warp-wide 8x4 ray packets
   streamed candidate-major, a producer warpgroup gathering the hash grid while a consumer
   warpgroup runs the tcgen05 MLP and composites, pipelined one round apart; the default) or
   LUMI_KERNEL_SIMT (thread-per-ray fp32 CUDA-core field with bit-exact features -- the
   numerical cross-check).  LUMI_KERNEL_TC / LUMI_KERNEL_PACKET name the round-1 kernels that
   LUMI_KERNEL_WS superseded; selecting them returns LUMI_ERR_UNSUPPORTED.  The environment
   variable LUMI_KERNEL=simt|ws sets the default. */
enum { LUMI_KERNEL_TC = 0, LUMI_KERNEL_SIMT = 1, LUMI_KERNEL_PACKET = 2, LUMI_KERNEL_WS = 3 };
int lumi_model_set_kernel(LumiModel* m, int kernel);
int lumi_model_destroy(LumiModel* m);
/* Kernel timing (bench/profiling aid, no reference counterpart): while enabled, every
 * render_rows launch records CUDA events around its march pass and its render kernel on the
 * launch stream.  take_timing synchronises those events, returns the summed milliseconds and
 * the number of render launches since the last take, and resets the accumulators. */
int lumi_model_set_timing(LumiModel* m, int enable);
int lumi_model_take_timing(LumiModel* m, double* march_ms, double* render_ms, int* launches);
/* Device-side memory footprint of the model in bytes. */
int lumi_model_bytes(const LumiModel* m, uint64_t* bytes);
/* The CUDA device the model lives on. */
int lumi_model_device(const LumiModel* m, int* device);

/* ---- rendering ------------------------------------------------------------------ */
/* Drop-in for render_rows (renderer.h:252-278): host planar buffers of the camera's
   full image size, rows [row_begin,row_end) written.  depth/opacity/stats may be NULL;
   stats receives (row_end-row_begin) entries.  Synchronous.  Page-locked (pinned) planes
   are written by the kernel directly (zero-copy, no device->host copy afterwards; set
   LUMI_ZERO_COPY=0 to disable); pageable planes go through a device staging copy. */
int lumi_render_rows(LumiModel* m, const LumiCameraDesc* cam, const LumiRenderOptions* opts,
                     int row_begin, int row_end, float* out, float* depth, float* opacity,
                     LumiRowStats* stats);
/* Same, into device memory, enqueued on `stream` (cudaStream_t or NULL). */
int lumi_render_rows_async(LumiModel* m, const LumiCameraDesc* cam,
                           const LumiRenderOptions* opts, int row_begin, int row_end,
                           const LumiFrameTarget* target, void* stream);
/* Occupancy-kept candidate bitmask per pixel, independent of the network (the set the
   reference marches with the early cut disabled).  mask: device, camera-sized
   [height][width][ceil(spp/32)] uint32; counts: device [height][width] int32. */
int lumi_march_kept_async(LumiModel* m, const LumiCameraDesc* cam, const LumiRenderOptions* opts,
                          int row_begin, int row_end, uint32_t* mask, int32_t* counts,
                          void* stream);

/* The renderer's tcgen05 MLP alone over a dense batch (RadianceField::forward_chunk after
   the encoding, field.h:114-136): features [n][32] fp16, view directions [n][3] fp32 -> out
   [n][4] fp32 (sigma, r, g, b).  Device pointers, enqueued on `stream`.  For measuring the
   tensor-core stage in isolation and checking it against the oracle. */
int lumi_mlp_batch_async(LumiModel* m, const void* features, const float* dirs, int n, float* out,
                         void* stream);

/* MultiResHashGrid::encode (grid.h:90-114) through the renderer's production gather (fp16 table
   copy, fp16 trilinear weights, packed-fp16 accumulation): n contracted positions pos [n][3]
   fp32, LOD weights as the renderer carries them, lod [n] = fl with w_l = clamp(fl - l, 0, 1)
   (fl = 1e-4 is the reference's L_eff < 0 case, only w_0 = 1e-4) -> out [n][2 * levels] fp32,
   zeros where w_l = 0.  Device pointers, enqueued on `stream`.  Parity tooling for the gather. */
int lumi_encode_async(LumiModel* m, int n, const float* pos, const float* lod, float* out,
                      void* stream);

/* The hash-grid gather alone (benchmark of the attainable gather rate): n points, every level
   of each through the renderer's gather (fp16 table); coherent != 0 gives each warp an 8x4
   patch of neighbouring points (like a ray packet), 0 uniform random points.  out: device
   [n] floats.  Level-samples gathered = n * levels. */
int lumi_gather_bench_async(LumiModel* m, int n, int coherent, float* out, void* stream);

/* ---- checkpoint ingest (host) ---------------------------------------------------- */
/* LUMICKPT v1 (proj/src/scene.cpp:286-394, occupancy.cpp:200-243). */
typedef struct LumiCheckpointInfo {
  LumiFieldDesc field;
  int32_t samples_per_ray;
  int32_t contraction; /* 0 = kNone, 1 = kLInfCubic */
  double background[3];
  int32_t occ_res;
  int32_t n_cameras;
  uint64_t table_floats;
  uint64_t density_params;
  uint64_t color_params;
} LumiCheckpointInfo;
/* Parses `path`.  Any output buffer may be NULL (call once with NULLs to learn the sizes in
   `info`, then again with table[table_floats], density[density_params],
   color[color_params], occupancy[occ_res^3]). */
int lumi_checkpoint_read(const char* path, LumiCheckpointInfo* info, float* table,
                         float* density_params, float* color_params, uint8_t* occupancy);
/* save_checkpoint (scene.cpp:320-351) of a rendering model: info->field / samples_per_ray /
   contraction / background / occ_res / n_cameras, the parameter arrays in the
   lumi_field_layout sizes, alpha_v [n_cameras] (NULL = zeros), occupancy [occ_res^3]
   (nonzero = occupied).  The occupancy grid's training trackers are written as zeros. */
int lumi_checkpoint_write(const char* path, const LumiCheckpointInfo* info, const float* table,
                          const float* density_params, const float* color_params,
                          const double* alpha_v, const uint8_t* occupancy);

/* ---- occupancy bake (GPU) ------------------------------------------------------- */
/* OccupancyGrid::probe(k) with the density head + prune(alpha), zero history, no
   carving; results to host buffers (probe_max may be NULL). */
int lumi_bake_occupancy(LumiModel* m, const LumiCameraDesc* cams, int ncams,
                        int samples_per_ray, int points_per_axis, int occ_res, float alpha,
                        uint8_t* occupancy_out, float* probe_max_out);

/* ---- training reverse path (GPU) ------------------------------------------------ */
/* TrainRay (trainer.h:90-97): the ray and its right-neighbour ray (generate_ray at
   x + 0.5 / generate_ray_unchecked at x + 1.5), the model-space target, the ground-truth
   depth (< 0: unavailable), the normalised vignetting radius and the camera index. */
typedef struct LumiTrainRay {
  double origin[3], dir[3];
  double norigin[3], ndir[3];
  float gt[3];
  int32_t camera;
  double gt_depth;
  double vignette_r;
} LumiTrainRay;

/* The TrainConfig fields ray_loss reads (trainer.h:18-60) and the per-iteration inputs. */
typedef struct LumiLossConfig {
  double lambda_depth, lambda_dvar, lambda_dist;
  double inv_batch;    /* 1 / batch size (trainer.cpp:544) */
  int32_t depth_active; /* iteration < depth window (trainer.cpp:545) */
  int32_t _pad;
} LumiLossConfig;

/* LossTerms (trainer.h:99-102), the ray-dependent part; total = image+depth+dvar+dist. */
typedef struct LumiLossTerms {
  double total, image, depth, dvar, dist;
} LumiLossTerms;

/* FieldGradients (field.h:48-62) + the per-camera vignetting gradient and loss sums.  All
   are ACCUMULATED (zero them per iteration, as trainer.cpp:547 does).  grid:
   [layout.total_floats], density: [layout.density_params], color: [layout.color_params]
   (weights then bias per layer), alpha_v: [ncams], loss: one LumiLossTerms. */
typedef struct LumiTrainGrads {
  float* grid;
  float* density;
  float* color;
  double* alpha_v;
  LumiLossTerms* loss;
} LumiTrainGrads;

/* For every ray: march_ray(record = true) through the model's occupancy grid, ray_loss, and
   backward_ray into `grads` -- the body of trainer.cpp:549-561.  cam_tnf ([ncams][2] t_near,
   t_far) and alpha_v ([ncams]) are host arrays.  Async form: rays, grads and the optional
   per-ray outputs (ray_evals = rec.t.size(), ray_contrib = rec.contributing) are device
   pointers, work is enqueued on `stream`; it synchronises the stream twice internally to
   size the per-sample buffers.  Sync form: the same with host buffers. */
int lumi_train_backward_async(LumiModel* m, const LumiTrainRay* rays, int nrays,
                              const double* cam_tnf, const double* alpha_v, int ncams,
                              const LumiRenderOptions* opts, const LumiLossConfig* loss,
                              const LumiTrainGrads* grads, int32_t* ray_evals,
                              int32_t* ray_contrib, void* stream);
int lumi_train_backward(LumiModel* m, const LumiTrainRay* rays, int nrays, const double* cam_tnf,
                        const double* alpha_v, int ncams, const LumiRenderOptions* opts,
                        const LumiLossConfig* loss, const LumiTrainGrads* grads,
                        int32_t* ray_evals, int32_t* ray_contrib);
/* The model's device-resident fp32 parameters (table in the grid.h:58-74 layout, density and
   colour nets weights-then-bias), for an in-place device optimizer.  After changing them,
   lumi_model_params_updated() rebuilds the derived copies the renderers read (fp16 table,
   fused density-L2/colour-L1 layer).  Synchronous. */
int lumi_model_device_params(LumiModel* m, float** table, float** density, float** color);
int lumi_model_params_updated(LumiModel* m);

/* ---- native multi-GPU frame driver -------------------------------------
   run_frame (scheduler.cpp:114-152) with GPUs as the workers.  models[i] is worker i's replica
   (one per GPU; the same model may appear several times to run several workers on one GPU,
   each on its own stream).  One persistent host thread per worker renders its contiguous band
   of the stacked image (eyes x eye_height rows of `width`; eye e's camera row y is stacked row
   e * eye_height + y) with lumi_render_rows_async; a band crossing the eye seam becomes one
   launch per eye.  The frame target is device memory on any GPU: workers on other GPUs store
   their pixels straight into it over NVLink (peer access enabled on first use) -- the gather
   is the render kernel's epilogue.  After each frame the per-worker CUDA-event ms drive
   next_assignment (scheduler.cpp:154-162, dampening lambda) for the next frame; the first frame
   uses equal_assignment.  lumi_frame_driver_render is synchronous; wall_ms is the host time of
   the frame, worker_ms / worker_rays ([workers], optional) the FrameStats fields.  A failing
   worker fails the frame with "run_frame: worker i failed: ..." (scheduler.cpp:137-139). */
typedef struct LumiFrameDriver LumiFrameDriver;
int lumi_frame_driver_create(LumiModel* const* models, int workers, int width, int eye_height,
                             int eyes, double dampening, LumiFrameDriver** out);
int lumi_frame_driver_render(LumiFrameDriver* d, const LumiCameraDesc* cams /* [eyes] */,
                             const LumiRenderOptions* opts, const LumiFrameTarget* target,
                             double* wall_ms, double* worker_ms, int64_t* worker_rays);
/* The same into a host planar image [3][eyes * eye_height][width] (the reference's shared
   Image<float>): the frame is rendered into a device frame on worker 0's GPU, then copied. */
int lumi_frame_driver_render_host(LumiFrameDriver* d, const LumiCameraDesc* cams,
                                  const LumiRenderOptions* opts, float* out, double* wall_ms,
                                  double* worker_ms, int64_t* worker_rays);
/* the assignment the NEXT frame will use: rows per worker (contiguous in worker order) */
int lumi_frame_driver_assignment(const LumiFrameDriver* d, int32_t* rows, double* shares);
int lumi_frame_driver_set_assignment(LumiFrameDriver* d, const int32_t* rows);
int lumi_frame_driver_destroy(LumiFrameDriver* d);

/* ---- peer-memory frame gather ------------------------------------------
   lumi_ipc_export: an inter-process handle (LUMI_IPC_HANDLE_BYTES opaque bytes) for the
   device allocation holding dev_ptr, plus dev_ptr's byte offset inside it.
   lumi_ipc_open: maps a handle exported by another process into this process on `device`
   (peer access enabled lazily); *dev_ptr = mapped base + offset, usable as the `rgb` /
   `depth` / `opacity` planes of a LumiFrameTarget, so the render kernel writes straight into
   the exporting GPU's memory.  lumi_ipc_close unmaps a pointer returned by lumi_ipc_open.
   A process cannot open its own handle (LUMI_ERR_CUDA). */
#define LUMI_IPC_HANDLE_BYTES 64
int lumi_ipc_export(const void* dev_ptr, void* handle, uint64_t* offset);
int lumi_ipc_open(int device, const void* handle, uint64_t offset, void** dev_ptr);
int lumi_ipc_close(int device, void* dev_ptr);

/* ---- row scheduler (host) ------------------------------------------------------- */
int lumi_equal_assignment(int height, int workers, int32_t* rows, double* shares);
int lumi_assign_rows(int height, int workers, const double* throughputs,
                     const double* prev_shares, double dampening, int32_t* rows,
                     double* shares);
int lumi_next_assignment(int height, int workers, const double* prev_shares,
                         const int32_t* prev_rows, const double* worker_ms, int width,
                         double dampening, int32_t* rows, double* shares);
int lumi_aggregate_stats(const double* wall_ms, int frames, double* mean_fps, double* std_fps,
                         double* p99_fps);

#ifdef __cplusplus
}
#endif
#endif /* LUMI_CUDA_H */
