/*
 * isg.h — the C-ABI drop-in boundary of the B200 isotropic-splat hot path.
 *
 * Every entry point is `extern "C"`, takes plain pointers and sizes, never
 * throws, and returns an isg_status.  The C++ host API in
 * paper_2403_14244_b200/csrc/isosplat_b200.hpp (a drop-in for the reference's
 * `isosplat::render`, /root/reference/proj/include/isosplat/splat3d.hpp:96-97)
 * and the Python binding (paper_2403_14244_b200/isg.py) are both thin layers
 * over these functions.  INTEGRATION.md shows the binding a maintainer of the
 * reference would add.
 *
 * Reference interfaces each entry replaces (file:line under /root/reference/proj):
 *   isg_camera          <- struct Camera                  include/isosplat/splat3d.hpp:37-53
 *   isg_set_scene       <- std::span<const IsoSplat3D>    include/isosplat/splat3d.hpp:13-22, 96
 *                          (+ IsoSplat3D::validate        src/splat3d.cpp:10-17, done on device)
 *   isg_render          <- isosplat::render(iso)          include/isosplat/splat3d.hpp:96-97,
 *                                                         src/splat3d.cpp:173-194
 *   isg_loss_backward   <- mse (L2)                       src/image.cpp:50-58, plus the 3D
 *                          backward the reference lacks (SPEC.md:484 non-goal; 2D pattern
 *                          loss_gradients src/loss.cpp:259-300)
 *   isg_adam_step       <- update_step(iso)               src/optimize.cpp:78-108 (optimizer slot;
 *                          log-sigma convention :93,:105; skip non-finite :87-90), Adam rule
 *   isg_debug_bins      <- sort_by_depth                  src/splat3d.cpp:164-169 (parity hook)
 *   isg_status codes    <- std::domain_error / std::invalid_argument / CLI exit codes
 *                          src/splat3d.cpp:10-37, tools/isosplat_main.cpp:30-33
 *
 * Data layout (host and device): scenes are SoA float4 arrays
 *   mu_sigma[n][4]    = (mu.x, mu.y, mu.z, sigma)       world units
 *   rgb_opacity[n][4] = (r, g, b, opacity)
 * images are row-major interleaved HWC float32 (ImageGrid, include/isosplat/image.hpp:11-31),
 * gradients are n x 8 float32: (dmu.x, dmu.y, dmu.z, dsigma, dr, dg, db, dopacity).
 */
#ifndef ISG_H_
#define ISG_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ISG_TILE 16 /* screen tiles are ISG_TILE x ISG_TILE pixels */
#define ISG_ABI_VERSION 2

typedef struct isg_ctx isg_ctx; /* one per device: device buffers, a stream, Adam state. NOT thread-safe. */

/* Camera (splat3d.hpp:37-53) in FP32: row-major world->camera rotation R, translation t,
 * pinhole focal length and principal point in pixels, image size. */
typedef struct {
  float R[9];
  float t[3];
  float focal;
  float cx, cy;
  int32_t width, height;
} isg_camera;

typedef enum {
  ISG_OK = 0,
  ISG_E_DOMAIN = 1,   /* invalid splat / camera: reference throws std::domain_error */
  ISG_E_ARG = 2,      /* invalid argument / config: std::invalid_argument */
  ISG_E_CUDA = 3,     /* CUDA runtime error (incl. no device) */
  ISG_E_OOM = 4,      /* device allocation failed */
  ISG_E_OVERFLOW = 5, /* internal capacity exceeded and could not grow */
  ISG_E_NCCL = 6,     /* NCCL unavailable or failed */
  ISG_E_STATE = 7     /* call out of order (e.g. adam before any backward) */
} isg_status;

typedef struct {
  int64_t n_gaussians;    /* scene size */
  int64_t n_visible;      /* splats with >= 1 tile in the last binning */
  int64_t n_keys;         /* (tile, splat) pairs in the last binning */
  int64_t key_capacity;   /* allocated key slots */
  int64_t n_tiles;        /* tiles of the last camera */
  int64_t adam_steps;     /* optimizer steps taken */
  int64_t skipped_updates;/* Gaussian updates skipped for non-finite gradients (optimize.cpp:87-90) */
  int64_t regrow_events;  /* frames re-run after key-capacity growth */
  int64_t kernel_launches;/* kernels launched by this context so far */
  int64_t overflowed_frames;/* frames skipped for key-capacity overflow (each reported once) */
} isg_stats;

/* ---- lifetime -------------------------------------------------------------------------- */
isg_status isg_create(int device, int64_t max_gaussians, int32_t max_width, int32_t max_height,
                      isg_ctx** out);
void isg_destroy(isg_ctx* ctx);
const char* isg_last_error(const isg_ctx* ctx);
const char* isg_status_string(isg_status s);
int isg_abi_version(void);
/* Run all work on an external cudaStream_t (e.g. torch's current stream); NULL = own stream. */
isg_status isg_set_stream(isg_ctx* ctx, void* cuda_stream);
isg_status isg_synchronize(isg_ctx* ctx);
isg_status isg_get_stats(const isg_ctx* ctx, isg_stats* out);

/* ---- scene ----------------------------------------------------------------------------- */
/* Host pointers.  Validation (IsoSplat3D::validate, splat3d.cpp:10-17) runs on the device and
 * surfaces as ISG_E_DOMAIN (with the reference's message) from the next render/backward. */
isg_status isg_set_scene(isg_ctx* ctx, int64_t n, const float* mu_sigma, const float* rgb_opacity);
/* Device pointers (already resident in HBM); copied device-to-device, stream-ordered. */
isg_status isg_set_scene_device(isg_ctx* ctx, int64_t n, const float* mu_sigma_dev,
                                const float* rgb_opacity_dev);
isg_status isg_get_scene(isg_ctx* ctx, float* mu_sigma, float* rgb_opacity);

/* ---- forward --------------------------------------------------------------------------- */
/* render (splat3d.cpp:173-194) into a host HWC3 float image.  t_min: early-termination
 * threshold on transmittance (0 = exact reference semantics, never terminate early). */
isg_status isg_render(isg_ctx* ctx, const isg_camera* cam, const float bg[3], float t_min,
                      float* out_hwc3);
/* Same, device output pointer, asynchronous on the context stream (no host sync). */
isg_status isg_render_device(isg_ctx* ctx, const isg_camera* cam, const float bg[3], float t_min,
                             float* out_hwc3_dev);

/* Host-buffer rendering without a host sync per frame: render into the context's image ring
 * slot `slot` (0..ISG_IMAGE_SLOTS-1, each allocated on first use) and enqueue the frame's
 * device-to-host copy into `host_dst` (page-locked H x W x 3) on the context's copy stream;
 * returns at once, so the next frames render while this one travels.  isg_image_wait blocks
 * until slot `slot`'s last copy has landed (then `host_dst` may be read or reused).  Overflow
 * of a frame's key capacity surfaces at the next synchronising call, as for the device form. */
#define ISG_IMAGE_SLOTS 8
isg_status isg_render_host_async(isg_ctx* ctx, const isg_camera* cam, const float bg[3],
                                 float t_min, int32_t slot, float* host_dst);
isg_status isg_image_wait(isg_ctx* ctx, int32_t slot);

/* ---- training -------------------------------------------------------------------------- */
/* Forward + L2 loss (weight * mse, image.cpp:50-58) + backward for one view.  Gradients
 * ACCUMULATE into the context's n x 8 buffer until isg_adam_step / isg_zero_grads.
 * target_hwc3: host pointer; *loss_out receives weight * mse (double). */
isg_status isg_loss_backward(isg_ctx* ctx, const isg_camera* cam, const float bg[3], float t_min,
                             const float* target_hwc3, float weight, double* loss_out);
/* Device target pointer; asynchronous; the loss accumulates on device (isg_read_loss). */
isg_status isg_loss_backward_device(isg_ctx* ctx, const isg_camera* cam, const float bg[3],
                                    float t_min, const float* target_hwc3_dev, float weight);
/* Host-buffer training without a host sync per view: a ring of ISG_TARGET_SLOTS device
 * target images owned by the context (each allocated on its first upload).
 * isg_upload_target_async enqueues the host-to-device copy of one view's HWC3 target into ring
 * slot `slot` on the context's copy stream and returns at once (`host_hwc3` should be page-locked and stay unchanged until the copy has run; the copy
 * first waits for the last enqueued frame that read the slot).  isg_loss_backward_slot is
 * isg_loss_backward_device on that slot: binning and the forward blend run while the upload
 * may still be in flight, only the backward waits for it.  A caller uploads view i + 2 while
 * view i trains (the pattern bench.py's end-to-end number uses: 3 slots per view of a step).
 * isg_loss_backward_slot may be captured (isg_graph_begin/end): the slot is fixed in the graph,
 * each replay waits for that slot's latest upload enqueued before the launch. */
#define ISG_TARGET_SLOTS 32
isg_status isg_upload_target_async(isg_ctx* ctx, int32_t slot, const float* host_hwc3,
                                   int32_t width, int32_t height);
isg_status isg_loss_backward_slot(isg_ctx* ctx, const isg_camera* cam, const float bg[3],
                                  float t_min, int32_t slot, float weight);
/* Sum of losses of the views since the last isg_adam_step/isg_zero_grads (syncs). */
isg_status isg_read_loss(isg_ctx* ctx, double* loss_out);
isg_status isg_zero_grads(isg_ctx* ctx);
isg_status isg_get_grads(isg_ctx* ctx, float* grads_nx8);
/* Replace the accumulated gradients with a host n x 8 buffer (a pending view is projected
 * first and then overwritten), e.g. after a reduction the caller ran itself; the next
 * isg_adam_step applies them.  Synchronous. */
isg_status isg_set_grads(isg_ctx* ctx, const float* grads_nx8);
/* Device pointer of the n x 8 gradient buffer (flushes pending per-view work first), e.g.
 * for an external all-reduce.  Valid until the next isg_set_scene. */
isg_status isg_grads_device(isg_ctx* ctx, float** grads_dev);
/* Adam (torch semantics) on (mu, log sigma, rgb, logit opacity) with per-group learning rates
 * lr = {lr_mu, lr_sigma, lr_color, lr_opacity}; consumes and zeroes the gradients.  Updates
 * with a non-finite gradient are skipped and counted (optimize.cpp:87-90). */
isg_status isg_adam_step(isg_ctx* ctx, const float lr[4], float beta1, float beta2, float eps);
/* Loss of the last Adam step's views (all-reduced over ranks when NCCL is attached; syncs). */
isg_status isg_last_step_loss(isg_ctx* ctx, double* loss_out);
/* Asynchronous form: enqueues the device-to-host transfer of the last Adam step's loss into
 * `host_dst` on the context stream and returns at once (no sync, no frame check; it can be
 * captured into a graph).  Page-locked `host_dst` is written by a one-thread kernel through its
 * mapped device address (no copy engine); pageable memory falls back to cudaMemcpyAsync.  The
 * value is valid once the stream has passed the transfer — the pipelined training loop reads
 * step i's loss while step i + 1 runs. */
isg_status isg_step_loss_async(isg_ctx* ctx, double* host_dst);
/* weight * mse of one view without gradients (forward + loss only; device target; syncs).
 * Pending per-view gradients are preserved. */
isg_status isg_eval_loss(isg_ctx* ctx, const isg_camera* cam, const float bg[3], float t_min,
                         const float* target_hwc3_dev, float weight, double* loss_out);
/* Save / restore the scene, Adam moments and step count (the reject-and-halve step of the
 * reference's fit loop, src/optimize.cpp:333-340, needs the pre-step state back). */
isg_status isg_snapshot(isg_ctx* ctx);
isg_status isg_restore(isg_ctx* ctx);

/* ---- image loss (the loss the training entry points use) --------------------------------
 * ISG_LOSS_L2 (default): weight * mse                          (image.cpp:50-58)
 * ISG_LOSS_L1_DSSIM:     weight * ((1-lambda) L1 + lambda (1 - SSIM)), 11-tap sigma-1.5
 *                        window on valid positions, and its pixel gradient
 *                        (loss <- loss.cpp:184-190, ssim :119-141, dL/dfhat :201-213,
 *                        ssim_gradient_wrt_second :143-182).  lambda outside [0,1] ->
 *                        ISG_E_DOMAIN "loss: lambda must be in [0,1]"; lambda > 0 needs
 *                        W, H >= 11 (ISG_E_DOMAIN "ssim: image smaller than the 11x11 window"). */
#define ISG_LOSS_L2 0
#define ISG_LOSS_L1_DSSIM 1
isg_status isg_set_loss(isg_ctx* ctx, int kind, float lambda);
/* The configured loss of a device image fhat against target (both HWC3), and optionally its
 * gradient dL/dfhat into dldc_dev (HWC3; NULL = loss only).  Syncs. */
isg_status isg_image_loss_device(isg_ctx* ctx, int32_t width, int32_t height,
                                 const float* fhat_dev, const float* target_dev, float weight,
                                 double* loss_out, float* dldc_dev);

/* ---- adaptive control (prune / merge / split of the splat set) ----------------------------
 * adaptive_control (src/optimize.cpp:221-284) for isotropic 3D splats, on the device:
 *   prune  opacity < prune_threshold (the first splat of maximal opacity always survives)
 *   merge  pairs with |mu_i - mu_j| < merge_distance_factor * min(sigma) and max colour
 *          difference < merge_color_tol, greedily nearest-first on (dist, i, j), one merge per
 *          splat; weights w = opacity * sigma^2, mu / sigma^2 / colour w-weighted, opacity =
 *          min(1, (w1 + w2) / sigma^2)
 *   split  sigma > split_sigma_max (world units), widest first, while count <= max_particles
 *          (<= 0: twice the current count); children at mu +- d sigma/2, sigma / sqrt(2), d a
 *          unit direction from (seed, round, parent index)
 * Parameter checks and messages follow AdaptiveControlParams::validate
 * (include/isosplat/optimize.hpp:21-27).  Adam moments and step restart at zero (the
 * reference clears its momentum, optimize.cpp:344).  Synchronises. */
typedef struct {
  double prune_threshold;       /* 1e-3 in the reference */
  double merge_distance_factor; /* 0.5 */
  double merge_color_tol;       /* 0.05 */
  double split_sigma_max;       /* world units */
  int64_t max_particles;        /* effective cap; <= 0: 2 x the current count */
} isg_adapt_params;
typedef struct {
  int64_t n_before, n_pruned, n_merged, n_split, n_after;
} isg_adapt_result;
isg_status isg_adaptive_control(isg_ctx* ctx, const isg_adapt_params* params, uint64_t seed,
                                uint64_t round, isg_adapt_result* out);

/* ---- CUDA graphs ------------------------------------------------------------------------
 * Capture the asynchronous calls of one train step (isg_loss_backward_device per view +
 * isg_adam_step, or isg_render_device) on the context stream and replay them with one launch.
 * Capture after a warm-up step (buffers must not grow inside the capture).  Synchronising
 * entry points return ISG_E_STATE while capturing.  The Adam step counter lives on the device,
 * so replays apply the correct bias corrections; the learning rates, cameras and device
 * pointers are the captured ones.  A replayed frame that overflows the key capacity is skipped
 * and reported by the next synchronising call (re-capture after it grows the buffers).
 * isg_graph_launch returns ISG_E_STATE for a graph captured before any device buffer it may
 * use was reallocated (larger scene, key capacity or image, adaptive control); isg_graph_end
 * returns it when a buffer grew inside the capture. */
typedef struct isg_graph isg_graph;
isg_status isg_graph_begin(isg_ctx* ctx);
isg_status isg_graph_end(isg_ctx* ctx, isg_graph** out);
isg_status isg_graph_launch(isg_ctx* ctx, isg_graph* graph);
void isg_graph_destroy(isg_graph* graph);

/* ---- multi-GPU (one process per GPU, views sharded, NCCL all-reduce before Adam) -------- */
/* NCCL is resolved at run time (dlopen libnccl.so.2, the copy torch already loaded if any).
 * Once a communicator is attached, isg_adam_step sums the n x 8 gradient buffer over ranks
 * (ncclAllReduce, in place) and every rank applies the identical Adam step, so replicas stay
 * bitwise identical.  The exchange is pipelined over splat chunks on a second stream (the
 * all-reduce of chunk c overlaps the projection backward of chunk c+1 and the Adam update of
 * chunk c-1); the step loss and every rank's key-overflow flag travel in front of chunk 0, so
 * a step is one all-reduce per chunk, and a view that overflowed on any rank skips the step
 * on every rank.  At most 64 ranks. */
isg_status isg_nccl_get_unique_id(void* out_128_bytes);
/* Create and own a communicator (ncclCommInitRank); destroyed by isg_nccl_detach. */
isg_status isg_nccl_init(isg_ctx* ctx, int nranks, int rank, const void* unique_id_128_bytes);
/* Use a caller-owned ncclComm_t (passed as void*); rank and size are read from it.  The
 * caller keeps ownership: isg_nccl_detach / isg_destroy do not destroy it. */
isg_status isg_nccl_attach(isg_ctx* ctx, void* nccl_comm);
/* Size and rank as the attached communicator reports them (1, 0 without one), and the
 * loaded NCCL's version code (0 if NCCL is not loadable); any pointer may be NULL. */
isg_status isg_nccl_info(isg_ctx* ctx, int* nranks, int* rank, int* nccl_version);
/* Pipeline depth of the exchange, 1..8 chunks (default 4; chunks are >= 128K splats). */
isg_status isg_set_exchange_chunks(isg_ctx* ctx, int chunks);
isg_status isg_nccl_detach(isg_ctx* ctx);

/* ---- parity hooks ---------------------------------------------------------------------- */
/* After the last render/backward: sorted (tile<<32 | float_bits(depth)) keys, the splat
 * index of each key, and per-tile [start,end) ranges (n_tiles x 2) in the oracle's form (an
 * empty tile gets (s, s), s = the position it would occupy).  Any output pointer may be NULL;
 * *n_keys always receives the key count. */
isg_status isg_debug_bins(isg_ctx* ctx, uint64_t* keys, uint32_t* vals, int64_t* n_keys,
                          uint32_t* ranges);
/* Measurement hook (bench.py's roofline): the last frame's algorithmic work as the
 * reference's per-pixel loop sees it -- each pixel walks its tile's depth-ordered list until
 * its transmittance drops to t_min; *evaluated = entries visited, *inside = entries inside
 * their 3-sigma circle (summed over pixels).  Slow (no culling): outside timed regions. */
isg_status isg_count_pairs(isg_ctx* ctx, int64_t* evaluated, int64_t* inside);
/* Per-pixel forward state of the last render (both H x W): the final transmittance — or,
 * negated, the transmittance before the last contributor in a tile where some pixel's final
 * transmittance is not a normal float — and 1 + the index of the last contributor. */
isg_status isg_debug_pixel_state(isg_ctx* ctx, float* t_last, uint32_t* n_proc);

/* ---- binning strategy (both produce bit-identical tile lists) ----------------------------
 * TILE_BUCKET: per-tile counters + bucket fill + per-tile bitonic sort by (depth bits, splat
 *   index) in shared memory.
 * RADIX (default): onesweep LSD radix sort of (depth, splat), tile-key emission in depth order
 *   and a stable onesweep radix sort of (tile, pair). */
#define ISG_BINNING_TILE_BUCKET 0
#define ISG_BINNING_RADIX 1
isg_status isg_set_binning(isg_ctx* ctx, int mode);

/* ---- gradient accumulation mode ---------------------------------------------------------
 * 0 (default, "direct"): the blend backward pre-reduces each (tile, splat) pair's gradients
 *   over warp lanes and adds them straight into a per-splat n x 8 buffer in L2
 *   (red.global.add.v2.f32); the projection backward / Adam read it densely.  Fastest; the
 *   summation order of a splat's tile contributions varies run to run (last-bit differences).
 * 1 ("deterministic"): every pair writes its own gradient slot and the projection backward
 *   sums a splat's slots in a fixed order -- bitwise-identical gradients and trajectories
 *   across runs, binning modes and CUDA-graph replays. */
isg_status isg_set_deterministic(isg_ctx* ctx, int on);

/* ---- stage timing (CUDA events on the context stream; for bench.py's roofline) ----------
 * While enabled, kernels are launched without programmatic dependent launch (process-wide),
 * so that the events between them time each kernel alone. */
isg_status isg_profile_enable(isg_ctx* ctx, int on);
int isg_profile_num_stages(void);
const char* isg_profile_stage_name(int stage);
/* Accumulated device milliseconds and launch counts per stage since the last read (syncs). */
isg_status isg_profile_read(isg_ctx* ctx, double* ms_per_stage, int64_t* calls_per_stage);

/* ---- synthetic workload "isg-synth v1" (host-side, no device needed) -------------------- */
isg_status isg_synth_scene(uint64_t seed, int64_t n, int32_t width, int32_t height,
                           float* mu_sigma, float* rgb_opacity);
/* Camera k of an n-view batch: yaw (k-(n-1)/2)*1.5 deg about y, t = (0.05*(k-(n-1)/2),0,0);
 * n = 1 gives the identity camera.  focal = 1000*W/1920, principal point at the centre. */
isg_status isg_synth_camera(int32_t width, int32_t height, int32_t view, int32_t n_views,
                            isg_camera* out);

#ifdef __cplusplus
}
#endif
#endif /* ISG_H_ */
