/*
 * fovnet.h -- C ABI of the B200-native FoVolNet per-frame hot path.
 *
 * One shared library (libfovnet.so, built from paper_2209_09965_b200/csrc)
 * exports these entry points. Signatures use plain pointers and sizes only;
 * device buffers are raw CUDA device pointers (e.g. a torch tensor's
 * data_ptr()), host buffers are borrowed for the duration of the call.
 *
 * Every function returns 0 on success or a negative FV_E* code; the message of
 * the last failure on the calling thread is available from fv_last_error().
 *
 * Each entry point replaces one reference function (pkg/src/fovray/...):
 *   fv_mask_compact     sample_maps.build_tau_map + build_sample_mask + compact_mask
 *                       (sample_maps.py:89-105, :128-132, :161-171)
 *   fv_render_sparse    renderer.render_sparse_compact (renderer.py:262-288)
 *   fv_render_full      renderer.render_full           (renderer.py:211-222)
 *   fv_volume_*         volume.VolumeGrid / make_procedural_volume / TransferFunction
 *                       (volume.py:47-72, :112-146, :184-242)
 *   fv_net_* / fv_state_* / fv_reconstruct
 *                       network.init_network/load_network + reset_state + forward_full
 *                       (network.py:162-180, :342-357, :118-119, :296-323)
 *   fv_pack_input       bench._reconstruct_frame input packing (bench.py:166-172)
 *   fv_frame            one body of bench.cmd_bench_throughput's loop (bench.py:194-209)
 */
#ifndef FOVNET_H
#define FOVNET_H

#include <stdint.h>

#if defined(__GNUC__)
#define FV_API __attribute__((visibility("default")))
#else
#define FV_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define FV_OK 0
#define FV_E_INVALID (-1)   /* argument validation failed (reference raises ValueError) */
#define FV_E_CUDA (-2)      /* CUDA runtime error */
#define FV_E_NOMEM (-3)     /* allocation failed */
#define FV_E_STATE (-4)     /* recurrent state does not match the film (reset the state) */
#define FV_E_UNSUPPORTED (-5)

typedef struct fv_ctx fv_ctx;       /* CUDA stream, workspace, noise stack, counters */
typedef struct fv_volume fv_volume; /* device-resident scalar grid + transfer function */
typedef struct fv_net fv_net;       /* device-resident W-Net weights (fp16 conv weights) */
typedef struct fv_state fv_state;   /* recurrent state + activation workspace for one film */

/* renderer.Camera (volume.py:246-276); basis computed by the library in fp64 */
typedef struct {
  double position[3];
  double look_at[3];
  double up[3];
  double fov_y; /* degrees */
  int32_t width;
  int32_t height;
} fv_camera;

/* volume.Light (volume.py:306-328) */
#define FV_LIGHT_NONE 0
#define FV_LIGHT_DIRECTIONAL 1
#define FV_LIGHT_POINT 2
typedef struct {
  int32_t kind;
  int32_t _pad;
  double vec[3];       /* propagation direction (directional) or position (point) */
  double intensity[3];
} fv_light;

/* renderer.RenderSettings (renderer.py:44-65); <=0 step/reference = resolve() default */
#define FV_PREC_FP32 0
#define FV_PREC_FP64 1
/* fp32 arithmetic with software trilinear quads in both passes (no hardware-filtered samples):
   the strict tier, <= ~2e-5 from the fp64 tier on every tested volume */
#define FV_PREC_FP32_STRICT 2
typedef struct {
  double step_size;
  double shadow_step_factor;
  double early_term_alpha;
  double background[4];
  double ambient;
  double reference_step;
  double shadow_min_transmittance;
  int32_t precision; /* FV_PREC_FP32 (default, the fast tier), FV_PREC_FP32_STRICT or FV_PREC_FP64 */
  int32_t _pad;
} fv_settings;

/* sample_maps.FoveaConfig (sample_maps.py:43-59) with scalar base density */
typedef struct {
  double focus[2]; /* (f_x, f_y) pixels */
  double sigma;
  double base_density;
  double pixel_scale;
} fv_fovea;

/* per-call work counters (a sample = one trilinear+TF evaluation) */
typedef struct {
  uint64_t rays;
  uint64_t hit_rays;
  uint64_t samples_main;
  uint64_t samples_shadow;
} fv_stats;

/* ---- context ----------------------------------------------------------- */
FV_API const char* fv_last_error(void);
FV_API int fv_version(void);
FV_API int fv_ctx_create(int device, fv_ctx** out);
FV_API int fv_ctx_destroy(fv_ctx* ctx);
/* use an external cudaStream_t (e.g. torch.cuda.current_stream().cuda_stream); NULL = legacy default stream */
FV_API int fv_ctx_set_stream(fv_ctx* ctx, void* cuda_stream);
FV_API void* fv_ctx_stream(fv_ctx* ctx);
FV_API int fv_sync(fv_ctx* ctx);
/* RNKSTACK payload (noise.py:432-453): T*H*W little-endian float32, (T,H,W) order, host memory */
FV_API int fv_noise_upload(fv_ctx* ctx, const float* host_vals, int T, int H, int W);
/* device counters accumulated by render calls since the last reset */
FV_API int fv_stats_read(fv_ctx* ctx, fv_stats* out_host);
FV_API int fv_stats_reset(fv_ctx* ctx);
/* number of library kernels launched on this ctx since creation */
FV_API uint64_t fv_launch_count(fv_ctx* ctx);
/* Per-kernel-class device timing: while enabled, every library launch on the context's stream is
 * bracketed by a pair of CUDA events; fv_ctx_kernel_time() synchronises on them and returns the
 * summed launch durations (ms), the summed algorithmic work of the class (FLOPs for FV_KC_CONV,
 * 0 elsewhere) and the launch count since timing was (re-)enabled. Costs an event pair per launch:
 * for measurement runs, not for the headline timed region. */
enum {
  FV_KC_MASK = 0,            /* mask_compact / tau */
  FV_KC_MARCH_MAIN = 1,      /* primary-ray march (wavefront main pass, or the fused single-pass tiers) */
  FV_KC_MARCH_SHADOW = 2,    /* wavefront shadow pass */
  FV_KC_MARCH_COMPOSITE = 3, /* wavefront composite pass */
  FV_KC_CONV = 4,            /* tcgen05 implicit-GEMM convolutions (W-Net D and K stages) */
  FV_KC_NETOPS = 5,          /* upsample / K filter application / pack / finalize */
  FV_KC_OTHER = 6,           /* volume bricking, procedural volumes */
  FV_KC_COUNT = 7
};
FV_API int fv_ctx_set_kernel_timing(fv_ctx* ctx, int enable);
FV_API int fv_ctx_kernel_time(fv_ctx* ctx, int kernel_class, double* ms, double* work, uint64_t* launches);

/* ---- foveated mask + compaction (device outputs) ------------------------ */
/* pb_map_dev: nullable (H,W) float64 per-pixel base density; bits_dev: nullable (H,W) uint8;
 * idx_dev: (H*W) int32 capacity, receives k flat indices v*W+u in row-major order;
 * k_dev: one int32 on device; net_state: nullable state whose film is (H,W): channels 0..4
 * (rgba*m, m) of its NHWC8 fp16 net input are written for unmasked pixels. */
FV_API int fv_mask_compact(fv_ctx* ctx, int frame, int H, int W, const fv_fovea* fovea,
                    const double* pb_map_dev, uint8_t* bits_dev, int32_t* idx_dev,
                    int32_t* k_dev, fv_state* net_state);
/* same, thresholding an explicit fp64 tau map (H,W) on device (TauMap given by value) */
FV_API int fv_mask_compact_tau(fv_ctx* ctx, int frame, int H, int W, const double* tau_dev,
                               uint8_t* bits_dev, int32_t* idx_dev, int32_t* k_dev,
                               fv_state* net_state);
/* fp64 tau map (H,W) on device -- the TauMap.values of sample_maps.py:89-105 */
FV_API int fv_tau_map(fv_ctx* ctx, int H, int W, const fv_fovea* fovea, const double* pb_map_dev,
               double* tau_dev);

/* ---- volume -------------------------------------------------------------- */
/* c_max (sample_maps.py:135-137): deterministic fp64 sum of tau over an (H, W) film into *sum_dev
 * (device); tau from the fovea (and optional per-pixel P_b map) or from a tau map (tau_dev) */
FV_API int fv_tau_sum(fv_ctx* ctx, int H, int W, const fv_fovea* fovea, const double* pb_map_dev,
                      const double* tau_dev, double* sum_dev);
/* draw_direct_samples (sample_maps.py:181-198): inverse-CDF draws over the fp64 tau map for `count`
 * caller-supplied uniforms in [0,1) -> flat pixel indices v*W+u (device int32) */
FV_API int fv_direct_draws(fv_ctx* ctx, int H, int W, const fv_fovea* fovea, const double* pb_map_dev,
                           const double* tau_dev, const double* uniforms_dev, int64_t count, int32_t* idx_dev);
/* foveal_density (sample_maps.py:62-68) over n broadcast pixel offsets (dx, dy), fp64 */
FV_API int fv_foveal_density(fv_ctx* ctx, const double* dx_dev, const double* dy_dev, int64_t n, double sigma,
                             double pixel_scale, double* out_dev);
FV_API int fv_volume_create(fv_ctx* ctx, int nx, int ny, int nz, const double spacing[3],
                     fv_volume** out);
/* same, over caller-owned device memory (nz,ny,nx) float32 that outlives the handle */
FV_API int fv_volume_wrap(fv_ctx* ctx, int nx, int ny, int nz, const double spacing[3],
                          float* data_dev, fv_volume** out);
FV_API int fv_volume_destroy(fv_volume* vol);
/* data: (nz,ny,nx) float32 already normalised to [0,1]; on_device selects the pointer kind */
FV_API int fv_volume_upload(fv_ctx* ctx, fv_volume* vol, const float* data, int on_device);
/* make_procedural_volume on the GPU (fp64 field, global min/max, f32 cast);
 * kind 0 sphere_shells, 1 vortex_field, 2 box_lattice; value_range_out: nullable host double[2] */
FV_API int fv_volume_procedural(fv_ctx* ctx, fv_volume* vol, int kind, double* value_range_out);
/* TransferFunction lut (K,4) float32 host */
/* load_raw_volume's normalisation (volume.py:75-109) on the device: raw_dev holds nx*ny*nz values
 * (dtype 0 = uint8, 1 = float32, x fastest); the volume's data receives (raw - lo) / (hi - lo) in fp64
 * cast to float32 (zeros when hi == lo); range = (lo, hi). Float data with a NaN fails with the
 * reference's message and *first_nan (nullable) = the first NaN's flat index (else -1). */
FV_API int fv_volume_from_raw(fv_ctx* ctx, fv_volume* vol, const void* raw_dev, int dtype, double* range,
                              int64_t* first_nan);
FV_API int fv_volume_set_tf(fv_ctx* ctx, fv_volume* vol, const float* lut_host, int K);
/* device pointer to the (nz,ny,nx) float32 grid */
FV_API float* fv_volume_data(fv_volume* vol);

/* ---- ray marching -------------------------------------------------------- */
/* idx_dev/k_dev from fv_mask_compact (k read on device; k_max bounds the launch).
 * rgba_dev (H,W,4) f32, depth_dev (H,W) f32: nullable, back-projected; must be zeroed by the
 * caller where the mask is unset. net_state: nullable; receives channels 0..3 of its net input.
 * stats_out: nullable; when given the call synchronises and returns this call's counters. */
FV_API int fv_render_sparse(fv_ctx* ctx, const fv_volume* vol, const fv_camera* cam,
                     const fv_light* light, const fv_settings* settings,
                     const int32_t* idx_dev, const int32_t* k_dev, int k_max,
                     float* rgba_dev, float* depth_dev, fv_state* net_state, fv_stats* stats_out);
/* renderer.render_sparse_naive (renderer.py:225-259): every pixel of each occupied 64-pixel chunk of
 * bits_dev ((H,W) uint8, device) is a lane of the thread-per-pixel marcher; lanes whose bit is clear
 * idle and receive zeros. idx_dev: (H*W) int32 device scratch receiving the lane list (idle lanes
 * as -(pix+1)); k_dev: one int32 on device receiving the lane count (= work_items). Pixels outside
 * occupied chunks are left untouched (the caller zero-fills the frame). */
FV_API int fv_render_sparse_naive(fv_ctx* ctx, const fv_volume* vol, const fv_camera* cam,
                                  const fv_light* light, const fv_settings* settings,
                                  const uint8_t* bits_dev, int32_t* idx_dev, int32_t* k_dev,
                                  float* rgba_dev, float* depth_dev, fv_stats* stats_out);
FV_API int fv_render_full(fv_ctx* ctx, const fv_volume* vol, const fv_camera* cam,
                   const fv_light* light, const fv_settings* settings, float* rgba_dev,
                   float* depth_dev, fv_stats* stats_out);

/* ---- reconstruction network ---------------------------------------------- */
/* block string as in network.NetConfig.from_string (network.py:46-53), e.g.
 * "e64-e64-e80-d96-d80-d64-d64"; recurrent/include_mask_channel as NetConfig. */
FV_API int fv_net_create(fv_ctx* ctx, const char* blocks, int predicted_kernel, int recurrent,
                  int include_mask_channel, fv_net** out);
FV_API int fv_net_destroy(fv_net* net);
/* set one parameter by its reference name ("D.block0.conv1.w", "K.block3.b", ...) from host
 * float32 in the reference layout ((oc,ic,kh,kw) weights, (oc,) biases). Weights are stored
 * as fp16 (truncate_fp16 semantics, autograd.py:499-503); biases stay fp32. */
FV_API int fv_net_set_param(fv_ctx* ctx, fv_net* net, const char* name, const float* host,
                     int64_t count);
FV_API int fv_state_create(fv_ctx* ctx, const fv_net* net, int H, int W, fv_state** out);
FV_API int fv_state_reset(fv_ctx* ctx, fv_state* st);
FV_API int fv_state_destroy(fv_state* st);
/* NHWC8 fp16 input buffer of the state (padded film), written by fv_mask_compact/fv_render_* */
FV_API void* fv_state_net_input(fv_state* st);
FV_API int fv_state_dims(const fv_state* st, int* H, int* W, int* Hp, int* Wp);
/* pack a host/device sparse frame into the state's input: x = rgba*m ++ m (bench.py:168-172) */
FV_API int fv_pack_input(fv_ctx* ctx, fv_state* st, const float* rgba_dev, const uint8_t* bits_dev);
/* forward_full's sparse input as given: (C,H,W) fp32 on device, C = 4 (+1 mask channel) */
FV_API int fv_state_set_input(fv_ctx* ctx, fv_state* st, const float* x_dev, int channels);
/* one forward_full; out_rgb_dev (H,W,3) f32 clipped to [0,1] (bench.py:175), out_o_dev /
 * out_od_dev nullable (3,H,W) f32 unclipped O and O_d (network.py:319-320). */
FV_API int fv_reconstruct(fv_ctx* ctx, const fv_net* net, fv_state* st, int use_kernel_stage,
                   float* out_rgb_dev, float* out_o_dev, float* out_od_dev);
/* read the carried state in the reference NCHW padded layout as float32 host arrays:
 * which = 0..n_dec-1 hidden[which], which = -1 prev_output; returns elements via *count */
FV_API int fv_state_read(fv_ctx* ctx, const fv_state* st, int which, float* host, int64_t cap,
                  int64_t* count);
/* overwrite the carried state from reference-layout NCHW float32 host arrays (same `which`) */
FV_API int fv_state_write(fv_ctx* ctx, fv_state* st, int which, const float* host, int64_t count);

/* diagnostic: one tcgen05 3x3 conv (+bias, optional ReLU, optional fused 2x2 avg-pool output)
 * over NC8HW8 fp16 device buffers; weights (cout,cin,3,3) float32 host (autograd.py:238-276) */
FV_API int fv_debug_conv3x3(fv_ctx* ctx, int cin, int cout, int H, int W, const void* x_nc8,
                            const float* w_host, const float* b_host, void* y_nc8,
                            void* pool_nc8, int relu);

/* ---- whole frame ---------------------------------------------------------- */
/* A camera path of n frames (bench.cmd_bench_throughput's loop, bench.py:194-209). Each frame --
 * frame t's network, with frame t+1's mask + compaction + march and frame t-1's K filter chain +
 * output stage forked off it (films above 4 Mpixel: frame t's march in line before its network) --
 * is replayed as ONE captured CUDA graph whose kernels read the per-frame camera / fovea / noise
 * frame from a device parameter block (fed by one small host->device copy per frame); frame t's
 * image is copied into host_rgb_out[t] on a copy stream while later frames compute. Every frame
 * equals the corresponding fv_frame call. cams, foveas, frame_ids: n entries each; host_rgb_out: nullable,
 * n pointers to (H,W,3) f32 buffers, each nullable (no copy for that frame), host (pinned for
 * overlap) or device memory; entries may repeat. Returns once every host copy has landed; device
 * copies are ordered on the context's stream. */
FV_API int fv_frames(fv_ctx* ctx, const fv_volume* vol, const fv_net* net, fv_state* st, int n,
                     const fv_camera* cams, const fv_light* light, const fv_settings* settings,
                     const fv_fovea* foveas, const int* frame_ids, float* const* host_rgb_out);
/* mask -> compact -> march -> reconstruct for one frame; host_rgb_out (H,W,3) f32 host (pinned
 * recommended) receives the clipped image; the copy is synchronous. timings_ms (nullable, 4
 * doubles) receives mask/render/reconstruct/total device times from CUDA events. */
FV_API int fv_frame(fv_ctx* ctx, const fv_volume* vol, const fv_net* net, fv_state* st,
             const fv_camera* cam, const fv_light* light, const fv_settings* settings,
             const fv_fovea* fovea, int frame, float* host_rgb_out, double* timings_ms);

/* pngio.to_uint8 (pngio.py:11-12) on the device: (clip(x,0,1)*255 + 0.5) truncated, fp32 without FMA
 * contraction; in_dev addressed by element strides (HWC RGB/RGBA or CHW), out_dev (H,W,3) uint8. */
/* forward_K (network.py:280-293): the K stage over the decoder hidden states the state holds and a
 * given O_d (3, Hp, Wp) fp32 on the device; out_dev (3, H, W) fp32 */
FV_API int fv_forward_k(fv_ctx* ctx, const fv_net* net, fv_state* st, const float* od_dev, float* out_dev);
/* predict_kernel_fields (network.py:268-277), one K block: logits (9, h, w) fp32 of the 1x1 conv
 * over hd (C, h, w) fp32; normalize = 1: softmax over the 9 taps (KernelField.normalized) */
FV_API int fv_kfield_logits(fv_ctx* ctx, const fv_net* net, int block, const float* hd_dev, int C, int h, int w,
                            int normalize, float* logits_dev);
/* Building blocks of the marcher as device calls (fp64, the reference's arithmetic):
 * volume.generate_rays (volume.py:293-303): n pixel centres -> origins (n,3), unit dirs (n,3) */
FV_API int fv_generate_rays(fv_ctx* ctx, const fv_camera* cam, const int32_t* us_dev, const int32_t* vs_dev,
                            int64_t n, double* origins_dev, double* dirs_dev);
/* volume.sample_trilinear (volume.py:149-180): n world points (n,3) -> values, 0 outside the box */
FV_API int fv_sample_trilinear(fv_ctx* ctx, const fv_volume* vol, const double* pts_dev, int64_t n,
                               double* out_dev);
/* TransferFunction.apply (volume.py:201-208): n scalars -> RGBA (n,4), lut (K,4) fp32 on the device */
FV_API int fv_tf_apply(fv_ctx* ctx, const float* lut_dev, int K, const double* s_dev, int64_t n, double* out_dev);
/* noise.tile_field (noise.py:378-384): frame `frame` of the uploaded stack tiled to (h, w) fp32 */
FV_API int fv_tile_field(fv_ctx* ctx, int frame, int h, int w, float* out_dev);
FV_API int fv_pack_rgb8(fv_ctx* ctx, const float* in_dev, int H, int W, int64_t stride_y, int64_t stride_x,
                        int64_t stride_c, uint8_t* out_dev);

/* ---- quality metrics on the device (metrics.py:40-148), fp64 ---------------------------- */
/* Images are (H,W,C) float64 device arrays, C >= 3 (RGB = channels 0..2; SSIM also takes C == 1
 * luma). fv_metric_sqdiff: sum over pixels and RGB of (a-b)^2 -> *sum_out (host); with a_prev and
 * b_prev it sums the tPSNR differences ((a-a_prev+1)/2 - (b-b_prev+1)/2)^2 (metrics.py:133-148).
 * fv_metric_ssim: mode 0 = mean SSIM over valid 11x11 windows of Rec.601 luma (metrics.py:74-87);
 * mode 1 = MS-SSIM over `scales` scales with the given renormalised weights (metrics.py:104-130).
 * Reductions are deterministic (fixed block partials summed in order). */
FV_API int fv_metric_sqdiff(fv_ctx* ctx, const double* a, const double* b, const double* a_prev,
                            const double* b_prev, int H, int W, int ca, int cb, double* sum_out);
FV_API int fv_metric_ssim(fv_ctx* ctx, const double* a, const double* b, int H, int W, int ca, int cb,
                          int mode, int scales, const double* weights, double* out);

/* ---- one frame across GPUs (config 5) ------------------------------------------- */
/* fv_shard_rays: the rank's share of the compacted ray list -- 32-ray packets dealt round-robin
 * (packet p belongs to rank p % world) -> out_idx_dev (capacity k_max), count -> out_k_dev.
 * fv_pack_records: (pixel, RGBA) records of the rays in idx_dev[0, *k_dev) read from the (H,W,4)
 * framebuffer into [0, cap) (pixel -1 past the count) -- the all-gather payload.
 * fv_scatter_records: n gathered records -> the network input channels 0..3 of st (fp16, exactly
 * as the marcher writes them) and/or an (H,W,4) framebuffer; records with pixel < 0 are skipped. */
FV_API int fv_shard_rays(fv_ctx* ctx, const int32_t* idx_dev, const int32_t* k_dev, int k_max, int rank,
                         int world, int32_t* out_idx_dev, int32_t* out_k_dev);
FV_API int fv_pack_records(fv_ctx* ctx, const float* rgba_dev, const int32_t* idx_dev, const int32_t* k_dev,
                           int cap, int32_t* rec_pix_dev, float* rec_rgba_dev);
FV_API int fv_scatter_records(fv_ctx* ctx, fv_state* st, const int32_t* rec_pix_dev, const float* rec_rgba_dev,
                              int64_t n, int W, float* rgba_out_dev);
/* Row-strip reconstruction (BASELINE config 5 across GPUs; sharded.py): marched rays as 12-byte
 * records (pix, RGBA fp16) -- rec (cap, 3) int32, pix = -1 past the rank's count */
FV_API int fv_pack_records16(fv_ctx* ctx, const float* rgba_dev, const int32_t* idx_dev, const int32_t* k_dev,
                             int cap, int32_t* rec_dev);
/* records -> channels 0..3 of a window state's input for frame rows [row0, row0 + H_window) */
FV_API int fv_scatter_records16(fv_ctx* ctx, fv_state* st, const int32_t* rec_dev, int64_t n, int W, int row0);
/* a window state's input channels 0..4 from the full-frame mask bits (H_full, W) uint8: zero RGBA +
 * the mask channel for frame rows [row0, row0 + H_window) (rows past the film: zero) */
FV_API int fv_window_input(fv_ctx* ctx, fv_state* st, const uint8_t* bits_dev, int H_full, int W, int row0);
/* the recurrent band [row0, row0 + rows) of a state (local L0 rows, multiples of the divisor): the
 * decoder hidden tensors + fp32 O_d, packed contiguously (pack = 1) or unpacked (pack = 0, then
 * the next input's O_d feedback channels of those rows); buf = null returns only *bytes */
FV_API int fv_state_band(fv_ctx* ctx, fv_state* st, int pack, int row0, int rows, void* buf_dev, int64_t* bytes);

#ifdef __cplusplus
}
#endif
#endif /* FOVNET_H */
