// C ABI entry points (include/fovnet.h): context, noise, volume, mask, render, whole frame.
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "internal.h"

namespace fv {

static thread_local char g_err[1024] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int cuda_fail(cudaError_t e, const char* what) {
  set_error("CUDA error %s (%s) in %s", cudaGetErrorName(e), cudaGetErrorString(e), what);
  return FV_E_CUDA;
}

int pack_input(fv_ctx* ctx, fv_state* st, const float* rgba, const uint8_t* bits);
int pack_rgb8(fv_ctx* ctx, const float* in, int h, int w, int64_t sy, int64_t sx, int64_t sc, uint8_t* out);

}  // namespace fv

using namespace fv;

namespace fv {
static cudaEvent_t kpool_get(fv_ctx* ctx) {
  if (ctx->kpool.empty()) {
    cudaEvent_t e = nullptr;
    if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
    return e;
  }
  cudaEvent_t e = ctx->kpool.back();
  ctx->kpool.pop_back();
  return e;
}

bool pdl_enabled() {
  static const bool on = !(getenv("FV_PDL") && atoi(getenv("FV_PDL")) == 0);
  return on;
}

void ktime_begin(fv_ctx* ctx) {
  if (!ctx->ktiming) return;
  if (!ctx->kopen) ctx->kopen = kpool_get(ctx);
  if (ctx->kopen) cudaEventRecord(ctx->kopen, ctx->stream);
}

void ktime_end(fv_ctx* ctx, int cls, double work) {
  if (!ctx->ktiming || !ctx->kopen) return;
  cudaEvent_t b = kpool_get(ctx);
  if (!b) return;
  cudaEventRecord(b, ctx->stream);
  ctx->kspans.push_back({ctx->kopen, b, cls, work});
  ctx->kopen = nullptr;
}
}  // namespace fv

extern "C" {

const char* fv_last_error(void) { return g_err; }
int fv_version(void) { return 1; }

int fv_ctx_create(int device, fv_ctx** out) {
  FV_REQUIRE(out, "null argument");
  FV_CUDA(cudaSetDevice(device));
  auto* ctx = new fv_ctx();
  ctx->device = device;
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) == cudaSuccess) ctx->num_sms = prop.multiProcessorCount;
  if (prop.major != 10) {
    delete ctx;
    set_error("device %d is sm_%d%d; libfovnet is built for sm_100a (B200) only", device, prop.major, prop.minor);
    return FV_E_UNSUPPORTED;
  }
  cudaError_t e = cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) { delete ctx; return cuda_fail(e, "cudaStreamCreate"); }
  ctx->own_stream = true;
  e = cudaMalloc(&ctx->counters, sizeof(DevCounters));
  if (e != cudaSuccess) { delete ctx; return cuda_fail(e, "cudaMalloc counters"); }
  cudaMemset(ctx->counters, 0, sizeof(DevCounters));
  for (auto& ev : ctx->ev) cudaEventCreate(&ev);
  *out = ctx;
  return 0;
}

int fv_ctx_destroy(fv_ctx* ctx) {
  if (!ctx) return 0;
  cudaStreamSynchronize(ctx->stream);
  if (ctx->noise) cudaFree(ctx->noise);
  if (ctx->scan_status) cudaFree(ctx->scan_status);
  if (ctx->counters) cudaFree(ctx->counters);
  if (ctx->k_scratch) cudaFree(ctx->k_scratch);
  if (ctx->idx_scratch) cudaFree(ctx->idx_scratch);
  if (ctx->rgb_scratch) cudaFree(ctx->rgb_scratch);
  if (ctx->wave_rec) cudaFree(ctx->wave_rec);
  if (ctx->wave_ray) cudaFree(ctx->wave_ray);
  if (ctx->wave_hits) cudaFree(ctx->wave_hits);
  if (ctx->wave_ovf) cudaFree(ctx->wave_ovf);
  if (ctx->wave_fb) cudaFreeHost(ctx->wave_fb);
  if (ctx->dyn_dev) cudaFree(ctx->dyn_dev);
  if (ctx->dyn_host) cudaFreeHost(ctx->dyn_host);
  for (auto& e : ctx->dyn_ev) if (e) cudaEventDestroy(e);
  if (ctx->wave_fb_ev) cudaEventDestroy(ctx->wave_fb_ev);
  for (auto& ev : ctx->ev) if (ev) cudaEventDestroy(ev);
  for (auto& sp : ctx->kspans) { cudaEventDestroy(sp.a); cudaEventDestroy(sp.b); }
  for (auto& ev : ctx->kpool) cudaEventDestroy(ev);
  if (ctx->kopen) cudaEventDestroy(ctx->kopen);
  for (auto& e : ctx->fev) if (e) cudaEventDestroy(e);
  for (auto& e : ctx->kev) if (e) cudaEventDestroy(e);
  if (ctx->scan_aux) cudaFree(ctx->scan_aux);
  for (auto& e : ctx->kdone) if (e) cudaEventDestroy(e);
  if (ctx->kstream) cudaStreamDestroy(ctx->kstream);
  for (auto& s : ctx->fstream) if (s) cudaStreamDestroy(s);
  if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
  return 0;
}

int fv_ctx_set_stream(fv_ctx* ctx, void* s) {
  FV_REQUIRE(ctx, "null ctx");
  if (ctx->own_stream) {
    cudaStreamSynchronize(ctx->stream);
    cudaStreamDestroy(ctx->stream);
    ctx->own_stream = false;
  }
  // NULL selects the legacy default stream (torch's default stream)
  ctx->stream = reinterpret_cast<cudaStream_t>(s);
  return 0;
}

void* fv_ctx_stream(fv_ctx* ctx) { return ctx ? (void*)ctx->stream : nullptr; }

int fv_sync(fv_ctx* ctx) {
  FV_REQUIRE(ctx, "null ctx");
  FV_CUDA(cudaStreamSynchronize(ctx->stream));
  return 0;
}

uint64_t fv_launch_count(fv_ctx* ctx) { return ctx ? ctx->launches : 0; }

int fv_ctx_set_kernel_timing(fv_ctx* ctx, int enable) {
  FV_REQUIRE(ctx, "null context");
  FV_CUDA(cudaStreamSynchronize(ctx->stream));
  for (auto& sp : ctx->kspans) {
    ctx->kpool.push_back(sp.a);
    ctx->kpool.push_back(sp.b);
  }
  ctx->kspans.clear();
  for (int c = 0; c < FV_KC_COUNT; ++c) {
    ctx->k_ms[c] = ctx->k_work[c] = 0.0;
    ctx->k_n[c] = 0;
  }
  ctx->ktiming = enable != 0;
  return 0;
}

int fv_ctx_kernel_time(fv_ctx* ctx, int cls, double* ms, double* work, uint64_t* launches) {
  FV_REQUIRE(ctx, "null context");
  FV_REQUIRE(cls >= 0 && cls < FV_KC_COUNT, "kernel class %d out of range", cls);
  // fold the pending spans into the totals (FV_KTIME_LOG=1: each span to stderr, for
  // tools/probes/launch_times.py)
  static const bool log = getenv("FV_KTIME_LOG") && atoi(getenv("FV_KTIME_LOG")) == 1;
  for (auto& sp : ctx->kspans) {
    FV_CUDA(cudaEventSynchronize(sp.b));
    float t = 0.f;
    FV_CUDA(cudaEventElapsedTime(&t, sp.a, sp.b));
    if (log) fprintf(stderr, "[kspan] %d %.0f %.5f\n", sp.cls, sp.work, t);
    ctx->k_ms[sp.cls] += t;
    ctx->k_work[sp.cls] += sp.work;
    ctx->k_n[sp.cls] += 1;
    ctx->kpool.push_back(sp.a);
    ctx->kpool.push_back(sp.b);
  }
  ctx->kspans.clear();
  if (ms) *ms = ctx->k_ms[cls];
  if (work) *work = ctx->k_work[cls];
  if (launches) *launches = ctx->k_n[cls];
  return 0;
}

int fv_noise_upload(fv_ctx* ctx, const float* vals, int T, int H, int W) {
  FV_REQUIRE(ctx && vals, "null argument");
  FV_REQUIRE(T >= 1 && H >= 1 && W >= 1, "noise stack must be (T>=1, H, W), got (%d, %d, %d)", T, H, W);
  if (ctx->noise) cudaFree(ctx->noise);
  ctx->noise = nullptr;
  const size_t bytes = sizeof(float) * (size_t)T * H * W;
  FV_CUDA(cudaMalloc(&ctx->noise, bytes));
  FV_CUDA(cudaMemcpy(ctx->noise, vals, bytes, cudaMemcpyHostToDevice));
  ctx->noise_T = T; ctx->noise_H = H; ctx->noise_W = W;
  return 0;
}

int fv_stats_read(fv_ctx* ctx, fv_stats* out) {
  FV_REQUIRE(ctx && out, "null argument");
  DevCounters c;
  FV_CUDA(cudaMemcpyAsync(&c, ctx->counters, sizeof(c), cudaMemcpyDeviceToHost, ctx->stream));
  FV_CUDA(cudaStreamSynchronize(ctx->stream));
  out->rays = c.rays; out->hit_rays = c.hit_rays;
  out->samples_main = c.samples_main; out->samples_shadow = c.samples_shadow;
  return 0;
}

int fv_stats_reset(fv_ctx* ctx) {
  FV_REQUIRE(ctx, "null ctx");
  FV_CUDA(cudaMemsetAsync(ctx->counters, 0, 4 * sizeof(unsigned long long), ctx->stream));
  return 0;
}

static int check_fovea(const fv_fovea* f) {
  FV_REQUIRE(f, "null fovea");
  FV_REQUIRE(f->sigma >= 0, "sigma must be >= 0, got %g", f->sigma);
  FV_REQUIRE(std::isfinite(f->focus[0]) && std::isfinite(f->focus[1]), "focus must be finite");
  FV_REQUIRE(f->base_density >= 0.0 && f->base_density <= 1.0, "base density must lie in [0,1]");
  return 0;
}

int fv_mask_compact(fv_ctx* ctx, int frame, int H, int W, const fv_fovea* fovea,
                    const double* pb_map_dev, uint8_t* bits_dev, int32_t* idx_dev, int32_t* k_dev,
                    fv_state* st) {
  FV_REQUIRE(ctx && idx_dev && k_dev, "null argument");
  FV_REQUIRE(H >= 1 && W >= 1, "dims must be positive, got (%d, %d)", H, W);
  int rc = check_fovea(fovea);
  if (rc) return rc;
  if (st && (st->H != H || st->W != W)) {
    set_error("carried state is for (%d, %d), input is (%d, %d); reset the state", st->H, st->W, H, W);
    return FV_E_STATE;
  }
  return launch_mask_compact(ctx, frame, H, W, fovea, pb_map_dev, bits_dev, idx_dev, k_dev,
                             st ? st->x.p : nullptr, st ? st->Wp : W);
}

int fv_mask_compact_tau(fv_ctx* ctx, int frame, int H, int W, const double* tau_dev, uint8_t* bits_dev,
                        int32_t* idx_dev, int32_t* k_dev, fv_state* st) {
  FV_REQUIRE(ctx && tau_dev && idx_dev && k_dev, "null argument");
  FV_REQUIRE(H >= 1 && W >= 1, "dims must be positive, got (%d, %d)", H, W);
  if (st && (st->H != H || st->W != W)) {
    set_error("carried state is for (%d, %d), input is (%d, %d); reset the state", st->H, st->W, H, W);
    return FV_E_STATE;
  }
  return launch_mask_compact(ctx, frame, H, W, nullptr, nullptr, bits_dev, idx_dev, k_dev,
                             st ? st->x.p : nullptr, st ? st->Wp : W, tau_dev);
}

int fv_tau_map(fv_ctx* ctx, int H, int W, const fv_fovea* fovea, const double* pb_map_dev,
               double* tau_dev) {
  FV_REQUIRE(ctx && tau_dev, "null argument");
  FV_REQUIRE(H >= 1 && W >= 1, "dims must be positive, got (%d, %d)", H, W);
  int rc = check_fovea(fovea);
  if (rc) return rc;
  return launch_tau_map(ctx, H, W, fovea, pb_map_dev, tau_dev);
}

int fv_tau_sum(fv_ctx* ctx, int H, int W, const fv_fovea* fovea, const double* pb_map_dev, const double* tau_dev,
               double* sum_dev) {
  FV_REQUIRE(ctx && sum_dev && (fovea || tau_dev), "null argument");
  FV_REQUIRE(H >= 1 && W >= 1, "dims must be positive, got (%d, %d)", H, W);
  fv_fovea dummy{};
  if (!tau_dev) {
    int rc = check_fovea(fovea);
    if (rc) return rc;
  }
  return launch_tau_sum(ctx, H, W, fovea ? fovea : &dummy, pb_map_dev, tau_dev, sum_dev);
}

int fv_direct_draws(fv_ctx* ctx, int H, int W, const fv_fovea* fovea, const double* pb_map_dev, const double* tau_dev,
                    const double* uniforms_dev, int64_t count, int32_t* idx_dev) {
  FV_REQUIRE(ctx && (fovea || tau_dev) && (count == 0 || (uniforms_dev && idx_dev)), "null argument");
  FV_REQUIRE(H >= 1 && W >= 1, "dims must be positive, got (%d, %d)", H, W);
  FV_REQUIRE(count >= 0, "count must be >= 0");
  fv_fovea dummy{};
  if (!tau_dev) {
    int rc = check_fovea(fovea);
    if (rc) return rc;
  }
  return launch_direct_draws(ctx, H, W, fovea ? fovea : &dummy, pb_map_dev, tau_dev, uniforms_dev, count, idx_dev);
}

int fv_foveal_density(fv_ctx* ctx, const double* dx_dev, const double* dy_dev, int64_t n, double sigma,
                      double pixel_scale, double* out_dev) {
  FV_REQUIRE(ctx && (n == 0 || (dx_dev && dy_dev && out_dev)), "null argument");
  FV_REQUIRE(n >= 0, "count must be >= 0");
  return launch_foveal_density(ctx, dx_dev, dy_dev, n, sigma, pixel_scale, out_dev);
}

int fv_volume_create(fv_ctx* ctx, int nx, int ny, int nz, const double spacing[3], fv_volume** out) {
  FV_REQUIRE(ctx && out, "null argument");
  FV_REQUIRE(nx >= 2 && ny >= 2 && nz >= 2, "volume dims must all be >= 2, got (%d, %d, %d)", nx, ny, nz);
  auto* v = new fv_volume();
  v->nx = nx; v->ny = ny; v->nz = nz;
  for (int a = 0; a < 3; ++a) v->spacing[a] = spacing ? spacing[a] : 1.0;
  const size_t bytes = sizeof(float) * (size_t)nx * ny * nz;
  cudaError_t e = cudaMalloc(&v->data, bytes);
  if (e != cudaSuccess) { delete v; return cuda_fail(e, "cudaMalloc volume"); }
  e = cudaMalloc(&v->lut_dev, sizeof(float) * 4 * 256);
  if (e != cudaSuccess) { cudaFree(v->data); delete v; return cuda_fail(e, "cudaMalloc lut"); }
  *out = v;
  return 0;
}

int fv_volume_wrap(fv_ctx* ctx, int nx, int ny, int nz, const double spacing[3], float* data_dev,
                   fv_volume** out) {
  FV_REQUIRE(ctx && out && data_dev, "null argument");
  FV_REQUIRE(nx >= 2 && ny >= 2 && nz >= 2, "volume dims must all be >= 2, got (%d, %d, %d)", nx, ny, nz);
  auto* v = new fv_volume();
  v->nx = nx; v->ny = ny; v->nz = nz;
  for (int a = 0; a < 3; ++a) v->spacing[a] = spacing ? spacing[a] : 1.0;
  v->data = data_dev;
  v->owns_data = false;
  cudaError_t e = cudaMalloc(&v->lut_dev, sizeof(float) * 4 * 256);
  if (e != cudaSuccess) { delete v; return cuda_fail(e, "cudaMalloc lut"); }
  *out = v;
  return 0;
}

int fv_volume_destroy(fv_volume* v) {
  if (!v) return 0;
  if (v->data && v->owns_data) cudaFree(v->data);
  if (v->lut_dev) cudaFree(v->lut_dev);
  if (v->bricks) cudaFree(v->bricks);
  if (v->qtex) cudaDestroyTextureObject((cudaTextureObject_t)v->qtex);
  if (v->qarr) cudaFreeArray(v->qarr);
  if (v->ltex) cudaDestroyTextureObject((cudaTextureObject_t)v->ltex);
  if (v->larr) cudaFreeArray(v->larr);
  delete v;
  return 0;
}

int fv_volume_upload(fv_ctx* ctx, fv_volume* v, const float* data, int on_device) {
  FV_REQUIRE(ctx && v && data, "null argument");
  const size_t bytes = sizeof(float) * (size_t)v->nx * v->ny * v->nz;
  FV_CUDA(cudaMemcpyAsync(v->data, data, bytes, on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                          ctx->stream));
  FV_CUDA(cudaStreamSynchronize(ctx->stream));
  ++v->version;
  return 0;
}

int fv_volume_procedural(fv_ctx* ctx, fv_volume* v, int kind, double* range) {
  FV_REQUIRE(ctx && v, "null argument");
  ++v->version;
  return launch_volume_procedural(ctx, v, kind, range);
}

int fv_volume_from_raw(fv_ctx* ctx, fv_volume* v, const void* raw_dev, int dtype, double* range,
                       int64_t* first_nan) {
  FV_REQUIRE(ctx && v && v->data && raw_dev, "null argument");
  return launch_volume_from_raw(ctx, v, raw_dev, dtype, range, first_nan);
}

int fv_volume_set_tf(fv_ctx* ctx, fv_volume* v, const float* lut, int K) {
  FV_REQUIRE(ctx && v && lut, "null argument");
  FV_REQUIRE(K >= 2 && K <= 256, "transfer function lut must be (K>=2, 4) with K <= 256, got K=%d", K);
  for (int i = 0; i < 4 * K; ++i)
    FV_REQUIRE(lut[i] >= 0.f && lut[i] <= 1.f, "transfer function entries must lie in [0,1]");
  FV_CUDA(cudaMemcpy(v->lut_dev, lut, sizeof(float) * 4 * K, cudaMemcpyHostToDevice));
  v->K = K;
  return 0;
}

float* fv_volume_data(fv_volume* v) { return v ? v->data : nullptr; }

static int finish_stats(fv_ctx* ctx, fv_stats* out, const DevCounters* before) {
  if (!out) return 0;
  DevCounters c;
  FV_CUDA(cudaMemcpyAsync(&c, ctx->counters, sizeof(c), cudaMemcpyDeviceToHost, ctx->stream));
  FV_CUDA(cudaStreamSynchronize(ctx->stream));
  out->rays = c.rays - before->rays;
  out->hit_rays = c.hit_rays - before->hit_rays;
  out->samples_main = c.samples_main - before->samples_main;
  out->samples_shadow = c.samples_shadow - before->samples_shadow;
  return 0;
}

static int snapshot(fv_ctx* ctx, fv_stats* want, DevCounters* before) {
  if (!want) return 0;
  FV_CUDA(cudaMemcpyAsync(before, ctx->counters, sizeof(*before), cudaMemcpyDeviceToHost, ctx->stream));
  FV_CUDA(cudaStreamSynchronize(ctx->stream));
  return 0;
}

int fv_render_sparse(fv_ctx* ctx, const fv_volume* vol, const fv_camera* cam, const fv_light* light,
                     const fv_settings* settings, const int32_t* idx_dev, const int32_t* k_dev,
                     int k_max, float* rgba_dev, float* depth_dev, fv_state* st,
                     fv_stats* stats_out) {
  FV_REQUIRE(ctx && vol && cam && settings && idx_dev && k_dev, "null argument");
  DevCounters before{};
  int rc = snapshot(ctx, stats_out, &before);
  if (rc) return rc;
  if (st && (st->H != cam->height || st->W != cam->width)) {
    set_error("carried state is for (%d, %d), input is (%d, %d); reset the state", st->H, st->W,
              cam->height, cam->width);
    return FV_E_STATE;
  }
  rc = launch_render(ctx, vol, cam, light, settings, idx_dev, k_dev, k_max, rgba_dev, depth_dev,
                     st ? st->x.p : nullptr, st ? st->Wp : cam->width);
  if (rc) return rc;
  return finish_stats(ctx, stats_out, &before);
}

int fv_render_sparse_naive(fv_ctx* ctx, const fv_volume* vol, const fv_camera* cam, const fv_light* light,
                           const fv_settings* settings, const uint8_t* bits_dev, int32_t* idx_dev,
                           int32_t* k_dev, float* rgba_dev, float* depth_dev, fv_stats* stats_out) {
  FV_REQUIRE(ctx && vol && cam && settings && bits_dev && idx_dev && k_dev, "null argument");
  DevCounters before{};
  int rc = snapshot(ctx, stats_out, &before);
  if (rc) return rc;
  rc = launch_naive_list(ctx, bits_dev, cam->height, cam->width, idx_dev, k_dev);
  if (rc) return rc;
  rc = launch_render(ctx, vol, cam, light, settings, idx_dev, k_dev, cam->width * cam->height, rgba_dev,
                     depth_dev, nullptr, cam->width, /*force_variant=*/2);
  if (rc) return rc;
  return finish_stats(ctx, stats_out, &before);
}

int fv_render_full(fv_ctx* ctx, const fv_volume* vol, const fv_camera* cam, const fv_light* light,
                   const fv_settings* settings, float* rgba_dev, float* depth_dev, fv_stats* stats_out) {
  FV_REQUIRE(ctx && vol && cam && settings, "null argument");
  DevCounters before{};
  int rc = snapshot(ctx, stats_out, &before);
  if (rc) return rc;
  rc = launch_render(ctx, vol, cam, light, settings, nullptr, nullptr, cam->width * cam->height,
                     rgba_dev, depth_dev, nullptr, cam->width);
  if (rc) return rc;
  return finish_stats(ctx, stats_out, &before);
}

int fv_pack_rgb8(fv_ctx* ctx, const float* in_dev, int H, int W, int64_t stride_y, int64_t stride_x,
                 int64_t stride_c, uint8_t* out_dev) {
  FV_REQUIRE(ctx && in_dev && out_dev, "null argument");
  FV_REQUIRE(H > 0 && W > 0, "dims must be positive, got (%d, %d)", H, W);
  return pack_rgb8(ctx, in_dev, H, W, stride_y, stride_x, stride_c, out_dev);
}

int fv_pack_input(fv_ctx* ctx, fv_state* st, const float* rgba_dev, const uint8_t* bits_dev) {
  FV_REQUIRE(ctx && st && rgba_dev && bits_dev, "null argument");
  return pack_input(ctx, st, rgba_dev, bits_dev);
}

int fv_frame(fv_ctx* ctx, const fv_volume* vol, const fv_net* net, fv_state* st, const fv_camera* cam,
             const fv_light* light, const fv_settings* settings, const fv_fovea* fovea, int frame,
             float* host_rgb_out, double* timings_ms) {
  FV_REQUIRE(ctx && vol && net && st && cam && settings && fovea && host_rgb_out, "null argument");
  const int H = cam->height, W = cam->width;
  if (st->H != H || st->W != W) {
    set_error("carried state is for (%d, %d), input is (%d, %d); reset the state", st->H, st->W, H, W);
    return FV_E_STATE;
  }
  int rc = check_fovea(fovea);
  if (rc) return rc;
  const int64_t npix = (int64_t)H * W;
  if (npix > ctx->idx_cap) {
    if (ctx->idx_scratch) cudaFree(ctx->idx_scratch);
    ctx->idx_scratch = nullptr;
    FV_CUDA(cudaMalloc(&ctx->idx_scratch, sizeof(int32_t) * npix));
    ctx->idx_cap = npix;
  }
  if (!ctx->k_scratch) FV_CUDA(cudaMalloc(&ctx->k_scratch, sizeof(int32_t) * 4));
  if (3 * npix > ctx->rgb_cap) {
    if (ctx->rgb_scratch) cudaFree(ctx->rgb_scratch);
    ctx->rgb_scratch = nullptr;
    FV_CUDA(cudaMalloc(&ctx->rgb_scratch, sizeof(float) * 3 * npix));
    ctx->rgb_cap = 3 * npix;
  }
  FV_CUDA(cudaEventRecord(ctx->ev[0], ctx->stream));
  rc = launch_mask_compact(ctx, frame, H, W, fovea, nullptr, nullptr, ctx->idx_scratch, ctx->k_scratch,
                           st->x.p, st->Wp);
  if (rc) return rc;
  FV_CUDA(cudaEventRecord(ctx->ev[1], ctx->stream));
  rc = launch_render(ctx, vol, cam, light, settings, ctx->idx_scratch, ctx->k_scratch, (int)npix, nullptr,
                     nullptr, st->x.p, st->Wp);
  if (rc) return rc;
  FV_CUDA(cudaEventRecord(ctx->ev[2], ctx->stream));
  rc = reconstruct(ctx, net, st, 1, ctx->rgb_scratch, nullptr, nullptr);
  if (rc) return rc;
  FV_CUDA(cudaEventRecord(ctx->ev[3], ctx->stream));
  FV_CUDA(cudaMemcpyAsync(host_rgb_out, ctx->rgb_scratch, sizeof(float) * 3 * npix, cudaMemcpyDeviceToHost,
                          ctx->stream));
  FV_CUDA(cudaStreamSynchronize(ctx->stream));
  if (timings_ms) {
    float a = 0, b = 0, c = 0;
    cudaEventElapsedTime(&a, ctx->ev[0], ctx->ev[1]);
    cudaEventElapsedTime(&b, ctx->ev[1], ctx->ev[2]);
    cudaEventElapsedTime(&c, ctx->ev[2], ctx->ev[3]);
    timings_ms[0] = a; timings_ms[1] = b; timings_ms[2] = c; timings_ms[3] = a + b + c;
  }
  return 0;
}

// ---- fv_frames, whole-frame graph path ------------------------------------------------------
// One frame = frame t's network with frame t+1's mask + march and frame t-1's K filter chain
// forked off it (frame_body_ahead; frame_body: the march of frame t in line, then its network next
// to frame t+1's mask), captured once per launch configuration as ONE CUDA graph and replayed with
// cudaGraphLaunch. The per-frame inputs -- frame t's camera basis and frame t+1's fovea, noise
// frame and scan epoch -- are read by the kernels from the context's FrameDyn block, which a
// pinned ring feeds with one small host->device copy ahead of each replay (no host round trip:
// the host only waits for a ring slot it is about to overwrite, kDynRing frames back).
constexpr int kDynRing = 8;

static int frame_body(fv_ctx* ctx, cudaStream_t s_main, cudaStream_t s_side, cudaEvent_t ev_fork, cudaEvent_t ev_join,
                      const fv_volume* vol, const fv_net* net, fv_state* st, const fv_camera* cam,
                      const fv_light* light, const fv_settings* settings, const fv_fovea* fovea_next, int frame_next,
                      float* img) {
  const int64_t npix = (int64_t)st->H * st->W;
  ctx->stream = s_main;
  int rc = launch_render(ctx, vol, cam, light, settings, ctx->idx_scratch, ctx->k_scratch, (int)npix, nullptr,
                         nullptr, st->x.p, st->Wp);
  if (rc) return rc;
  FV_CUDA(cudaEventRecord(ev_fork, s_main));
  FV_CUDA(cudaStreamWaitEvent(s_side, ev_fork, 0));
  ctx->stream = s_side;
  // the next frame's mask writes channels 0..4 of the other input buffer (the network below writes
  // its feedback channels 5..7 of the same buffer: disjoint bytes)
  rc = launch_mask_compact(ctx, frame_next, st->H, st->W, fovea_next, nullptr, nullptr, ctx->idx_scratch,
                           ctx->k_scratch, st->xalt.p, st->Wp);
  if (rc) return rc;
  FV_CUDA(cudaEventRecord(ev_join, s_side));
  ctx->stream = s_main;
  rc = reconstruct_launches(ctx, const_cast<fv_net*>(net), st, 1, img, nullptr, nullptr);
  if (rc) return rc;
  FV_CUDA(cudaStreamWaitEvent(s_main, ev_join, 0));
  return 0;
}

// March-ahead variant (FV_MARCH_AHEAD=k): the graph of frame t holds frame t's network and, forked
// after its k-th conv launch, frame t+1's mask + march into the other input buffer -- the render of
// the next frame fills the SMs the network's small levels leave idle. (Both write disjoint bytes of
// that buffer: the mask channels 0..4, the march channels 0..3 of active pixels, the network's
// D.head feedback channels 5..7; the network reads only the current buffer.)
// The previous frame's K filter chain + output stage (FV_KCHAIN_SPLIT=2), forked off this frame's
// network after its chain_at-th conv: it reads the previous frame's O_d and weight planes (the
// other parity's buffers, which this frame's network does not touch).
struct ChainFork {
  cudaStream_t s_main, s_side;
  cudaEvent_t fork, join;
  fv_net* net;
  fv_state* st;
  float* img;
  const float* od;
  const std::vector<kw_t*>* kw;
  cudaEvent_t done;  // recorded (an external record node when captured) once the chain is complete
};

static int chain_fork_hook(fv_ctx* ctx, void* arg) {
  const ChainFork& c = *static_cast<const ChainFork*>(arg);
  FV_CUDA(cudaEventRecord(c.fork, c.s_main));
  FV_CUDA(cudaStreamWaitEvent(c.s_side, c.fork, 0));
  const cudaStream_t keep = ctx->stream;
  ctx->stream = c.s_side;
  const int rc = kfilter_launches(ctx, c.net, c.st, 1, c.od, c.img, nullptr, nullptr, c.kw);
  ctx->stream = keep;
  if (rc) return rc;
  // (the external record first: the join below then covers it, so the capture stays joined)
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  FV_CUDA(cudaStreamIsCapturing(c.s_side, &cs));
  FV_CUDA(cudaEventRecordWithFlags(c.done, c.s_side,
                                   cs == cudaStreamCaptureStatusActive ? cudaEventRecordExternal : 0));
  FV_CUDA(cudaEventRecord(c.join, c.s_side));
  return 0;
}

static int frame_body_ahead(fv_ctx* ctx, cudaStream_t s_main, cudaStream_t s_side, cudaEvent_t ev_fork,
                            cudaEvent_t ev_join, const fv_volume* vol, const fv_net* net, fv_state* st,
                            const fv_camera* cam_next, const fv_light* light, const fv_settings* settings,
                            const fv_fovea* fovea_next, int frame_next, float* img, int fork_at,
                            const ChainFork* chain = nullptr, int chain_at = 0) {
  const int64_t npix = (int64_t)st->H * st->W;
  ctx->stream = s_main;
  ctx->conv_fork_ev = ev_fork;
  ctx->conv_fork_at = fork_at;
  ctx->conv_count = 0;
  if (chain) {
    ctx->conv_hook = chain_fork_hook;
    ctx->conv_hook_arg = const_cast<ChainFork*>(chain);
    ctx->conv_hook_at = chain_at;
  }
  int rc = reconstruct_launches(ctx, const_cast<fv_net*>(net), st, 1, img, nullptr, nullptr);
  const bool hook_missed = ctx->conv_hook != nullptr;
  ctx->conv_fork_ev = nullptr;
  ctx->conv_hook = nullptr;
  ctx->kw_wait_ev = nullptr;
  if (rc) return rc;
  if (chain && hook_missed) {
    set_error("fv_frames: the filter chain fork point (conv %d) lies past the network's convs", chain_at);
    return FV_E_INVALID;
  }
  if (chain) FV_CUDA(cudaStreamWaitEvent(s_main, chain->join, 0));
  if (ctx->conv_count < fork_at) FV_CUDA(cudaEventRecord(ev_fork, s_main));
  FV_CUDA(cudaStreamWaitEvent(s_side, ev_fork, 0));
  ctx->stream = s_side;
  rc = launch_mask_compact(ctx, frame_next, st->H, st->W, fovea_next, nullptr, nullptr, ctx->idx_scratch,
                           ctx->k_scratch, st->xalt.p, st->Wp);
  if (!rc)
    rc = launch_render(ctx, vol, cam_next, light, settings, ctx->idx_scratch, ctx->k_scratch, (int)npix, nullptr,
                       nullptr, st->xalt.p, st->Wp);
  if (rc) return rc;
  FV_CUDA(cudaEventRecord(ev_join, s_side));
  ctx->stream = s_main;
  FV_CUDA(cudaStreamWaitEvent(s_main, ev_join, 0));
  return 0;
}

static int frames_graph(fv_ctx* ctx, const fv_volume* vol, const fv_net* net, fv_state* st, int n,
                        const fv_camera* cams, const fv_light* light, const fv_settings* settings,
                        const fv_fovea* foveas, const int* frame_ids, float* const* host_rgb_out) {
  const int H = st->H, W = st->W;
  const int64_t npix = (int64_t)H * W;
  int rc = prepare_net(ctx, net);
  if (rc) return rc;
  if (!ctx->dyn_dev) {
    FV_CUDA(cudaMalloc(&ctx->dyn_dev, sizeof(FrameDyn)));
    FV_CUDA(cudaMallocHost(&ctx->dyn_host, sizeof(FrameDyn) * kDynRing));
    for (auto& e : ctx->dyn_ev) FV_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  for (int i = 0; i < 3; ++i)
    if (!st->fcap[i]) FV_CUDA(cudaStreamCreateWithFlags(&st->fcap[i], cudaStreamNonBlocking));
  for (int i = 0; i < 4; ++i)
    if (!st->fcap_ev[i]) FV_CUDA(cudaEventCreateWithFlags(&st->fcap_ev[i], cudaEventDisableTiming));
  static const bool no_graph = getenv("FV_FRAME_GRAPH") && atoi(getenv("FV_FRAME_GRAPH")) == 0;
  const cudaStream_t own = ctx->stream;
  cudaStream_t s_n = ctx->fstream[1], s_m = ctx->fstream[3], s_c = ctx->fstream[2];
  cudaEvent_t* net_done = ctx->fev + 2;  // [2]
  cudaEvent_t* copied = ctx->fev + 4;    // [2]
  cudaEvent_t fork = ctx->fev[8], join = ctx->fev[9];
  // The K filter chain + output stage of frame t (10 launches) reads frame t's O_d and K weight
  // planes, which are double-buffered by hidden parity, so it can run next to frame t+1's network:
  //   FV_KCHAIN_SPLIT=2 (default): folded into frame t+1's graph, forked after its FV_KCHAIN_AT-th
  //     conv (default 12: next to the level-0 upsample and D6.conv1); frame t's image is copied after
  //     frame t+1's graph (one frame of output latency; the last frame's chain runs after the loop);
  //   =1: its own graph on a chain stream right after frame t's graph;  =0: in the frame graph.
  // Measured on the C3 frame timeline (median us per frame): chain stream 1539 / 1542, folded after
  // conv 1 / 9 / 12 / 13: 1543 / 1541 / 1533 (1535) / 1537; in the frame graph (round-2 first pass) ~1610.
  static const int split_env = getenv("FV_KCHAIN_SPLIT") ? atoi(getenv("FV_KCHAIN_SPLIT")) : 2;
  static const int chain_at = std::min(14, std::max(1, getenv("FV_KCHAIN_AT") ? atoi(getenv("FV_KCHAIN_AT")) : 12));
  const bool fold = split_env == 2;  // (needs march-ahead; checked below)
  const bool split = split_env == 1;
  if ((split || fold) && !ctx->kstream) {
    int lo = 0, hi = 0;
    FV_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    int prio = 0;
    FV_CUDA(cudaStreamGetPriority(s_n, &prio));
    FV_CUDA(cudaStreamCreateWithPriority(&ctx->kstream, cudaStreamNonBlocking, prio));
    for (auto& e : ctx->kev) FV_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    for (auto& e : ctx->kdone) FV_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  cudaStream_t s_k = split ? ctx->kstream : s_n;
  cudaEvent_t* chain_done = ctx->kev;  // [2]
  cudaEvent_t chain_last = ctx->kev[2];
  FV_CUDA(cudaEventRecord(ctx->fev[6], own));
  for (cudaStream_t s_ : {s_n, s_m, s_c, s_k}) FV_CUDA(cudaStreamWaitEvent(s_, ctx->fev[6], 0));
  if (split) FV_CUDA(cudaEventRecord(chain_last, s_k));  // nothing pending: the first network need not wait
  // frame t+1's mask + march forked off frame t's network after its k-th conv launch (the march
  // then runs next to the network's level 1-3 convs, which leave SMs idle). A/B at C3 (frames/s,
  // e2e), fork after conv 0 (off) / 2 / 4 / 6 / 8: 547.8 / 559.6 / 579.1 / 583.0 / 585.4 and e2e
  // 498 / 506 / 520 / 514 / 492 (later forks collide with the level-0 decoder convs); frames are
  // bit-identical for every fork point. FV_MARCH_AHEAD=0: the march in line before the network.
  // With the K filter chain split off (it overlaps the frame's first convs), re-measured on the
  // frame timeline (median us per frame), fork after conv 2 / 3 / 4 / 5 / 6 / 8: 1579 / 1590 / 1566 /
  // 1575 / 1553 / 1558 -- after E2.conv2 (6) by default.
  // At 4K (C5) every network conv fills the GPU, so there is no idle capacity for the march: the
  // march in line measured 124.4 / 125.6 against 123.3 / 123.5 frames/s forked after conv 6 --
  // films above 4 Mpixel march in line by default.
  static const int ahead_env = getenv("FV_MARCH_AHEAD") ? atoi(getenv("FV_MARCH_AHEAD")) : -1;
  const int ahead = ahead_env >= 0 ? ahead_env : (npix > 4000000 ? 0 : 6);
  const bool folded = fold && ahead > 0;
  // prologue: frame 0's mask (and with march-ahead its march), by-value parameters
  ctx->stream = s_n;
  rc = launch_mask_compact(ctx, frame_ids[0], H, W, &foveas[0], nullptr, nullptr, ctx->idx_scratch, ctx->k_scratch,
                           st->x.p, st->Wp);
  if (!rc && ahead > 0)
    rc = launch_render(ctx, vol, &cams[0], light, settings, ctx->idx_scratch, ctx->k_scratch, (int)npix, nullptr,
                       nullptr, st->x.p, st->Wp);
  static uint64_t dyn_seq = 0;
// inside the frame loop: record the failure and leave the loop (streams are restored below)
#define FG_TRY(call)                 \
  {                                  \
    const cudaError_t e_ = (call);   \
    if (e_ != cudaSuccess) {         \
      rc = cuda_fail(e_, #call);     \
      break;                         \
    }                                \
  }
  for (int t = 0; t < n && !rc; ++t) {
    const int b = t & 1;
    float* img = ctx->rgb_scratch + (int64_t)b * 3 * npix;
    const int tn = t + 1 < n ? t + 1 : t;
    // this frame's FrameDyn: camera t, fovea / noise frame / epoch of frame t+1's mask
    const int slot = (int)(dyn_seq++ % kDynRing);
    FG_TRY(cudaEventSynchronize(ctx->dyn_ev[slot]));
    FrameDyn& d = ctx->dyn_host[slot];
    rc = fill_camera_dyn(&cams[ahead > 0 ? tn : t], &d);
    if (rc) break;
    d.fx = foveas[tn].focus[0]; d.fy = foveas[tn].focus[1]; d.sigma = foveas[tn].sigma;
    d.pb = foveas[tn].base_density; d.scale = foveas[tn].pixel_scale;
    d.frame = frame_ids[tn];
    if (++ctx->epoch == 0) ctx->epoch = 1;
    d.epoch = ctx->epoch;
    FG_TRY(cudaMemcpyAsync(ctx->dyn_dev, &d, sizeof(FrameDyn), cudaMemcpyHostToDevice, s_n));
    FG_TRY(cudaEventRecord(ctx->dyn_ev[slot], s_n));
    if (!folded && t >= 2) FG_TRY(cudaStreamWaitEvent(s_k, copied[b], 0));  // frame t-2's copy read image b
    // folded: this graph's chain writes frame t-1's image, whose buffer frame t-3's copy read
    float* prev_img = folded && t >= 1 ? ctx->rgb_scratch + (int64_t)((t - 1) & 1) * 3 * npix : nullptr;
    if (folded && t >= 3) FG_TRY(cudaStreamWaitEvent(s_n, copied[(t - 1) & 1], 0));
    ctx->kchain_split = split || folded;
    ctx->kw_wait_ev = split ? chain_last : nullptr;
    ctx->kw_wait_external = split;
    // the frame's launch configuration
    fv_state::FrameGraph* g = nullptr;
    for (auto& e : st->fgraphs)
      if (e.vol == vol && e.net == net && e.version == net->version && e.wave_version == ctx->wave_version &&
          e.x == st->x.p && e.parity == st->parity && e.ahead == ahead && e.img == img && e.prev_img == prev_img &&
          e.has_light == (light != nullptr) &&
          (!light || memcmp(&e.light, light, sizeof(fv_light)) == 0) &&
          memcmp(&e.settings, settings, sizeof(fv_settings)) == 0) {
        g = &e;
        break;
      }
    if (!g && !no_graph) {
      if (st->fgraphs.size() >= 8) {
        for (auto& e : st->fgraphs)
          if (e.exec) cudaGraphExecDestroy(e.exec);
        st->fgraphs.clear();
      }
      fv_state::FrameGraph e;
      e.vol = vol; e.net = net; e.version = net->version; e.wave_version = ctx->wave_version; e.x = st->x.p;
      e.parity = st->parity; e.ahead = ahead; e.img = img; e.prev_img = prev_img; e.has_light = light != nullptr;
      if (light) e.light = *light;
      e.settings = *settings;
      st->fgraphs.push_back(e);
      g = &st->fgraphs.back();
    }
    ctx->dyn_active = ctx->dyn_dev;
    if (g && g->exec) {
      const cudaError_t e = cudaGraphLaunch(g->exec, s_n);
      if (e != cudaSuccess) rc = cuda_fail(e, "cudaGraphLaunch (frame)");
      ctx->launches += g->n_launches;
    } else if (g && g->uses >= 1) {
      // capture this configuration (second use), then replay it for this frame
      cudaGraph_t graph = nullptr;
      const unsigned long long before = ctx->launches;
      cudaError_t e = cudaStreamBeginCapture(st->fcap[0], cudaStreamCaptureModeThreadLocal);
      if (e == cudaSuccess) {
        const ChainFork cf{st->fcap[0], st->fcap[2], st->fcap_ev[2], st->fcap_ev[3], const_cast<fv_net*>(net), st,
                           prev_img, st->od_buf[st->parity], &st->kw_buf[st->parity], ctx->kdone[(t - 1) & 1]};
        rc = ahead > 0 ? frame_body_ahead(ctx, st->fcap[0], st->fcap[1], st->fcap_ev[0], st->fcap_ev[1], vol, net, st,
                                          &cams[tn], light, settings, &foveas[tn], frame_ids[tn], img, ahead,
                                          prev_img ? &cf : nullptr, chain_at)
                       : frame_body(ctx, st->fcap[0], st->fcap[1], st->fcap_ev[0], st->fcap_ev[1], vol, net, st,
                                    &cams[t], light, settings, &foveas[tn], frame_ids[tn], img);
        e = cudaStreamEndCapture(st->fcap[0], &graph);
      }
      if (!rc && e != cudaSuccess) rc = cuda_fail(e, "frame graph capture");
      if (!rc) {
        e = cudaGraphInstantiate(&g->exec, graph, 0);
        if (e != cudaSuccess) { g->exec = nullptr; rc = cuda_fail(e, "cudaGraphInstantiate (frame)"); }
      }
      if (graph) cudaGraphDestroy(graph);
      g->n_launches = ctx->launches - before;
      if (!rc) {
        e = cudaGraphLaunch(g->exec, s_n);
        if (e != cudaSuccess) rc = cuda_fail(e, "cudaGraphLaunch (frame)");
      }
    } else if (ahead > 0) {
      const ChainFork cf{s_n, s_k, ctx->kev[0], ctx->kev[1], const_cast<fv_net*>(net), st, prev_img,
                         st->od_buf[st->parity], &st->kw_buf[st->parity], ctx->kdone[(t - 1) & 1]};
      rc = frame_body_ahead(ctx, s_n, s_m, fork, join, vol, net, st, &cams[tn], light, settings, &foveas[tn],
                            frame_ids[tn], img, ahead, prev_img ? &cf : nullptr, chain_at);
    } else {
      rc = frame_body(ctx, s_n, s_m, fork, join, vol, net, st, &cams[t], light, settings, &foveas[tn],
                      frame_ids[tn], img);
    }
    ctx->dyn_active = nullptr;
    ctx->kchain_split = false;
    ctx->kw_wait_ev = nullptr;
    ctx->kw_wait_external = false;
    if (g) ++g->uses;
    if (rc) break;
    // reconstruct()'s host-side state change: the input buffers swap, the hidden parity flips
    state_advance(st);
    FG_TRY(cudaEventRecord(net_done[b], s_n));
    if (split) {
      // the filter chain of frame t into image b (reads O_d and the weight planes of frame t)
      FG_TRY(cudaStreamWaitEvent(s_k, net_done[b], 0));
      fv_state::ChainGraph* cg = nullptr;
      for (auto& e : st->cgraphs)
        if (e.net == net && e.version == net->version && e.img == img && e.od == st->od) cg = &e;
      if (!cg) {
        fv_state::ChainGraph e;
        e.net = net; e.version = net->version; e.img = img; e.od = st->od;
        st->cgraphs.push_back(e);
        cg = &st->cgraphs.back();
      }
      ctx->stream = s_k;
      if (cg->exec) {
        const cudaError_t e = cudaGraphLaunch(cg->exec, s_k);
        if (e != cudaSuccess) rc = cuda_fail(e, "cudaGraphLaunch (filter chain)");
        ctx->launches += cg->n_launches;
      } else if (cg->uses >= 1 && !no_graph) {
        cudaGraph_t graph = nullptr;
        const unsigned long long before = ctx->launches;
        cudaError_t e = cudaStreamBeginCapture(st->fcap[0], cudaStreamCaptureModeThreadLocal);
        if (e == cudaSuccess) {
          ctx->stream = st->fcap[0];
          rc = kfilter_launches(ctx, const_cast<fv_net*>(net), st, 1, st->od, img, nullptr, nullptr);
          ctx->stream = s_k;
          e = cudaStreamEndCapture(st->fcap[0], &graph);
        }
        if (!rc && e != cudaSuccess) rc = cuda_fail(e, "filter chain graph capture");
        if (!rc) {
          e = cudaGraphInstantiate(&cg->exec, graph, 0);
          if (e != cudaSuccess) { cg->exec = nullptr; rc = cuda_fail(e, "cudaGraphInstantiate (filter chain)"); }
        }
        if (graph) cudaGraphDestroy(graph);
        cg->n_launches = ctx->launches - before;
        if (!rc) {
          e = cudaGraphLaunch(cg->exec, s_k);
          if (e != cudaSuccess) rc = cuda_fail(e, "cudaGraphLaunch (filter chain)");
        }
      } else {
        rc = kfilter_launches(ctx, const_cast<fv_net*>(net), st, 1, st->od, img, nullptr, nullptr);
      }
      ctx->stream = s_n;
      ++cg->uses;
      if (rc) break;
      FG_TRY(cudaEventRecord(chain_done[b], s_k));
      FG_TRY(cudaEventRecord(chain_last, s_k));
    }
    if (folded) {
      // frame t-1's image is complete once this graph's chain branch is (its external record node)
      if (t >= 1) {
        const bool out = host_rgb_out && host_rgb_out[t - 1];
        if (out) {
          FG_TRY(cudaStreamWaitEvent(s_c, ctx->kdone[(t - 1) & 1], 0));
          FG_TRY(cudaMemcpyAsync(host_rgb_out[t - 1], prev_img, sizeof(float) * 3 * npix, cudaMemcpyDefault, s_c));
        }
        FG_TRY(cudaEventRecord(copied[(t - 1) & 1], out ? s_c : s_n));
      }
      if (t == n - 1) {
        // the last frame's chain after its own graph
        ctx->stream = s_n;
        rc = kfilter_launches(ctx, const_cast<fv_net*>(net), st, 1, st->od, img, nullptr, nullptr);
        if (rc) break;
        FG_TRY(cudaEventRecord(net_done[b], s_n));
        const bool out = host_rgb_out && host_rgb_out[t];
        if (out) {
          FG_TRY(cudaStreamWaitEvent(s_c, net_done[b], 0));
          FG_TRY(cudaMemcpyAsync(host_rgb_out[t], img, sizeof(float) * 3 * npix, cudaMemcpyDefault, s_c));
        }
        FG_TRY(cudaEventRecord(copied[b], out ? s_c : s_n));
      }
      continue;
    }
    cudaEvent_t img_ready = split ? chain_done[b] : net_done[b];
    const bool out = host_rgb_out && host_rgb_out[t];
    if (out) {
      FG_TRY(cudaStreamWaitEvent(s_c, img_ready, 0));
      FG_TRY(cudaMemcpyAsync(host_rgb_out[t], img, sizeof(float) * 3 * npix, cudaMemcpyDefault, s_c));
    }
    FG_TRY(cudaEventRecord(copied[b], out ? s_c : s_k));
  }
#undef FG_TRY
  ctx->dyn_active = nullptr;
  ctx->kchain_split = false;
  ctx->kw_wait_ev = nullptr;
  ctx->stream = own;
  for (cudaStream_t s_ : {s_n, s_m, s_c, s_k}) {
    cudaError_t e = cudaEventRecord(ctx->fev[7], s_);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(own, ctx->fev[7], 0);
    if (e != cudaSuccess && !rc) rc = cuda_fail(e, "fv_frames rejoin");
  }
  if (rc) return rc;
  // host outputs are complete on return; device outputs are stream-ordered on the context's stream
  bool any_host = false;
  for (int t = 0; host_rgb_out && t < n; ++t) {
    cudaPointerAttributes pa{};
    if (host_rgb_out[t] && cudaPointerGetAttributes(&pa, host_rgb_out[t]) == cudaSuccess && pa.type != cudaMemoryTypeDevice)
      any_host = true;
    (void)cudaGetLastError();
  }
  if (any_host) FV_CUDA(cudaStreamSynchronize(s_c));
  return 0;
}

// fv_frames: the whole-frame graph path above (frames_graph) by default; the stream-juggling path
// below serves FV_PIPE_OVERLAP=1, FV_MASK_AHEAD=0, FV_FRAME_GRAPH=2, kernel timing and fp64 renders.
// A path of frames with host outputs, pipelined over four streams:
//   mask stream   : mask + compaction of frame t+1 (FV_MASK_AHEAD, default on) next to frame t's
//                   network; waits for rendered[t] (the march of frame t, the last reader of the ray
//                   list) and net_done[t-1] (the last reader of the input buffer it fills), signals
//                   masked[t+1]. With FV_MASK_AHEAD=0 the mask runs in line on the render stream.
//   render stream : the march of frame t (waits for masked[t] and net_done[t-2]); by default this
//                   IS the network stream (render and network in frame order: the marcher's and the
//                   convs' persistent grids do not share SMs well); FV_PIPE_OVERLAP=1 gives it its
//                   own stream so render t+1 overlaps reconstruct t. Signals rendered[t].
//   network stream: reconstruction of frame t into device image t%2 (waits for rendered[t] and
//                   copied[t-2], the last reader of that image); signals net_done[t].
//   copy stream   : device image t%2 -> host_rgb_out[t] (waits for net_done[t]); signals copied[t].
// The host enqueues in frame order, so every kernel sees exactly the buffers fv_frame would. On an
// error the loop stops, the context's own stream is restored and rejoined with all four streams.
int fv_frames(fv_ctx* ctx, const fv_volume* vol, const fv_net* net, fv_state* st, int n,
              const fv_camera* cams, const fv_light* light, const fv_settings* settings,
              const fv_fovea* foveas, const int* frame_ids, float* const* host_rgb_out) {
  FV_REQUIRE(ctx && vol && net && st && cams && settings && foveas && frame_ids, "null argument");
  FV_REQUIRE(n >= 0, "frame count must be >= 0 (got %d)", n);
  if (n == 0) return 0;
  const int H = st->H, W = st->W;
  for (int t = 0; t < n; ++t) {
    if (cams[t].height != H || cams[t].width != W) {
      set_error("carried state is for (%d, %d), input is (%d, %d); reset the state", H, W, cams[t].height,
                cams[t].width);
      return FV_E_STATE;
    }
    const int rc = check_fovea(&foveas[t]);
    if (rc) return rc;
  }
  const int64_t npix = (int64_t)H * W;
  if (npix > ctx->idx_cap) {
    if (ctx->idx_scratch) cudaFree(ctx->idx_scratch);
    ctx->idx_scratch = nullptr;
    FV_CUDA(cudaMalloc(&ctx->idx_scratch, sizeof(int32_t) * npix));
    ctx->idx_cap = npix;
  }
  if (!ctx->k_scratch) FV_CUDA(cudaMalloc(&ctx->k_scratch, sizeof(int32_t) * 4));
  if (6 * npix > ctx->rgb_cap) {
    if (ctx->rgb_scratch) cudaFree(ctx->rgb_scratch);
    ctx->rgb_scratch = nullptr;
    FV_CUDA(cudaMalloc(&ctx->rgb_scratch, sizeof(float) * 6 * npix));
    ctx->rgb_cap = 6 * npix;
  }
  if (!ctx->fstream[0]) {
    // the network is the critical path: its stream gets the highest priority, so the marcher's
    // blocks fill the SMs the convs leave idle instead of delaying them
    int lo = 0, hi = 0;
    FV_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    const char* e = getenv("FV_PIPE_PRIORITY");
    const bool prio = !(e && atoi(e) == 0);
    FV_CUDA(cudaStreamCreateWithPriority(&ctx->fstream[0], cudaStreamNonBlocking, lo));
    FV_CUDA(cudaStreamCreateWithPriority(&ctx->fstream[1], cudaStreamNonBlocking, prio ? hi : lo));
    FV_CUDA(cudaStreamCreateWithPriority(&ctx->fstream[2], cudaStreamNonBlocking, lo));
    FV_CUDA(cudaStreamCreateWithPriority(&ctx->fstream[3], cudaStreamNonBlocking, lo));
  }
  for (auto& e : ctx->fev)
    if (!e) FV_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  // FV_PIPE_OVERLAP=1: render t+1 on its own stream next to reconstruct t; by default both run
  // in order on the network stream (only the copy-out overlaps): the marcher's persistent grids
  // and the convs' persistent CTAs do not share SMs well (C5: 71 frames/s overlapped against 95
  // in order), and the two barely overlap at C3
  static const bool overlap = getenv("FV_PIPE_OVERLAP") && atoi(getenv("FV_PIPE_OVERLAP")) == 1;
  // frame t+1's mask + compaction on a fourth stream next to frame t's network (after frame t's
  // march, the last reader of the ray list, and frame t-1's network, the last reader of the input
  // buffer it fills); FV_MASK_AHEAD=0 keeps it in line. Measured +0.5% frames/s, +1% e2e at C3.
  static const bool ahead = !(getenv("FV_MASK_AHEAD") && atoi(getenv("FV_MASK_AHEAD")) == 0);
  // default: the whole-frame graph path (FV_FRAME_GRAPH=0 keeps it eager but with the same
  // FrameDyn launches); the stream-juggling path below serves FV_PIPE_OVERLAP=1, FV_MASK_AHEAD=0,
  // kernel timing and fp64 renders
  static const bool legacy = getenv("FV_FRAME_GRAPH") && atoi(getenv("FV_FRAME_GRAPH")) == 2;
  if (!overlap && ahead && !legacy && !ctx->ktiming && settings->precision != FV_PREC_FP64)
    return frames_graph(ctx, vol, net, st, n, cams, light, settings, foveas, frame_ids, host_rgb_out);
  cudaStream_t s_r = overlap ? ctx->fstream[0] : ctx->fstream[1], s_n = ctx->fstream[1], s_c = ctx->fstream[2];
  cudaStream_t s_m = ctx->fstream[3];
  cudaEvent_t* masked = ctx->fev + 8;  // [2]
  cudaEvent_t* rendered = ctx->fev;      // [2]
  cudaEvent_t* net_done = ctx->fev + 2;  // [2]
  cudaEvent_t* copied = ctx->fev + 4;    // [2]
  cudaEvent_t start = ctx->fev[6];
  const cudaStream_t own = ctx->stream;
  FV_CUDA(cudaEventRecord(start, own));
  for (cudaStream_t s : {s_r, s_n, s_c, s_m}) FV_CUDA(cudaStreamWaitEvent(s, start, 0));
  int rc = 0;
  if (ahead) {
    ctx->stream = s_m;
    rc = launch_mask_compact(ctx, frame_ids[0], H, W, &foveas[0], nullptr, nullptr, ctx->idx_scratch,
                             ctx->k_scratch, st->x.p, st->Wp);
    if (!rc) {
      const cudaError_t e = cudaEventRecord(masked[0], s_m);
      if (e != cudaSuccess) rc = cuda_fail(e, "cudaEventRecord (mask ahead)");
    }
  }
// inside the frame loop: record the failure and leave the loop (the stream state is restored below)
#define FV_TRY(call)                                   \
  {                                                    \
    const cudaError_t e_ = (call);                     \
    if (e_ != cudaSuccess) {                           \
      rc = cuda_fail(e_, #call);                       \
      break;                                           \
    }                                                  \
  }
  for (int t = 0; t < n && !rc; ++t) {
    const int b = t & 1;
    float* img = ctx->rgb_scratch + (int64_t)b * 3 * npix;
    // render
    if (t >= 2) FV_TRY(cudaStreamWaitEvent(s_r, net_done[b], 0));
    ctx->stream = s_r;
    if (ahead) {
      FV_TRY(cudaStreamWaitEvent(s_r, masked[b], 0));
    } else {
      rc = launch_mask_compact(ctx, frame_ids[t], H, W, &foveas[t], nullptr, nullptr, ctx->idx_scratch,
                               ctx->k_scratch, st->x.p, st->Wp);
    }
    if (!rc)
      rc = launch_render(ctx, vol, &cams[t], light, settings, ctx->idx_scratch, ctx->k_scratch, (int)npix,
                         nullptr, nullptr, st->x.p, st->Wp);
    if (rc) break;
    FV_TRY(cudaEventRecord(rendered[b], s_r));
    // network
    FV_TRY(cudaStreamWaitEvent(s_n, rendered[b], 0));
    if (t >= 2) FV_TRY(cudaStreamWaitEvent(s_n, copied[b], 0));
    ctx->stream = s_n;
    rc = reconstruct(ctx, net, st, 1, img, nullptr, nullptr);
    if (rc) break;
    FV_TRY(cudaEventRecord(net_done[b], s_n));
    if (ahead && t + 1 < n) {
      // reconstruct() swapped the state's input buffers: st->x is frame t+1's now
      FV_TRY(cudaStreamWaitEvent(s_m, rendered[b], 0));
      if (t >= 1) FV_TRY(cudaStreamWaitEvent(s_m, net_done[b ^ 1], 0));
      ctx->stream = s_m;
      rc = launch_mask_compact(ctx, frame_ids[t + 1], H, W, &foveas[t + 1], nullptr, nullptr, ctx->idx_scratch,
                               ctx->k_scratch, st->x.p, st->Wp);
      if (rc) break;
      FV_TRY(cudaEventRecord(masked[b ^ 1], s_m));
    }
    // copy out
    FV_TRY(cudaStreamWaitEvent(s_c, net_done[b], 0));
    if (host_rgb_out && host_rgb_out[t])
      FV_TRY(cudaMemcpyAsync(host_rgb_out[t], img, sizeof(float) * 3 * npix, cudaMemcpyDefault, s_c));
    FV_TRY(cudaEventRecord(copied[b], s_c));
  }
  ctx->stream = own;
  // rejoin: the context's own stream continues after every frame and copy (also after an error)
  for (cudaStream_t s : {s_r, s_n, s_c, s_m}) {
    cudaError_t e = cudaEventRecord(ctx->fev[7], s);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(own, ctx->fev[7], 0);
    if (e != cudaSuccess && !rc) rc = cuda_fail(e, "fv_frames rejoin");
  }
#undef FV_TRY
  if (rc) return rc;
  FV_CUDA(cudaStreamSynchronize(s_c));
  return 0;
}

}  // extern "C"
