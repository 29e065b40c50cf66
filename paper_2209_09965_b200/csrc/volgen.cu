// Procedural test volumes generated on the GPU.
//
// Reference: volume.make_procedural_volume (volume.py:112-146) + _normalize (volume.py:75-81).
// Raw fields are evaluated in fp64 at voxel centres u,v,w = (i+0.5)/n*2-1 with numpy's
// left-to-right operation order, min-max normalised with the global extremes and cast to
// float32. fp64 sin/cos differ from numpy's by at most an ulp, which survives the f32 cast only
// for a vanishing fraction of voxels (the tests bound it).
#include "internal.h"

namespace fv {
namespace {

constexpr double kPi = 3.141592653589793;

__device__ __forceinline__ double raw_field(int kind, int x, int y, int z, int nx, int ny, int nz) {
  const double u = ((double)x + 0.5) / nx * 2.0 - 1.0;
  const double v = ((double)y + 0.5) / ny * 2.0 - 1.0;
  const double w = ((double)z + 0.5) / nz * 2.0 - 1.0;
  if (kind == 2) {  // box_lattice
    const double par = fmod(floor(2.0 * (u + 1.0)) + floor(2.0 * (v + 1.0)) + floor(2.0 * (w + 1.0)), 2.0);
    return __dadd_rn(__dmul_rn(0.7, par), __dmul_rn(0.3, u + 1.0) / 2.0);
  }
  const double r = sqrt(__dadd_rn(__dadd_rn(__dmul_rn(u, u), __dmul_rn(v, v)), __dmul_rn(w, w)));
  if (kind == 0) {  // sphere_shells
    return 0.5 * (1.0 + cos(__dmul_rn(2.0 * kPi * 3.0, r)));
  }
  // vortex_field
  const double a = __dadd_rn(__dmul_rn(3.0 * kPi, u), __dmul_rn(__dmul_rn(2.0, v), w));
  const double b = __dsub_rn(__dmul_rn(2.0 * kPi, v), __dmul_rn(__dmul_rn(1.5, u), w));
  const double raw = __dmul_rn(sin(a), cos(b));
  return __dadd_rn(raw, __dmul_rn(0.5, cos(__dmul_rn(4.0 * kPi, r))));
}

__global__ void minmax_kernel(int kind, int nx, int ny, int nz, double* partial) {
  const int64_t n = (int64_t)nx * ny * nz;
  double lo = INFINITY, hi = -INFINITY;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int x = (int)(i % nx);
    const int y = (int)((i / nx) % ny);
    const int z = (int)(i / ((int64_t)nx * ny));
    const double r = raw_field(kind, x, y, z, nx, ny, nz);
    lo = fmin(lo, r);
    hi = fmax(hi, r);
  }
  __shared__ double slo[32], shi[32];
  for (int o = 16; o > 0; o >>= 1) {
    lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  if ((threadIdx.x & 31) == 0) { slo[threadIdx.x >> 5] = lo; shi[threadIdx.x >> 5] = hi; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) { lo = fmin(lo, slo[w]); hi = fmax(hi, shi[w]); }
    partial[2 * blockIdx.x] = lo;
    partial[2 * blockIdx.x + 1] = hi;
  }
}

__global__ void minmax_final(const double* partial, int n, double* out) {
  double lo = INFINITY, hi = -INFINITY;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    lo = fmin(lo, partial[2 * i]);
    hi = fmax(hi, partial[2 * i + 1]);
  }
  for (int o = 16; o > 0; o >>= 1) {
    lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  if (threadIdx.x == 0) { out[0] = lo; out[1] = hi; }
}

__global__ void normalize_kernel(int kind, int nx, int ny, int nz, const double* range, float* out) {
  const int64_t n = (int64_t)nx * ny * nz;
  const double lo = range[0], hi = range[1];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int x = (int)(i % nx);
    const int y = (int)((i / nx) % ny);
    const int z = (int)(i / ((int64_t)nx * ny));
    const double r = raw_field(kind, x, y, z, nx, ny, nz);
    out[i] = hi > lo ? (float)(__dsub_rn(r, lo) / __dsub_rn(hi, lo)) : 0.0f;
  }
}

// ---- raw volumes (load_raw_volume, volume.py:84-109): NaN scan, global min/max, normalisation ----
template <typename T>
__global__ void raw_scan_kernel(const T* __restrict__ raw, int64_t n, double* partial,
                                unsigned long long* first_nan) {
  double lo = INFINITY, hi = -INFINITY;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double r = (double)raw[i];
    if (r != r) {
      atomicMin(first_nan, (unsigned long long)i);
      continue;
    }
    lo = fmin(lo, r);
    hi = fmax(hi, r);
  }
  __shared__ double slo[32], shi[32];
  for (int o = 16; o > 0; o >>= 1) {
    lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  if ((threadIdx.x & 31) == 0) { slo[threadIdx.x >> 5] = lo; shi[threadIdx.x >> 5] = hi; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) { lo = fmin(lo, slo[w]); hi = fmax(hi, shi[w]); }
    partial[2 * blockIdx.x] = lo;
    partial[2 * blockIdx.x + 1] = hi;
  }
}

// (raw - lo) / (hi - lo) in fp64 -> float32 (volume.py:75-81); zeros for a constant volume
template <typename T>
__global__ void raw_normalize_kernel(const T* __restrict__ raw, int64_t n, const double* range, float* out) {
  const double lo = range[0], hi = range[1];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = hi > lo ? (float)(__dsub_rn((double)raw[i], lo) / __dsub_rn(hi, lo)) : 0.0f;
}

}  // namespace

int launch_volume_from_raw(fv_ctx* ctx, fv_volume* vol, const void* raw, int dtype, double* range_out,
                           int64_t* first_nan_out) {
  FV_REQUIRE(dtype == 0 || dtype == 1, "raw dtype code %d (0 = uint8, 1 = float32)", dtype);
  const int64_t n = (int64_t)vol->nx * vol->ny * vol->nz;
  const int blocks = ctx->num_sms * 8;
  double* tmp = nullptr;
  FV_CUDA(cudaMallocAsync(&tmp, sizeof(double) * (2 * blocks + 3), ctx->stream));
  unsigned long long* nan_at = reinterpret_cast<unsigned long long*>(tmp + 2 * blocks + 2);
  FV_CUDA(cudaMemsetAsync(nan_at, 0xff, sizeof(unsigned long long), ctx->stream));
  if (dtype == 0)
    FV_TIMED(ctx, FV_KC_OTHER, raw_scan_kernel<uint8_t><<<blocks, 256, 0, ctx->stream>>>(
                                   static_cast<const uint8_t*>(raw), n, tmp + 2, nan_at));
  else
    FV_TIMED(ctx, FV_KC_OTHER, raw_scan_kernel<float><<<blocks, 256, 0, ctx->stream>>>(
                                   static_cast<const float*>(raw), n, tmp + 2, nan_at));
  FV_TIMED(ctx, FV_KC_OTHER, minmax_final<<<1, 32, 0, ctx->stream>>>(tmp + 2, blocks, tmp));
  unsigned long long nan_host = ~0ull;
  FV_CUDA(cudaMemcpyAsync(&nan_host, nan_at, sizeof(nan_host), cudaMemcpyDeviceToHost, ctx->stream));
  double r[2];
  FV_CUDA(cudaMemcpyAsync(r, tmp, sizeof(r), cudaMemcpyDeviceToHost, ctx->stream));
  FV_CUDA(cudaStreamSynchronize(ctx->stream));
  if (first_nan_out) *first_nan_out = nan_host == ~0ull ? -1 : (int64_t)nan_host;
  if (nan_host != ~0ull) {
    cudaFreeAsync(tmp, ctx->stream);
    const int64_t i = (int64_t)nan_host;
    set_error("NaN in volume data at flat index %lld (voxel x=%lld, y=%lld, z=%lld)", (long long)i,
              (long long)(i % vol->nx), (long long)((i / vol->nx) % vol->ny),
              (long long)(i / ((int64_t)vol->nx * vol->ny)));
    return FV_E_INVALID;
  }
  if (dtype == 0)
    FV_TIMED(ctx, FV_KC_OTHER, raw_normalize_kernel<uint8_t><<<blocks, 256, 0, ctx->stream>>>(
                                   static_cast<const uint8_t*>(raw), n, tmp, vol->data));
  else
    FV_TIMED(ctx, FV_KC_OTHER, raw_normalize_kernel<float><<<blocks, 256, 0, ctx->stream>>>(
                                   static_cast<const float*>(raw), n, tmp, vol->data));
  FV_CHECK_LAUNCH("raw volume kernels");
  ctx->launches += 3;
  FV_CUDA(cudaFreeAsync(tmp, ctx->stream));
  vol->value_range[0] = r[0];
  vol->value_range[1] = r[1];
  ++vol->version;
  if (range_out) { range_out[0] = r[0]; range_out[1] = r[1]; }
  return 0;
}

int launch_volume_procedural(fv_ctx* ctx, fv_volume* vol, int kind, double* range_out) {
  FV_REQUIRE(kind >= 0 && kind <= 2, "unknown procedural volume kind %d", kind);
  FV_REQUIRE(vol->nx >= 8 && vol->ny >= 8 && vol->nz >= 8,
             "procedural dims must be >= 8 per axis, got (%d, %d, %d)", vol->nx, vol->ny, vol->nz);
  const int blocks = ctx->num_sms * 8;
  double* tmp = nullptr;
  FV_CUDA(cudaMallocAsync(&tmp, sizeof(double) * (2 * blocks + 2), ctx->stream));
  FV_TIMED(ctx, FV_KC_OTHER, minmax_kernel<<<blocks, 256, 0, ctx->stream>>>(kind, vol->nx, vol->ny, vol->nz, tmp + 2));
  FV_TIMED(ctx, FV_KC_OTHER, minmax_final<<<1, 32, 0, ctx->stream>>>(tmp + 2, blocks, tmp));
  FV_TIMED(ctx, FV_KC_OTHER, normalize_kernel<<<blocks, 256, 0, ctx->stream>>>(kind, vol->nx, vol->ny, vol->nz, tmp, vol->data));
  FV_CHECK_LAUNCH("procedural volume kernels");
  ctx->launches += 3;
  double r[2];
  FV_CUDA(cudaMemcpyAsync(r, tmp, sizeof(r), cudaMemcpyDeviceToHost, ctx->stream));
  FV_CUDA(cudaFreeAsync(tmp, ctx->stream));
  FV_CUDA(cudaStreamSynchronize(ctx->stream));
  vol->value_range[0] = r[0];
  vol->value_range[1] = r[1];
  if (range_out) { range_out[0] = r[0]; range_out[1] = r[1]; }
  return 0;
}

}  // namespace fv
