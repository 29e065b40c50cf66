// Image-quality metrics on the device, fp64 like the reference.
//
// Reference (pkg/src/fovray/metrics.py):
//   psnr      metrics.py:40-49   joint RGB mean squared error, 100 dB cap
//   ssim      metrics.py:74-87   Rec.601 luma, 11x11 Gaussian window (sigma 1.5) as a separable
//                                'valid' correlation (rows first), K1=0.01, K2=0.03, mean over
//                                valid windows
//   msssim    metrics.py:104-130 5-scale weights renormalised to the usable scales, contrast-
//                                structure means clamped at 0, 2x2 mean downsampling
//   tpsnr     metrics.py:133-148 PSNR of (d+1)/2 temporal differences
//
// Reductions are deterministic: fixed per-block partial sums, then one block adds them in order.
// Images are (H, W, C) float64 with C >= 3 (RGB = channels 0..2) or C == 1 (already luma).
#include <cmath>
#include <vector>

#include "internal.h"

namespace fv {
namespace {

constexpr int kWin = 11;
constexpr int kRed = 256;      // threads per reduction block
constexpr int kRedBlocks = 592;  // 4 x 148 partial sums

__constant__ double c_gauss[kWin];

__device__ __forceinline__ double block_sum(double v, double* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) sh[w] = v;
  __syncthreads();
  v = 0.0;
  if (threadIdx.x < 32) {
    v = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  }
  __syncthreads();
  return v;  // valid in thread 0
}

// partial[b] (q per block) -> out[q] in block order
__global__ void sum_partials_kernel(const double* __restrict__ partial, int nblocks, int q, double* out) {
  __shared__ double sh[32];
  for (int k = 0; k < q; ++k) {
    double v = 0.0;
    for (int i = threadIdx.x; i < nblocks; i += blockDim.x) v += partial[(int64_t)i * q + k];
    v = block_sum(v, sh);
    if (threadIdx.x == 0) out[k] = v;
  }
}

// sum over pixels and channels 0..2 of (a - b)^2, or of the tPSNR difference when a0/b0 are given
__global__ void __launch_bounds__(kRed) sqdiff_kernel(const double* __restrict__ a, const double* __restrict__ b,
                                                      const double* __restrict__ a0, const double* __restrict__ b0,
                                                      int64_t npix, int ca, int cb, double* partial) {
  __shared__ double sh[32];
  double acc = 0.0;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < npix; p += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      double x = a[p * ca + c], y = b[p * cb + c];
      if (a0) {  // (d + 1) / 2 of the temporal differences (metrics.py:145-146)
        x = (x - a0[p * ca + c] + 1.0) / 2.0;
        y = (y - b0[p * cb + c] + 1.0) / 2.0;
      }
      const double d = x - y;
      acc += d * d;
    }
  }
  acc = block_sum(acc, sh);
  if (threadIdx.x == 0) partial[blockIdx.x] = acc;
}

// Rec.601 luma (metrics.py:32-37); C == 1 passes through
__global__ void luma_kernel(const double* __restrict__ img, int c, int64_t npix, double* __restrict__ out) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < npix; p += (int64_t)gridDim.x * blockDim.x)
    out[p] = c == 1 ? img[p] : 0.299 * img[p * c] + 0.587 * img[p * c + 1] + 0.114 * img[p * c + 2];
}

// vertical 11-tap pass of the five SSIM fields: (H-10, W) x 5 planes
__global__ void ssim_vert_kernel(const double* __restrict__ la, const double* __restrict__ lb, int h, int w,
                                 double* __restrict__ v5) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y;
  if (x >= w) return;
  double s[5] = {0, 0, 0, 0, 0};
#pragma unroll
  for (int k = 0; k < kWin; ++k) {
    const double g = c_gauss[k];
    const double pa = la[(int64_t)(y + k) * w + x], pb = lb[(int64_t)(y + k) * w + x];
    s[0] += pa * g;
    s[1] += pb * g;
    s[2] += (pa * pa) * g;
    s[3] += (pb * pb) * g;
    s[4] += (pa * pb) * g;
  }
  const int64_t n = (int64_t)(h - kWin + 1) * w, i = (int64_t)y * w + x;
#pragma unroll
  for (int f = 0; f < 5; ++f) v5[f * n + i] = s[f];
}

// horizontal pass + per-window statistics; per-block partial sums of (ssim, cs, lum*cs)
__global__ void __launch_bounds__(kRed) ssim_horiz_kernel(const double* __restrict__ v5, int hv, int w,
                                                          double* partial) {
  __shared__ double sh[32];
  const int wo = w - kWin + 1;
  const int64_t n = (int64_t)hv * w, no = (int64_t)hv * wo;
  const double c1 = 0.01 * 0.01, c2 = 0.03 * 0.03;
  double acc_s = 0.0, acc_cs = 0.0, acc_lcs = 0.0;
  for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < no; o += (int64_t)gridDim.x * blockDim.x) {
    const int64_t y = o / wo, x = o % wo;
    double s[5] = {0, 0, 0, 0, 0};
#pragma unroll
    for (int k = 0; k < kWin; ++k) {
      const double g = c_gauss[k];
#pragma unroll
      for (int f = 0; f < 5; ++f) s[f] += v5[f * n + y * w + x + k] * g;
    }
    const double mu_a = s[0], mu_b = s[1];
    const double var_a = s[2] - mu_a * mu_a, var_b = s[3] - mu_b * mu_b, cov = s[4] - mu_a * mu_b;
    const double cs = (2 * cov + c2) / (var_a + var_b + c2);
    const double lum = (2 * mu_a * mu_b + c1) / (mu_a * mu_a + mu_b * mu_b + c1);
    acc_s += ((2 * mu_a * mu_b + c1) * (2 * cov + c2)) / ((mu_a * mu_a + mu_b * mu_b + c1) * (var_a + var_b + c2));
    acc_cs += cs;
    acc_lcs += lum * cs;
  }
  acc_s = block_sum(acc_s, sh);
  acc_cs = block_sum(acc_cs, sh);
  acc_lcs = block_sum(acc_lcs, sh);
  if (threadIdx.x == 0) {
    partial[blockIdx.x * 3 + 0] = acc_s;
    partial[blockIdx.x * 3 + 1] = acc_cs;
    partial[blockIdx.x * 3 + 2] = acc_lcs;
  }
}

// 2x2 mean downsampling with the odd row/column cropped (metrics.py:90-93)
__global__ void down2_kernel(const double* __restrict__ in, int h, int w, double* __restrict__ out) {
  const int wo = w / 2;
  const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y;
  if (x >= wo) return;
  const double* r0 = in + (int64_t)(2 * y) * w + 2 * x;
  const double* r1 = r0 + w;
  out[(int64_t)y * wo + x] = 0.25 * (((r0[0] + r1[0]) + r0[1]) + r1[1]);
}

struct Scratch {
  double* p = nullptr;
  size_t cap = 0;
};

int scratch_get(Scratch& s, size_t n, double** out) {
  if (n > s.cap) {
    if (s.p) cudaFree(s.p);
    s.p = nullptr;
    FV_CUDA(cudaMalloc(&s.p, n * sizeof(double)));
    s.cap = n;
  }
  *out = s.p;
  return 0;
}

thread_local Scratch g_scratch;
bool g_gauss_ready = false;

int upload_gauss() {
  if (g_gauss_ready) return 0;
  double k[kWin], sum = 0.0;
  for (int i = 0; i < kWin; ++i) {
    const double d = (double)i - (kWin - 1) / 2.0;
    k[i] = std::exp(-(d * d) / (2.0 * 1.5 * 1.5));
  }
  for (int i = 0; i < kWin; ++i) sum += k[i];
  for (int i = 0; i < kWin; ++i) k[i] /= sum;
  FV_CUDA(cudaMemcpyToSymbol(c_gauss, k, sizeof(k)));
  g_gauss_ready = true;
  return 0;
}

// sums of (ssim, cs, lum*cs) over the valid windows of luma planes la, lb (h x w)
int ssim_sums(fv_ctx* ctx, const double* la, const double* lb, int h, int w, double* work, double* part,
              double* dsum, double host[3], int64_t* count) {
  const int hv = h - kWin + 1;
  ssim_vert_kernel<<<dim3((w + 127) / 128, hv), 128, 0, ctx->stream>>>(la, lb, h, w, work);
  FV_CHECK_LAUNCH("ssim_vert_kernel");
  ssim_horiz_kernel<<<kRedBlocks, kRed, 0, ctx->stream>>>(work, hv, w, part);
  FV_CHECK_LAUNCH("ssim_horiz_kernel");
  sum_partials_kernel<<<1, kRed, 0, ctx->stream>>>(part, kRedBlocks, 3, dsum);
  FV_CHECK_LAUNCH("sum_partials_kernel");
  ctx->launches += 3;
  FV_CUDA(cudaMemcpyAsync(host, dsum, 3 * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  FV_CUDA(cudaStreamSynchronize(ctx->stream));
  *count = (int64_t)hv * (w - kWin + 1);
  return 0;
}

}  // namespace
}  // namespace fv

using namespace fv;

extern "C" {

int fv_metric_sqdiff(fv_ctx* ctx, const double* a, const double* b, const double* a_prev, const double* b_prev,
                     int H, int W, int ca, int cb, double* sum_out) {
  FV_REQUIRE(ctx && a && b && sum_out, "null argument");
  FV_REQUIRE(H > 0 && W > 0 && ca >= 3 && cb >= 3, "images must be (H,W,C>=3), got %dx%d C=%d/%d", H, W, ca, cb);
  FV_REQUIRE((a_prev == nullptr) == (b_prev == nullptr), "temporal differences need both previous frames");
  double* buf = nullptr;
  int rc = scratch_get(g_scratch, kRedBlocks + 4, &buf);
  if (rc) return rc;
  sqdiff_kernel<<<kRedBlocks, kRed, 0, ctx->stream>>>(a, b, a_prev, b_prev, (int64_t)H * W, ca, cb, buf);
  FV_CHECK_LAUNCH("sqdiff_kernel");
  sum_partials_kernel<<<1, kRed, 0, ctx->stream>>>(buf, kRedBlocks, 1, buf + kRedBlocks);
  FV_CHECK_LAUNCH("sum_partials_kernel");
  ctx->launches += 2;
  FV_CUDA(cudaMemcpyAsync(sum_out, buf + kRedBlocks, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  FV_CUDA(cudaStreamSynchronize(ctx->stream));
  return 0;
}

// mode 0: SSIM; mode 1: MS-SSIM with `scales` scales and renormalised `weights` (host, scales entries)
int fv_metric_ssim(fv_ctx* ctx, const double* a, const double* b, int H, int W, int ca, int cb, int mode,
                   int scales, const double* weights, double* out) {
  FV_REQUIRE(ctx && a && b && out, "null argument");
  FV_REQUIRE((ca == 1 || ca >= 3) && (cb == 1 || cb >= 3), "images must be (H,W) luma or (H,W,C>=3)");
  FV_REQUIRE(H >= kWin && W >= kWin, "frames smaller than the %dpx SSIM window: (%d, %d)", kWin, H, W);
  FV_REQUIRE(mode == 0 || (scales >= 1 && weights), "MS-SSIM needs its scale weights");
  int rc = upload_gauss();
  if (rc) return rc;
  const int64_t np0 = (int64_t)H * W;
  // scratch: la, lb, la2, lb2 (half size), 5 vertical planes, partials, sums
  const size_t need = 2 * np0 + 2 * (np0 / 4 + 1) + 5 * np0 + 3 * kRedBlocks + 8;
  double* s = nullptr;
  rc = scratch_get(g_scratch, need, &s);
  if (rc) return rc;
  double *la = s, *lb = la + np0, *la2 = lb + np0, *lb2 = la2 + np0 / 4 + 1, *work = lb2 + np0 / 4 + 1;
  double* part = work + 5 * np0;
  double* dsum = part + 3 * kRedBlocks;
  const int g = (int)std::min<int64_t>((np0 + 255) / 256, (int64_t)ctx->num_sms * 8);
  luma_kernel<<<g, 256, 0, ctx->stream>>>(a, ca, np0, la);
  luma_kernel<<<g, 256, 0, ctx->stream>>>(b, cb, np0, lb);
  FV_CHECK_LAUNCH("luma_kernel");
  ctx->launches += 2;
  double sums[3];
  int64_t cnt = 0;
  if (mode == 0) {
    rc = ssim_sums(ctx, la, lb, H, W, work, part, dsum, sums, &cnt);
    if (rc) return rc;
    *out = sums[0] / (double)cnt;
    return 0;
  }
  double value = 1.0;
  int h = H, w = W;
  for (int j = 0; j < scales; ++j) {
    rc = ssim_sums(ctx, la, lb, h, w, work, part, dsum, sums, &cnt);
    if (rc) return rc;
    const double stat = (j == scales - 1 ? sums[2] : sums[1]) / (double)cnt;
    value *= std::pow(stat > 0.0 ? stat : 0.0, weights[j]);
    if (j < scales - 1) {
      down2_kernel<<<dim3((w / 2 + 127) / 128, h / 2), 128, 0, ctx->stream>>>(la, h, w, la2);
      down2_kernel<<<dim3((w / 2 + 127) / 128, h / 2), 128, 0, ctx->stream>>>(lb, h, w, lb2);
      FV_CHECK_LAUNCH("down2_kernel");
      ctx->launches += 2;
      // the next scale reads la2/lb2; copy back into la/lb (sizes shrink, so they fit)
      FV_CUDA(cudaMemcpyAsync(la, la2, sizeof(double) * (h / 2) * (w / 2), cudaMemcpyDeviceToDevice, ctx->stream));
      FV_CUDA(cudaMemcpyAsync(lb, lb2, sizeof(double) * (h / 2) * (w / 2), cudaMemcpyDeviceToDevice, ctx->stream));
      h /= 2;
      w /= 2;
    }
  }
  *out = value;
  return 0;
}

}  // extern "C"
