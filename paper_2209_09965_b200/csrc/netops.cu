// Memory-bound W-Net operators around the tcgen05 convolutions.
//
// Reference (pkg/src/fovray):
//   upsample_bilinear2   autograd.py:294-305, :322-329 (half-pixel, edge clamp, rows then cols)
//   avg_pool2            autograd.py:279-291
//   softmax_channels     autograd.py:188-199 (max-subtracted softmax over the 9 taps)
//   apply_kernel_field   autograd.py:332-359 (tap j = (dy, dx) = divmod(j, 3), zero padding,
//                                             accumulated in tap order)
//   predict_kernel_fields network.py:268-277 (1x1 conv of the decoder hidden state)
//   forward_K            network.py:280-293 (pool after e-blocks, upsample after d-blocks)
//   _reconstruct_frame   bench.py:166-175   (x = rgba*m ++ m; output clipped to [0,1])
#include <cooperative_groups.h>

#include "internal.h"

namespace cg = cooperative_groups;

namespace fv {

namespace {

// ---- D-path 2x bilinear upsample, fp16 NC8HW8 -> fp16 NC8HW8 -------------------------------
// (FV_UP_ROWS=1; the default is upsample2_nc8_rows_kernel<2> below)
// grid: (ceil(w / 128), h, groups); one thread per INPUT pixel (i, j) writes the 2x2 output
// block (2i..2i+1, 2j..2j+1) of its 8 channels from the clamped 3x3 input neighbourhood.
__device__ __forceinline__ void load8(const __half* p, float (&v)[8]) {
  const uint4 q = *reinterpret_cast<const uint4*>(p);
  const __half2* h2 = reinterpret_cast<const __half2*>(&q);
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const float2 t = __half22float2(h2[e]);
    v[2 * e] = t.x;
    v[2 * e + 1] = t.y;
  }
}

__global__ void __launch_bounds__(128) upsample2_nc8_kernel(const __half* __restrict__ in,
                                                            __half* __restrict__ out, int h, int w) {
  fv::pdl_wait();
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y, g = blockIdx.z;
  if (j >= w) return;
  const __half* pl = in + (int64_t)g * h * w * 8;
  const int rows[3] = {max(i - 1, 0), i, min(i + 1, h - 1)};
  const int cols[3] = {max(j - 1, 0), j, min(j + 1, w - 1)};
  // rows first (axis 2): even output row = 0.25*prev + 0.75*self, odd = 0.75*self + 0.25*next
  float re[3][8], ro[3][8];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    float a[8], b[8], d[8];
    load8(pl + ((int64_t)rows[0] * w + cols[c]) * 8, a);
    load8(pl + ((int64_t)rows[1] * w + cols[c]) * 8, b);
    load8(pl + ((int64_t)rows[2] * w + cols[c]) * 8, d);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      re[c][e] = 0.25f * a[e] + 0.75f * b[e];
      ro[c][e] = 0.75f * b[e] + 0.25f * d[e];
    }
  }
  const int W2 = 2 * w;
  __half* ob = out + (int64_t)g * (2 * h) * W2 * 8;
#pragma unroll
  for (int rr = 0; rr < 2; ++rr) {
    const float (&r)[3][8] = rr ? ro : re;
    uint4 q0, q1;
    __half2* o0 = reinterpret_cast<__half2*>(&q0);
    __half2* o1 = reinterpret_cast<__half2*>(&q1);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      // then columns (axis 3)
      o0[e] = __floats2half2_rn(0.25f * r[0][2 * e] + 0.75f * r[1][2 * e],
                                0.25f * r[0][2 * e + 1] + 0.75f * r[1][2 * e + 1]);
      o1[e] = __floats2half2_rn(0.75f * r[1][2 * e] + 0.25f * r[2][2 * e],
                                0.75f * r[1][2 * e + 1] + 0.25f * r[2][2 * e + 1]);
    }
    uint4* dst = reinterpret_cast<uint4*>(ob + ((int64_t)(2 * i + rr) * W2 + 2 * j) * 8);
    dst[0] = q0;
    dst[1] = q1;
  }
}

// RP input rows per thread (i0 .. i0 + RP - 1 -> output rows 2 i0 .. 2 i0 + 2 RP - 1): the RP + 2
// input rows i0 - 1 .. i0 + RP are loaded once (3 (RP + 2) loads instead of 9 RP), kept as packed
// halves; the arithmetic per output is the one-row kernel's (bit-identical).
// grid: (ceil(w / 128), ceil(h / RP), groups).
template <int RP>
__global__ void __launch_bounds__(128) upsample2_nc8_rows_kernel(const __half* __restrict__ in,
                                                                 __half* __restrict__ out, int h, int w) {
  fv::pdl_wait();
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int i0 = RP * blockIdx.y, g = blockIdx.z;
  if (j >= w) return;
  const __half* pl = in + (int64_t)g * h * w * 8;
  const int cols[3] = {max(j - 1, 0), j, min(j + 1, w - 1)};
  const int W2 = 2 * w;
  __half* ob = out + (int64_t)g * (2 * h) * W2 * 8;
  uint4 q[RP + 2][3];
#pragma unroll
  for (int r = 0; r < RP + 2; ++r) {
    const int row = min(max(i0 - 1 + r, 0), h - 1);
#pragma unroll
    for (int c = 0; c < 3; ++c) q[r][c] = *reinterpret_cast<const uint4*>(pl + ((int64_t)row * w + cols[c]) * 8);
  }
#pragma unroll
  for (int ii = 0; ii < RP; ++ii) {
    if (i0 + ii >= h) break;
#pragma unroll
    for (int rr = 0; rr < 2; ++rr) {
      // rows first: even output row = 0.25*prev + 0.75*self, odd = 0.75*self + 0.25*next
      float r[3][8];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const __half2* p0 = reinterpret_cast<const __half2*>(&q[ii + rr][c]);
        const __half2* p1 = reinterpret_cast<const __half2*>(&q[ii + rr + 1][c]);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 u = __half22float2(p0[e]), v = __half22float2(p1[e]);
          r[c][2 * e] = rr ? 0.75f * u.x + 0.25f * v.x : 0.25f * u.x + 0.75f * v.x;
          r[c][2 * e + 1] = rr ? 0.75f * u.y + 0.25f * v.y : 0.25f * u.y + 0.75f * v.y;
        }
      }
      uint4 q0, q1;
      __half2* o0 = reinterpret_cast<__half2*>(&q0);
      __half2* o1 = reinterpret_cast<__half2*>(&q1);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        o0[e] = __floats2half2_rn(0.25f * r[0][2 * e] + 0.75f * r[1][2 * e],
                                  0.25f * r[0][2 * e + 1] + 0.75f * r[1][2 * e + 1]);
        o1[e] = __floats2half2_rn(0.75f * r[1][2 * e] + 0.25f * r[2][2 * e],
                                  0.75f * r[1][2 * e + 1] + 0.25f * r[2][2 * e + 1]);
      }
      uint4* dst = reinterpret_cast<uint4*>(ob + ((int64_t)(2 * (i0 + ii) + rr) * W2 + 2 * j) * 8);
      dst[0] = q0;
      dst[1] = q1;
    }
  }
}

// ---- K stage: apply the per-pixel 3x3 filters ------------------------------------------------
// out[c,y,x] = sum_j k[j,y,x] * img[c, y+j/3-1, x+j%3-1], zero padding, taps in order
// (apply_kernel_field, autograd.py:332-359). The softmax-normalised weights k come from the
// tcgen05 logits conv's epilogue (conv_tc.cu), so this pass only streams 9 + 3 planes.
__device__ __forceinline__ void kapply_at(const kw_t* __restrict__ kw, const float* __restrict__ img,
                                          float* __restrict__ out, int h, int w, int x, int y) {
  const int64_t n = (int64_t)h * w, pix = (int64_t)y * w + x;
  float k[9];
#pragma unroll
  for (int j = 0; j < 9; ++j) k[j] = kw_load(kw + j * n + pix);
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const float* pl = img + (int64_t)c * n;
    float acc = 0.f;
#pragma unroll
    for (int j = 0; j < 9; ++j) {
      const int yy = y + j / 3 - 1, xx = x + j % 3 - 1;
      const float v = (yy >= 0 && yy < h && xx >= 0 && xx < w) ? __ldg(pl + (int64_t)yy * w + xx) : 0.f;
      acc = acc + k[j] * v;
    }
    out[(int64_t)c * n + pix] = acc;
  }
}

__global__ void __launch_bounds__(128) kapply_kernel(const kw_t* __restrict__ kw, const float* __restrict__ img,
                                                     float* __restrict__ out, int h, int w) {
  fv::pdl_wait();
  const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y;
  if (x >= w) return;
  kapply_at(kw, img, out, h, w, x, y);
}

// One pixel of apply_kernel_field for the 3 channels (same tap order and zero padding as above).
__device__ __forceinline__ void kapply_px(const kw_t* __restrict__ kw, const float* __restrict__ img, int h, int w,
                                          int y, int x, float (&o)[3]) {
  const int64_t n = (int64_t)h * w, pix = (int64_t)y * w + x;
  float k[9];
#pragma unroll
  for (int j = 0; j < 9; ++j) k[j] = kw_load(kw + j * n + pix);
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const float* pl = img + (int64_t)c * n;
    float acc = 0.f;
#pragma unroll
    for (int j = 0; j < 9; ++j) {
      const int yy = y + j / 3 - 1, xx = x + j % 3 - 1;
      const float v = (yy >= 0 && yy < h && xx >= 0 && xx < w) ? __ldg(pl + (int64_t)yy * w + xx) : 0.f;
      acc = acc + k[j] * v;
    }
    o[c] = acc;
  }
}

// K block on an encoder level fused with the avg_pool2 that follows it (forward_K, network.py:280-293):
// one thread per POOLED pixel computes the 2x2 filtered pixels and averages them, so the level-L
// filtered image is never written. h, w: level-L dims (even).
__global__ void __launch_bounds__(128) kapply_pool_kernel(const kw_t* __restrict__ kw, const float* __restrict__ img,
                                                          float* __restrict__ out, int h, int w) {
  fv::pdl_wait();
  const int ho = h >> 1, wo = w >> 1;
  const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y;
  if (x >= wo) return;
  float p00[3], p10[3], p01[3], p11[3];
  kapply_px(kw, img, h, w, 2 * y, 2 * x, p00);
  kapply_px(kw, img, h, w, 2 * y + 1, 2 * x, p10);
  kapply_px(kw, img, h, w, 2 * y, 2 * x + 1, p01);
  kapply_px(kw, img, h, w, 2 * y + 1, 2 * x + 1, p11);
  const int64_t no = (int64_t)ho * wo;
#pragma unroll
  for (int c = 0; c < 3; ++c)  // 0.25 * (p00 + p10 + p01 + p11), left to right as autograd.avg_pool2
    out[c * no + (int64_t)y * wo + x] = 0.25f * (((p00[c] + p10[c]) + p01[c]) + p11[c]);
}

// Last K block (level 0) fused with the output stage: crop, clip to [0,1] and interleave (rgb), plus
// the optional raw outputs (bench._reconstruct_frame, bench.py:166-175).
__global__ void __launch_bounds__(128) kapply_final_kernel(const kw_t* __restrict__ kw, const float* __restrict__ img,
                                                           const float* __restrict__ od, int H, int W, int Hp, int Wp,
                                                           float* __restrict__ rgb, float* __restrict__ o_raw,
                                                           float* __restrict__ od_raw) {
  fv::pdl_wait();
  const int u = blockIdx.x * blockDim.x + threadIdx.x, v = blockIdx.y;
  if (u >= W) return;
  float o[3];
  kapply_px(kw, img, Hp, Wp, v, u, o);
  const int64_t n = (int64_t)H * W, i = (int64_t)v * W + u, pp = (int64_t)Hp * Wp, j = (int64_t)v * Wp + u;
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    if (rgb) rgb[i * 3 + c] = fminf(fmaxf(o[c], 0.f), 1.f);
    if (o_raw) o_raw[c * n + i] = o[c];
    if (od_raw) od_raw[c * n + i] = od[c * pp + j];
  }
}

// The same two passes with 8-byte loads: a thread handles two horizontally adjacent pixels, so its
// filter weights come as float2 and its 3 x 4 (or, pooled, 4 x 4) image window as three float2 per
// row and channel -- all independent loads, issued together (the per-pixel kernels above: 80
// registers, four dependent rounds of 36 loads, ncu 31% occupancy and 31% DRAM). Taps are summed in
// the same order, so results are identical.
__device__ __forceinline__ float2 ld2_or0(const float* p, bool ok) {
  return ok ? __ldg(reinterpret_cast<const float2*>(p)) : make_float2(0.f, 0.f);
}

// window win[r][c] = img[c0 + ...]: rows y0-1 .. y0+nr-2, columns x0-1 .. x0+2 (zero outside)
template <int NR>
__device__ __forceinline__ void load_win(const float* pl, int h, int w, int y0, int x0, float (&win)[NR][4]) {
#pragma unroll
  for (int r = 0; r < NR; ++r) {
    const int yy = y0 - 1 + r;
    const bool rin = yy >= 0 && yy < h;
    const float* row = pl + (int64_t)(rin ? yy : 0) * w;
    const float2 a = ld2_or0(row + x0 - 2, rin && x0 - 2 >= 0);   // columns x0-2, x0-1
    const float2 b = ld2_or0(row + x0, rin);                      // x0, x0+1
    const float2 c = ld2_or0(row + x0 + 2, rin && x0 + 2 < w);    // x0+2, x0+3
    win[r][0] = a.y; win[r][1] = b.x; win[r][2] = b.y; win[r][3] = c.x;
  }
}

// grid (ceil(w/2/128), h/2): one thread per POOLED pixel = the 2x2 filtered pixels (2x .. 2x+1)
__device__ __forceinline__ void kapply_pool2_at(const kw_t* __restrict__ kw, const float* __restrict__ img,
                                                float* __restrict__ out, int h, int w, int x, int y) {
  const int ho = h >> 1, wo = w >> 1;
  const int X0 = 2 * x, Y0 = 2 * y;
  const int64_t n = (int64_t)h * w;
  float2 k[9][2];
#pragma unroll
  for (int j = 0; j < 9; ++j)
#pragma unroll
    for (int r = 0; r < 2; ++r) k[j][r] = __ldg(reinterpret_cast<const float2*>(kw + j * n + (int64_t)(Y0 + r) * w + X0));
  const int64_t no = (int64_t)ho * wo;
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    float win[4][4];
    load_win<4>(img + (int64_t)c * n, h, w, Y0, X0, win);
    float p[2][2];
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        float acc = 0.f;
#pragma unroll
        for (int j = 0; j < 9; ++j) acc = acc + (q ? k[j][r].y : k[j][r].x) * win[r + j / 3][q + j % 3];
        p[r][q] = acc;
      }
    // 0.25 * (p00 + p10 + p01 + p11), left to right as autograd.avg_pool2
    out[c * no + (int64_t)y * wo + x] = 0.25f * (((p[0][0] + p[1][0]) + p[0][1]) + p[1][1]);
  }
}

__global__ void __launch_bounds__(128) kapply_pool2_kernel(const kw_t* __restrict__ kw, const float* __restrict__ img,
                                                           float* __restrict__ out, int h, int w) {
  fv::pdl_wait();
  const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y;
  if (x >= (w >> 1)) return;
  kapply_pool2_at(kw, img, out, h, w, x, y);
}

// grid (ceil(W/2/128), H): pixels (2x, 2x+1) of row v of the cropped film
__global__ void __launch_bounds__(128) kapply_final2_kernel(const kw_t* __restrict__ kw, const float* __restrict__ img,
                                                            const float* __restrict__ od, int H, int W, int Hp, int Wp,
                                                            float* __restrict__ rgb, float* __restrict__ o_raw,
                                                            float* __restrict__ od_raw) {
  fv::pdl_wait();
  const int x = blockIdx.x * blockDim.x + threadIdx.x, v = blockIdx.y;
  const int u0 = 2 * x;
  if (u0 >= W) return;
  const int64_t pp = (int64_t)Hp * Wp, n = (int64_t)H * W;
  float2 k[9];
#pragma unroll
  for (int j = 0; j < 9; ++j) k[j] = __ldg(reinterpret_cast<const float2*>(kw + j * pp + (int64_t)v * Wp + u0));
  float o[2][3];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    float win[3][4];
    load_win<3>(img + (int64_t)c * pp, Hp, Wp, v, u0, win);
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      float acc = 0.f;
#pragma unroll
      for (int j = 0; j < 9; ++j) acc = acc + (q ? k[j].y : k[j].x) * win[j / 3][q + j % 3];
      o[q][c] = acc;
    }
  }
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int u = u0 + q;
    if (u >= W) break;
    const int64_t i = (int64_t)v * W + u, jp = (int64_t)v * Wp + u;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      if (rgb) rgb[i * 3 + c] = fminf(fmaxf(o[q][c], 0.f), 1.f);
      if (o_raw) o_raw[c * n + i] = o[q][c];
      if (od_raw) od_raw[c * n + i] = od[c * pp + jp];
    }
  }
}

// pngio.to_uint8 (pngio.py:11-12): (clip(x, 0, 1) * 255 + 0.5) truncated, in fp32 without FMA
// contraction like NumPy; input addressed by element strides so HWC (RGB / RGBA) and CHW both work.
__global__ void rgb8_kernel(const float* __restrict__ in, int h, int w, int64_t sy, int64_t sx, int64_t sc,
                            uint8_t* __restrict__ out) {
  const int64_t n = (int64_t)h * w;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
    const int64_t y = p / w, x = p % w;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const float v = fminf(fmaxf(in[y * sy + x * sx + c * sc], 0.f), 1.f);
      out[p * 3 + c] = (uint8_t)__float2uint_rz(__fadd_rn(__fmul_rn(v, 255.f), 0.5f));
    }
  }
}

// 3-channel fp32 avg_pool2; grid (ceil(w/128), h, 3), h, w the OUTPUT dims
__global__ void __launch_bounds__(128) pool3_kernel(const float* __restrict__ in, float* __restrict__ out,
                                                    int h, int w) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y, c = blockIdx.z;
  if (x >= w) return;
  const int W2 = 2 * w;
  const float* p = in + (int64_t)c * 4 * h * w;
  const float2 r0 = *reinterpret_cast<const float2*>(p + (int64_t)(2 * y) * W2 + 2 * x);
  const float2 r1 = *reinterpret_cast<const float2*>(p + (int64_t)(2 * y + 1) * W2 + 2 * x);
  // 0.25 * (p00 + p10 + p01 + p11), left to right as autograd.avg_pool2
  out[(int64_t)c * h * w + (int64_t)y * w + x] = 0.25f * (((r0.x + r1.x) + r0.y) + r1.y);
}

// 3-channel fp32 2x bilinear upsample; grid (ceil(w/128), h, 3), h, w the INPUT dims; one thread
// writes the 2x2 output block of one input pixel
__device__ __forceinline__ void up3_at(const float* __restrict__ in, float* __restrict__ out, int h, int w,
                                       int j, int i, int c) {
  const float* p = in + (int64_t)c * h * w;
  const int rows[3] = {max(i - 1, 0), i, min(i + 1, h - 1)};
  const int cols[3] = {max(j - 1, 0), j, min(j + 1, w - 1)};
  float re[3], ro[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const float a = p[(int64_t)rows[0] * w + cols[k]], b = p[(int64_t)rows[1] * w + cols[k]],
                d = p[(int64_t)rows[2] * w + cols[k]];
    re[k] = 0.25f * a + 0.75f * b;
    ro[k] = 0.75f * b + 0.25f * d;
  }
  float* o = out + (int64_t)c * 4 * h * w;
  const int W2 = 2 * w;
  *reinterpret_cast<float2*>(o + (int64_t)(2 * i) * W2 + 2 * j) =
      make_float2(0.25f * re[0] + 0.75f * re[1], 0.75f * re[1] + 0.25f * re[2]);
  *reinterpret_cast<float2*>(o + (int64_t)(2 * i + 1) * W2 + 2 * j) =
      make_float2(0.25f * ro[0] + 0.75f * ro[1], 0.75f * ro[1] + 0.25f * ro[2]);
}

__global__ void __launch_bounds__(128) up3_kernel(const float* __restrict__ in, float* __restrict__ out,
                                                  int h, int w) {
  fv::pdl_wait();
  const int j = blockIdx.x * blockDim.x + threadIdx.x, i = blockIdx.y, c = blockIdx.z;
  if (j >= w) return;
  up3_at(in, out, h, w, j, i, c);
}

// The K stage between its first and last block (forward_K, network.py:280-293) in ONE cooperative
// launch: the small levels' filter / pool / upsample passes (each a few us of work at L1..L3, but
// a launch and a ramp apiece) run as grid-stride loops separated by grid-wide barriers. Every
// element is computed by the same device function as the separate kernels, so results are identical.
__global__ void __launch_bounds__(128) kchain_kernel(KChain ch) {
  cg::grid_group grid = cg::this_grid();
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nthr = (int64_t)gridDim.x * blockDim.x;
  for (int s = 0; s < ch.n; ++s) {
    const KChainStage st = ch.s[s];
    if (st.op == 0) {
      const int wo = st.w >> 1;
      const int64_t n = (int64_t)(st.h >> 1) * wo;
      for (int64_t i = tid; i < n; i += nthr) kapply_pool2_at(st.kw, st.in, st.out, st.h, st.w, (int)(i % wo), (int)(i / wo));
    } else if (st.op == 1) {
      const int64_t n = (int64_t)st.h * st.w;
      for (int64_t i = tid; i < n; i += nthr) kapply_at(st.kw, st.in, st.out, st.h, st.w, (int)(i % st.w), (int)(i / st.w));
    } else {
      const int64_t hw = (int64_t)st.h * st.w;
      for (int64_t i = tid; i < 3 * hw; i += nthr) {
        const int c = (int)(i / hw);
        const int64_t r = i - c * hw;
        up3_at(st.in, st.out, st.h, st.w, (int)(r % st.w), (int)(r / st.w), c);
      }
    }
    if (s + 1 < ch.n) grid.sync();
  }
}

// x = rgba*m ++ m: group 0 of the input (channels 0..4, film region only; internal.h kInGroups)
__global__ void pack_input_kernel(const float* __restrict__ rgba, const uint8_t* __restrict__ bits,
                                  __half* __restrict__ x, int H, int W, int Wp) {
  const int64_t n = (int64_t)H * W;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int u = (int)(i % W), v = (int)(i / W);
    const float m = bits[i] ? 1.f : 0.f;
    const float4 c = *reinterpret_cast<const float4*>(rgba + i * 4);
    uint4 q;
    __half2* p2 = reinterpret_cast<__half2*>(&q);
    p2[0] = __floats2half2_rn(c.x * m, c.y * m);
    p2[1] = __floats2half2_rn(c.z * m, c.w * m);
    p2[2] = __floats2half2_rn(m, 0.f);
    p2[3] = __floats2half2_rn(0.f, 0.f);
    *reinterpret_cast<uint4*>(x + ((int64_t)v * Wp + u) * 8) = q;  // the whole group-0 pixel
  }
}

// forward_full input: NCHW (C,H,W) fp32 -> channels 0..C-1 of the input's group 0 (C = 4 or 5)
__global__ void set_input_kernel(const float* __restrict__ xin, int C, __half* __restrict__ x, int H,
                                 int W, int Wp) {
  const int64_t n = (int64_t)H * W;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int u = (int)(i % W), v = (int)(i / W);
    uint4 q;
    __half* h = reinterpret_cast<__half*>(&q);
#pragma unroll
    for (int c = 0; c < 8; ++c) h[c] = __float2half_rn(c < C && c < 5 ? xin[c * n + i] : 0.f);
    *reinterpret_cast<uint4*>(x + ((int64_t)v * Wp + u) * 8) = q;
  }
}

// crop (3,Hp,Wp) -> (H,W,3) clipped, (3,H,W) raw O and O_d
__global__ void finalize_kernel(const float* __restrict__ img, const float* __restrict__ od, int H,
                                int W, int Hp, int Wp, float* __restrict__ rgb, float* __restrict__ o_raw,
                                float* __restrict__ od_raw) {
  fv::pdl_wait();
  const int64_t n = (int64_t)H * W;
  const int64_t pp = (int64_t)Hp * Wp;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int u = (int)(i % W), v = (int)(i / W);
    const int64_t j = (int64_t)v * Wp + u;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const float o = img[c * pp + j];
      if (rgb) rgb[i * 3 + c] = fminf(fmaxf(o, 0.f), 1.f);
      if (o_raw) o_raw[c * n + i] = o;
      if (od_raw) od_raw[c * n + i] = od[c * pp + j];
    }
  }
}

// NC8HW8 fp16 -> NCHW fp32
__global__ void nc8_to_nchw_kernel(const __half* __restrict__ in, float* __restrict__ out, int C,
                                   int h, int w) {
  const int64_t n = (int64_t)C * h * w;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = i % ((int64_t)h * w);
    const int c = (int)(i / ((int64_t)h * w));
    out[i] = __half2float(in[(int64_t)(c >> 3) * h * w * 8 + p * 8 + (c & 7)]);
  }
}

// NCHW fp32 -> NC8HW8 fp16
__global__ void nchw_to_nc8_kernel(const float* __restrict__ in, __half* __restrict__ out, int C,
                                   int h, int w) {
  const int64_t n = (int64_t)C * h * w;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = i % ((int64_t)h * w);
    const int c = (int)(i / ((int64_t)h * w));
    out[(int64_t)(c >> 3) * h * w * 8 + p * 8 + (c & 7)] = __float2half_rn(in[i]);
  }
}

// O_d (3,H,W) fp32 -> the input's feedback group [O_d, 0 x 5] (fb = its base)
__global__ void od_to_feedback_kernel(const float* __restrict__ od, __half* __restrict__ fb, int h, int w) {
  const int64_t n = (int64_t)h * w;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint4 q;
    __half2* p2 = reinterpret_cast<__half2*>(&q);
    p2[0] = __floats2half2_rn(od[i], od[n + i]);
    p2[1] = __floats2half2_rn(od[2 * n + i], 0.f);
    q.z = q.w = 0u;
    *reinterpret_cast<uint4*>(fb + i * 8) = q;
  }
}

inline int grid_for(fv_ctx* ctx, int64_t n, int threads = 256) {
  int64_t b = (n + threads - 1) / threads;
  const int64_t cap = (int64_t)ctx->num_sms * 16;
  if (b > cap) b = cap;
  return (int)(b < 1 ? 1 : b);
}

}  // namespace

int upsample2_nc8(fv_ctx* ctx, const fv_act& in, fv_act& out) {
  // input rows per thread (FV_UP_ROWS = 1 / 2 / 4), measured at C3 (L1 -> L0): 74.3 / 66.1 / 69.7 us
  static const int rp = getenv("FV_UP_ROWS") ? atoi(getenv("FV_UP_ROWS")) : 2;
  if (rp == 2 || rp == 4) {
    const dim3 grid((in.W + 127) / 128, (in.H + rp - 1) / rp, in.C / 8);
    FV_TIMED(ctx, FV_KC_NETOPS, fv::launch_pdl(rp == 2 ? upsample2_nc8_rows_kernel<2> : upsample2_nc8_rows_kernel<4>,
                                               grid, 128, 0, ctx->stream, in.p, out.p, in.H, in.W));
    FV_CHECK_LAUNCH("upsample2_nc8_rows_kernel");
    ctx->launches += 1;
    return 0;
  }
  const dim3 grid((in.W + 127) / 128, in.H, in.C / 8);
  FV_TIMED(ctx, FV_KC_NETOPS, fv::launch_pdl(upsample2_nc8_kernel, grid, 128, 0, ctx->stream, in.p, out.p, in.H, in.W));
  FV_CHECK_LAUNCH("upsample2_nc8_kernel");
  ctx->launches += 1;
  return 0;
}

int kapply(fv_ctx* ctx, const kw_t* kw, const float* img, float* out, int h, int w) {
  const dim3 g((w + 127) / 128, h);
  FV_TIMED(ctx, FV_KC_NETOPS, fv::launch_pdl(kapply_kernel, g, 128, 0, ctx->stream, kw, img, out, h, w));
  FV_CHECK_LAUNCH("kapply_kernel");
  ctx->launches += 1;
  return 0;
}

static bool kapply_v1() {  // FV_KAPPLY_V=1: the per-pixel kernels (A/B)
  static const bool v1 = getenv("FV_KAPPLY_V") && atoi(getenv("FV_KAPPLY_V")) == 1;
  return v1;
}

int kapply_pool(fv_ctx* ctx, const kw_t* kw, const float* img, float* out, int h, int w) {
  const dim3 g(((w >> 1) + 127) / 128, h >> 1);
  if (kapply_v1() || (w & 1))
    FV_TIMED(ctx, FV_KC_NETOPS, fv::launch_pdl(kapply_pool_kernel, g, 128, 0, ctx->stream, kw, img, out, h, w));
  else
    FV_TIMED(ctx, FV_KC_NETOPS, fv::launch_pdl(kapply_pool2_kernel, g, 128, 0, ctx->stream, kw, img, out, h, w));
  FV_CHECK_LAUNCH("kapply_pool_kernel");
  ctx->launches += 1;
  return 0;
}

int kapply_final(fv_ctx* ctx, fv_state* st, const kw_t* kw, const float* img, float* rgb, float* o_raw,
                 float* od_raw) {
  if (kapply_v1() || (st->Wp & 1)) {
    const dim3 g((st->W + 127) / 128, st->H);
    FV_TIMED(ctx, FV_KC_NETOPS, fv::launch_pdl(kapply_final_kernel, g, 128, 0, ctx->stream, kw, img, st->od, st->H, st->W, st->Hp,
                                                                            st->Wp, rgb, o_raw, od_raw));
  } else {
    const dim3 g(((st->W + 1) / 2 + 127) / 128, st->H);
    FV_TIMED(ctx, FV_KC_NETOPS, fv::launch_pdl(kapply_final2_kernel, g, 128, 0, ctx->stream, kw, img, st->od, st->H, st->W, st->Hp,
                                                                             st->Wp, rgb, o_raw, od_raw));
  }
  FV_CHECK_LAUNCH("kapply_final_kernel");
  ctx->launches += 1;
  return 0;
}

int pack_rgb8(fv_ctx* ctx, const float* in, int h, int w, int64_t sy, int64_t sx, int64_t sc, uint8_t* out) {
  const int64_t n = (int64_t)h * w;
  FV_TIMED(ctx, FV_KC_NETOPS, rgb8_kernel<<<grid_for(ctx, n), 256, 0, ctx->stream>>>(in, h, w, sy, sx, sc, out));
  FV_CHECK_LAUNCH("rgb8_kernel");
  ctx->launches += 1;
  return 0;
}

int pool3(fv_ctx* ctx, const float* in, float* out, int h_out, int w_out) {
  FV_TIMED(ctx, FV_KC_NETOPS, pool3_kernel<<<dim3((w_out + 127) / 128, h_out, 3), 128, 0, ctx->stream>>>(in, out, h_out, w_out));
  FV_CHECK_LAUNCH("pool3_kernel");
  ctx->launches += 1;
  return 0;
}

int up3(fv_ctx* ctx, const float* in, float* out, int h_in, int w_in) {
  FV_TIMED(ctx, FV_KC_NETOPS, fv::launch_pdl(up3_kernel, dim3((w_in + 127) / 128, h_in, 3), 128, 0, ctx->stream, in, out, h_in, w_in));
  FV_CHECK_LAUNCH("up3_kernel");
  ctx->launches += 1;
  return 0;
}

int kchain(fv_ctx* ctx, const KChain& ch) {
  if (ch.n == 0) return 0;
  static int per_sm = 0;
  if (!per_sm) {
    FV_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kchain_kernel, 128, 0));
    const char* e = getenv("FV_KCHAIN_BPS");  // blocks per SM cap (A/B)
    const int cap = e ? atoi(e) : 4;
    if (per_sm > cap) per_sm = cap;
    if (per_sm < 1) per_sm = 1;
  }
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ctx->num_sms * per_sm);
  cfg.blockDim = dim3(128);
  cfg.stream = ctx->stream;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  FV_TIMED(ctx, FV_KC_NETOPS, cudaLaunchKernelEx(&cfg, kchain_kernel, ch));
  FV_CHECK_LAUNCH("kchain_kernel");
  ctx->launches += 1;
  return 0;
}

// opt-in (FV_KCHAIN=1): measured -1.2% frames/s at C3 against the separate launches replayed from
// the graph (the grid-stride loops with index divisions and 6 grid barriers take 62 us; the ten
// separate launches cost less than that inside the graph)
bool kchain_enabled() {
  static const bool on = getenv("FV_KCHAIN") && atoi(getenv("FV_KCHAIN")) == 1 && !kapply_v1();
  return on;
}

int pack_input(fv_ctx* ctx, fv_state* st, const float* rgba, const uint8_t* bits) {
  const int64_t n = (int64_t)st->H * st->W;
  FV_TIMED(ctx, FV_KC_NETOPS, pack_input_kernel<<<grid_for(ctx, n), 256, 0, ctx->stream>>>(rgba, bits, st->x.p, st->H, st->W, st->Wp));
  FV_CHECK_LAUNCH("pack_input_kernel");
  ctx->launches += 1;
  return 0;
}

int set_input(fv_ctx* ctx, fv_state* st, const float* xin, int C) {
  const int64_t n = (int64_t)st->H * st->W;
  FV_TIMED(ctx, FV_KC_NETOPS, set_input_kernel<<<grid_for(ctx, n), 256, 0, ctx->stream>>>(xin, C, st->x.p, st->H, st->W, st->Wp));
  FV_CHECK_LAUNCH("set_input_kernel");
  ctx->launches += 1;
  return 0;
}

int finalize(fv_ctx* ctx, fv_state* st, const float* img, float* rgb, float* o_raw, float* od_raw) {
  const int64_t n = (int64_t)st->H * st->W;
  FV_TIMED(ctx, FV_KC_NETOPS, fv::launch_pdl(finalize_kernel, grid_for(ctx, n), 256, 0, ctx->stream, img, st->od, st->H, st->W, st->Hp, st->Wp,
                                                              rgb, o_raw, od_raw));
  FV_CHECK_LAUNCH("finalize_kernel");
  ctx->launches += 1;
  return 0;
}

int nc8_to_nchw(fv_ctx* ctx, const fv_act& a, float* out) {
  const int64_t n = (int64_t)a.C * a.H * a.W;
  FV_TIMED(ctx, FV_KC_NETOPS, nc8_to_nchw_kernel<<<grid_for(ctx, n), 256, 0, ctx->stream>>>(a.p, out, a.C, a.H, a.W));
  FV_CHECK_LAUNCH("nc8_to_nchw_kernel");
  ctx->launches += 1;
  return 0;
}

int nchw_to_nc8(fv_ctx* ctx, const float* in, fv_act& a) {
  const int64_t n = (int64_t)a.C * a.H * a.W;
  FV_TIMED(ctx, FV_KC_NETOPS, nchw_to_nc8_kernel<<<grid_for(ctx, n), 256, 0, ctx->stream>>>(in, a.p, a.C, a.H, a.W));
  FV_CHECK_LAUNCH("nchw_to_nc8_kernel");
  ctx->launches += 1;
  return 0;
}

// predict_kernel_fields' 1x1 conv for one block in fp32 (a checking/API path, not the hot path:
// the hot path computes these logits on the tensor cores inside the K-stage conv epilogue)
__global__ void kfield_logits_kernel(const float* __restrict__ w, const float* __restrict__ b,
                                     const float* __restrict__ hd, int C, int64_t n, int normalize,
                                     float* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    float acc[9];
#pragma unroll
    for (int j = 0; j < 9; ++j) acc[j] = 0.f;
    for (int c = 0; c < C; ++c) {
      const float v = hd[(int64_t)c * n + i];
#pragma unroll
      for (int j = 0; j < 9; ++j) acc[j] = fmaf(w[j * C + c], v, acc[j]);
    }
#pragma unroll
    for (int j = 0; j < 9; ++j) acc[j] += b[j];
    if (normalize) {  // softmax_channels (autograd.py:188-199): max-subtracted, then normalised
      float m = acc[0];
#pragma unroll
      for (int j = 1; j < 9; ++j) m = fmaxf(m, acc[j]);
      float sum = 0.f;
#pragma unroll
      for (int j = 0; j < 9; ++j) {
        acc[j] = expf(acc[j] - m);
        sum += acc[j];
      }
#pragma unroll
      for (int j = 0; j < 9; ++j) acc[j] /= sum;
    }
#pragma unroll
    for (int j = 0; j < 9; ++j) out[(int64_t)j * n + i] = acc[j];
  }
}

int kfield_logits(fv_ctx* ctx, const float* w_host, const float* b_host, const float* hd, int C, int h, int w,
                  int normalize, float* out) {
  const int64_t n = (int64_t)h * w;
  float* wb = nullptr;
  FV_CUDA(cudaMallocAsync(&wb, sizeof(float) * (9 * C + 9), ctx->stream));
  FV_CUDA(cudaMemcpyAsync(wb, w_host, sizeof(float) * 9 * C, cudaMemcpyHostToDevice, ctx->stream));
  FV_CUDA(cudaMemcpyAsync(wb + 9 * C, b_host, sizeof(float) * 9, cudaMemcpyHostToDevice, ctx->stream));
  kfield_logits_kernel<<<grid_for(ctx, n), 256, 0, ctx->stream>>>(wb, wb + 9 * C, hd, C, n, normalize, out);
  FV_CHECK_LAUNCH("kfield_logits_kernel");
  ctx->launches += 1;
  FV_CUDA(cudaFreeAsync(wb, ctx->stream));
  FV_CUDA(cudaStreamSynchronize(ctx->stream));  // the host weight pointers are borrowed for the call
  return 0;
}

int od_to_feedback(fv_ctx* ctx, fv_state* st) {
  const int64_t n = (int64_t)st->Hp * st->Wp;
  FV_TIMED(ctx, FV_KC_NETOPS, od_to_feedback_kernel<<<grid_for(ctx, n), 256, 0, ctx->stream>>>(st->od, feedback_plane(st->x), st->Hp, st->Wp));
  FV_CHECK_LAUNCH("od_to_feedback_kernel");
  ctx->launches += 1;
  return 0;
}

}  // namespace fv
