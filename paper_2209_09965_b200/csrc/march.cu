// Sparse / dense ray marcher over a device-resident scalar grid.
//
// Reference semantics (pkg/src/fovray):
//   generate_rays        volume.py:293-303   (pinhole through pixel centres, v down)
//   _ray_box             renderer.py:88-98   (slab test on [0, ext])
//   sample_trilinear     volume.py:149-180   (q = p/spacing - 0.5, clipped i0/i1, 0 outside)
//   TransferFunction     volume.py:201-208   (clip, x = s*(K-1), clipped i0, linear lerp)
//   _march               renderer.py:150-195 (front-to-back, 1-(1-a)^(dt/ref), depth at A>=0.5,
//                                             stop at t >= t_end-1e-12 or A >= early_term_alpha)
//   shadow_transmittance renderer.py:109-147 (march toward the light at step*factor, exit at
//                                             T <= shadow_min_transmittance)
//   render_sparse_compact renderer.py:262-288 (one work item per compacted pixel)
//
// Step control (t, dt, mid and the world position of every sample) always runs in fp64, so the
// sequence of sample points and the termination tests on t are the reference's. The per-sample
// arithmetic (trilinear lerps, transfer function, compositing) runs in `Real`: float for the
// default fast path, double for the exact tier. One thread marches one compacted ray; its
// shadow rays are marched inline. The TF LUT lives in shared memory.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "internal.h"

namespace fv {

namespace {

struct MarchParams {
  // camera
  double pos[3], right[3], up[3], fwd[3];
  double tan_half, aspect;
  int W, H;
  // volume
  const float* data;
  int nx, ny, nz;
  double sp[3], ext[3];
  int K;
  const float* lut;
  // light
  int light_kind;
  double lvec[3];   // directional: unit direction toward the light; point: light position
  double intensity[3];
  // settings
  double step, ref, step_sh, early, ambient, min_trans;
  double bg[4];
  // work
  const int32_t* idx;
  const int32_t* k_dev;
  int k_max;
  float* rgba;
  float* depth;
  __half* net_in;
  int net_wp;
  DevCounters* counters;
  const FrameDyn* dyn;  // non-null: the camera basis comes from device memory (graph replay)
};

// The camera of a ray-generating kernel: the launch's by-value basis, or the FrameDyn block.
struct CamView {
  double pos[3], right[3], up[3], fwd[3], tan_half, aspect;
};
__device__ __forceinline__ CamView load_cam(const MarchParams& P) {
  CamView c;
  if (P.dyn) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      c.pos[a] = P.dyn->pos[a]; c.right[a] = P.dyn->right[a]; c.up[a] = P.dyn->up[a]; c.fwd[a] = P.dyn->fwd[a];
    }
    c.tan_half = P.dyn->tan_half;
    c.aspect = P.dyn->aspect;
  } else {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      c.pos[a] = P.pos[a]; c.right[a] = P.right[a]; c.up[a] = P.up[a]; c.fwd[a] = P.fwd[a];
    }
    c.tan_half = P.tan_half;
    c.aspect = P.aspect;
  }
  return c;
}

__device__ __forceinline__ void ray_box(const double o[3], const double d[3], const double ext[3],
                                        double& t0, double& t1, bool& hit) {
  double tmin = -INFINITY, tmax = INFINITY;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    double da = d[a];
    if (fabs(da) < 1e-30) da = da < 0.0 ? -1e-30 : 1e-30;
    const double inv = 1.0 / da;
    const double ta = (0.0 - o[a]) * inv;
    const double tb = (ext[a] - o[a]) * inv;
    tmin = fmax(tmin, fmin(ta, tb));
    tmax = fmin(tmax, fmax(ta, tb));
  }
  t0 = fmax(tmin, 0.0);
  t1 = tmax;
  hit = tmax > t0;
}

template <typename Real>
__device__ __forceinline__ Real trilinear(const MarchParams& P, const double p[3]) {
  if (!(p[0] >= 0.0 && p[0] <= P.ext[0] && p[1] >= 0.0 && p[1] <= P.ext[1] && p[2] >= 0.0 &&
        p[2] <= P.ext[2]))
    return Real(0);
  const double qx = p[0] / P.sp[0] - 0.5, qy = p[1] / P.sp[1] - 0.5, qz = p[2] / P.sp[2] - 0.5;
  const double fx = floor(qx), fy = floor(qy), fz = floor(qz);
  const Real tx = (Real)(qx - fx), ty = (Real)(qy - fy), tz = (Real)(qz - fz);
  const int x0 = min(max((int)fx, 0), P.nx - 1), y0 = min(max((int)fy, 0), P.ny - 1),
            z0 = min(max((int)fz, 0), P.nz - 1);
  const int x1 = min(x0 + 1, P.nx - 1), y1 = min(y0 + 1, P.ny - 1), z1 = min(z0 + 1, P.nz - 1);
  const int64_t sy = P.nx, sz = (int64_t)P.nx * P.ny;
  const float* d = P.data;
  const Real d000 = __ldg(d + z0 * sz + y0 * sy + x0), d001 = __ldg(d + z0 * sz + y0 * sy + x1);
  const Real d010 = __ldg(d + z0 * sz + y1 * sy + x0), d011 = __ldg(d + z0 * sz + y1 * sy + x1);
  const Real d100 = __ldg(d + z1 * sz + y0 * sy + x0), d101 = __ldg(d + z1 * sz + y0 * sy + x1);
  const Real d110 = __ldg(d + z1 * sz + y1 * sy + x0), d111 = __ldg(d + z1 * sz + y1 * sy + x1);
  const Real one = Real(1);
  const Real c00 = d000 * (one - tx) + d001 * tx;
  const Real c10 = d010 * (one - tx) + d011 * tx;
  const Real c01 = d100 * (one - tx) + d101 * tx;
  const Real c11 = d110 * (one - tx) + d111 * tx;
  const Real c0 = c00 * (one - ty) + c10 * ty;
  const Real c1 = c01 * (one - ty) + c11 * ty;
  return c0 * (one - tz) + c1 * tz;
}

__device__ __forceinline__ int ifloor(float x) { return (int)floorf(x); }
__device__ __forceinline__ int ifloor(double x) { return (int)floor(x); }

template <typename Real>
__device__ __forceinline__ void tf_apply(const float* lut, int K, Real s, Real out[4]) {
  s = s < Real(0) ? Real(0) : (s > Real(1) ? Real(1) : s);
  const Real x = s * (Real)(K - 1);
  int i0 = ifloor(x);
  i0 = min(max(i0, 0), K - 2);
  const Real t = x - (Real)i0;
#pragma unroll
  for (int c = 0; c < 4; ++c)
    out[c] = (Real)lut[i0 * 4 + c] * (Real(1) - t) + (Real)lut[(i0 + 1) * 4 + c] * t;
}

template <typename Real>
__device__ __forceinline__ Real tf_alpha(const float* lut, int K, Real s) {
  s = s < Real(0) ? Real(0) : (s > Real(1) ? Real(1) : s);
  const Real x = s * (Real)(K - 1);
  int i0 = ifloor(x);
  i0 = min(max(i0, 0), K - 2);
  const Real t = x - (Real)i0;
  return (Real)lut[i0 * 4 + 3] * (Real(1) - t) + (Real)lut[(i0 + 1) * 4 + 3] * t;
}

// (1-a)^(dt/ref) with the exponents that occur on full steps special-cased.
template <typename Real>
__device__ __forceinline__ Real keep_fraction(Real one_minus_a, double e) {
  if (e == 0.5) return sqrt(one_minus_a);
  if (e == 2.0) return one_minus_a * one_minus_a;
  if (e == 1.0) return one_minus_a;
  return (Real)pow((double)one_minus_a, e);
}
template <>
__device__ __forceinline__ float keep_fraction<float>(float one_minus_a, double e) {
  if (e == 0.5) return sqrtf(one_minus_a);
  if (e == 2.0) return one_minus_a * one_minus_a;
  if (e == 1.0) return one_minus_a;
  return powf(one_minus_a, (float)e);
}

template <typename Real>
__device__ Real shadow_T(const MarchParams& P, const float* lut, const double pt[3],
                         unsigned int& nsamp) {
  double dir[3], dist = INFINITY;
  if (P.light_kind == FV_LIGHT_DIRECTIONAL) {
    dir[0] = P.lvec[0]; dir[1] = P.lvec[1]; dir[2] = P.lvec[2];
  } else {
    const double dx = P.lvec[0] - pt[0], dy = P.lvec[1] - pt[1], dz = P.lvec[2] - pt[2];
    dist = sqrt(dx * dx + dy * dy + dz * dz);
    const double m = fmax(dist, 1e-30);
    dir[0] = dx / m; dir[1] = dy / m; dir[2] = dz / m;
  }
  double t0, t1;
  bool hit;
  ray_box(pt, dir, P.ext, t0, t1, hit);
  const double t_end = fmin(t1, dist);
  Real trans = Real(1);
  if (!(hit && t_end > t0)) return trans;
  double t = t0;
  const Real mt = (Real)P.min_trans;
  while (true) {
    const double dt = fmin(P.step_sh, t_end - t);
    const double mid = t + 0.5 * dt;
    const double p[3] = {pt[0] + dir[0] * mid, pt[1] + dir[1] * mid, pt[2] + dir[2] * mid};
    const Real a = tf_alpha<Real>(lut, P.K, trilinear<Real>(P, p));
    const Real a_step = Real(1) - keep_fraction<Real>(Real(1) - a, dt / P.ref);
    trans = trans * (Real(1) - a_step);
    ++nsamp;
    t = t + dt;
    if (!(t < t_end - 1e-12) || !(trans > mt)) break;
  }
  return trans;
}

template <typename Real>
__global__ void __launch_bounds__(128) march_kernel(MarchParams P) {
  __shared__ float lut[4 * 256];
  for (int i = threadIdx.x; i < 4 * P.K; i += blockDim.x) lut[i] = P.lut[i];
  __syncthreads();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int k = P.k_dev ? *P.k_dev : P.k_max;
  unsigned int n_main = 0, n_shadow = 0, hitc = 0;
  // naive renderer lists idle lanes of occupied chunks as -(pix+1): out[~active] = 0 (renderer.py:195-197)
  const int raw = (i < k) ? (P.idx ? P.idx[i] : i) : 0;
  if (i < k && raw < 0) {
    const int q = -raw - 1;
    if (P.rgba) *reinterpret_cast<float4*>(P.rgba + (int64_t)q * 4) = make_float4(0.f, 0.f, 0.f, 0.f);
    if (P.depth) P.depth[q] = 0.f;
  }
  if (i < k && raw >= 0) {
    const int pix = raw;
    const int u = pix % P.W, v = pix / P.W;
    // generate_rays (volume.py:293-303)
    const double sx = (((double)u + 0.5) / P.W * 2.0 - 1.0) * P.tan_half * P.aspect;
    const double sy = (1.0 - ((double)v + 0.5) / P.H * 2.0) * P.tan_half;
    double d[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) d[a] = P.fwd[a] + sx * P.right[a] + sy * P.up[a];
    const double nrm = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
    d[0] /= nrm; d[1] /= nrm; d[2] /= nrm;
    double t0, t_end;
    bool hit;
    ray_box(P.pos, d, P.ext, t0, t_end, hit);
    Real rgb[3] = {Real(0), Real(0), Real(0)};
    Real trans = Real(1);
    double depth = 0.0;
    const bool lit = P.light_kind != FV_LIGHT_NONE;
    const Real amb = lit ? (Real)P.ambient : Real(1);
    const Real I[3] = {(Real)P.intensity[0], (Real)P.intensity[1], (Real)P.intensity[2]};
    const Real early = (Real)P.early;
    if (hit) {
      hitc = 1;
      double t = t0;
      while (true) {
        const double dt = fmin(P.step, t_end - t);
        const double mid = t + 0.5 * dt;
        const double p[3] = {P.pos[0] + d[0] * mid, P.pos[1] + d[1] * mid, P.pos[2] + d[2] * mid};
        Real c[4];
        tf_apply<Real>(lut, P.K, trilinear<Real>(P, p), c);
        ++n_main;
        const Real a_step = Real(1) - keep_fraction<Real>(Real(1) - c[3], dt / P.ref);
        Real shade = Real(1);
        if (lit && a_step > Real(0)) {
          const Real ts = shadow_T<Real>(P, lut, p, n_shadow);
          shade = amb + (Real(1) - amb) * ts;
        }
        const Real contrib = trans * a_step;
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) rgb[ch] += contrib * (c[ch] * (shade * I[ch]));
        trans = trans * (Real(1) - a_step);
        const Real acc = Real(1) - trans;
        if (depth == 0.0 && acc >= Real(0.5)) depth = mid;
        t = t + dt;
        if (!(t < t_end - 1e-12) || !(acc < early)) break;
      }
    }
    const Real bga = (Real)P.bg[3];
    float out[4];
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) out[ch] = (float)(rgb[ch] + (trans * bga) * (Real)P.bg[ch]);
    out[3] = (float)((Real(1) - trans) + trans * bga);
    if (P.rgba)
      *reinterpret_cast<float4*>(P.rgba + (int64_t)pix * 4) = make_float4(out[0], out[1], out[2], out[3]);
    if (P.depth) P.depth[pix] = (float)depth;
    if (P.net_in) {
      __half2* px = reinterpret_cast<__half2*>(P.net_in + ((int64_t)v * P.net_wp + u) * 8);
      px[0] = __floats2half2_rn(out[0], out[1]);
      px[1] = __floats2half2_rn(out[2], out[3]);
    }
  }
  // counters: warp reduce, one atomic per warp
  unsigned int r = (i < k && raw >= 0) ? 1u : 0u;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    r += __shfl_xor_sync(0xffffffffu, r, o);
    hitc += __shfl_xor_sync(0xffffffffu, hitc, o);
    n_main += __shfl_xor_sync(0xffffffffu, n_main, o);
    n_shadow += __shfl_xor_sync(0xffffffffu, n_shadow, o);
  }
  if ((threadIdx.x & 31) == 0 && r) {
    atomicAdd(&P.counters->rays, (unsigned long long)r);
    atomicAdd(&P.counters->hit_rays, (unsigned long long)hitc);
    atomicAdd(&P.counters->samples_main, (unsigned long long)n_main);
    atomicAdd(&P.counters->samples_shadow, (unsigned long long)n_shadow);
  }
}

// ---------------------------------------------------------------------------------------------
// Fast tier: fp32 inner loops over a bricked copy of the volume.
//
// Per ray the setup (direction, slab test, entry point, main-step count) is fp64; the samples are
// then generated as p = entry + d * (i*step + dt/2) in fp32 (<=1e-4 voxel from the reference's
// fp64 positions) and the trilinear weights, TF and compositing run in fp32.
//
// Volume layout for the fast tier ("quads"): every voxel (x,y,z) stores the float4
//   (v[z][y][x], v[z][y][x1], v[z][y1][x], v[z][y1][x1]),  x1 = min(x+1,nx-1), y1 = min(y+1,ny-1)
// -- the reference's clamped neighbours (volume.py:167-168) -- so the 8 trilinear corners are two
// 16-byte loads (planes z0 and z1) instead of eight scalar gathers; that cuts the L1 wavefronts
// per sample 4x, which is what bounds a gather-heavy marcher (ncu: L1/TEX 67% busy, DRAM idle).
// Quads are stored in 8x8x8 bricks (8 KB, z-y-x inside a brick) so consecutive samples of a ray
// in any direction -- shadow rays run diagonally toward the light -- stay in the same lines.
struct FastVol {
  cudaTextureObject_t tex;  // non-zero: fetch quads from the 3D texture (unnormalised, point, clamp)
  cudaTextureObject_t ltex;  // non-zero: the shadow pass samples the hardware-filtered scalar texture
  const float4* quads;
  int nx, ny, nz;
  int sby, sbz;        // brick strides (quads) in y and z
  float ext[3];
  float inv_sp[3];
  float qmax[3];       // n - 0.5
};

// Morton order inside a brick: a 128-byte line holds a 2x2x2 block of quads, so a step in any
// direction (and the z0/z1 pair of one sample) usually stays in the same line.
// (Measured: the Morton order costs ~10 ALU ops per sample and the shadow pass is ALU-bound,
// so the default is z-y-x inside a brick; FV_BRICK_MORTON=1 restores the Morton layout.)
#ifndef FV_BRICK_MORTON
#define FV_BRICK_MORTON 0
#endif
__host__ __device__ __forceinline__ int spread3(int v) { return (v & 1) | ((v & 2) << 2) | ((v & 4) << 4); }
__host__ __device__ __forceinline__ int morton_xy(int x, int y) {
  return FV_BRICK_MORTON ? (spread3(x) | (spread3(y) << 1)) : (x | (y << 3));
}
__host__ __device__ __forceinline__ int morton_z(int z) { return FV_BRICK_MORTON ? (spread3(z) << 2) : (z << 6); }

// Texel coordinate offset of the point-sampled quad texture: texel i is returned for any coordinate
// in [i, i+1); floor(q) is an exact integer, so it addresses texel floor(q) itself (no +0.5 add).
#ifndef FV_TEX_OFF
#define FV_TEX_OFF 0.0f
#endif
constexpr float kTexOff = FV_TEX_OFF;

// Two-phase trilinear: tri_issue computes the weights and issues both loads, tri_finish blends.
struct TriFetch {
  float4 A, B;
  float tx, ty, tz;
  bool inside;
};

// Hardware-filtered sample (TEX == 2, the fast tier): trilinear at q + 1/2 from the scalar texture;
// q < 0 (the lower half-voxel shell) maps to q + 1, which addresses the reference's texels 0, 1
// with its weight q + 1 (see volume_ltex).
__device__ __forceinline__ float tex_lin(const FastVol& V, float qx, float qy, float qz) {
  return tex3D<float>(V.ltex, qx + (qx < 0.f ? 1.5f : 0.5f), qy + (qy < 0.f ? 1.5f : 0.5f),
                      qz + (qz < 0.f ? 1.5f : 0.5f));
}

// Same, from continuous voxel coordinates q = p/spacing - 0.5 (rays stepped directly in q-space;
// p in [0, ext] <=> q in [-0.5, n-0.5]).
template <int TEX = 0>
__device__ __forceinline__ TriFetch tri_issue_q(const FastVol& V, float qx, float qy, float qz) {
  TriFetch f;
  f.inside = qx >= -0.5f && qx <= V.qmax[0] && qy >= -0.5f && qy <= V.qmax[1] && qz >= -0.5f &&
             qz <= V.qmax[2];
  if constexpr (TEX == 2) {
    f.A.x = tex_lin(V, qx, qy, qz);
    return f;
  }
  const float fx = floorf(qx), fy = floorf(qy), fz = floorf(qz);
  f.tx = qx - fx; f.ty = qy - fy; f.tz = qz - fz;
  if constexpr (TEX) {
    // texel (i, j, k) is sampled at (i + .5, j + .5, k + .5); clamp addressing = the reference's
    // clamped i0; the second plane is clamp(max(floor, 0) + 1) as the reference's i1
    if constexpr (kTexOff == 0.f) {
      f.A = tex3D<float4>(V.tex, fx, fy, fz);
      f.B = tex3D<float4>(V.tex, fx, fy, fmaxf(fz, 0.f) + 1.f);
    } else {
      f.A = tex3D<float4>(V.tex, fx + kTexOff, fy + kTexOff, fz + kTexOff);
      f.B = tex3D<float4>(V.tex, fx + kTexOff, fy + kTexOff, fmaxf(fz, 0.f) + (1.f + kTexOff));
    }
    return f;
  }
  const int x0 = min(max((int)fx, 0), V.nx - 1), y0 = min(max((int)fy, 0), V.ny - 1),
            z0 = min(max((int)fz, 0), V.nz - 1);
  const int z1 = min(z0 + 1, V.nz - 1);
  const int xy = (y0 >> 3) * V.sby + ((x0 >> 3) << 9) + morton_xy(x0 & 7, y0 & 7);
  f.A = __ldg(V.quads + xy + (z0 >> 3) * V.sbz + morton_z(z0 & 7));
  f.B = __ldg(V.quads + xy + (z1 >> 3) * V.sbz + morton_z(z1 & 7));
  return f;
}

template <int TEX = 0>
__device__ __forceinline__ TriFetch tri_issue(const FastVol& V, float px, float py, float pz) {
  TriFetch f;
  f.inside = px >= 0.f && px <= V.ext[0] && py >= 0.f && py <= V.ext[1] && pz >= 0.f && pz <= V.ext[2];
  const float qx = px * V.inv_sp[0] - 0.5f, qy = py * V.inv_sp[1] - 0.5f, qz = pz * V.inv_sp[2] - 0.5f;
  if constexpr (TEX == 2) {
    f.A.x = tex_lin(V, qx, qy, qz);
    return f;
  }
  const float fx = floorf(qx), fy = floorf(qy), fz = floorf(qz);
  f.tx = qx - fx; f.ty = qy - fy; f.tz = qz - fz;
  if constexpr (TEX) {
    if constexpr (kTexOff == 0.f) {
      f.A = tex3D<float4>(V.tex, fx, fy, fz);
      f.B = tex3D<float4>(V.tex, fx, fy, fmaxf(fz, 0.f) + 1.f);
    } else {
      f.A = tex3D<float4>(V.tex, fx + kTexOff, fy + kTexOff, fz + kTexOff);
      f.B = tex3D<float4>(V.tex, fx + kTexOff, fy + kTexOff, fmaxf(fz, 0.f) + (1.f + kTexOff));
    }
    return f;
  }
  const int x0 = min(max((int)fx, 0), V.nx - 1), y0 = min(max((int)fy, 0), V.ny - 1),
            z0 = min(max((int)fz, 0), V.nz - 1);
  const int z1 = min(z0 + 1, V.nz - 1);
  const int xy = (y0 >> 3) * V.sby + ((x0 >> 3) << 9) + morton_xy(x0 & 7, y0 & 7);
  f.A = __ldg(V.quads + xy + (z0 >> 3) * V.sbz + morton_z(z0 & 7));
  f.B = __ldg(V.quads + xy + (z1 >> 3) * V.sbz + morton_z(z1 & 7));
  return f;
}

__device__ __forceinline__ float tri_finish(const TriFetch& f) {
  if (!f.inside) return 0.f;
  const float tx = f.tx, ty = f.ty, tz = f.tz;
  const float c00 = f.A.x * (1.f - tx) + f.A.y * tx;
  const float c10 = f.A.z * (1.f - tx) + f.A.w * tx;
  const float c01 = f.B.x * (1.f - tx) + f.B.y * tx;
  const float c11 = f.B.z * (1.f - tx) + f.B.w * tx;
  const float c0 = c00 * (1.f - ty) + c10 * ty;
  const float c1 = c01 * (1.f - ty) + c11 * ty;
  return c0 * (1.f - tz) + c1 * tz;
}

// texture quads hold (v00, v01 - v00, v10, v11 - v10) per plane
template <int TEX>
__device__ __forceinline__ float tri_finish_t(const TriFetch& f) {
  if constexpr (!TEX) {
    return tri_finish(f);
  } else if constexpr (TEX == 2) {
    return f.inside ? f.A.x : 0.f;
  } else {
    if (!f.inside) return 0.f;
    const float c00 = fmaf(f.tx, f.A.y, f.A.x), c10 = fmaf(f.tx, f.A.w, f.A.z);
    const float c01 = fmaf(f.tx, f.B.y, f.B.x), c11 = fmaf(f.tx, f.B.w, f.B.z);
    const float c0 = fmaf(f.ty, c10 - c00, c00), c1 = fmaf(f.ty, c11 - c01, c01);
    return fmaf(f.tz, c1 - c0, c0);
  }
}

__device__ __forceinline__ float tri_fast(const FastVol& V, float px, float py, float pz) {
  if (!(px >= 0.f && px <= V.ext[0] && py >= 0.f && py <= V.ext[1] && pz >= 0.f && pz <= V.ext[2]))
    return 0.f;
  const float qx = px * V.inv_sp[0] - 0.5f, qy = py * V.inv_sp[1] - 0.5f, qz = pz * V.inv_sp[2] - 0.5f;
  const float fx = floorf(qx), fy = floorf(qy), fz = floorf(qz);
  const float tx = qx - fx, ty = qy - fy, tz = qz - fz;
  const int x0 = min(max((int)fx, 0), V.nx - 1), y0 = min(max((int)fy, 0), V.ny - 1),
            z0 = min(max((int)fz, 0), V.nz - 1);
  const int z1 = min(z0 + 1, V.nz - 1);
  const int xy = (y0 >> 3) * V.sby + ((x0 >> 3) << 9) + morton_xy(x0 & 7, y0 & 7);
  const float4 A = __ldg(V.quads + xy + (z0 >> 3) * V.sbz + morton_z(z0 & 7));
  const float4 B = __ldg(V.quads + xy + (z1 >> 3) * V.sbz + morton_z(z1 & 7));
  const float c00 = A.x * (1.f - tx) + A.y * tx;
  const float c10 = A.z * (1.f - tx) + A.w * tx;
  const float c01 = B.x * (1.f - tx) + B.y * tx;
  const float c11 = B.z * (1.f - tx) + B.w * tx;
  const float c0 = c00 * (1.f - ty) + c10 * ty;
  const float c1 = c01 * (1.f - ty) + c11 * ty;
  return c0 * (1.f - tz) + c1 * tz;
}

// (1-a)^(dt/ref) of a ray's last, partial step (and of unusual full-step exponents). Not inlined:
// the call forces a real branch -- inlined, the compiler evaluated powf for every sample and
// selected (ncu: 26% of the shadow pass's instructions on that line).
__device__ __noinline__ float keep_partial(float x, float e) { return powf(x, e); }

// exponent classes of (1-a)^(dt/ref) on full steps: 0 sqrt, 1 identity, 2 square, 3 general
__device__ __forceinline__ float keep_cls(float x, int cls, float e) {
  if (cls == 0) return sqrtf(x);
  if (cls == 1) return x;
  if (cls == 2) return x * x;
  return keep_partial(x, e);
}

struct FastParams {
  MarchParams P;
  FastVol V;
  float ld[3], ld_inv[3];  // directional light: unit direction toward the light (+ guarded inverse)
  float lpos[3];
  int cls_main, cls_sh;
  float e_main, e_sh, inv_ref;
  // shadow pass (directional light): q-space step toward the light, fp32 copies of the settings
  float qs_sh[3];
  float step_sh, inv_step_sh, min_trans, ambient;
};

template <int TEX = 0>
__device__ float shadow_fast(const FastParams& F, const float* lut, float px, float py, float pz,
                             unsigned int& nsamp) {
  const MarchParams& P = F.P;
  float dir[3], inv[3], dist = INFINITY;
  if (P.light_kind == FV_LIGHT_DIRECTIONAL) {
#pragma unroll
    for (int a = 0; a < 3; ++a) { dir[a] = F.ld[a]; inv[a] = F.ld_inv[a]; }
  } else {
    const float dx = F.lpos[0] - px, dy = F.lpos[1] - py, dz = F.lpos[2] - pz;
    dist = sqrtf(dx * dx + dy * dy + dz * dz);
    const float m = fmaxf(dist, 1e-30f);
    dir[0] = dx / m; dir[1] = dy / m; dir[2] = dz / m;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      float s = dir[a];
      if (fabsf(s) < 1e-30f) s = s < 0.f ? -1e-30f : 1e-30f;
      inv[a] = 1.f / s;
    }
  }
  const float p[3] = {px, py, pz};
  float tmin = -INFINITY, tmax = INFINITY;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const float ta = (0.f - p[a]) * inv[a], tb = (F.V.ext[a] - p[a]) * inv[a];
    tmin = fmaxf(tmin, fminf(ta, tb));
    tmax = fminf(tmax, fmaxf(ta, tb));
  }
  const float t0 = fmaxf(tmin, 0.f);
  const float tend = fminf(tmax, dist);
  float trans = 1.f;
  if (!(tmax > t0 && tend > t0)) return trans;
  const float step = (float)P.step_sh, mt = (float)P.min_trans;
  // The sample positions do not depend on the data, so kShadowU samples are addressed and their
  // loads issued before any of them is consumed: one lane keeps 2*kShadowU 16-byte loads in
  // flight. That shortens the longest rays, whose serial chains of L2 round trips otherwise set
  // the kernel's tail. Samples past the exit are discarded, so results are unchanged.
  constexpr int kShadowU = 4;
  // step in voxel coordinates: q(mid) = q0 + qd * mid
  const float q0x = px * F.V.inv_sp[0] - 0.5f, q0y = py * F.V.inv_sp[1] - 0.5f, q0z = pz * F.V.inv_sp[2] - 0.5f;
  const float qdx = dir[0] * F.V.inv_sp[0], qdy = dir[1] * F.V.inv_sp[1], qdz = dir[2] * F.V.inv_sp[2];
  float t = t0;
#pragma unroll 1
  while (true) {
    TriFetch f[kShadowU];
    float dts[kShadowU];
    float tj = t;
#pragma unroll
    for (int j = 0; j < kShadowU; ++j) {
      const float dt = fminf(step, tend - tj);
      const float mid = tj + 0.5f * dt;
      dts[j] = dt;
      f[j] = tri_issue_q<TEX>(F.V, q0x + qdx * mid, q0y + qdy * mid, q0z + qdz * mid);
      tj = tj + dt;
    }
    bool stop = false;
#pragma unroll
    for (int j = 0; j < kShadowU; ++j) {
      const float dt = dts[j];
      const float a = tf_alpha<float>(lut, P.K, tri_finish_t<TEX>(f[j]));
      const float keep = dt == step ? keep_cls(1.f - a, F.cls_sh, F.e_sh) : keep_partial(1.f - a, dt * F.inv_ref);
      trans = trans * (1.f - (1.f - keep));
      ++nsamp;
      t = t + dt;
      if (!(t < tend) || !(trans > mt)) { stop = true; break; }
    }
    if (stop) break;
  }
  return trans;
}

// ---- shadow pass fast path ---------------------------------------------------------------------
// The wavefront shadow pass is issue-bound (ncu: 78% issue slots, ~140 instructions per sample), so
// its per-sample path is specialised: the full-step exponent class is a template parameter (no
// per-sample switch), lerps are single FMAs, and the TF alpha comes from a (a_i, a_{i+1} - a_i)
// float2 table in shared memory (one LDS.64). All fp32-tier rounding changes (~1e-7).
__device__ __forceinline__ float lerp_fma(float a, float b, float t) { return fmaf(t, b - a, a); }

__device__ __forceinline__ float tri_finish_fma(const TriFetch& f) {
  if (!f.inside) return 0.f;
  const float c00 = lerp_fma(f.A.x, f.A.y, f.tx), c10 = lerp_fma(f.A.z, f.A.w, f.tx);
  const float c01 = lerp_fma(f.B.x, f.B.y, f.tx), c11 = lerp_fma(f.B.z, f.B.w, f.tx);
  return lerp_fma(lerp_fma(c00, c10, f.ty), lerp_fma(c01, c11, f.ty), f.tz);
}

// alpha LUT: lut2[i] = (a_i, a_{i+1} - a_i), i < K-1
__device__ __forceinline__ float tf_alpha2(const float2* lut2, int K, float s) {
  s = fminf(fmaxf(s, 0.f), 1.f);
  const float x = s * (float)(K - 1);
  const int i0 = min((int)x, K - 2);  // x >= 0: truncation == floor
  const float2 v = lut2[i0];
  return fmaf(x - (float)i0, v.y, v.x);
}

template <int CLS>
__device__ __forceinline__ float keep_t(float x, float e) {
  if constexpr (CLS == 0) return sqrtf(x);
  else if constexpr (CLS == 1) return x;
  else if constexpr (CLS == 2) return x * x;
  else return keep_partial(x, e);
}

template <int CLS, int TEX>
__device__ float shadow_fast_t(const FastParams& F, const float2* lut2, float px, float py, float pz,
                               unsigned int& nsamp) {
  const MarchParams& P = F.P;
  float dir[3], inv[3], dist = INFINITY;
  if (P.light_kind == FV_LIGHT_DIRECTIONAL) {
#pragma unroll
    for (int a = 0; a < 3; ++a) { dir[a] = F.ld[a]; inv[a] = F.ld_inv[a]; }
  } else {
    const float dx = F.lpos[0] - px, dy = F.lpos[1] - py, dz = F.lpos[2] - pz;
    dist = sqrtf(dx * dx + dy * dy + dz * dz);
    const float m = fmaxf(dist, 1e-30f);
    dir[0] = dx / m; dir[1] = dy / m; dir[2] = dz / m;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      float s = dir[a];
      if (fabsf(s) < 1e-30f) s = s < 0.f ? -1e-30f : 1e-30f;
      inv[a] = 1.f / s;
    }
  }
  const float p[3] = {px, py, pz};
  float tmin = -INFINITY, tmax = INFINITY;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const float ta = (0.f - p[a]) * inv[a], tb = (F.V.ext[a] - p[a]) * inv[a];
    tmin = fmaxf(tmin, fminf(ta, tb));
    tmax = fminf(tmax, fmaxf(ta, tb));
  }
  const float t0 = fmaxf(tmin, 0.f);
  const float tend = fminf(tmax, dist);
  float trans = 1.f;
  if (!(tmax > t0 && tend > t0)) return trans;
  const float step = (float)P.step_sh, mt = (float)P.min_trans;
  constexpr int kU = 4;
  const float q0x = px * F.V.inv_sp[0] - 0.5f, q0y = py * F.V.inv_sp[1] - 0.5f, q0z = pz * F.V.inv_sp[2] - 0.5f;
  const float qdx = dir[0] * F.V.inv_sp[0], qdy = dir[1] * F.V.inv_sp[1], qdz = dir[2] * F.V.inv_sp[2];
  float t = t0;
#pragma unroll 1
  while (true) {
    TriFetch f[kU];
    float dts[kU];
    float tj = t;
#pragma unroll
    for (int j = 0; j < kU; ++j) {
      const float dt = fminf(step, tend - tj);
      const float mid = tj + 0.5f * dt;
      dts[j] = dt;
      f[j] = tri_issue_q<TEX>(F.V, fmaf(qdx, mid, q0x), fmaf(qdy, mid, q0y), fmaf(qdz, mid, q0z));
      tj = tj + dt;
    }
    bool stop = false;
#pragma unroll
    for (int j = 0; j < kU; ++j) {
      const float dt = dts[j];
      const float om = 1.f - tf_alpha2(lut2, P.K, TEX ? tri_finish_t<TEX>(f[j]) : tri_finish_fma(f[j]));
      const float keep = dt == step ? keep_t<CLS>(om, F.e_sh) : keep_partial(om, dt * F.inv_ref);
      trans = trans * keep;
      ++nsamp;
      t = t + dt;
      if (!(t < tend) || !(trans > mt)) { stop = true; break; }
    }
    if (stop) break;
  }
  return trans;
}

// One thread per ray, shadows inline; grid-stride over the list. Used by the naive renderer (bricks)
// and, on the texture path, for the rays the wavefront main pass could not record (count_rays =
// false: the setup pass counted them already).
template <int TEX>
__global__ void __launch_bounds__(128) march_fast_kernel(FastParams F, bool count_rays) {
  const MarchParams& P = F.P;
  __shared__ float lut[4 * 256];
  const int k = P.k_dev ? *P.k_dev : P.k_max;
  if ((int64_t)blockIdx.x * blockDim.x >= k) return;  // (the overflow list is usually empty)
  for (int i = threadIdx.x; i < 4 * P.K; i += blockDim.x) lut[i] = P.lut[i];
  __syncthreads();
  unsigned int n_main = 0, n_shadow = 0, hitc = 0, nr = 0;
  for (int i0 = blockIdx.x * blockDim.x; i0 < k; i0 += gridDim.x * blockDim.x) {
  const int i = i0 + threadIdx.x;
  // naive renderer lists idle lanes of occupied chunks as -(pix+1): out[~active] = 0 (renderer.py:195-197)
  const int raw = (i < k) ? (P.idx ? P.idx[i] : i) : 0;
  if (i < k && raw < 0) {
    const int q = -raw - 1;
    if (P.rgba) *reinterpret_cast<float4*>(P.rgba + (int64_t)q * 4) = make_float4(0.f, 0.f, 0.f, 0.f);
    if (P.depth) P.depth[q] = 0.f;
  }
  if (i < k && raw >= 0) {
    const int pix = raw;
    const int u = pix % P.W, v = pix / P.W;
    const CamView cam = load_cam(P);
    const double sx = (((double)u + 0.5) / P.W * 2.0 - 1.0) * cam.tan_half * cam.aspect;
    const double sy = (1.0 - ((double)v + 0.5) / P.H * 2.0) * cam.tan_half;
    double d[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) d[a] = cam.fwd[a] + sx * cam.right[a] + sy * cam.up[a];
    const double nrm = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
    d[0] /= nrm; d[1] /= nrm; d[2] /= nrm;
    double t0, t_end;
    bool hit;
    ray_box(cam.pos, d, P.ext, t0, t_end, hit);
    float rgb[3] = {0.f, 0.f, 0.f};
    float trans = 1.f;
    double depth = 0.0;
    const bool lit = P.light_kind != FV_LIGHT_NONE;
    const float amb = lit ? (float)P.ambient : 1.f;
    const float I0 = (float)P.intensity[0], I1 = (float)P.intensity[1], I2 = (float)P.intensity[2];
    const float early = (float)P.early;
    if (hit) {
      ++hitc;
      // iterations of the reference loop: t_{i+1} = t0 + (i+1)*step, stop once >= t_end - 1e-12
      const double L = t_end - t0;
      int n = (int)ceil((L - 1e-12) / P.step);
      if (n < 1) n = 1;
      const float last_dt = (float)(L - (double)(n - 1) * P.step);
      const float ex = (float)(cam.pos[0] + d[0] * t0), ey = (float)(cam.pos[1] + d[1] * t0),
                  ez = (float)(cam.pos[2] + d[2] * t0);
      const float dx = (float)d[0], dy = (float)d[1], dz = (float)d[2];
      const float stepf = (float)P.step;
#pragma unroll 1
      for (int s = 0; s < n; ++s) {
        const bool last = s == n - 1;
        const float dt = last ? last_dt : stepf;
        const float mid = (float)s * stepf + 0.5f * dt;
        const float px = ex + dx * mid, py = ey + dy * mid, pz = ez + dz * mid;
        float c[4];
        tf_apply<float>(lut, P.K, TEX ? tri_finish_t<TEX>(tri_issue<TEX>(F.V, px, py, pz)) : tri_fast(F.V, px, py, pz), c);
        ++n_main;
        const float keep = last ? keep_partial(1.f - c[3], dt * F.inv_ref) : keep_cls(1.f - c[3], F.cls_main, F.e_main);
        const float a_step = 1.f - keep;
        float shade = 1.f;
        if (lit && a_step > 0.f) shade = amb + (1.f - amb) * shadow_fast<TEX>(F, lut, px, py, pz, n_shadow);
        const float contrib = trans * a_step;
        rgb[0] += contrib * (c[0] * (shade * I0));
        rgb[1] += contrib * (c[1] * (shade * I1));
        rgb[2] += contrib * (c[2] * (shade * I2));
        trans = trans * (1.f - a_step);
        const float acc = 1.f - trans;
        if (depth == 0.0 && acc >= 0.5f) depth = t0 + (double)mid;
        if (!(acc < early)) break;
      }
    }
    const float bga = (float)P.bg[3];
    float out[4];
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) out[ch] = rgb[ch] + (trans * bga) * (float)P.bg[ch];
    out[3] = (1.f - trans) + trans * bga;
    if (P.rgba)
      *reinterpret_cast<float4*>(P.rgba + (int64_t)pix * 4) = make_float4(out[0], out[1], out[2], out[3]);
    if (P.depth) P.depth[pix] = (float)depth;
    if (P.net_in) {
      __half2* px = reinterpret_cast<__half2*>(P.net_in + ((int64_t)v * P.net_wp + u) * 8);
      px[0] = __floats2half2_rn(out[0], out[1]);
      px[1] = __floats2half2_rn(out[2], out[3]);
    }
  }
  nr += (i < k && raw >= 0) ? 1u : 0u;
  }
  unsigned int r = count_rays ? nr : 0u;
  if (!count_rays) hitc = 0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    r += __shfl_xor_sync(0xffffffffu, r, o);
    hitc += __shfl_xor_sync(0xffffffffu, hitc, o);
    n_main += __shfl_xor_sync(0xffffffffu, n_main, o);
    n_shadow += __shfl_xor_sync(0xffffffffu, n_shadow, o);
  }
  if ((threadIdx.x & 31) == 0 && (r || n_main)) {
    if (r) atomicAdd(&P.counters->rays, (unsigned long long)r);
    if (hitc) atomicAdd(&P.counters->hit_rays, (unsigned long long)hitc);
    atomicAdd(&P.counters->samples_main, (unsigned long long)n_main);
    atomicAdd(&P.counters->samples_shadow, (unsigned long long)n_shadow);
  }
}

// ---------------------------------------------------------------------------------------------
// Wavefront marcher (default fast tier): main rays, shadow rays and compositing as three passes.
//
// In _march the shade of a sample enters only the colour sum (renderer.py:181-182); opacity,
// depth and early termination never depend on it. So the main pass marches every compacted ray
// once, without shadows, and records for each sample with a_step > 0 its position, its weight
// T*a_step and its TF colour; the shadow pass then marches all those shadow rays as independent
// work items (4.6M per C3 frame instead of 117k hit rays, so no ray's serial chain sets the
// tail); the composite pass sums contrib*(c*(shade*I)) per ray. Records are appended to 32-slot
// chunks taken from a global counter (a ray's chunks form a linked list), so one march suffices.
// A ray that cannot get a chunk (buffer full) is listed and re-marched by march_fast_kernel with
// inline shadows after the main pass.
constexpr int kChunk = 32;

struct WaveBufs {
  float4* rec0;            // (px, py, pz, -): shadow-ray origin
  float4* rec1;            // (c0, c1, c2, contrib = T * a_step)
  float* shade;            // written by the shadow pass
  int* chunk_next;         // next chunk of the same ray (-1 = last)
  int* chunk_fill;         // used slots of a chunk
  int n_chunks_cap;
  unsigned int* chunk_count;
  unsigned int* next;      // work counter of the shadow pass
  int4* ray;               // per compacted ray: (first chunk, record count, trans, depth) bits
  int* ord;                // nullable: chunk ids in shadow-pass visiting order (order_*_kernel)
  unsigned int* ord_count;
  int cap_a;               // > 0 (warp main pass): chunk r < cap_a is the FIRST chunk of ray r; later
                           // chunks come from pools at ids cap_a + counter (see march_wave_shadow_kernel)
  int chunk_pool;          // warp main pass: chunks claimed per counter round trip
  int claim;               // main pass: rays claimed per counter round trip (<= 32)
  float4* hits;            // setup pass -> main pass: 3 float4 per hitting ray
  int* ovf;                // pixels of the rays that found the record buffer full
  unsigned int* ovf_count;
  unsigned int* hit_count;
  unsigned int* hit_next;
  int by_hit;              // ray[] indexed by hit-list position (the composite walks the hits only)
};

__device__ __forceinline__ void write_pixel(const MarchParams& P, int pix, float r0, float r1, float r2,
                                            float trans, float depth) {
  const float bga = (float)P.bg[3];
  const float o0 = r0 + (trans * bga) * (float)P.bg[0], o1 = r1 + (trans * bga) * (float)P.bg[1],
              o2 = r2 + (trans * bga) * (float)P.bg[2], o3 = (1.f - trans) + trans * bga;
  if (P.rgba) *reinterpret_cast<float4*>(P.rgba + (int64_t)pix * 4) = make_float4(o0, o1, o2, o3);
  if (P.depth) P.depth[pix] = depth;
  if (P.net_in) {
    const int u = pix % P.W, v = pix / P.W;
    __half2* hp = reinterpret_cast<__half2*>(P.net_in + ((int64_t)v * P.net_wp + u) * 8);
    hp[0] = __floats2half2_rn(o0, o1);
    hp[1] = __floats2half2_rn(o2, o3);
  }
}

// March the hitting rays of a claimed set (one ray's setup per lane, hit_mask = lanes holding a
// hitting ray) one at a time, the whole warp on each. The samples of a primary ray do not depend on
// the data, so lane l evaluates samples s0 + u*32 + l (all texture loads issued first); the
// transmittance in front of each sample is an inclusive product scan over the lanes, and early
// termination cuts the block after the first sample whose accumulated opacity reaches
// early_term_alpha -- the samples the sequential loop evaluates, with the products associated
// differently (fp32 rounding). Records of the lit samples are compacted into the ray's 32-slot chunks
// with ballot/popc, so all chunks but the last are full (the composite pass relies on it). The
// first chunk of ray r is chunk r (first_list_kernel); later ones come from per-warp pools of
// chunk_pool chunks, the next pool claimed when the current one opens. A ray that finds the record
// buffer full releases its chunks and goes to the overflow list (march_fast_kernel marches those
// with inline shadow rays afterwards): keeping that code out of this pass leaves it at 64 registers.
template <int kU, int TEX>
__device__ __forceinline__ void march_hits(const FastParams& F, const WaveBufs& B, const float* lut,
                                           unsigned hit_mask, int n, float last_dt, float ex, float ey,
                                           float ez, float dx, float dy, float dz, double t0, int pix,
                                           int rid, int hid, int& pool_cur, int& pool_end, unsigned int& pool_pref,
                                           unsigned int& n_main) {
  const MarchParams& P = F.P;
  const int lane = threadIdx.x & 31;
  const unsigned lt_mask = (1u << lane) - 1u;
  const bool lit = P.light_kind != FV_LIGHT_NONE;
  const float I0 = (float)P.intensity[0], I1 = (float)P.intensity[1], I2 = (float)P.intensity[2];
  const float early = (float)P.early, stepf = (float)P.step;
  const int kPool = B.chunk_pool;
  // ---- march the hitting rays one at a time, the whole warp on each ----
  while (hit_mask) {
    const int src = __ffs(hit_mask) - 1;
    hit_mask &= hit_mask - 1;
    const int rn = __shfl_sync(0xffffffffu, n, src);
    const float rl = __shfl_sync(0xffffffffu, last_dt, src);
    const float rex = __shfl_sync(0xffffffffu, ex, src), rey = __shfl_sync(0xffffffffu, ey, src),
                rez = __shfl_sync(0xffffffffu, ez, src);
    const float rdx = __shfl_sync(0xffffffffu, dx, src), rdy = __shfl_sync(0xffffffffu, dy, src),
                rdz = __shfl_sync(0xffffffffu, dz, src);
    const double rt0 = __shfl_sync(0xffffffffu, t0, src);
    const int rpix = __shfl_sync(0xffffffffu, pix, src);
    const int rray = __shfl_sync(0xffffffffu, rid, src);
    const int rslot = B.by_hit ? __shfl_sync(0xffffffffu, hid, src) : rray;  // this ray's header in ray[]
    // (a loop of one pass: `continue` below abandons the ray when the record buffer is full)
    for (int pass = 0; pass < 1; ++pass) {
      float trans = 1.f, depth = 0.f;
      float rgb0 = 0.f, rgb1 = 0.f, rgb2 = 0.f;  // per-lane partial sums
      int first = -1, chunk = -1, fill = kChunk, m = 0;
      bool overflow = false;
      unsigned int n_main_ray = 0;
      for (int s0 = 0; s0 < rn; s0 += 32 * kU) {
        TriFetch f[kU];
#pragma unroll
        for (int uu = 0; uu < kU; ++uu) {
          const int s = s0 + uu * 32 + lane;
          const float dt = s == rn - 1 ? rl : stepf;
          const float mid = (float)s * stepf + 0.5f * dt;
          f[uu] = tri_issue<TEX>(F.V, rex + rdx * mid, rey + rdy * mid, rez + rdz * mid);
        }
        bool done = false;
#pragma unroll
        for (int uu = 0; uu < kU; ++uu) {
          const int s = s0 + uu * 32 + lane;
          const bool active = s < rn;
          const unsigned act = __ballot_sync(0xffffffffu, active);
          if (!act) { done = true; break; }
          const bool last = s == rn - 1;
          const float dt = last ? rl : stepf;
          const float mid = (float)s * stepf + 0.5f * dt;
          float c[4];
          tf_apply<float>(lut, P.K, tri_finish_t<TEX>(f[uu]), c);
          const float keep = last ? keep_partial(1.f - c[3], dt * F.inv_ref) : keep_cls(1.f - c[3], F.cls_main, F.e_main);
          const float a_step = active ? 1.f - keep : 0.f;
          // transmittance in front of / behind each sample: product scan of (1 - a_step)
          const float om = 1.f - a_step;
          float incl = om;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const float v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl *= v;
          }
          float excl = __shfl_up_sync(0xffffffffu, incl, 1);
          if (lane == 0) excl = 1.f;
          const float t_in = trans * excl, t_out = trans * incl;
          const float acc = 1.f - t_out;
          // the sequential loop stops after the first sample with !(acc < early) (or the last)
          const unsigned term = __ballot_sync(0xffffffffu, active && !(acc < early));
          const int stop_lane = term ? __ffs(term) - 1 : 31 - __clz(act);
          const bool use = active && lane <= stop_lane;
          if (depth == 0.f) {
            const unsigned dm = __ballot_sync(0xffffffffu, use && acc >= 0.5f);
            if (dm) {
              const int dl = __ffs(dm) - 1;
              const float mid_d = __shfl_sync(0xffffffffu, mid, dl);
              depth = (float)(rt0 + (double)mid_d);
            }
          }
          const float contrib = t_in * a_step;
          const bool needs_shadow = use && lit && a_step > 0.f;
          if (!lit) {
            if (use) {
              rgb0 += contrib * (c[0] * I0);
              rgb1 += contrib * (c[1] * I1);
              rgb2 += contrib * (c[2] * I2);
            }
          } else {
            const unsigned lm = __ballot_sync(0xffffffffu, needs_shadow);
            const int cnt = __popc(lm);
            if (cnt) {
              const int room = kChunk - fill;
              int nc = -1;
              if (cnt > room) {
                if (chunk < 0 && rray < B.cap_a) {
                  nc = rray;  // the ray's first chunk: fixed id, so the shadow pass meets first chunks in ray order
                } else {
                  if (pool_cur >= pool_end) {
                    pool_cur = B.cap_a + (int)__shfl_sync(0xffffffffu, pool_pref, 0);
                    pool_end = pool_cur + kPool;
                    if (lane == 0) pool_pref = atomicAdd(B.chunk_count, (unsigned)kPool);
                  }
                  nc = pool_cur++;
                  if (nc >= B.n_chunks_cap) overflow = true;
                }
              }
              if (!overflow) {
                const int rank = __popc(lm & lt_mask);
                if (needs_shadow) {
                  const int slot = rank < room ? chunk * kChunk + fill + rank : nc * kChunk + (rank - room);
                  B.rec0[slot] = make_float4(rex + rdx * mid, rey + rdy * mid, rez + rdz * mid, 0.f);
                  B.rec1[slot] = make_float4(c[0], c[1], c[2], contrib);
                }
                if (nc >= 0) {
                  if (lane == 0) {
                    if (chunk >= 0) { B.chunk_fill[chunk] = kChunk; B.chunk_next[chunk] = nc; }
                  }
                  if (chunk < 0) first = nc;
                  chunk = nc;
                  fill = cnt - room;
                } else {
                  fill += cnt;
                }
                m += cnt;
              }
            }
          }
          n_main_ray += __popc(__ballot_sync(0xffffffffu, use));
          trans = __shfl_sync(0xffffffffu, t_out, stop_lane);
          if (term || overflow) { done = true; break; }
        }
        if (done) break;
      }
      if (overflow) {
        // release this ray's chunks; march_fast_kernel re-marches it with inline shadow rays after
        // this pass (the overflow list), so neither this pass's samples nor its pixel count
        if (lane == 0) {
          for (int cc = first; cc >= 0; cc = (cc == chunk) ? -1 : B.chunk_next[cc]) B.chunk_fill[cc] = 0;
          B.ray[rslot] = make_int4(-1, 0, 0, 0);
          B.ovf[atomicAdd(B.ovf_count, 1u)] = rpix;
        }
        continue;
      }
      n_main += n_main_ray;
      if (lit && m > 0) {
        if (lane == 0) {
          B.chunk_fill[chunk] = fill;
          B.chunk_next[chunk] = -1;
          B.ray[rslot] = make_int4(first, m, __float_as_int(trans), __float_as_int(depth));
        }
      } else {
        if (lane == 0 && rray < B.cap_a) B.chunk_fill[rray] = 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          rgb0 += __shfl_xor_sync(0xffffffffu, rgb0, o);
          rgb1 += __shfl_xor_sync(0xffffffffu, rgb1, o);
          rgb2 += __shfl_xor_sync(0xffffffffu, rgb2, o);
        }
        if (lane == 0) {
          write_pixel(P, rpix, rgb0, rgb1, rgb2, trans, depth);
          B.ray[rslot] = make_int4(-1, 0, 0, 0);
        }
      }
      break;
    }
  }
}

// ---- ray setup pass + main pass over the list of hitting rays ------------------------------------
// With the setup inside the main pass, a warp claims 32 compacted rays, sets them up one per lane and
// then marches the ~10 that hit the volume one by one: per-warp work comes in lumps of 32 rays, and
// the last lumps leave a tail in which most warps have exited (ncu: 19% achieved occupancy against
// 31% theoretical; claiming 4 rays per round trip cut the pass 262 -> 185 us, but then 28 of 32 lanes
// idle through every fp64 setup). Here a thread-per-ray pass does the fp64 setup (ray through the
// pixel centre, slab test, step count), writes the pixels of missing rays, and lists the hitting rays
// (warp-aggregated appends, so the list keeps the compacted order within each warp); the main pass
// then claims hitting rays a few at a time. A/B on B200 at C3 (main pass incl. setup, us):
// in-kernel setup 262; list with 1 / 2 / 4 / 8 rays per claim: 171 / 168 / 180 / 211. Two per claim
// also gave the best pipelined frame rate (the pass then co-runs with the network's convs).
// one compacted ray's fp64 setup; misses write their pixel here
__device__ __forceinline__ bool setup_ray(const MarchParams& P, const WaveBufs& B, int r, float4& h0, float4& h1,
                                          double& t0, int& pix) {
  pix = P.idx ? P.idx[r] : r;
  const int u = pix % P.W, v = pix / P.W;
  const CamView cam = load_cam(P);
  const double sx = (((double)u + 0.5) / P.W * 2.0 - 1.0) * cam.tan_half * cam.aspect;
  const double sy = (1.0 - ((double)v + 0.5) / P.H * 2.0) * cam.tan_half;
  double d[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) d[a] = cam.fwd[a] + sx * cam.right[a] + sy * cam.up[a];
  const double nrm = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
  d[0] /= nrm; d[1] /= nrm; d[2] /= nrm;
  double tend;
  bool hit;
  ray_box(cam.pos, d, P.ext, t0, tend, hit);
  if (!hit) {
    write_pixel(P, pix, 0.f, 0.f, 0.f, 1.f, 0.f);
    if (!B.by_hit) B.ray[r] = make_int4(-1, 0, 0, 0);
    if (r < B.cap_a) B.chunk_fill[r] = 0;
    return false;
  }
  const double L = tend - t0;
  int n = (int)ceil((L - 1e-12) / P.step);
  if (n < 1) n = 1;
  const float last_dt = (float)(L - (double)(n - 1) * P.step);
  h0 = make_float4((float)(cam.pos[0] + d[0] * t0), (float)(cam.pos[1] + d[1] * t0),
                   (float)(cam.pos[2] + d[2] * t0), (float)d[0]);
  h1 = make_float4((float)d[1], (float)d[2], last_dt, __int_as_float(n));
  return true;
}

// RPT compacted rays per thread per round (r, r + 256, ...): their fp64 chains are independent, so
// they overlap; a block's hits are appended with one atomic per round.
template <int RPT>
__global__ void __launch_bounds__(256) ray_setup_kernel(FastParams F, WaveBufs B) {
  const MarchParams& P = F.P;
  __shared__ unsigned s_cnt[8], s_off[8], s_base;
  const int k = P.k_dev ? *P.k_dev : P.k_max;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned lt_mask = (1u << lane) - 1u;
  unsigned int nrays = 0, hitc = 0;
  for (int r0 = blockIdx.x * blockDim.x * RPT; r0 < k; r0 += gridDim.x * blockDim.x * RPT) {
    bool hit[RPT];
    int pix[RPT];
    float4 h0[RPT], h1[RPT];
    double t0[RPT];
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
      const int r = r0 + q * blockDim.x + threadIdx.x;
      hit[q] = false;
      pix[q] = 0;
      t0[q] = 0.0;
      if (r < k) {
        ++nrays;
        hit[q] = setup_ray(P, B, r, h0[q], h1[q], t0[q], pix[q]);
        hitc += hit[q] ? 1u : 0u;
      }
    }
    // one append per block (the shared list counter is contended: one atomic per warp cost ~2x)
    unsigned hm[RPT], wcnt = 0;
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
      hm[q] = __ballot_sync(0xffffffffu, hit[q]);
      wcnt += __popc(hm[q]);
    }
    if (lane == 0) s_cnt[warp] = wcnt;
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned t = 0;
      for (int w2 = 0; w2 < 8; ++w2) { s_off[w2] = t; t += s_cnt[w2]; }
      s_base = t ? atomicAdd(B.hit_count, t) : 0u;
    }
    __syncthreads();
    unsigned base = s_base + s_off[warp];
    __syncthreads();  // (s_cnt / s_off / s_base are rewritten by the next round)
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
      if (hit[q]) {
        const int r = r0 + q * blockDim.x + threadIdx.x;
        float4* e = B.hits + 3 * (int64_t)(base + __popc(hm[q] & lt_mask));
        e[0] = h0[q];
        e[1] = h1[q];
        e[2] = make_float4(__int_as_float(__double2loint(t0[q])), __int_as_float(__double2hiint(t0[q])),
                           __int_as_float(r), __int_as_float(pix[q]));
      }
      base += __popc(hm[q]);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    nrays += __shfl_xor_sync(0xffffffffu, nrays, o);
    hitc += __shfl_xor_sync(0xffffffffu, hitc, o);
  }
  if (lane == 0 && nrays) {
    atomicAdd(&P.counters->rays, (unsigned long long)nrays);
    atomicAdd(&P.counters->hit_rays, (unsigned long long)hitc);
  }
}

template <int kU, int TEX, int MINB>
__global__ void __launch_bounds__(128, MINB) march_wave_main_list_kernel(FastParams F, WaveBufs B) {
  const MarchParams& P = F.P;
  B.cap_a = min(P.k_dev ? *P.k_dev : P.k_max, B.cap_a);  // first chunks for this frame's k rays
  __shared__ float lut[4 * 256];
  for (int i = threadIdx.x; i < 4 * P.K; i += blockDim.x) lut[i] = P.lut[i];
  __syncthreads();
  const int nhit = (int)*B.hit_count;
  const int lane = threadIdx.x & 31;
  const bool lit = P.light_kind != FV_LIGHT_NONE;
  unsigned int n_main = 0;
  const int kPool = B.chunk_pool;
  int pool_cur = 0, pool_end = 0;  // warp-uniform
  unsigned int pool_pref = 0;      // lane 0: base of the prefetched pool
  if (lit && lane == 0) pool_pref = atomicAdd(B.chunk_count, (unsigned)kPool);
  while (true) {
    unsigned int base = 0;
    if (lane == 0) base = atomicAdd(B.hit_next, (unsigned)B.claim);
    base = __shfl_sync(0xffffffffu, base, 0);
    if ((int)base >= nhit) break;
    const int i = (int)base + lane;
    const bool valid = lane < B.claim && i < nhit;
    float4 h0 = make_float4(0.f, 0.f, 0.f, 0.f), h1 = h0, h2 = h0;
    if (valid) {
      const float4* e = B.hits + 3 * (int64_t)i;
      h0 = e[0]; h1 = e[1]; h2 = e[2];
    }
    const double t0 = __hiloint2double(__float_as_int(h2.y), __float_as_int(h2.x));
    march_hits<kU, TEX>(F, B, lut, __ballot_sync(0xffffffffu, valid), __float_as_int(h1.w), h1.z, h0.x, h0.y,
                        h0.z, h0.w, h1.x, h1.y, t0, __float_as_int(h2.w), __float_as_int(h2.z), i, pool_cur,
                        pool_end, pool_pref, n_main);
  }
  if (lit) {
    const int pref = B.cap_a + (int)__shfl_sync(0xffffffffu, pool_pref, 0);
    for (int c = pool_cur + lane; c < pool_end; c += 32)
      if (c < B.n_chunks_cap) B.chunk_fill[c] = 0;
    for (int c = lane; c < kPool; c += 32)
      if (pref + c < B.n_chunks_cap) B.chunk_fill[pref + c] = 0;
  }
  if (lane == 0 && n_main) atomicAdd(&P.counters->samples_main, (unsigned long long)n_main);
}

// With cap_a: list the rays whose first chunk (id = ray index) holds records, in ray order (one
// atomic per block; blocks cover consecutive rays) -- the shadow pass visits these first, then the
// pooled later chunks. No chain walks, so this is a few microseconds.
__global__ void __launch_bounds__(256) first_list_kernel(FastParams F, WaveBufs B) {
  const MarchParams& P = F.P;
  __shared__ int s_cnt[8], s_pre[8];
  __shared__ unsigned s_base;
  const int n = min(P.k_dev ? *P.k_dev : P.k_max, B.cap_a);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned lt_mask = (1u << lane) - 1u;
  for (int r0 = blockIdx.x * blockDim.x; r0 < n; r0 += gridDim.x * blockDim.x) {
    const int r = r0 + threadIdx.x;
    const bool has = r < n && B.chunk_fill[r] > 0;
    const unsigned m = __ballot_sync(0xffffffffu, has);
    if (lane == 0) s_cnt[warp] = __popc(m);
    __syncthreads();
    if (threadIdx.x == 0) {
      int t = 0;
#pragma unroll
      for (int w = 0; w < 8; ++w) { s_pre[w] = t; t += s_cnt[w]; }
      s_base = t ? atomicAdd(B.ord_count, (unsigned)t) : 0u;
    }
    __syncthreads();
    if (has) B.ord[s_base + s_pre[warp] + __popc(m & lt_mask)] = r;
    __syncthreads();
  }
}

// One shadow ray per record slot (empty tail slots of a ray's last chunk are skipped); lanes
// refill from a work counter so long shadow rays do not idle their warp's neighbours.
template <int CLS, int TEX>
__global__ void __launch_bounds__(128, 8) march_wave_shadow_kernel(FastParams F, WaveBufs B) {
  const MarchParams& P = F.P;
  B.cap_a = min(P.k_dev ? *P.k_dev : P.k_max, B.cap_a);  // first chunks for this frame's k rays
  __shared__ float2 lut2[256];
  for (int i = threadIdx.x; i < P.K - 1; i += blockDim.x)
    lut2[i] = make_float2(P.lut[4 * i + 3], P.lut[4 * (i + 1) + 3] - P.lut[4 * i + 3]);
  __syncthreads();
  // chunks to visit: with cap_a, first the listed non-empty first chunks (ord) then the pooled ones
  // slots: first the listed non-empty first chunks (ord), then the pooled chunks
  const int n_a = (int)*B.ord_count;
  const int n_b = (int)min(*B.chunk_count, (unsigned)(B.n_chunks_cap - B.cap_a));
  const int nslots = (n_a + n_b) * kChunk;
  const int lane = threadIdx.x & 31;
  const unsigned lt_mask = (1u << lane) - 1u;
  const float amb = (float)P.ambient;
  unsigned int n_shadow = 0;
  bool exhausted = false;
  int my = -1;
  while (true) {
    // refill until every lane holds a used slot (or the slots ran out), then march
    while (true) {
      const bool need = my < 0 && !exhausted;
      const unsigned msk = __ballot_sync(0xffffffffu, need);
      if (!msk) break;
      const int leader = __ffs(msk) - 1;
      unsigned base = 0;
      if (lane == leader) base = atomicAdd(B.next, (unsigned)__popc(msk));
      base = __shfl_sync(0xffffffffu, base, leader);
      if (need) {
        int i = (int)(base + __popc(msk & lt_mask));
        if (i >= nslots) {
          exhausted = true;
        } else {
          {
            const int q = i / kChunk;
            i = (q < n_a ? B.ord[q] : B.cap_a + q - n_a) * kChunk + (i % kChunk);
          }
          if ((i % kChunk) < B.chunk_fill[i / kChunk]) my = i;
        }
      }
    }
    if (!__any_sync(0xffffffffu, my >= 0)) break;
    if (my >= 0) {
      const float4 r0 = B.rec0[my];
      const float ts = shadow_fast_t<CLS, TEX>(F, lut2, r0.x, r0.y, r0.z, n_shadow);
      B.shade[my] = amb + (1.f - amb) * ts;
      my = -1;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) n_shadow += __shfl_xor_sync(0xffffffffu, n_shadow, o);
  if (lane == 0 && n_shadow) atomicAdd(&P.counters->samples_shadow, (unsigned long long)n_shadow);
}

// ---- shadow pass, directional light, partial refill ------------------------------------------
// The pass above marches all 32 lanes' shadow rays to the end of the longest before it refills
// (ncu: 17 of 32 lanes active) and pays ~76 instructions per sample. This version:
//  * steps by sample index: sample s < last sits at q = qa + qs*s (qs = the warp-uniform q-space
//    step toward the light), the final partial sample at q = qa + qs*fl with its own exponent --
//    no per-sample dt/min/compare chain, no fp64->fp32 parameter conversions in the loop;
//  * drops the inside-the-box test: the shadow ray is clipped to the box, so every midpoint lies
//    inside it in exact arithmetic (the fp64 reference never sees an outside sample there); the
//    texture's clamp addressing gives the edge value for the fp32 points that land a rounding
//    error outside;
//  * marches U samples per lane per round and, between rounds, hands a finished lane the next
//    record slot once at least `refill_min` lanes of the warp are free -- refilled lanes take
//    consecutive slots (neighbouring samples of one primary ray, whose light rays overlap) from a
//    warp-private range, so refills neither lose that coherence nor wait on a shared counter.
// Results match march_wave_shadow_kernel to fp32 rounding (same samples, same termination rule).
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float lg2_approx(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

template <int U, int MINB, bool LIN = false>
__global__ void __launch_bounds__(128, MINB) march_wave_shadow_dir_kernel(FastParams F, WaveBufs B, int refill_min,
                                                                          unsigned claim_blk) {
  const MarchParams& P = F.P;
  B.cap_a = min(P.k_dev ? *P.k_dev : P.k_max, B.cap_a);  // first chunks for this frame's k rays
  // om table: (1 - a_i, -(a_{i+1} - a_i)), padded with (1 - a_{K-1}, 0) so that the index may
  // round to K-1 at s = 1 (w = 0 there)
  __shared__ float2 lut_om[257];
  for (int i = threadIdx.x; i < P.K; i += blockDim.x)
    lut_om[i] = i < P.K - 1 ? make_float2(1.f - P.lut[4 * i + 3], -(P.lut[4 * (i + 1) + 3] - P.lut[4 * i + 3]))
                            : make_float2(1.f - P.lut[4 * i + 3], 0.f);
  __syncthreads();
  // slots: first the listed non-empty first chunks (ord), then the pooled chunks
  const int n_a = (int)*B.ord_count;
  const int n_b = (int)min(*B.chunk_count, (unsigned)(B.n_chunks_cap - B.cap_a));
  const int nslots = (n_a + n_b) * kChunk;
  const int lane = threadIdx.x & 31;
  const unsigned lt_mask = (1u << lane) - 1u;
  const float amb = F.ambient;
  const float step = F.step_sh, inv_step = F.inv_step_sh, mt = F.min_trans;
  const float lmt = mt > 0.f ? log2f(mt) : -INFINITY;  // LIN: the threshold on log2 T
  const float qsx = F.qs_sh[0], qsy = F.qs_sh[1], qsz = F.qs_sh[2];
  const float kscale = (float)(P.K - 1), e_full = F.e_sh;
  constexpr float kMagic = 12582912.f;  // 1.5 * 2^23: x + kMagic rounds x to an integer
  unsigned int n_shadow = 0;
  bool exhausted = false;
  int my = -1, s = 0, last = -1;  // free lanes keep last = -1, so none of their samples is live
  float qax = 0.f, qay = 0.f, qaz = 0.f, fl = 0.f, el = 0.f, trans = 1.f;
  // Record slots come from a warp-private range [lb, le) of claim_blk slots; the next range is
  // claimed (lane 0) when the current one opens, so a refill never waits on the shared counter
  // (one contended atomic per claim_blk slots instead of one per refill).
  unsigned lb = 0, le = 0, pend = 0;
  if (lane == 0) pend = atomicAdd(B.next, claim_blk);
  while (true) {
    while (true) {
      const bool need = my < 0 && !exhausted;
      const unsigned msk = __ballot_sync(0xffffffffu, need);
      const unsigned busy = __ballot_sync(0xffffffffu, my >= 0);
      if (!msk || (busy && __popc(msk) < refill_min)) break;
      const unsigned cnt = (unsigned)__popc(msk), rank = (unsigned)__popc(msk & lt_mask);
      const unsigned take = min(cnt, le - lb);
      unsigned slot = lb + rank;
      lb += take;
      if (take < cnt) {
        const unsigned nb = __shfl_sync(0xffffffffu, pend, 0);
        if (lane == 0) pend = atomicAdd(B.next, claim_blk);
        if (rank >= take) slot = nb + (rank - take);
        lb = nb + (cnt - take);
        le = nb + claim_blk;
      }
      if (need) {
        int i = slot < (unsigned)nslots ? (int)slot : nslots;
        if (i >= nslots) {
          exhausted = true;
        } else {
          {
            const int q = i / kChunk;
            i = (q < n_a ? B.ord[q] : B.cap_a + q - n_a) * kChunk + (i % kChunk);
          }
          if ((i % kChunk) < B.chunk_fill[i / kChunk]) {
            const float4 r0 = B.rec0[i];
            const float p[3] = {r0.x, r0.y, r0.z};
            float tmin = -INFINITY, tmax = INFINITY;
#pragma unroll
            for (int a = 0; a < 3; ++a) {
              const float ta = (0.f - p[a]) * F.ld_inv[a], tb = (F.V.ext[a] - p[a]) * F.ld_inv[a];
              tmin = fmaxf(tmin, fminf(ta, tb));
              tmax = fminf(tmax, fmaxf(ta, tb));
            }
            const float t0 = fmaxf(tmin, 0.f);
            if (!(tmax > t0)) {
              B.shade[i] = amb + (1.f - amb) * 1.f;
            } else {
              const float L = tmax - t0;
              int n = max(1, (int)ceilf(L * inv_step));
              float ldt = L - (float)(n - 1) * step;
              if (ldt <= 0.f && n > 1) { --n; ldt += step; }
              ldt = fminf(ldt, step);
              const float m0 = t0 + 0.5f * step;
              // (LIN: q + 1/2, the texel-centre offset, folded into the base)
              constexpr float kQ0 = LIN ? 0.f : -0.5f;
              qax = fmaf(F.ld[0] * F.V.inv_sp[0], m0, fmaf(p[0], F.V.inv_sp[0], kQ0));
              qay = fmaf(F.ld[1] * F.V.inv_sp[1], m0, fmaf(p[1], F.V.inv_sp[1], kQ0));
              qaz = fmaf(F.ld[2] * F.V.inv_sp[2], m0, fmaf(p[2], F.V.inv_sp[2], kQ0));
              last = n - 1;
              fl = (float)(n - 1) + 0.5f * (ldt - step) * inv_step;
              el = ldt * F.inv_ref;
              s = 0;
              trans = LIN ? 0.f : 1.f;  // LIN: log2 of the transmittance
              my = i;
            }
          }
        }
      }
    }
    if (!__any_sync(0xffffffffu, my >= 0)) break;
    if constexpr (LIN) {
      // Filtered samples with a lean per-sample path (the pass is issue-bound: ~37 -> ~28
      // instructions per sample): the sample index clamps to the partial last step with one min;
      // q < 0 (the half-voxel shell) -> q + 1 through a saturated FMA; the transmittance is kept as
      // log2 T = sum e_j log2(1 - a_j) (one MUFU per sample) against log2 of the threshold.
      const float sf = (float)s;
      float vl[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const float fs = fminf(sf + (float)u, fl);
        const float cx = fmaf(qsx, fs, qax), cy = fmaf(qsy, fs, qay), cz = fmaf(qsz, fs, qaz);
        // c + [c < 1/2]: (1/2 - c) * 2^126 saturates to 1 for every c < 1/2 down to ~1e-38 below
        vl[u] = tex3D<float>(F.V.ltex, cx + __saturatef(fmaf(-cx, 8.5070592e37f, 4.2535296e37f)),
                             cy + __saturatef(fmaf(-cy, 8.5070592e37f, 4.2535296e37f)),
                             cz + __saturatef(fmaf(-cz, 8.5070592e37f, 4.2535296e37f)));
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int si = s + u;
        const float v = __saturatef(vl[u]);
        const float xh = fmaf(v, kscale, -0.5f);
        const float r = xh + kMagic;
        const int i0 = __float_as_int(r) - __float_as_int(kMagic);
        const float w = fmaf(v, kscale, -(r - kMagic));
        const float2 lv = lut_om[i0];
        const float om = fmaf(w, lv.y, lv.x);
        if (si <= last && trans > lmt) {
          trans = fmaf(si == last ? el : e_full, lg2_approx(om), trans);
          ++n_shadow;
        }
      }
      s += U;
      if (my >= 0 && (s > last || !(trans > lmt))) {
        B.shade[my] = amb + (1.f - amb) * ex2_approx(trans);
        my = -1;
        last = -1;
      }
      continue;
    }
    // U samples per lane: positions first (all texture loads in flight), then the products
    float4 A[U], Bq[U];
    float tx[U], ty[U], tz[U];
    float vl[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int si = s + u;
      const float fs = si == last ? fl : (float)si;
      const float qx = fmaf(qsx, fs, qax), qy = fmaf(qsy, fs, qay), qz = fmaf(qsz, fs, qaz);
      if constexpr (LIN) {
        // hardware trilinear at q + 1/2; q < 0 (the lower half-voxel shell) maps to q + 1, which
        // addresses the reference's texels 0, 1 with its weight q + 1 (see volume_ltex)
        vl[u] = tex3D<float>(F.V.ltex, qx + (qx < 0.f ? 1.5f : 0.5f), qy + (qy < 0.f ? 1.5f : 0.5f),
                             qz + (qz < 0.f ? 1.5f : 0.5f));
        continue;
      }
      const float fx = floorf(qx), fy = floorf(qy), fz = floorf(qz);
      tx[u] = qx - fx; ty[u] = qy - fy; tz[u] = qz - fz;
      if constexpr (kTexOff == 0.f) {
        A[u] = tex3D<float4>(F.V.tex, fx, fy, fz);
        Bq[u] = tex3D<float4>(F.V.tex, fx, fy, fmaxf(fz, 0.f) + 1.f);
      } else {
        A[u] = tex3D<float4>(F.V.tex, fx + kTexOff, fy + kTexOff, fz + kTexOff);
        Bq[u] = tex3D<float4>(F.V.tex, fx + kTexOff, fy + kTexOff, fmaxf(fz, 0.f) + (1.f + kTexOff));
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int si = s + u;
      float v;
      if constexpr (LIN) {
        v = __saturatef(vl[u]);
      } else {
        // quads hold (v00, v01 - v00, v10, v11 - v10)
        const float c00 = fmaf(tx[u], A[u].y, A[u].x), c10 = fmaf(tx[u], A[u].w, A[u].z);
        const float c01 = fmaf(tx[u], Bq[u].y, Bq[u].x), c11 = fmaf(tx[u], Bq[u].w, Bq[u].z);
        const float c0 = fmaf(ty[u], c10 - c00, c00), c1 = fmaf(ty[u], c11 - c01, c01);
        v = __saturatef(fmaf(tz[u], c1 - c0, c0));
      }
      // TF alpha: x = v (K-1); i = rint(x - 1/2) in [0, K-1], w = x - i in [0, 1]
      const float xh = fmaf(v, kscale, -0.5f);
      const float r = xh + kMagic;
      const int i0 = __float_as_int(r) - __float_as_int(kMagic);
      const float w = fmaf(v, kscale, -(r - kMagic));
      const float2 lv = lut_om[i0];
      const float om = fmaf(w, lv.y, lv.x);
      // (1 - a)^(dt/ref): e = e_full on full steps, dt_last/ref on the final partial one
      const float keep = ex2_approx((si == last ? el : e_full) * lg2_approx(om));
      if (si <= last && trans > mt) {
        trans *= keep;
        ++n_shadow;
      }
    }
    s += U;
    if (my >= 0 && (s > last || !(trans > mt))) {
      B.shade[my] = amb + (1.f - amb) * trans;
      my = -1;
      last = -1;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) n_shadow += __shfl_xor_sync(0xffffffffu, n_shadow, o);
  if (lane == 0 && n_shadow) atomicAdd(&P.counters->samples_shadow, (unsigned long long)n_shadow);
}

// rgb = sum_j contrib_j * (c_j * (shade_j * I)), then the background blend. One warp per ray,
// one chunk (32 records) per step of the chain; lane sums then a fixed xor tree -- deterministic;
// the reordering versus the reference's sequential sum is an fp32 rounding effect (~1e-7).
__global__ void __launch_bounds__(128) march_wave_composite_kernel(FastParams F, WaveBufs B) {
  const MarchParams& P = F.P;
  const int k = P.k_dev ? *P.k_dev : P.k_max;
  const float I0 = (float)P.intensity[0], I1 = (float)P.intensity[1], I2 = (float)P.intensity[2];
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  // Latency-bound: a chain of dependent loads per ray, one warp per ray and many warps in flight
  // (A/B: a warp walking 32 rays' records in turn took 143 us against 65). All of a ray's chunks but
  // the last are full (the main pass compacts records with ballots), so the fill of chunk j is
  // min(32, records - 32 j): chunk_fill is not read, and a chunk's records, shades and successor
  // link come back in one round trip.
  // by_hit: the headers sit at hit-list positions (the rays that miss the volume were written by
  // the setup pass and are not visited; the pixel comes from the hit entry, loaded with the header)
  const int n = B.by_hit ? (int)*B.hit_count : k;
  for (int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < n; r += warps) {
    const int4 v = B.ray[r];
    const int hpix = B.by_hit && lane == 0 ? __float_as_int(B.hits[3 * (int64_t)r + 2].w) : 0;
    if (v.x < 0) continue;
    float rgb0 = 0.f, rgb1 = 0.f, rgb2 = 0.f;
    for (int c = v.x, jj = 0; jj < v.y; jj += kChunk) {
      const int nxt = jj + kChunk < v.y ? B.chunk_next[c] : -1;
      if (lane < v.y - jj) {
        const int slot = c * kChunk + lane;
        const float4 q = B.rec1[slot];
        const float sh = B.shade[slot];
        rgb0 += q.w * (q.x * (sh * I0));
        rgb1 += q.w * (q.y * (sh * I1));
        rgb2 += q.w * (q.z * (sh * I2));
      }
      c = nxt;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      rgb0 += __shfl_xor_sync(0xffffffffu, rgb0, o);
      rgb1 += __shfl_xor_sync(0xffffffffu, rgb1, o);
      rgb2 += __shfl_xor_sync(0xffffffffu, rgb2, o);
    }
    if (lane == 0)
      write_pixel(P, B.by_hit ? hpix : (P.idx ? P.idx[r] : r), rgb0, rgb1, rgb2, __int_as_float(v.z),
                  __int_as_float(v.w));
  }
}

// linear (nz,ny,nx) -> bricked quads (see FastVol)
__global__ void brick_kernel(const float* __restrict__ lin, float4* __restrict__ quads, int nx, int ny,
                             int nz, int nbx, int nby, int nbz) {
  const int64_t n = (int64_t)nbx * nby * nbz * 512;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int e = (int)(i & 511);
    const int64_t b = i >> 9;
    const int bx = (int)(b % nbx), by = (int)((b / nbx) % nby), bz = (int)(b / ((int64_t)nbx * nby));
    // inverse of the in-brick Morton order (bits x: 0,3,6  y: 1,4,7  z: 2,5,8)
    const int lx = FV_BRICK_MORTON ? ((e & 1) | ((e >> 2) & 2) | ((e >> 4) & 4)) : (e & 7);
    const int ly = FV_BRICK_MORTON ? (((e >> 1) & 1) | ((e >> 3) & 2) | ((e >> 5) & 4)) : ((e >> 3) & 7);
    const int lz = FV_BRICK_MORTON ? (((e >> 2) & 1) | ((e >> 4) & 2) | ((e >> 6) & 4)) : (e >> 6);
    const int x = bx * 8 + lx, y = by * 8 + ly, z = bz * 8 + lz;
    float4 q = make_float4(0.f, 0.f, 0.f, 0.f);
    if (x < nx && y < ny && z < nz) {
      const int x1 = min(x + 1, nx - 1), y1 = min(y + 1, ny - 1);
      const float* pl = lin + (int64_t)z * ny * nx;
      q = make_float4(pl[(int64_t)y * nx + x], pl[(int64_t)y * nx + x1], pl[(int64_t)y1 * nx + x],
                      pl[(int64_t)y1 * nx + x1]);
    }
    quads[i] = q;
  }
}

int exp_class(double e) {
  if (e == 0.5) return 0;
  if (e == 1.0) return 1;
  if (e == 2.0) return 2;
  return 3;
}

void normalize3(double v[3]) {
  const double n = sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
  v[0] /= n; v[1] /= n; v[2] /= n;
}

}  // namespace

// quads -> 3D surface (texel (x,y,z) = the quad of voxel (x,y,z) as brick_kernel's, x pairs stored
// as value + difference)
__global__ void quad_surface_kernel(const float* __restrict__ lin, cudaSurfaceObject_t surf, int nx, int ny, int nz) {
  const int64_t n = (int64_t)nx * ny * nz;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int x = (int)(i % nx), y = (int)((i / nx) % ny), z = (int)(i / ((int64_t)nx * ny));
    const int x1 = min(x + 1, nx - 1), y1 = min(y + 1, ny - 1);
    const float* pl = lin + (int64_t)z * ny * nx;
    // (v00, v01 - v00, v10, v11 - v10): the x lerps become one FMA each (tri_finish_t<true>)
    const float v00 = pl[(int64_t)y * nx + x], v01 = pl[(int64_t)y * nx + x1];
    const float v10 = pl[(int64_t)y1 * nx + x], v11 = pl[(int64_t)y1 * nx + x1];
    const float4 q = make_float4(v00, v01 - v00, v10, v11 - v10);
    surf3Dwrite(q, surf, x * (int)sizeof(float4), y, z);
  }
}

int volume_texture(fv_ctx* ctx, fv_volume* vol) {
  if (vol->qtex && vol->tex_version == vol->version) return 0;
  if (!vol->qarr) {
    const cudaChannelFormatDesc fd = cudaCreateChannelDesc<float4>();
    FV_CUDA(cudaMalloc3DArray(&vol->qarr, &fd, make_cudaExtent(vol->nx, vol->ny, vol->nz), cudaArraySurfaceLoadStore));
  }
  cudaResourceDesc rd{};
  rd.resType = cudaResourceTypeArray;
  rd.res.array.array = vol->qarr;
  cudaSurfaceObject_t surf = 0;
  FV_CUDA(cudaCreateSurfaceObject(&surf, &rd));
  const int64_t n = (int64_t)vol->nx * vol->ny * vol->nz;
  const int blocks = (int)std::min<int64_t>((n + 255) / 256, (int64_t)ctx->num_sms * 16);
  FV_TIMED(ctx, FV_KC_OTHER, quad_surface_kernel<<<blocks, 256, 0, ctx->stream>>>(vol->data, surf, vol->nx, vol->ny, vol->nz));
  FV_CHECK_LAUNCH("quad_surface_kernel");
  ctx->launches += 1;
  FV_CUDA(cudaStreamSynchronize(ctx->stream));
  cudaDestroySurfaceObject(surf);
  if (!vol->qtex) {
    cudaTextureDesc td{};
    td.addressMode[0] = td.addressMode[1] = td.addressMode[2] = cudaAddressModeClamp;
    td.filterMode = cudaFilterModePoint;
    td.readMode = cudaReadModeElementType;
    td.normalizedCoords = 0;
    cudaTextureObject_t t = 0;
    FV_CUDA(cudaCreateTextureObject(&t, &rd, &td, nullptr));
    vol->qtex = (unsigned long long)t;
  }
  vol->tex_version = vol->version;
  return 0;
}

// The voxels as a 3D float texture with hardware trilinear filtering (unnormalised coordinates,
// clamp addressing). tex3D(q + 0.5) = lerp over texels floor(q), floor(q)+1 with weights
// frac(q) quantised to 8 fractional bits (the SURVEY's fast tier) -- the reference's
// sample_trilinear (volume.py:149-180) except in the half-voxel shell q < 0, where the reference
// keeps i0 = 0, i1 = 1 and t = q + 1; the caller maps q -> q + 1 there (same texels and weight).
// unorm16 texels of voxels in [0, 1] (round to nearest; *oob set when any voxel lies outside)
__global__ void unorm16_kernel(const float* __restrict__ in, uint16_t* __restrict__ out, int64_t n, int* oob) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float v = in[i];
    if (!(v >= 0.f && v <= 1.f)) *oob = 1;
    out[i] = (uint16_t)__float2uint_rn(__saturatef(v) * 65535.f);
  }
}

int volume_ltex(fv_ctx* ctx, fv_volume* vol) {
  if (vol->ltex && vol->ltex_version == vol->version) return 0;
  // Texel format (FV_LTEX_BITS, default 16): 16-bit texels filter at the texture unit's full rate
  // (32-bit float texels at half rate); unorm16 holds a voxel in [0, 1] to 7.6e-6, far below the
  // 8-bit fractional filter weights' 1/256. A volume with any voxel outside [0, 1] (the shadow
  // pass clamps AFTER interpolation) keeps float texels.
  static const int bits_env = getenv("FV_LTEX_BITS") ? atoi(getenv("FV_LTEX_BITS")) : 16;
  const int64_t n = (int64_t)vol->nx * vol->ny * vol->nz;
  const cudaExtent ext = make_cudaExtent(vol->nx, vol->ny, vol->nz);
  int bits = 32;
  uint16_t* u16 = nullptr;
  if (bits_env == 16) {
    int* oob = nullptr;
    FV_CUDA(cudaMalloc(&u16, (size_t)n * sizeof(uint16_t) + 16));
    oob = reinterpret_cast<int*>(reinterpret_cast<uint8_t*>(u16) + (((size_t)n * sizeof(uint16_t) + 7) & ~size_t(7)));
    FV_CUDA(cudaMemsetAsync(oob, 0, sizeof(int), ctx->stream));
    unorm16_kernel<<<4 * ctx->num_sms, 256, 0, ctx->stream>>>(vol->data, u16, n, oob);
    FV_CHECK_LAUNCH("unorm16_kernel");
    int h_oob = 1;
    FV_CUDA(cudaMemcpyAsync(&h_oob, oob, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    FV_CUDA(cudaStreamSynchronize(ctx->stream));
    if (!h_oob) bits = 16;
  }
  if (vol->larr && vol->ltex_bits != bits) {
    if (vol->ltex) cudaDestroyTextureObject((cudaTextureObject_t)vol->ltex);
    cudaFreeArray(vol->larr);
    vol->ltex = 0;
    vol->larr = nullptr;
  }
  int rc = 0;
  if (!vol->larr) {
    const cudaChannelFormatDesc fd =
        bits == 16 ? cudaCreateChannelDesc<unsigned short>() : cudaCreateChannelDesc<float>();
    const cudaError_t e = cudaMalloc3DArray(&vol->larr, &fd, ext);
    if (e != cudaSuccess) {
      vol->larr = nullptr;
      cudaFree(u16);
      set_error("cudaMalloc3DArray: %s", cudaGetErrorString(e));
      return FV_E_CUDA;
    }
    vol->ltex_bits = bits;
  }
  cudaMemcpy3DParms cp{};
  if (bits == 16)
    cp.srcPtr = make_cudaPitchedPtr(u16, (size_t)vol->nx * sizeof(uint16_t), vol->nx, vol->ny);
  else
    cp.srcPtr = make_cudaPitchedPtr(vol->data, (size_t)vol->nx * sizeof(float), vol->nx, vol->ny);
  cp.dstArray = vol->larr;
  cp.extent = ext;
  cp.kind = cudaMemcpyDeviceToDevice;
  cudaError_t e = cudaMemcpy3DAsync(&cp, ctx->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
  cudaFree(u16);
  if (e != cudaSuccess) {
    set_error("volume texture copy: %s", cudaGetErrorString(e));
    return FV_E_CUDA;
  }
  if (!vol->ltex) {
    cudaResourceDesc rd{};
    rd.resType = cudaResourceTypeArray;
    rd.res.array.array = vol->larr;
    cudaTextureDesc td{};
    td.addressMode[0] = td.addressMode[1] = td.addressMode[2] = cudaAddressModeClamp;
    td.filterMode = cudaFilterModeLinear;
    td.readMode = bits == 16 ? cudaReadModeNormalizedFloat : cudaReadModeElementType;
    td.normalizedCoords = 0;
    cudaTextureObject_t t = 0;
    FV_CUDA(cudaCreateTextureObject(&t, &rd, &td, nullptr));
    vol->ltex = (unsigned long long)t;
  }
  vol->ltex_version = vol->version;
  return rc;
}

int volume_bricks(fv_ctx* ctx, fv_volume* vol) {
  if (vol->bricks && vol->bricks_version == vol->version) return 0;
  const int nbx = (vol->nx + 7) / 8, nby = (vol->ny + 7) / 8, nbz = (vol->nz + 7) / 8;
  const int64_t n = (int64_t)nbx * nby * nbz * 512;
  FV_REQUIRE(n < (1ll << 31), "volume too large for 32-bit brick addressing");
  if (!vol->bricks) FV_CUDA(cudaMalloc(&vol->bricks, sizeof(float4) * n));
  int blocks = (int)std::min<int64_t>((n + 255) / 256, (int64_t)ctx->num_sms * 16);
  FV_TIMED(ctx, FV_KC_OTHER, brick_kernel<<<blocks, 256, 0, ctx->stream>>>(vol->data, reinterpret_cast<float4*>(vol->bricks), vol->nx,
                                                vol->ny, vol->nz, nbx, nby, nbz));
  FV_CHECK_LAUNCH("brick_kernel");
  ctx->launches += 1;
  vol->bricks_version = vol->version;
  return 0;
}

// resident blocks per SM the main pass's registers are capped for (A/B on B200 at C3)
#ifndef FV_MAIN_MINB
#define FV_MAIN_MINB 6
#endif

// wavefront passes, instantiated for quads from the bricked buffer (TEX = false) or the texture
template <int TEX>
int launch_main(fv_ctx* ctx, const FastParams& F, const WaveBufs& B, int threads) {
  const int blocks = std::max(1, std::min((F.P.k_max + 255) / 256, ctx->num_sms * 8));
  static bool co = false;
  if (!co) {
    render_carveout(ray_setup_kernel<1>);
    render_carveout(ray_setup_kernel<2>);
    render_carveout(march_wave_main_list_kernel<2, TEX, FV_MAIN_MINB>);
    render_carveout(first_list_kernel);
    render_carveout(march_wave_composite_kernel);
    co = true;
  }
  // rays per thread (FV_SETUP_RPT): 2 overlaps two fp64 setups per thread (C3 23.0 -> 18.9 us)
  static const int rpt = getenv("FV_SETUP_RPT") ? atoi(getenv("FV_SETUP_RPT")) : 2;
  if (rpt == 2)
    FV_TIMED(ctx, FV_KC_MARCH_MAIN, ray_setup_kernel<2><<<blocks, 256, 0, ctx->stream>>>(F, B));
  else
    FV_TIMED(ctx, FV_KC_MARCH_MAIN, ray_setup_kernel<1><<<blocks, 256, 0, ctx->stream>>>(F, B));
  ctx->launches += 1;
  static int per_sm = 0;
  if (!per_sm) {
    FV_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, march_wave_main_list_kernel<2, TEX, FV_MAIN_MINB>, threads, 0));
    per_sm = render_occ(std::max(per_sm, 1));
  }
  // samples per lane per warp block (FV_MAIN_U): 1 = 32-sample blocks (C3 main pass 102.8 ->
  // 97.6 us: a hitting ray takes ~40 samples, so 64-sample blocks fetched many past its end)
  static const int main_u = getenv("FV_MAIN_U") ? atoi(getenv("FV_MAIN_U")) : 1;
  if (main_u == 1) {
    static int per_sm1 = 0;
    if (!per_sm1) {
      render_carveout(march_wave_main_list_kernel<1, TEX, FV_MAIN_MINB>);
      FV_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm1, march_wave_main_list_kernel<1, TEX, FV_MAIN_MINB>, threads, 0));
      per_sm1 = render_occ(std::max(per_sm1, 1));
    }
    FV_TIMED(ctx, FV_KC_MARCH_MAIN, march_wave_main_list_kernel<1, TEX, FV_MAIN_MINB><<<ctx->num_sms * per_sm1, threads, 0, ctx->stream>>>(F, B));
    return 0;
  }
  FV_TIMED(ctx, FV_KC_MARCH_MAIN, march_wave_main_list_kernel<2, TEX, FV_MAIN_MINB><<<ctx->num_sms * per_sm, threads, 0, ctx->stream>>>(F, B));
  return 0;
}

template <int TEX>
int launch_shadow(fv_ctx* ctx, const FastParams& F, const WaveBufs& B, int threads) {
  static int per_sm = 0;
  if (!per_sm) {
    FV_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, march_wave_shadow_kernel<2, TEX>, threads, 0));
    per_sm = std::max(per_sm, 1);
  }
  const int g = ctx->num_sms * per_sm;
  switch (F.cls_sh) {
    case 0: FV_TIMED(ctx, FV_KC_MARCH_SHADOW, march_wave_shadow_kernel<0, TEX><<<g, threads, 0, ctx->stream>>>(F, B)); break;
    case 1: FV_TIMED(ctx, FV_KC_MARCH_SHADOW, march_wave_shadow_kernel<1, TEX><<<g, threads, 0, ctx->stream>>>(F, B)); break;
    case 2: FV_TIMED(ctx, FV_KC_MARCH_SHADOW, march_wave_shadow_kernel<2, TEX><<<g, threads, 0, ctx->stream>>>(F, B)); break;
    default: FV_TIMED(ctx, FV_KC_MARCH_SHADOW, march_wave_shadow_kernel<3, TEX><<<g, threads, 0, ctx->stream>>>(F, B)); break;
  }
  return 0;
}

// directional light on the texture path: the partial-refill pass (FV_SHADOW_V=1 keeps the
// all-lane-refill pass for A/B runs; FV_SHADOW_REFILL tunes it)
template <int U, int MINB, bool LIN = false>
int launch_shadow_dir_t(fv_ctx* ctx, const FastParams& F, const WaveBufs& B, int threads, int refill) {
  static int per_sm = 0;
  if (!per_sm) {
    FV_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, march_wave_shadow_dir_kernel<U, MINB, LIN>, threads, 0));
    per_sm = render_occ(std::max(per_sm, 1));
    render_carveout(march_wave_shadow_dir_kernel<U, MINB, LIN>);
  }
  static const unsigned blk = getenv("FV_SHADOW_CLAIM") ? (unsigned)std::max(32, atoi(getenv("FV_SHADOW_CLAIM"))) : 64u;
  FV_TIMED(ctx, FV_KC_MARCH_SHADOW, march_wave_shadow_dir_kernel<U, MINB, LIN><<<ctx->num_sms * per_sm, threads, 0, ctx->stream>>>(F, B, refill, blk));
  return 0;
}

// Refill threshold (free lanes) and private slot-range size, A/B on B200 at C3 (shadow pass, us):
// with one shared-counter atomic per refill, 1 / 4 / 8 / 16 / 24 / 32 free lanes gave 632 / 517 /
// 434 / 372 / 359 / 376 (each refill waited on the contended counter); with warp-private ranges of
// 64 slots, 1 / 2 / 4 / 8 / 16 / 24 gave 386 / 364 / 345 / 335 / 371 / 395, ranges of 32 / 48 / 128 /
// 256 slots at 8 free lanes 345 / 335 / 374 / 441. 4 samples per round and 8 blocks/SM beat 2
// samples and 6 blocks/SM (+37% / +17%).
int launch_shadow_dir(fv_ctx* ctx, const FastParams& F, const WaveBufs& B, int threads) {
  static const int refill = getenv("FV_SHADOW_REFILL") ? std::min(32, std::max(1, atoi(getenv("FV_SHADOW_REFILL")))) : 8;
  // filtered samples: (samples in flight per lane, resident blocks per SM) -- FV_SHADOW_LIN=U,B (A/B)
  // (6, 10) since the leaner per-sample path: C3 frame timeline 1529 against 1537 us for (4, 8),
  // three A/B pairs on one box (shadow 225 against 233 us)
  static const int lin_cfg = getenv("FV_SHADOW_LIN") ? atoi(getenv("FV_SHADOW_LIN")) * 100 +
                                                           atoi(strchr(getenv("FV_SHADOW_LIN"), ',') + 1)
                                                     : 610;
  if (F.V.ltex) {
    switch (lin_cfg) {
      case 808: return launch_shadow_dir_t<8, 8, true>(ctx, F, B, threads, refill);
      case 412: return launch_shadow_dir_t<4, 12, true>(ctx, F, B, threads, refill);
      case 812: return launch_shadow_dir_t<8, 12, true>(ctx, F, B, threads, refill);
      case 416: return launch_shadow_dir_t<4, 16, true>(ctx, F, B, threads, refill);
      case 408: return launch_shadow_dir_t<4, 8, true>(ctx, F, B, threads, refill);
      default: return launch_shadow_dir_t<6, 10, true>(ctx, F, B, threads, refill);
    }
  }
  return launch_shadow_dir_t<4, 8>(ctx, F, B, threads, refill);
}

int launch_render(fv_ctx* ctx, const fv_volume* vol, const fv_camera* cam, const fv_light* light,
                  const fv_settings* s, const int32_t* idx, const int32_t* k, int k_max,
                  float* rgba, float* depth, __half* net_in, int net_wp, int force_variant) {
  FV_REQUIRE(vol && vol->data, "volume has no data");
  FV_REQUIRE(vol->K >= 2, "transfer function not set");
  FV_REQUIRE(cam->width >= 1 && cam->height >= 1, "film dims must be positive");
  FV_REQUIRE(cam->fov_y > 0.0 && cam->fov_y < 180.0, "fov_y must be in (0, 180) degrees, got %g",
             cam->fov_y);
  MarchParams P{};
  // Camera.basis (volume.py:269-276)
  double fwd[3] = {cam->look_at[0] - cam->position[0], cam->look_at[1] - cam->position[1],
                   cam->look_at[2] - cam->position[2]};
  FV_REQUIRE(fwd[0] != 0 || fwd[1] != 0 || fwd[2] != 0, "camera position and look_at coincide");
  normalize3(fwd);
  double right[3] = {fwd[1] * cam->up[2] - fwd[2] * cam->up[1], fwd[2] * cam->up[0] - fwd[0] * cam->up[2],
                     fwd[0] * cam->up[1] - fwd[1] * cam->up[0]};
  const double rn = sqrt(right[0] * right[0] + right[1] * right[1] + right[2] * right[2]);
  FV_REQUIRE(rn >= 1e-9 * sqrt(cam->up[0] * cam->up[0] + cam->up[1] * cam->up[1] + cam->up[2] * cam->up[2]) && rn > 0,
             "up vector is parallel to the view direction");
  normalize3(right);
  double up[3] = {right[1] * fwd[2] - right[2] * fwd[1], right[2] * fwd[0] - right[0] * fwd[2],
                  right[0] * fwd[1] - right[1] * fwd[0]};
  for (int a = 0; a < 3; ++a) {
    P.pos[a] = cam->position[a]; P.fwd[a] = fwd[a]; P.right[a] = right[a]; P.up[a] = up[a];
  }
  P.tan_half = tan(cam->fov_y * (M_PI / 180.0) * 0.5);
  P.aspect = (double)cam->width / (double)cam->height;
  P.W = cam->width; P.H = cam->height;
  P.data = vol->data; P.nx = vol->nx; P.ny = vol->ny; P.nz = vol->nz;
  for (int a = 0; a < 3; ++a) {
    P.sp[a] = vol->spacing[a];
  }
  P.ext[0] = vol->nx * vol->spacing[0]; P.ext[1] = vol->ny * vol->spacing[1];
  P.ext[2] = vol->nz * vol->spacing[2];
  P.K = vol->K;
  P.lut = vol->lut_dev;
  // light
  P.light_kind = light ? light->kind : FV_LIGHT_NONE;
  if (P.light_kind == FV_LIGHT_DIRECTIONAL) {
    double dv[3] = {-light->vec[0], -light->vec[1], -light->vec[2]};
    FV_REQUIRE(dv[0] != 0 || dv[1] != 0 || dv[2] != 0, "light direction must be nonzero");
    normalize3(dv);
    for (int a = 0; a < 3; ++a) P.lvec[a] = dv[a];
  } else if (P.light_kind == FV_LIGHT_POINT) {
    for (int a = 0; a < 3; ++a) P.lvec[a] = light->vec[a];
  }
  for (int a = 0; a < 3; ++a) P.intensity[a] = light && P.light_kind ? light->intensity[a] : 1.0;
  // RenderSettings.resolve (renderer.py:60-65)
  const double base = fmin(vol->spacing[0], fmin(vol->spacing[1], vol->spacing[2]));
  P.step = s->step_size > 0 ? s->step_size : 0.5 * base;
  P.ref = s->reference_step > 0 ? s->reference_step : base;
  FV_REQUIRE(s->shadow_step_factor >= 1, "shadow_step_factor must be >= 1");
  FV_REQUIRE(s->precision == FV_PREC_FP32 || s->precision == FV_PREC_FP32_STRICT || s->precision == FV_PREC_FP64,
             "precision must be FV_PREC_FP32, FV_PREC_FP32_STRICT or FV_PREC_FP64, got %d", (int)s->precision);
  P.step_sh = P.step * s->shadow_step_factor;
  P.early = s->early_term_alpha;
  P.ambient = s->ambient;
  P.min_trans = s->shadow_min_transmittance;
  for (int a = 0; a < 4; ++a) P.bg[a] = s->background[a];
  P.idx = idx; P.k_dev = k; P.k_max = k_max;
  P.rgba = rgba; P.depth = depth; P.net_in = net_in; P.net_wp = net_wp;
  P.counters = ctx->counters;
  // graph replays read the camera from the FrameDyn block (the wavefront fp32 path: its ray setup
  // and the overflow re-march are the only ray-generating kernels there)
  P.dyn = s->precision == FV_PREC_FP64 ? nullptr : ctx->dyn_active;
  if (k_max <= 0) return 0;
  const int threads = 128;
  const int blocks = (k_max + threads - 1) / threads;
  if (s->precision == FV_PREC_FP64) {
    FV_TIMED(ctx, FV_KC_MARCH_MAIN, march_kernel<double><<<blocks, threads, 0, ctx->stream>>>(P));
  } else {
    fv_volume* mv = const_cast<fv_volume*>(vol);  // the quad copy is a cache of the grid
    // variant 3: the wavefront passes; 2: one thread per ray (march_fast_kernel), which the naive
    // renderer forces (its idle lanes are the point) and FV_MARCH_KERNEL=ray selects everywhere
    static const bool env_ray = getenv("FV_MARCH_KERNEL") && strcmp(getenv("FV_MARCH_KERNEL"), "ray") == 0;
    const int variant = force_variant >= 0 ? force_variant : env_ray ? 2 : 3;
    // Quads come from a point-sampled 3D texture (block-linear layout, hardware clamp addressing:
    // A/B -43 us per C3 frame versus the bricked buffer, which the thread-per-ray variants and
    // FV_VOL_TEX=0 still use).
    static const bool use_tex = !(getenv("FV_VOL_TEX") && atoi(getenv("FV_VOL_TEX")) == 0);
    const bool tex_path = use_tex && variant == 3;
    // Sample source of the wavefront passes (`src`, the kernels' TEX parameter):
    //   1  quads (v00, v01-v00, v10, v11-v10) from a point-sampled float4 texture, software
    //      trilinear in fp32 (two 16-byte returns per sample; 4 floats per voxel)
    //   2  a hardware-filtered float texture: trilinear with 8-bit fractional weights (one 4-byte
    //      return per sample; 1 float per voxel) -- the SURVEY's fast tier
    // FV_TEX_FILTER: 0 = quads everywhere, 1 = filtered shadow samples only, 2 = filtered
    // everywhere (the quad texture is then never built). Default: 2 when the call asks for no depth
    // output (the frame loop: the network input is RGBA only) or the volume's quad copy would exceed
    // 4 GiB, else 1. The filtered main pass keeps the fast tier on colour (tests/test_headline_parity:
    // RGBA max |err| and PSNR per C3 / C2 frame); its first-hit depth is one step off on ~0.03% of
    // the active pixels, so calls that return depth keep the quads. Measured at C3 on the frame
    // timeline: main pass 117.5 -> 103.5 us, frame 1594 -> 1575 us; at 1024^3 30.6 instead of 47.8 GB.
    // The 8-bit weights cost more on coarse grids (features span few voxels): measured over the
    // active pixels of a foveated frame, filtered main-pass samples reach 76.9 / 89.0 / 95.6 dB at
    // 40x36x32 / 128^3 / 256^3 (quads 85.6 / 97.6 / 100), so volumes below 128 voxels per axis
    // keep the quads in the main pass.
    static const int tex_filter_env = getenv("FV_TEX_FILTER") ? atoi(getenv("FV_TEX_FILTER")) : -1;
    const bool big = 16.0 * vol->nx * vol->ny * vol->nz > 4.0 * 1024 * 1024 * 1024;
    const bool fine = std::min(vol->nx, std::min(vol->ny, vol->nz)) >= 128;
    const int tex_filter = s->precision == FV_PREC_FP32_STRICT ? 0
                           : tex_filter_env >= 0                ? tex_filter_env
                           : (big || (!P.depth && fine))        ? 2
                                                                : 1;
    const int src = !tex_path ? 0 : tex_filter >= 2 ? 2 : 1;
    int rc = src == 0 ? volume_bricks(ctx, mv) : src == 1 ? volume_texture(ctx, mv) : 0;
    if (rc) return rc;
    FastParams F;
    F.P = P;
    F.V.quads = reinterpret_cast<const float4*>(mv->bricks);
    F.V.tex = src == 1 ? (cudaTextureObject_t)mv->qtex : 0;
    F.V.ltex = 0;
    if (tex_path && tex_filter >= 1) {
      rc = volume_ltex(ctx, mv);
      if (rc) return rc;
      F.V.ltex = (cudaTextureObject_t)mv->ltex;
    }
    F.V.nx = vol->nx; F.V.ny = vol->ny; F.V.nz = vol->nz;
    const int nbx = (vol->nx + 7) / 8, nby = (vol->ny + 7) / 8;
    F.V.sby = nbx * 512;
    F.V.sbz = nbx * nby * 512;
    for (int a = 0; a < 3; ++a) {
      F.V.ext[a] = (float)P.ext[a];
      F.V.inv_sp[a] = (float)(1.0 / vol->spacing[a]);
      F.V.qmax[a] = (float)((a == 0 ? vol->nx : a == 1 ? vol->ny : vol->nz) - 0.5);
      F.ld[a] = (float)P.lvec[a];
      F.lpos[a] = (float)P.lvec[a];
      float sdir = F.ld[a];
      if (fabsf(sdir) < 1e-30f) sdir = sdir < 0.f ? -1e-30f : 1e-30f;
      F.ld_inv[a] = 1.f / sdir;
    }
    F.e_main = (float)(P.step / P.ref);
    F.e_sh = (float)(P.step_sh / P.ref);
    F.cls_main = exp_class(P.step / P.ref);
    F.cls_sh = exp_class(P.step_sh / P.ref);
    F.inv_ref = (float)(1.0 / P.ref);
    F.step_sh = (float)P.step_sh;
    F.inv_step_sh = 1.f / F.step_sh;
    F.min_trans = (float)P.min_trans;
    F.ambient = (float)P.ambient;
    for (int a = 0; a < 3; ++a) F.qs_sh[a] = F.ld[a] * F.V.inv_sp[a] * F.step_sh;
    if (variant == 3) {
      // wavefront: main -> shadow -> composite
      // Record buffer, in chunks of kChunk slots (36 B per slot). The first min(k, n_chunks / 2)
      // chunks are the first chunks of rays 0..k-1 (chunk id = ray index; k = this frame's ray
      // count, read on the device); the rest is the pool for later chunks (and the first chunks of
      // any rays beyond). Initial size 32 slots per film pixel (at least 8M, at most 128M): a C3 frame
      // writes ~24 records per film pixel, so foveated frames never overflow and their results do
      // not depend on the buffer's history. The buffer then follows this context's usage -- the
      // previous render's pooled-chunk and overflow counts are read back asynchronously into pinned
      // memory (a readback still in flight is not waited for) -- and never shrinks. A frame whose
      // records do not fit is still correct: its overflowing rays are re-marched one thread per ray
      // (inline shadows) after the main pass. FV_WAVE_REC_PER_RAY fixes the size at that many
      // slots per film pixel, FV_WAVE_REC_CAP at an absolute slot count (tests force the overflow
      // fallback with a tiny one); both disable the feedback.
      static const int64_t per_ray_env = getenv("FV_WAVE_REC_PER_RAY") ? std::max(1, atoi(getenv("FV_WAVE_REC_PER_RAY"))) : 0;
      static const int64_t cap_env = getenv("FV_WAVE_REC_CAP") ? std::max(2 * kChunk, atoi(getenv("FV_WAVE_REC_CAP"))) : 0;
      {
        cudaStreamCaptureStatus cap_st = cudaStreamCaptureStatusNone;
        FV_CUDA(cudaStreamIsCapturing(ctx->stream, &cap_st));
        const bool capturing = cap_st != cudaStreamCaptureStatusNone;
        const int64_t have = ctx->wave_cap / kChunk;
        int64_t need = have;
        if (cap_env || per_ray_env) {
          need = (cap_env ? cap_env : per_ray_env * k_max) / kChunk;
        } else if (have == 0) {
          // 32 slots per film pixel, at least 8M and at most 128M slots (4.6 GB) to start with
          need = std::min<int64_t>(std::max<int64_t>((8 << 20) / kChunk, (int64_t)k_max), (128 << 20) / kChunk);
        } else if (ctx->wave_fb_pending && !capturing && cudaEventQuery(ctx->wave_fb_ev) == cudaSuccess) {
          ctx->wave_fb_pending = false;
          const int64_t k_prev = ctx->wave_fb[0], pooled = ctx->wave_fb[1 + 1], ovf = ctx->wave_fb[1 + 6];
          const int64_t first = std::min(k_prev, have / 2), pool = have - first;
          // grow in large steps: a reallocation synchronises the device and maps new pages (a C4
          // dense zoomed frame that grew the buffer took ~0.3 s), so it should happen rarely
          if (ovf) need = 2 * have;
          else if (pooled > pool - pool / 8) need = std::max(first + 2 * pooled, 2 * have);
        } else {
          (void)cudaGetLastError();  // cudaEventQuery's cudaErrorNotReady is not an error here
        }
        need = std::min<int64_t>(need, INT32_MAX / kChunk);
        if (need > have || (cap_env || per_ray_env) && need != have) {
          if (ctx->wave_rec) cudaFree(ctx->wave_rec);
          ctx->wave_rec = nullptr;
          ctx->wave_cap = 0;
          // on an allocation failure retry smaller (the overflow path handles what does not fit)
          for (int64_t n = need; n >= 64 && !ctx->wave_rec; n /= 2) {
            const size_t bytes = (sizeof(float4) * 2 + sizeof(float)) * (size_t)(n * kChunk) + 3 * sizeof(int) * (size_t)n +
                                 64 * sizeof(int);
            if (cudaMalloc(&ctx->wave_rec, bytes) == cudaSuccess) {
              ctx->wave_cap = n * kChunk;
              ++ctx->wave_version;
            } else {
              ctx->wave_rec = nullptr;
              (void)cudaGetLastError();
            }
          }
          FV_REQUIRE(ctx->wave_rec, "cudaMalloc of the marcher record buffer failed");
        }
        if (!ctx->wave_fb) {
          FV_CUDA(cudaMallocHost(&ctx->wave_fb, 8 * sizeof(unsigned int)));
          FV_CUDA(cudaEventCreateWithFlags(&ctx->wave_fb_ev, cudaEventDisableTiming));
        }
      }
      if (k_max > ctx->wave_ray_cap) {
        if (ctx->wave_ray) cudaFree(ctx->wave_ray);
        ctx->wave_ray = nullptr;
        FV_CUDA(cudaMalloc(&ctx->wave_ray, sizeof(int4) * k_max));
        ctx->wave_ray_cap = k_max;
      }
      WaveBufs B;
      B.rec0 = reinterpret_cast<float4*>(ctx->wave_rec);
      B.rec1 = B.rec0 + ctx->wave_cap;
      B.shade = reinterpret_cast<float*>(B.rec1 + ctx->wave_cap);
      B.n_chunks_cap = (int)std::min<int64_t>(ctx->wave_cap / kChunk, INT32_MAX / kChunk);
      B.chunk_next = reinterpret_cast<int*>(B.shade + ctx->wave_cap);
      B.chunk_fill = B.chunk_next + ctx->wave_cap / kChunk;
      B.chunk_count = &ctx->counters->wave_rec;
      B.next = &ctx->counters->wave_next;
      B.ray = reinterpret_cast<int4*>(ctx->wave_ray);
      static const int chunk_pool = getenv("FV_CHUNK_POOL") ? std::max(1, atoi(getenv("FV_CHUNK_POOL"))) : 8;
      B.chunk_pool = chunk_pool;
      static const int claim = getenv("FV_MAIN_CLAIM") ? std::min(32, std::max(1, atoi(getenv("FV_MAIN_CLAIM")))) : 2;
      B.claim = claim;
      if (k_max > ctx->wave_hits_cap) {
        if (ctx->wave_hits) cudaFree(ctx->wave_hits);
        ctx->wave_hits = nullptr;
        FV_CUDA(cudaMalloc(&ctx->wave_hits, 3 * sizeof(float4) * (size_t)k_max));
        ctx->wave_hits_cap = k_max;
      }
      B.hits = reinterpret_cast<float4*>(ctx->wave_hits);
      B.hit_count = &ctx->counters->hit_count;
      // headers at hit-list positions, composite over the hits only (FV_COMP_HITS=0: by compacted
      // ray, every ray visited; C3 composite 56.5 -> 42.2 us)
      static const bool by_hit = !(getenv("FV_COMP_HITS") && atoi(getenv("FV_COMP_HITS")) == 0);
      B.by_hit = by_hit ? 1 : 0;
      B.hit_next = &ctx->counters->hit_next;
      if (k_max > ctx->wave_ovf_cap) {
        if (ctx->wave_ovf) cudaFree(ctx->wave_ovf);
        ctx->wave_ovf = nullptr;
        FV_CUDA(cudaMalloc(&ctx->wave_ovf, sizeof(int) * (size_t)k_max));
        ctx->wave_ovf_cap = k_max;
      }
      B.ovf = reinterpret_cast<int*>(ctx->wave_ovf);
      B.ovf_count = &ctx->counters->ovf_count;
      // half of the chunk space holds first chunks at id = ray index (k_max may exceed it: later
      // rays then take pooled first chunks); ord lists the non-empty ones in ray order
      B.cap_a = B.n_chunks_cap / 2;  // at most; the kernels take min(k, cap_a) on the device
      B.ord = B.chunk_fill + ctx->wave_cap / kChunk;
      B.ord_count = &ctx->counters->wave_ord;
      // ray_next, wave_rec, wave_next, wave_ord, hit_count, hit_next, ovf_count are consecutive
      FV_CUDA(cudaMemsetAsync(&ctx->counters->ray_next, 0, 7 * sizeof(unsigned int), ctx->stream));
      rc = src == 2 ? launch_main<2>(ctx, F, B, threads) : src == 1 ? launch_main<1>(ctx, F, B, threads)
                                                            : launch_main<0>(ctx, F, B, threads);
      if (rc) return rc;
      if (P.light_kind != FV_LIGHT_NONE) {
        // rays that found the record buffer full: inline shadows, one thread per ray (a grid that
        // exits at once when the list is empty)
        FastParams Fo = F;
        Fo.P.idx = B.ovf;
        Fo.P.k_dev = reinterpret_cast<const int32_t*>(B.ovf_count);
        if (src == 2)
          FV_TIMED(ctx, FV_KC_MARCH_MAIN, march_fast_kernel<2><<<ctx->num_sms, threads, 0, ctx->stream>>>(Fo, false));
        else if (src == 1)
          FV_TIMED(ctx, FV_KC_MARCH_MAIN, march_fast_kernel<1><<<ctx->num_sms, threads, 0, ctx->stream>>>(Fo, false));
        else
          FV_TIMED(ctx, FV_KC_MARCH_MAIN, march_fast_kernel<0><<<ctx->num_sms, threads, 0, ctx->stream>>>(Fo, false));
        ctx->launches += 1;
      }
      if (P.light_kind != FV_LIGHT_NONE) {
        // blocks per SM (FV_FIRST_BPS): 8 covers the compacted rays in ~1 round (C3 10.7 -> 8.6 us vs 2)
        static const int fl_bps = getenv("FV_FIRST_BPS") ? std::max(1, atoi(getenv("FV_FIRST_BPS"))) : 8;
        FV_TIMED(ctx, FV_KC_MARCH_COMPOSITE, first_list_kernel<<<ctx->num_sms * fl_bps, 256, 0, ctx->stream>>>(F, B));
        ctx->launches += 1;
        // directional lights on the texture path: the partial-refill pass (FV_SHADOW_V=1: the
        // all-lane-refill pass, which point lights and the bricked path use)
        static const int shadow_v = getenv("FV_SHADOW_V") ? atoi(getenv("FV_SHADOW_V")) : 2;
        if (src && P.light_kind == FV_LIGHT_DIRECTIONAL && shadow_v == 2)
          rc = launch_shadow_dir(ctx, F, B, threads);  // (filtered samples whenever F.V.ltex is set)
        else
          rc = src == 2 ? launch_shadow<2>(ctx, F, B, threads) : src == 1 ? launch_shadow<1>(ctx, F, B, threads)
                                                                : launch_shadow<0>(ctx, F, B, threads);
        if (rc) return rc;
        FV_TIMED(ctx, FV_KC_MARCH_COMPOSITE, march_wave_composite_kernel<<<ctx->num_sms * 16, threads, 0, ctx->stream>>>(F, B));
        ctx->launches += 2;
      }
      // record usage of this frame for the next one's buffer sizing (not inside a graph capture,
      // and not while the previous readback is still unread)
      cudaStreamCaptureStatus cap_st = cudaStreamCaptureStatusNone;
      FV_CUDA(cudaStreamIsCapturing(ctx->stream, &cap_st));
      if (cap_st == cudaStreamCaptureStatusNone && !ctx->wave_fb_pending) {
        if (P.k_dev)
          FV_CUDA(cudaMemcpyAsync(ctx->wave_fb, P.k_dev, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
        else
          ctx->wave_fb[0] = (unsigned)k_max;
        FV_CUDA(cudaMemcpyAsync(ctx->wave_fb + 1, &ctx->counters->ray_next, 7 * sizeof(unsigned int),
                                cudaMemcpyDeviceToHost, ctx->stream));
        FV_CUDA(cudaEventRecord(ctx->wave_fb_ev, ctx->stream));
        ctx->wave_fb_pending = true;
      }
    } else {
      FV_TIMED(ctx, FV_KC_MARCH_MAIN, march_fast_kernel<false><<<blocks, threads, 0, ctx->stream>>>(F, true));
    }
  }
  FV_CHECK_LAUNCH("march_kernel");
  ctx->launches += 1;
  return 0;
}

}  // namespace fv

// ---- Boundary ops: the reference's per-sample building blocks as device calls ------------------
// (volume.generate_rays :293-303, volume.sample_trilinear :149-180, TransferFunction.apply
// :201-208, noise.tile_field :378-384), fp64 like the reference. The marcher inlines the same
// arithmetic; these entry points serve callers of the individual functions.
namespace fv {
namespace {

__global__ void generate_rays_kernel(MarchParams P, const int32_t* __restrict__ us, const int32_t* __restrict__ vs,
                                     int64_t n, double* __restrict__ orig, double* __restrict__ dirs) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double sx = (((double)us[i] + 0.5) / P.W * 2.0 - 1.0) * P.tan_half * P.aspect;
    const double sy = (1.0 - ((double)vs[i] + 0.5) / P.H * 2.0) * P.tan_half;
    double d[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) d[a] = P.fwd[a] + sx * P.right[a] + sy * P.up[a];
    const double nrm = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      dirs[3 * i + a] = d[a] / nrm;
      orig[3 * i + a] = P.pos[a];
    }
  }
}

__global__ void sample_trilinear_kernel(MarchParams P, const double* __restrict__ pts, int64_t n,
                                        double* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double p[3] = {pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]};
    out[i] = trilinear<double>(P, p);
  }
}

__global__ void tf_apply_kernel(const float* __restrict__ lut, int K, const double* __restrict__ s, int64_t n,
                                double* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double c[4];
    // np.clip propagates NaN; tf_apply's comparisons would map it to 0 -- keep the reference's NaN
    if (s[i] != s[i]) {
      for (int a = 0; a < 4; ++a) out[4 * i + a] = s[i];
      continue;
    }
    tf_apply<double>(lut, K, s[i], c);
#pragma unroll
    for (int a = 0; a < 4; ++a) out[4 * i + a] = c[a];
  }
}

__global__ void tile_field_kernel(const float* __restrict__ noise, int T, int th, int tw, int frame, int h, int w,
                                  float* __restrict__ out) {
  const float* f = noise + (int64_t)(frame % T) * th * tw;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (int64_t)h * w; i += (int64_t)gridDim.x * blockDim.x) {
    const int u = (int)(i % w), v = (int)(i / w);
    out[i] = f[(v % th) * tw + (u % tw)];
  }
}

int grid_for(const fv_ctx* ctx, int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, ctx->num_sms * 16)); }

int camera_params(const fv_camera* cam, MarchParams& P) {
  FV_REQUIRE(cam->width >= 1 && cam->height >= 1, "film dims must be positive");
  FV_REQUIRE(cam->fov_y > 0.0 && cam->fov_y < 180.0, "fov_y must be in (0, 180) degrees, got %g", cam->fov_y);
  double fwd[3] = {cam->look_at[0] - cam->position[0], cam->look_at[1] - cam->position[1],
                   cam->look_at[2] - cam->position[2]};
  FV_REQUIRE(fwd[0] != 0 || fwd[1] != 0 || fwd[2] != 0, "camera position and look_at coincide");
  normalize3(fwd);
  double right[3] = {fwd[1] * cam->up[2] - fwd[2] * cam->up[1], fwd[2] * cam->up[0] - fwd[0] * cam->up[2],
                     fwd[0] * cam->up[1] - fwd[1] * cam->up[0]};
  FV_REQUIRE(sqrt(right[0] * right[0] + right[1] * right[1] + right[2] * right[2]) > 0,
             "up vector is parallel to the view direction");
  normalize3(right);
  const double up[3] = {right[1] * fwd[2] - right[2] * fwd[1], right[2] * fwd[0] - right[0] * fwd[2],
                        right[0] * fwd[1] - right[1] * fwd[0]};
  for (int a = 0; a < 3; ++a) {
    P.pos[a] = cam->position[a]; P.fwd[a] = fwd[a]; P.right[a] = right[a]; P.up[a] = up[a];
  }
  P.tan_half = tan(cam->fov_y * (M_PI / 180.0) * 0.5);
  P.aspect = (double)cam->width / (double)cam->height;
  P.W = cam->width;
  P.H = cam->height;
  return 0;
}

}  // namespace
}  // namespace fv

extern "C" {

int fv_generate_rays(fv_ctx* ctx, const fv_camera* cam, const int32_t* us_dev, const int32_t* vs_dev, int64_t n,
                     double* origins_dev, double* dirs_dev) {
  FV_REQUIRE(ctx && cam && (n == 0 || (us_dev && vs_dev && origins_dev && dirs_dev)), "null argument");
  fv::MarchParams P{};
  const int rc = fv::camera_params(cam, P);
  if (rc) return rc;
  if (n == 0) return 0;
  fv::generate_rays_kernel<<<fv::grid_for(ctx, n), 256, 0, ctx->stream>>>(P, us_dev, vs_dev, n, origins_dev, dirs_dev);
  FV_CHECK_LAUNCH("generate_rays_kernel");
  ctx->launches += 1;
  return 0;
}

int fv_sample_trilinear(fv_ctx* ctx, const fv_volume* vol, const double* pts_dev, int64_t n, double* out_dev) {
  FV_REQUIRE(ctx && vol && vol->data && (n == 0 || (pts_dev && out_dev)), "null argument");
  fv::MarchParams P{};
  P.data = vol->data; P.nx = vol->nx; P.ny = vol->ny; P.nz = vol->nz;
  for (int a = 0; a < 3; ++a) P.sp[a] = vol->spacing[a];
  P.ext[0] = vol->nx * vol->spacing[0]; P.ext[1] = vol->ny * vol->spacing[1]; P.ext[2] = vol->nz * vol->spacing[2];
  if (n == 0) return 0;
  fv::sample_trilinear_kernel<<<fv::grid_for(ctx, n), 256, 0, ctx->stream>>>(P, pts_dev, n, out_dev);
  FV_CHECK_LAUNCH("sample_trilinear_kernel");
  ctx->launches += 1;
  return 0;
}

int fv_tf_apply(fv_ctx* ctx, const float* lut_dev, int K, const double* s_dev, int64_t n, double* out_dev) {
  FV_REQUIRE(ctx && lut_dev && (n == 0 || (s_dev && out_dev)), "null argument");
  FV_REQUIRE(K >= 2 && K <= 256, "transfer function lut must be (K>=2, 4), got K=%d", K);
  if (n == 0) return 0;
  fv::tf_apply_kernel<<<fv::grid_for(ctx, n), 256, 0, ctx->stream>>>(lut_dev, K, s_dev, n, out_dev);
  FV_CHECK_LAUNCH("tf_apply_kernel");
  ctx->launches += 1;
  return 0;
}

int fv_tile_field(fv_ctx* ctx, int frame, int h, int w, float* out_dev) {
  FV_REQUIRE(ctx && out_dev, "null argument");
  FV_REQUIRE(ctx->noise, "no noise stack uploaded (fv_noise_upload)");
  FV_REQUIRE(h >= 1 && w >= 1, "dims must be positive, got (%d, %d)", h, w);
  FV_REQUIRE(frame >= 0, "frame must be >= 0");
  fv::tile_field_kernel<<<fv::grid_for(ctx, (int64_t)h * w), 256, 0, ctx->stream>>>(
      ctx->noise, ctx->noise_T, ctx->noise_H, ctx->noise_W, frame, h, w, out_dev);
  FV_CHECK_LAUNCH("tile_field_kernel");
  ctx->launches += 1;
  return 0;
}

}  // extern "C"

namespace fv {
// Camera.basis (volume.py:269-276) and the generate_rays constants into a FrameDyn block.
int fill_camera_dyn(const fv_camera* cam, FrameDyn* d) {
  MarchParams P{};
  const int rc = camera_params(cam, P);
  if (rc) return rc;
  for (int a = 0; a < 3; ++a) {
    d->pos[a] = P.pos[a]; d->right[a] = P.right[a]; d->up[a] = P.up[a]; d->fwd[a] = P.fwd[a];
  }
  d->tan_half = P.tan_half;
  d->aspect = P.aspect;
  return 0;
}
}  // namespace fv

