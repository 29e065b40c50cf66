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
};

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

template <typename Real>
__device__ __forceinline__ void tf_apply(const float* lut, int K, Real s, Real out[4]) {
  s = s < Real(0) ? Real(0) : (s > Real(1) ? Real(1) : s);
  const Real x = s * (Real)(K - 1);
  int i0 = (int)floor((double)x);
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
  int i0 = (int)floor((double)x);
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
  if (i < k) {
    const int pix = P.idx ? P.idx[i] : i;
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
  unsigned int r = (i < k) ? 1u : 0u;
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

void normalize3(double v[3]) {
  const double n = sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
  v[0] /= n; v[1] /= n; v[2] /= n;
}

}  // namespace

int launch_render(fv_ctx* ctx, const fv_volume* vol, const fv_camera* cam, const fv_light* light,
                  const fv_settings* s, const int32_t* idx, const int32_t* k, int k_max,
                  float* rgba, float* depth, __half* net_in, int net_wp) {
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
  P.step_sh = P.step * s->shadow_step_factor;
  P.early = s->early_term_alpha;
  P.ambient = s->ambient;
  P.min_trans = s->shadow_min_transmittance;
  for (int a = 0; a < 4; ++a) P.bg[a] = s->background[a];
  P.idx = idx; P.k_dev = k; P.k_max = k_max;
  P.rgba = rgba; P.depth = depth; P.net_in = net_in; P.net_wp = net_wp;
  P.counters = ctx->counters;
  if (k_max <= 0) return 0;
  const int threads = 128;
  const int blocks = (k_max + threads - 1) / threads;
  if (s->precision == FV_PREC_FP64)
    march_kernel<double><<<blocks, threads, 0, ctx->stream>>>(P);
  else
    march_kernel<float><<<blocks, threads, 0, ctx->stream>>>(P);
  FV_CHECK_LAUNCH("march_kernel");
  ctx->launches += 1;
  return 0;
}

}  // namespace fv
