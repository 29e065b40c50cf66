/*
 * CPU ORACLE -- test infrastructure only (tests/, __graft_entry__.smoke(), bench.py's
 * cpu_baseline / --impl reference legs). Never linked into the product library.
 *
 * Scalar fp64 restatement of the reference ray marcher, one ray at a time:
 *   generate_rays          pkg/src/fovray/volume.py:293-303
 *   _ray_box               pkg/src/fovray/renderer.py:88-98
 *   sample_trilinear       pkg/src/fovray/volume.py:149-180
 *   TransferFunction.apply pkg/src/fovray/volume.py:201-208
 *   shadow_transmittance   pkg/src/fovray/renderer.py:109-147
 *   _march                 pkg/src/fovray/renderer.py:150-195
 * The reference advances a batch of rays in lockstep with NumPy, but every lane's arithmetic
 * depends only on that lane (renderer.py:3-7), so marching rays one by one with the same
 * operation order reproduces its float64 results; pow() is the same libm call NumPy makes.
 * Parity with the reference is pinned by tests/test_oracle.py against the golden renders
 * (including the reference's own SHA-256 golden image, tests/test_renderer.py:109-114).
 *
 * Build: see oracle/Makefile (gcc -O2 -pthread -ffp-contract=off).
 */
#include <math.h>
#include <pthread.h>
#include <stdatomic.h>
#include <stdint.h>
#include <string.h>

typedef struct {
  const float* data; /* (nz, ny, nx) */
  int n[3];          /* nx, ny, nz */
  double sp[3];
  double ext[3];
  const float* lut; /* (K, 4) */
  int K;
  int light_kind; /* 0 none, 1 directional, 2 point */
  double ldir[3]; /* directional: unit vector toward the light */
  double lpos[3];
  double intensity[3];
  double step, ref, step_sh, early, ambient, min_trans;
  double bg[4];
} scene_t;

static void ray_box(const double o[3], const double d[3], const double ext[3], double* t0,
                    double* t1, int* hit) {
  double tmin = -INFINITY, tmax = INFINITY;
  for (int a = 0; a < 3; ++a) {
    double s = d[a];
    if (fabs(s) < 1e-30) s = s < 0 ? -1e-30 : 1e-30;
    double inv = 1.0 / s;
    double ta = (0.0 - o[a]) * inv;
    double tb = (ext[a] - o[a]) * inv;
    double lo = ta < tb ? ta : tb, hi = ta > tb ? ta : tb;
    if (a == 0 || lo > tmin) tmin = lo;
    if (a == 0 || hi < tmax) tmax = hi;
  }
  *t0 = tmin > 0.0 ? tmin : 0.0;
  *t1 = tmax;
  *hit = tmax > *t0;
}

static double trilinear(const scene_t* s, const double p[3]) {
  for (int a = 0; a < 3; ++a)
    if (!(p[a] >= 0.0 && p[a] <= s->ext[a])) return 0.0;
  int i0[3], i1[3];
  double t[3];
  for (int a = 0; a < 3; ++a) {
    double q = p[a] / s->sp[a] - 0.5;
    double f = floor(q);
    t[a] = q - f;
    long long fi = (long long)f;
    if (fi < 0) fi = 0;
    if (fi > s->n[a] - 1) fi = s->n[a] - 1;
    i0[a] = (int)fi;
    i1[a] = i0[a] + 1 > s->n[a] - 1 ? s->n[a] - 1 : i0[a] + 1;
  }
  const int64_t sy = s->n[0], sz = (int64_t)s->n[0] * s->n[1];
#define D(z, y, x) ((double)s->data[(int64_t)(z) * sz + (int64_t)(y) * sy + (x)])
  const double tx = t[0], ty = t[1], tz = t[2];
  double c00 = D(i0[2], i0[1], i0[0]) * (1 - tx) + D(i0[2], i0[1], i1[0]) * tx;
  double c10 = D(i0[2], i1[1], i0[0]) * (1 - tx) + D(i0[2], i1[1], i1[0]) * tx;
  double c01 = D(i1[2], i0[1], i0[0]) * (1 - tx) + D(i1[2], i0[1], i1[0]) * tx;
  double c11 = D(i1[2], i1[1], i0[0]) * (1 - tx) + D(i1[2], i1[1], i1[0]) * tx;
#undef D
  double c0 = c00 * (1 - ty) + c10 * ty;
  double c1 = c01 * (1 - ty) + c11 * ty;
  return c0 * (1 - tz) + c1 * tz;
}

static void tf(const scene_t* s, double v, double out[4]) {
  if (v < 0.0) v = 0.0;
  if (v > 1.0) v = 1.0;
  double x = v * (s->K - 1);
  long long i0 = (long long)floor(x);
  if (i0 < 0) i0 = 0;
  if (i0 > s->K - 2) i0 = s->K - 2;
  double t = x - (double)i0;
  for (int c = 0; c < 4; ++c)
    out[c] = (double)s->lut[i0 * 4 + c] * (1 - t) + (double)s->lut[(i0 + 1) * 4 + c] * t;
}

static double shadow_T(const scene_t* s, const double pt[3], int64_t* nsamp) {
  double dir[3], dist = INFINITY;
  if (s->light_kind == 1) {
    memcpy(dir, s->ldir, sizeof(dir));
  } else {
    double dl[3] = {s->lpos[0] - pt[0], s->lpos[1] - pt[1], s->lpos[2] - pt[2]};
    dist = sqrt(dl[0] * dl[0] + dl[1] * dl[1] + dl[2] * dl[2]);
    double m = dist > 1e-30 ? dist : 1e-30;
    for (int a = 0; a < 3; ++a) dir[a] = dl[a] / m;
  }
  double t0, t1;
  int hit;
  ray_box(pt, dir, s->ext, &t0, &t1, &hit);
  double t_end = t1 < dist ? t1 : dist;
  double trans = 1.0, t = t0;
  int live = hit && (t_end > t0);
  while (live) {
    double dt = t_end - t;
    if (s->step_sh < dt) dt = s->step_sh;
    double mid = t + 0.5 * dt;
    double p[3] = {pt[0] + dir[0] * mid, pt[1] + dir[1] * mid, pt[2] + dir[2] * mid};
    double c[4];
    tf(s, trilinear(s, p), c);
    double a_step = 1.0 - pow(1.0 - c[3], dt / s->ref);
    trans = trans * (1.0 - a_step);
    ++*nsamp;
    t = t + dt;
    live = (t < t_end - 1e-12) && (trans > s->min_trans);
  }
  return trans;
}

static void march_ray(const scene_t* s, const double o[3], const double d[3], float out[4],
                      float* depth_out, int64_t* nmain, int64_t* nshadow) {
  double t0, t_end;
  int hit;
  ray_box(o, d, s->ext, &t0, &t_end, &hit);
  const int lit = s->light_kind != 0;
  const double amb = lit ? s->ambient : 1.0;
  double rgb[3] = {0, 0, 0}, trans = 1.0, depth = 0.0, t = t0;
  int live = hit;
  while (live) {
    double dt = t_end - t;
    if (s->step < dt) dt = s->step;
    double mid = t + 0.5 * dt;
    double p[3] = {o[0] + d[0] * mid, o[1] + d[1] * mid, o[2] + d[2] * mid};
    double c[4];
    tf(s, trilinear(s, p), c);
    ++*nmain;
    double a_step = 1.0 - pow(1.0 - c[3], dt / s->ref);
    double shade = 1.0;
    if (lit && a_step > 0.0) shade = amb + (1.0 - amb) * shadow_T(s, p, nshadow);
    double contrib = trans * a_step;
    for (int ch = 0; ch < 3; ++ch) rgb[ch] += contrib * (c[ch] * (shade * s->intensity[ch]));
    trans = trans * (1.0 - a_step);
    double acc = 1.0 - trans;
    if (depth == 0.0 && acc >= 0.5) depth = mid;
    t = t + dt;
    live = (t < t_end - 1e-12) && (acc < s->early);
  }
  for (int ch = 0; ch < 3; ++ch) out[ch] = (float)(rgb[ch] + (trans * s->bg[3]) * s->bg[ch]);
  out[3] = (float)((1.0 - trans) + trans * s->bg[3]);
  *depth_out = (float)depth;
}

typedef struct {
  const scene_t* s;
  const double* cam;
  int W, H;
  const int64_t* pix;
  int64_t npix;
  float* rgba;
  float* depth;
  int64_t* counts;
  atomic_llong next;
} job_t;

static void* worker(void* arg) {
  job_t* j = (job_t*)arg;
  const double* cam = j->cam;
  for (;;) {
    long long start = atomic_fetch_add(&j->next, 64);
    if (start >= j->npix) break;
    long long end = start + 64 < j->npix ? start + 64 : j->npix;
    for (long long i = start; i < end; ++i) {
      const int64_t px = j->pix[i];
      const int u = (int)(px % j->W), v = (int)(px / j->W);
      const double sx = (((double)u + 0.5) / j->W * 2.0 - 1.0) * cam[12] * cam[13];
      const double sy = (1.0 - ((double)v + 0.5) / j->H * 2.0) * cam[12];
      double d[3];
      for (int a = 0; a < 3; ++a) d[a] = cam[9 + a] + sx * cam[3 + a] + sy * cam[6 + a];
      const double nrm = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
      for (int a = 0; a < 3; ++a) d[a] /= nrm;
      int64_t nm = 0, ns = 0;
      march_ray(j->s, cam, d, j->rgba + 4 * i, j->depth + i, &nm, &ns);
      if (j->counts) {
        j->counts[2 * i] = nm;
        j->counts[2 * i + 1] = ns;
      }
    }
  }
  return NULL;
}

/*
 * Render the pixels `pix` (flat v*W+u) of a W x H film on `nthreads` host threads.
 * cam: pos[3], right[3], up[3], fwd[3], tan_half, aspect (Camera.basis computed by the caller).
 * cfg: step, ref, step_sh, early, ambient, min_trans, bg[4].
 * counts: nullable, receives per-ray (main, shadow) sample counts.
 */
void oracle_render(const float* data, const int n[3], const double sp[3], const float* lut, int K,
                   int light_kind, const double lvec[3], const double intensity[3],
                   const double cfg[10], const double cam[14], int W, int H, const int64_t* pix,
                   int64_t npix, float* rgba, float* depth, int64_t* counts, int nthreads) {
  scene_t s;
  s.data = data;
  for (int a = 0; a < 3; ++a) {
    s.n[a] = n[a];
    s.sp[a] = sp[a];
    s.ext[a] = (double)n[a] * sp[a];
    s.intensity[a] = intensity[a];
    s.ldir[a] = lvec[a];
    s.lpos[a] = lvec[a];
  }
  s.lut = lut;
  s.K = K;
  s.light_kind = light_kind;
  s.step = cfg[0]; s.ref = cfg[1]; s.step_sh = cfg[2]; s.early = cfg[3];
  s.ambient = cfg[4]; s.min_trans = cfg[5];
  for (int a = 0; a < 4; ++a) s.bg[a] = cfg[6 + a];
  job_t job = {&s, cam, W, H, pix, npix, rgba, depth, counts, 0};
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  pthread_t th[256];
  for (int i = 1; i < nthreads; ++i) pthread_create(&th[i], NULL, worker, &job);
  worker(&job);
  for (int i = 1; i < nthreads; ++i) pthread_join(th[i], NULL);
}
