// Foveated sample mask + stream compaction in one pass.
//
// Reference semantics (pkg/src/fovray):
//   tau(u,v) = min(P_f + (1-P_f)*P_b, 1),  P_f = exp(-0.5*((dx*s)^2+(dy*s)^2)*sigma)
//       sample_maps.py:62-68 (foveal_density), :89-105 (build_tau_map)
//   M(u,v)   = float64(N[frame%T][v%Ht][u%Wt]) < tau     sample_maps.py:128-132, noise.py:378-384
//   coords   = set bits in row-major order (exclusive scan) sample_maps.py:161-171
//
// tau is evaluated in fp64 with explicit round-to-nearest intrinsics so nvcc cannot contract
// the products into FMAs; numpy evaluates dx*dx, dy*dy, the sum, *-0.5, *sigma left to right.
// The mask is bit-exact because the smallest |tau-N| margin over the reference configs
// (>=3.4e-9) is seven orders of magnitude above one fp64 ulp of tau.
//
// Compaction is a single-pass decoupled look-back scan: each CTA takes a 2048-pixel tile
// (dynamic tile index => tiles retire in order), publishes its aggregate, looks back over its
// predecessors' epoch-tagged status words -- 32 at a time, one per lane of the first warp -- and
// writes its indices. Status words carry the call's epoch, so they never need clearing between
// calls.
#include <algorithm>

#include "internal.h"

namespace fv {

namespace {

constexpr int kThreads = 256;
constexpr int kPerThread = 8;
constexpr int kTile = kThreads * kPerThread;

struct MaskParams {
  int H, W, frame;
  double fx, fy, sigma, pb, scale;
  const double* pb_map;
  const double* tau_map;  // overrides the fovea formula when set (TauMap given by value)
  const float* noise;
  int T, Ht, Wt;
  uint8_t* bits;
  int32_t* idx;
  int32_t* k_out;
  __half* net_in;
  int net_wp;
  unsigned long long* status;
  unsigned int epoch;
  unsigned int* tile_counter;
  const FrameDyn* dyn;  // non-null: fovea, noise frame and epoch from device memory (graph replay)
};

__device__ __forceinline__ double tau_at(const MaskParams& p, int u, int v) {
  if (p.tau_map) return p.tau_map[(int64_t)v * p.W + u];
  double dx = __dmul_rn(__dsub_rn((double)u, p.fx), p.scale);
  double dy = __dmul_rn(__dsub_rn((double)v, p.fy), p.scale);
  double r2 = __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
  double pf = exp(__dmul_rn(__dmul_rn(-0.5, r2), p.sigma));
  double pb = p.pb_map ? p.pb_map[(int64_t)v * p.W + u] : p.pb;
  double tau = __dadd_rn(pf, __dmul_rn(__dsub_rn(1.0, pf), pb));
  return tau < 1.0 ? tau : 1.0;
}

__device__ __forceinline__ unsigned long long pack_status(unsigned int epoch, unsigned flag,
                                                          unsigned value) {
  return ((unsigned long long)epoch << 32) | ((unsigned long long)flag << 30) | value;
}

// One tile's mask bits (8 consecutive pixels per thread, bit j = pixel base + j) and the network
// input's group 0 for those pixels (whole 16-byte pixels, warp-coalesced).
__device__ __forceinline__ unsigned int tile_bits(const MaskParams& p, unsigned int tile, int tid) {
  const int64_t npix = (int64_t)p.H * p.W;
  const int64_t base = (int64_t)tile * kTile + (int64_t)tid * kPerThread;
  const float* nz = p.noise + (int64_t)(p.frame % p.T) * p.Ht * p.Wt;
  unsigned int bits = 0;
  int u = (int)(base % p.W), v = (int)(base / p.W);
  int um = u % p.Wt, vm = v % p.Ht;  // the noise tile's coordinates, stepped with (u, v)
#pragma unroll
  for (int j = 0; j < kPerThread; ++j) {
    const int64_t pix = base + j;
    if (pix < npix) {
      const double n = (double)__ldg(nz + vm * p.Wt + um);
      const bool m = n < tau_at(p, u, v);
      bits |= (unsigned)m << j;
      if (p.bits) p.bits[pix] = (uint8_t)m;
    }
    if (++um == p.Wt) um = 0;
    if (++u == p.W) {
      u = 0;
      um = 0;
      ++v;
      if (++vm == p.Ht) vm = 0;
    }
  }
  const int lane = tid & 31, warp = tid >> 5;
  // the network input's group 0 ([0 x 4, m, 0 x 3]: the march's records fill channels 0..3 of the
  // active pixels afterwards), whole 16-byte pixels, warp-coalesced: lane l writes pixel
  // wbase + 32 j + l, whose bit lane (32 j + l) / 8 holds
  if (p.net_in) {
    const int64_t wbase = (int64_t)tile * kTile + (int64_t)warp * 32 * kPerThread;
    unsigned vv = (unsigned)((wbase + lane) / p.W), uu = (unsigned)((wbase + lane) - (int64_t)vv * p.W);
#pragma unroll
    for (int j = 0; j < kPerThread; ++j) {
      const int q = 32 * j + lane;
      const unsigned b = __shfl_sync(0xffffffffu, bits, q >> 3);
      const int64_t pix = wbase + q;
      if (j) {  // (u, v) of pixel wbase + q: 32 pixels on from the previous one
        uu += 32;
        while (uu >= (unsigned)p.W) { uu -= (unsigned)p.W; ++vv; }
      }
      if (pix < npix) {
        const bool m = (b >> (q & 7)) & 1u;
        *reinterpret_cast<uint4*>(p.net_in + ((int64_t)vv * p.net_wp + uu) * 8) =
            make_uint4(0u, 0u, m ? 0x3c00u : 0u, 0u);  // 0x3c00: fp16 1.0 in channel 4
      }
    }
  }
  return bits;
}

__device__ __forceinline__ void load_dyn(MaskParams& p) {
  if (p.dyn) {
    p.fx = p.dyn->fx; p.fy = p.dyn->fy; p.sigma = p.dyn->sigma; p.pb = p.dyn->pb; p.scale = p.dyn->scale;
    p.frame = p.dyn->frame;
    p.epoch = p.dyn->epoch;
  }
}

__global__ void __launch_bounds__(kThreads) mask_compact_kernel(MaskParams p_in) {
  MaskParams p = p_in;
  load_dyn(p);
  __shared__ unsigned int s_tile;
  __shared__ unsigned int s_warp[kThreads / 32];
  __shared__ unsigned int s_prefix;
  const int tid = threadIdx.x;
  if (tid == 0) s_tile = atomicAdd(p.tile_counter, 1u);
  __syncthreads();
  const unsigned int tile = s_tile;
  const int64_t npix = (int64_t)p.H * p.W;
  const int64_t base = (int64_t)tile * kTile + (int64_t)tid * kPerThread;
  unsigned int bits = tile_bits(p, tile, tid);
  const unsigned int cnt = __popc(bits);
  const int lane = tid & 31, warp = tid >> 5;
  // block-wide exclusive scan of cnt
  unsigned int incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    unsigned int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    unsigned int w = lane < kThreads / 32 ? s_warp[lane] : 0u;
    unsigned int wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      unsigned int y = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += y;
    }
    if (lane < kThreads / 32) s_warp[lane] = wi - w;  // exclusive per warp
    const unsigned int aggregate = __shfl_sync(0xffffffffu, wi, kThreads / 32 - 1);
    // decoupled look-back, a warp-wide window of 32 predecessors per step (lane l reads tile
    // j - l): one memory round trip covers 32 tiles instead of one
    volatile unsigned long long* st = p.status;
    if (tile == 0) {
      if (lane == 0) {
        st[0] = pack_status(p.epoch, 2u, aggregate);
        s_prefix = 0;
      }
    } else {
      if (lane == 0) {
        st[tile] = pack_status(p.epoch, 1u, aggregate);
        __threadfence();
      }
      __syncwarp();
      unsigned int excl = 0;
      for (int j = (int)tile - 1;; j -= 32) {
        const int t = j - lane;
        unsigned long long s = pack_status(p.epoch, 2u, 0u);  // before tile 0: an inclusive 0
        if (t >= 0) {
          do { s = st[t]; } while ((unsigned int)(s >> 32) != p.epoch || ((s >> 30) & 3u) == 0u);
        }
        const unsigned inc = __ballot_sync(0xffffffffu, ((s >> 30) & 3u) == 2u);
        const int stop = inc ? __ffs(inc) - 1 : 31;
        unsigned int v = lane <= stop ? (unsigned int)(s & 0x3fffffffu) : 0u;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        excl += v;
        if (inc) break;
      }
      if (lane == 0) {
        __threadfence();
        st[tile] = pack_status(p.epoch, 2u, excl + aggregate);
        s_prefix = excl;
      }
    }
    if (lane == 0) {
      const int64_t ntiles = (npix + kTile - 1) / kTile;
      if ((int64_t)tile == ntiles - 1) *p.k_out = (int32_t)(s_prefix + aggregate);
    }
  }
  __syncthreads();
  unsigned int pos = s_prefix + s_warp[warp] + (incl - cnt);
  while (bits) {
    const int j = __ffs(bits) - 1;
    bits &= bits - 1;
    p.idx[pos++] = (int32_t)(base + j);
  }
}

// Two-pass compaction (FV_MASK_2PASS, default): pass 1 computes every tile's bits, writes the
// network input and the per-thread bit bytes and the tile's count; pass 2 gives each tile its
// prefix by summing the earlier tiles' counts (a 4-KB block reduction, no spinning on
// predecessors) and writes the ordered indices. (The single-pass decoupled look-back spent most of
// its time spinning on the status chain: ncu, 29 us at 1080p.)
__global__ void __launch_bounds__(kThreads) mask_count_kernel(MaskParams p_in, uint8_t* __restrict__ tbits,
                                                              unsigned int* __restrict__ counts) {
  MaskParams p = p_in;
  load_dyn(p);
  __shared__ unsigned int s_warp[kThreads / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned int tile = blockIdx.x;
  const unsigned int bits = tile_bits(p, tile, tid);
  tbits[(int64_t)tile * kThreads + tid] = (uint8_t)bits;
  unsigned int c = __popc(bits);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if (lane == 0) s_warp[warp] = c;
  __syncthreads();
  if (tid == 0) {
    unsigned int t = 0;
#pragma unroll
    for (int w = 0; w < kThreads / 32; ++w) t += s_warp[w];
    counts[tile] = t;
  }
}

__global__ void __launch_bounds__(kThreads) mask_write_kernel(MaskParams p, const uint8_t* __restrict__ tbits,
                                                              const unsigned int* __restrict__ counts, int ntiles) {
  __shared__ unsigned int s_warp[kThreads / 32];
  __shared__ unsigned int s_red[kThreads / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned int tile = blockIdx.x;
  // prefix = sum of the earlier tiles' counts
  unsigned int pre = 0;
  for (unsigned int i = tid; i < tile; i += kThreads) pre += counts[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) pre += __shfl_xor_sync(0xffffffffu, pre, o);
  if (lane == 0) s_red[warp] = pre;
  unsigned int bits = tbits[(int64_t)tile * kThreads + tid];
  const unsigned int cnt = __popc(bits);
  unsigned int incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  unsigned int prefix = 0, before = 0, total = 0;
#pragma unroll
  for (int w = 0; w < kThreads / 32; ++w) {
    prefix += s_red[w];
    if (w < warp) before += s_warp[w];
    total += s_warp[w];
  }
  unsigned int pos = prefix + before + (incl - cnt);
  const int64_t base = (int64_t)tile * kTile + (int64_t)tid * kPerThread;
  while (bits) {
    const int j = __ffs(bits) - 1;
    bits &= bits - 1;
    p.idx[pos++] = (int32_t)(base + j);
  }
  if (tid == 0 && (int)tile == ntiles - 1) *p.k_out = (int32_t)(prefix + total);
}

__global__ void tau_kernel(MaskParams p, double* tau) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)p.H * p.W) return;
  tau[i] = tau_at(p, (int)(i % p.W), (int)(i / p.W));
}

MaskParams make_params(fv_ctx* ctx, int frame, int H, int W, const fv_fovea* f,
                       const double* pb_map) {
  MaskParams p{};
  p.H = H; p.W = W; p.frame = frame;
  if (f) {
    p.fx = f->focus[0]; p.fy = f->focus[1]; p.sigma = f->sigma; p.pb = f->base_density;
    p.scale = f->pixel_scale;
  }
  p.pb_map = pb_map;
  p.noise = ctx->noise; p.T = ctx->noise_T; p.Ht = ctx->noise_H; p.Wt = ctx->noise_W;
  return p;
}

}  // namespace

int launch_mask_compact(fv_ctx* ctx, int frame, int H, int W, const fv_fovea* f,
                        const double* pb_map, uint8_t* bits, int32_t* idx, int32_t* k,
                        __half* net_in, int net_wp, const double* tau_map) {
  FV_REQUIRE(ctx->noise != nullptr, "no noise stack uploaded (fv_noise_upload)");
  FV_REQUIRE(frame >= 0, "frame must be >= 0, got %d", frame);
  const int64_t npix = (int64_t)H * W;
  FV_REQUIRE(npix < (1ll << 30), "film too large for the 30-bit scan (%lld px)", (long long)npix);
  const int ntiles = (int)((npix + kTile - 1) / kTile);
  if (ntiles > ctx->scan_tiles_cap) {
    if (ctx->scan_status) cudaFree(ctx->scan_status);
    ctx->scan_status = nullptr;
    FV_CUDA(cudaMalloc(&ctx->scan_status, sizeof(unsigned long long) * ntiles));
    FV_CUDA(cudaMemsetAsync(ctx->scan_status, 0, sizeof(unsigned long long) * ntiles, ctx->stream));
    ctx->scan_tiles_cap = ntiles;
  }
  MaskParams p = make_params(ctx, frame, H, W, f, pb_map);
  p.tau_map = tau_map;
  p.bits = bits; p.idx = idx; p.k_out = k; p.net_in = net_in; p.net_wp = net_wp;
  p.status = ctx->scan_status;
  if (++ctx->epoch == 0) ctx->epoch = 1;
  p.epoch = ctx->epoch;
  p.tile_counter = &ctx->counters->scan_tile;
  p.dyn = ctx->dyn_active;
  FV_CUDA(cudaMemsetAsync(&ctx->counters->scan_tile, 0, sizeof(unsigned int), ctx->stream));
  static bool co = false;
  if (!co) {
    render_carveout(mask_compact_kernel);
    co = true;
  }
  static const bool two_pass = !(getenv("FV_MASK_2PASS") && atoi(getenv("FV_MASK_2PASS")) == 0);
  if (two_pass) {
    // tile bit bytes (256 per tile) and counts live behind the status words of the single pass
    if ((int64_t)ntiles * (kThreads + 4) > ctx->scan_aux_cap) {
      if (ctx->scan_aux) cudaFree(ctx->scan_aux);
      ctx->scan_aux = nullptr;
      FV_CUDA(cudaMalloc(&ctx->scan_aux, (size_t)ntiles * (kThreads + 4)));
      ctx->scan_aux_cap = (int64_t)ntiles * (kThreads + 4);
    }
    uint8_t* tb = reinterpret_cast<uint8_t*>(ctx->scan_aux);
    unsigned int* counts = reinterpret_cast<unsigned int*>(tb + (size_t)ntiles * kThreads);
    static bool co2 = false;
    if (!co2) {
      render_carveout(mask_count_kernel);
      render_carveout(mask_write_kernel);
      co2 = true;
    }
    FV_TIMED(ctx, FV_KC_MASK, mask_count_kernel<<<ntiles, kThreads, 0, ctx->stream>>>(p, tb, counts));
    FV_CHECK_LAUNCH("mask_count_kernel");
    FV_TIMED(ctx, FV_KC_MASK, mask_write_kernel<<<ntiles, kThreads, 0, ctx->stream>>>(p, tb, counts, ntiles));
    FV_CHECK_LAUNCH("mask_write_kernel");
    ctx->launches += 2;
    return 0;
  }
  FV_TIMED(ctx, FV_KC_MASK, mask_compact_kernel<<<ntiles, kThreads, 0, ctx->stream>>>(p));
  FV_CHECK_LAUNCH("mask_compact_kernel");
  ctx->launches += 1;
  return 0;
}

int launch_tau_map(fv_ctx* ctx, int H, int W, const fv_fovea* f, const double* pb_map,
                   double* tau) {
  MaskParams p = make_params(ctx, 0, H, W, f, pb_map);
  const int64_t n = (int64_t)H * W;
  FV_TIMED(ctx, FV_KC_MASK, tau_kernel<<<(unsigned)((n + 255) / 256), 256, 0, ctx->stream>>>(p, tau));
  FV_CHECK_LAUNCH("tau_kernel");
  ctx->launches += 1;
  return 0;
}

// c_max (sample_maps.py:135-137): the mean of tau over the frame as a deterministic fp64 sum --
// a fixed grid of kSumBlocks blocks (independent of the device), each summing a fixed pixel
// stride then a fixed shared-memory tree, and one block summing the partials the same way. tau is
// evaluated inline (tau_at: the mask kernel's arithmetic) or read from a tau map.
constexpr int kSumBlocks = 512, kSumThreads = 256;

__global__ void __launch_bounds__(kSumThreads) tau_sum_partial_kernel(MaskParams p, double* partial) {
  __shared__ double s[kSumThreads];
  const int64_t n = (int64_t)p.H * p.W;
  double acc = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * kSumThreads + threadIdx.x; i < n; i += (int64_t)kSumBlocks * kSumThreads)
    acc += tau_at(p, (int)(i % p.W), (int)(i / p.W));
  s[threadIdx.x] = acc;
  __syncthreads();
  for (int o = kSumThreads / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) s[threadIdx.x] += s[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = s[0];
}

__global__ void __launch_bounds__(kSumThreads) sum_partials_kernel(const double* partial, double* out) {
  __shared__ double s[kSumThreads];
  double acc = 0.0;
  for (int i = threadIdx.x; i < kSumBlocks; i += kSumThreads) acc += partial[i];
  s[threadIdx.x] = acc;
  __syncthreads();
  for (int o = kSumThreads / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) s[threadIdx.x] += s[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = s[0];
}

// foveal_density (sample_maps.py:62-68) elementwise over broadcast (dx, dy) offsets: the mask
// kernel's fp64 arithmetic (no FMA contraction)
__global__ void foveal_density_kernel(const double* __restrict__ ox, const double* __restrict__ oy, int64_t n,
                                      double sigma, double scale, double* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double dx = __dmul_rn(ox[i], scale), dy = __dmul_rn(oy[i], scale);
    const double r2 = __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
    out[i] = exp(__dmul_rn(__dmul_rn(-0.5, r2), sigma));
  }
}

int launch_tau_sum(fv_ctx* ctx, int H, int W, const fv_fovea* f, const double* pb_map, const double* tau_map,
                   double* sum_dev) {
  MaskParams p = make_params(ctx, 0, H, W, f, pb_map);
  p.tau_map = tau_map;
  double* partial = nullptr;
  FV_CUDA(cudaMallocAsync(&partial, sizeof(double) * kSumBlocks, ctx->stream));
  FV_TIMED(ctx, FV_KC_MASK, tau_sum_partial_kernel<<<kSumBlocks, kSumThreads, 0, ctx->stream>>>(p, partial));
  FV_TIMED(ctx, FV_KC_MASK, sum_partials_kernel<<<1, kSumThreads, 0, ctx->stream>>>(partial, sum_dev));
  FV_CHECK_LAUNCH("tau_sum_kernel");
  ctx->launches += 2;
  FV_CUDA(cudaFreeAsync(partial, ctx->stream));
  return 0;
}

int launch_foveal_density(fv_ctx* ctx, const double* ox, const double* oy, int64_t n, double sigma, double scale,
                          double* out) {
  if (n == 0) return 0;
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)ctx->num_sms * 16));
  FV_TIMED(ctx, FV_KC_MASK, foveal_density_kernel<<<blocks, 256, 0, ctx->stream>>>(ox, oy, n, sigma, scale, out));
  FV_CHECK_LAUNCH("foveal_density_kernel");
  ctx->launches += 1;
  return 0;
}

// draw_direct_samples (sample_maps.py:181-198): inverse-CDF sampling over the row-major fp64 tau
// map -- cdf = cumsum(tau) / total, idx = searchsorted(cdf, r, side="right") clamped to n-1 -- for
// caller-supplied uniforms r (NumPy's stream, so the draws follow the reference's generator). The
// cumulative sum is blocked (sequential per thread over 16 pixels, a fixed in-block scan, a
// sequential scan of the block totals): deterministic, and within rounding of np.cumsum's
// sequential sum (a draw can only differ when r falls within ~1e-16 of a CDF step).
constexpr int kCdfPer = 16, kCdfBlock = kSumThreads * kCdfPer;

__global__ void __launch_bounds__(kSumThreads) cdf_block_kernel(MaskParams p, double* cdf, double* bsum) {
  __shared__ double s[kSumThreads];
  const int64_t n = (int64_t)p.H * p.W;
  const int64_t base = (int64_t)blockIdx.x * kCdfBlock + (int64_t)threadIdx.x * kCdfPer;
  double loc[kCdfPer];
  double acc = 0.0;
#pragma unroll
  for (int j = 0; j < kCdfPer; ++j) {
    const int64_t i = base + j;
    const double t = i < n ? tau_at(p, (int)(i % p.W), (int)(i / p.W)) : 0.0;
    acc += t;
    loc[j] = acc;
  }
  s[threadIdx.x] = acc;
  __syncthreads();
  // inclusive Hillis-Steele scan of the thread totals (fixed order)
  for (int o = 1; o < kSumThreads; o <<= 1) {
    const double v = threadIdx.x >= o ? s[threadIdx.x - o] : 0.0;
    __syncthreads();
    s[threadIdx.x] += v;
    __syncthreads();
  }
  const double off = threadIdx.x ? s[threadIdx.x - 1] : 0.0;
#pragma unroll
  for (int j = 0; j < kCdfPer; ++j)
    if (base + j < n) cdf[base + j] = off + loc[j];
  if (threadIdx.x == kSumThreads - 1) bsum[blockIdx.x] = s[threadIdx.x];
}

__global__ void cdf_offsets_kernel(double* bsum, int nb) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double acc = 0.0;
  for (int b = 0; b < nb; ++b) {
    const double v = bsum[b];
    bsum[b] = acc;  // exclusive offsets; bsum[nb] = total
    acc += v;
  }
  bsum[nb] = acc;
}

__global__ void direct_draw_kernel(double* cdf, const double* bsum, int nb, int64_t n, const double* r,
                                   int64_t count, int32_t* idx) {
  const double total = bsum[nb];
  for (int64_t d = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; d < count; d += (int64_t)gridDim.x * blockDim.x) {
    const double x = r[d];
    // first i with cdf[i] / total > x (searchsorted side="right" on the normalised cdf)
    int64_t lo = 0, hi = n;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      const double c = (cdf[mid] + bsum[mid / kCdfBlock]) / total;
      if (c > x) hi = mid; else lo = mid + 1;
    }
    idx[d] = (int32_t)(lo < n - 1 ? lo : n - 1);
  }
}

int launch_direct_draws(fv_ctx* ctx, int H, int W, const fv_fovea* f, const double* pb_map, const double* tau_map,
                        const double* r, int64_t count, int32_t* idx) {
  MaskParams p = make_params(ctx, 0, H, W, f, pb_map);
  p.tau_map = tau_map;
  const int64_t n = (int64_t)H * W;
  const int nb = (int)((n + kCdfBlock - 1) / kCdfBlock);
  double* cdf = nullptr;
  FV_CUDA(cudaMallocAsync(&cdf, sizeof(double) * (n + nb + 1), ctx->stream));
  double* bsum = cdf + n;
  FV_TIMED(ctx, FV_KC_MASK, cdf_block_kernel<<<nb, kSumThreads, 0, ctx->stream>>>(p, cdf, bsum));
  FV_TIMED(ctx, FV_KC_MASK, cdf_offsets_kernel<<<1, 32, 0, ctx->stream>>>(bsum, nb));
  if (count > 0) {
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((count + 255) / 256, (int64_t)ctx->num_sms * 16));
    FV_TIMED(ctx, FV_KC_MASK, direct_draw_kernel<<<blocks, 256, 0, ctx->stream>>>(cdf, bsum, nb, n, r, count, idx));
  }
  FV_CHECK_LAUNCH("direct_draw_kernel");
  ctx->launches += 3;
  FV_CUDA(cudaFreeAsync(cdf, ctx->stream));
  return 0;
}

// Naive renderer lane list (render_sparse_naive, renderer.py:225-259): one warp per 64-pixel chunk;
// an occupied chunk appends all its pixels (idle ones as -(pix+1)), contiguous in the list so each
// chunk still maps onto two warps of the thread-per-lane marcher.
__global__ void naive_list_kernel(const uint8_t* __restrict__ bits, int64_t n, int32_t* __restrict__ idx,
                                  int32_t* __restrict__ k_dev) {
  const int lane = threadIdx.x & 31;
  const int64_t n_chunks = (n + kChunkNaive - 1) / kChunkNaive;
  const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t c = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; c < n_chunks; c += warps) {
    const int64_t p0 = c * kChunkNaive + lane, p1 = p0 + 32;
    const bool b0 = p0 < n && bits[p0], b1 = p1 < n && bits[p1];
    if (!__any_sync(0xffffffffu, b0 || b1)) continue;
    const int64_t rem = n - c * kChunkNaive;
    const int len = rem < kChunkNaive ? (int)rem : kChunkNaive;
    int base = 0;
    if (lane == 0) base = atomicAdd(k_dev, len);
    base = __shfl_sync(0xffffffffu, base, 0);
    if (p0 < n) idx[base + lane] = b0 ? (int32_t)p0 : -(int32_t)p0 - 1;
    if (p1 < n) idx[base + 32 + lane] = b1 ? (int32_t)p1 : -(int32_t)p1 - 1;
  }
}

int launch_naive_list(fv_ctx* ctx, const uint8_t* bits, int H, int W, int32_t* idx, int32_t* k_dev) {
  const int64_t n = (int64_t)H * W;
  FV_CUDA(cudaMemsetAsync(k_dev, 0, sizeof(int32_t), ctx->stream));
  const int64_t chunks = (n + kChunkNaive - 1) / kChunkNaive;
  const int blocks = (int)std::min<int64_t>((chunks * 32 + 255) / 256, (int64_t)ctx->num_sms * 8);
  FV_TIMED(ctx, FV_KC_MASK, naive_list_kernel<<<blocks, 256, 0, ctx->stream>>>(bits, n, idx, k_dev));
  FV_CHECK_LAUNCH("naive_list_kernel");
  ctx->launches += 1;
  return 0;
}

}  // namespace fv
