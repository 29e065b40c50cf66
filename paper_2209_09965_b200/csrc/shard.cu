// Ray-list sharding for a frame split across GPUs (BASELINE config 5: 1024^3 at
// 3840x2160 sharded over 2/4/8 B200 with a framebuffer all-gather).
//
// Every rank builds the full mask (microseconds) and marches only its share of the compacted
// active-ray list: 32-ray packets dealt round-robin (rank r takes packets p with p % world == r),
// which balances samples statistically where fixed screen tiles would be unbalanced by the fovea.
// The marched RGBA of the rank's rays is packed into fixed-capacity records (pixel, RGBA); the
// records of all ranks are all-gathered (NCCL over NVLink; torch.distributed in the host code) and
// scattered into the network input exactly as the marcher would have written it, so the
// reconstruction that follows sees the same input as the unsharded frame (bit-exact).
#include <algorithm>

#include "internal.h"

namespace fv {
namespace {

constexpr int kPacket = 32;

// out = entries of idx[0, k) whose packet index (i / 32) % world == rank, in list order
__global__ void shard_rays_kernel(const int32_t* __restrict__ idx, const int32_t* __restrict__ k_dev, int k_max,
                                  int rank, int world, int32_t* __restrict__ out, int32_t* __restrict__ out_k) {
  const int k = k_dev ? min(*k_dev, k_max) : k_max;
  const int n_packets = (k + kPacket - 1) / kPacket;
  const int mine = n_packets > rank ? (n_packets - rank + world - 1) / world : 0;  // packets of this rank
  const int64_t total = (int64_t)mine * kPacket;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < total; j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = (int64_t)rank + (j / kPacket) * world;  // global packet
    const int64_t i = p * kPacket + (j % kPacket);
    if (i < k) out[j] = idx[i];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    // the last packet overall may be partial; only the rank that owns it is short
    int64_t cnt = total;
    if (mine > 0) {
      const int64_t last_p = (int64_t)rank + (int64_t)(mine - 1) * world;
      const int64_t end = (last_p + 1) * kPacket < (int64_t)k ? (last_p + 1) * kPacket : (int64_t)k;
      cnt = (int64_t)(mine - 1) * kPacket + (end - last_p * kPacket);
    }
    *out_k = (int32_t)cnt;
  }
}

// records [0, cap): (pix, rgba) of the rank's marched rays, pix = -1 past the rank's count
__global__ void pack_records_kernel(const float* __restrict__ rgba, const int32_t* __restrict__ idx,
                                    const int32_t* __restrict__ k_dev, int cap, int32_t* __restrict__ rec_pix,
                                    float4* __restrict__ rec_rgba) {
  const int k = min(*k_dev, cap);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < cap; i += gridDim.x * blockDim.x) {
    if (i < k) {
      const int pix = idx[i];
      rec_pix[i] = pix;
      rec_rgba[i] = *reinterpret_cast<const float4*>(rgba + (int64_t)pix * 4);
    } else {
      rec_pix[i] = -1;
    }
  }
}

// gathered records -> network input channels 0..3 (fp16, as the marcher writes them) and an
// optional full (H,W,4) framebuffer
__global__ void scatter_records_kernel(const int32_t* __restrict__ rec_pix, const float4* __restrict__ rec_rgba,
                                       int64_t n, int W, __half* __restrict__ net_in, int net_wp,
                                       float* __restrict__ rgba_out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int pix = rec_pix[i];
    if (pix < 0) continue;
    const float4 c = rec_rgba[i];
    if (net_in) {
      const int u = pix % W, v = pix / W;
      __half2* hp = reinterpret_cast<__half2*>(net_in + ((int64_t)v * net_wp + u) * 8);
      hp[0] = __floats2half2_rn(c.x, c.y);
      hp[1] = __floats2half2_rn(c.z, c.w);
    }
    if (rgba_out) *reinterpret_cast<float4*>(rgba_out + (int64_t)pix * 4) = c;
  }
}

// ---- row-strip reconstruction (see sharded.py): record exchange in fp16 and window inputs ----

// records as (pix, rgba half2 x2) int32 triples: 12 bytes per marched ray
__global__ void pack_records16_kernel(const float* __restrict__ rgba, const int32_t* __restrict__ idx,
                                      const int32_t* __restrict__ k_dev, int cap, int32_t* __restrict__ rec) {
  const int k = min(*k_dev, cap);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < cap; i += gridDim.x * blockDim.x) {
    int3 r = make_int3(-1, 0, 0);
    if (i < k) {
      const int pix = idx[i];
      const float4 c = *reinterpret_cast<const float4*>(rgba + (int64_t)pix * 4);
      const __half2 a = __floats2half2_rn(c.x, c.y), b = __floats2half2_rn(c.z, c.w);
      r = make_int3(pix, *reinterpret_cast<const int*>(&a), *reinterpret_cast<const int*>(&b));
    }
    rec[3 * (int64_t)i] = r.x;
    rec[3 * (int64_t)i + 1] = r.y;
    rec[3 * (int64_t)i + 2] = r.z;
  }
}

// fp16 records -> network input channels 0..3 of rows [row0, row0 + rows) (window-local rows)
__global__ void scatter_records16_kernel(const int32_t* __restrict__ rec, int64_t n, int W, int row0, int rows,
                                         __half* __restrict__ net_in, int net_wp) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int pix = rec[3 * i];
    if (pix < 0) continue;
    const int u = pix % W, v = pix / W - row0;
    if (v < 0 || v >= rows) continue;
    int2* hp = reinterpret_cast<int2*>(net_in + ((int64_t)v * net_wp + u) * 8);
    *hp = make_int2(rec[3 * i + 1], rec[3 * i + 2]);
  }
}

// window input channels 0..4 from the full-frame mask bits: 0 RGBA (the records fill the active
// pixels) and the mask channel; rows past the film (the padded bottom) are zero
__global__ void window_input_kernel(const uint8_t* __restrict__ bits, int H_full, int W, int row0, int rows,
                                    __half* __restrict__ net_in, int net_wp) {
  const int64_t n = (int64_t)rows * W;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int u = (int)(i % W), y = (int)(i / W), v = row0 + y;
    const bool m = v < H_full && bits[(int64_t)v * W + u];
    // the whole group-0 pixel [0 x 4, m, 0 x 3] (the records fill channels 0..3 afterwards)
    *reinterpret_cast<uint4*>(net_in + ((int64_t)y * net_wp + u) * 8) = make_uint4(0u, 0u, m ? 0x3c00u : 0u, 0u);
  }
}

// the input's feedback group (fb = its base: [O_d, 0 x 5]) for rows [r0, r0 + rows) from the fp32 O_d planes
__global__ void feedback_rows_kernel(const float* __restrict__ od, __half* __restrict__ fb, int Hp, int Wp, int r0,
                                     int rows) {
  const int64_t n = (int64_t)rows * Wp, plane = (int64_t)Hp * Wp;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t pix = (int64_t)r0 * Wp + i;
    uint4 q;
    __half2* p2 = reinterpret_cast<__half2*>(&q);
    p2[0] = __floats2half2_rn(od[pix], od[plane + pix]);
    p2[1] = __floats2half2_rn(od[2 * plane + pix], 0.f);
    q.z = q.w = 0u;
    *reinterpret_cast<uint4*>(fb + pix * 8) = q;
  }
}

int grid_of(fv_ctx* ctx, int64_t n) {
  const int64_t b = (n + 255) / 256;
  return (int)std::max<int64_t>(1, std::min<int64_t>(b, (int64_t)ctx->num_sms * 8));
}

}  // namespace
}  // namespace fv

using namespace fv;

extern "C" {

int fv_shard_rays(fv_ctx* ctx, const int32_t* idx_dev, const int32_t* k_dev, int k_max, int rank, int world,
                  int32_t* out_idx_dev, int32_t* out_k_dev) {
  FV_REQUIRE(ctx && idx_dev && out_idx_dev && out_k_dev, "null argument");
  FV_REQUIRE(world >= 1 && rank >= 0 && rank < world, "rank %d outside world %d", rank, world);
  FV_TIMED(ctx, FV_KC_MASK, shard_rays_kernel<<<grid_of(ctx, k_max), 256, 0, ctx->stream>>>(
                                idx_dev, k_dev, k_max, rank, world, out_idx_dev, out_k_dev));
  FV_CHECK_LAUNCH("shard_rays_kernel");
  ctx->launches += 1;
  return 0;
}

int fv_pack_records(fv_ctx* ctx, const float* rgba_dev, const int32_t* idx_dev, const int32_t* k_dev, int cap,
                    int32_t* rec_pix_dev, float* rec_rgba_dev) {
  FV_REQUIRE(ctx && rgba_dev && idx_dev && k_dev && rec_pix_dev && rec_rgba_dev, "null argument");
  FV_REQUIRE(cap >= 0, "record capacity must be >= 0");
  FV_TIMED(ctx, FV_KC_NETOPS, pack_records_kernel<<<grid_of(ctx, cap), 256, 0, ctx->stream>>>(
                                  rgba_dev, idx_dev, k_dev, cap, rec_pix_dev, reinterpret_cast<float4*>(rec_rgba_dev)));
  FV_CHECK_LAUNCH("pack_records_kernel");
  ctx->launches += 1;
  return 0;
}

int fv_scatter_records(fv_ctx* ctx, fv_state* st, const int32_t* rec_pix_dev, const float* rec_rgba_dev, int64_t n,
                       int W, float* rgba_out_dev) {
  FV_REQUIRE(ctx && rec_pix_dev && rec_rgba_dev, "null argument");
  FV_REQUIRE(st || rgba_out_dev, "nothing to scatter into");
  FV_REQUIRE(!st || st->W == W, "state film width %d != %d", st ? st->W : 0, W);
  FV_TIMED(ctx, FV_KC_NETOPS, scatter_records_kernel<<<grid_of(ctx, n), 256, 0, ctx->stream>>>(
                                  rec_pix_dev, reinterpret_cast<const float4*>(rec_rgba_dev), n, W,
                                  st ? st->x.p : nullptr, st ? st->Wp : W, rgba_out_dev));
  FV_CHECK_LAUNCH("scatter_records_kernel");
  ctx->launches += 1;
  return 0;
}


int fv_pack_records16(fv_ctx* ctx, const float* rgba_dev, const int32_t* idx_dev, const int32_t* k_dev, int cap,
                      int32_t* rec_dev) {
  FV_REQUIRE(ctx && rgba_dev && idx_dev && k_dev && rec_dev, "null argument");
  FV_REQUIRE(cap >= 0, "record capacity must be >= 0");
  FV_TIMED(ctx, FV_KC_NETOPS, pack_records16_kernel<<<grid_of(ctx, cap), 256, 0, ctx->stream>>>(
                                  rgba_dev, idx_dev, k_dev, cap, rec_dev));
  FV_CHECK_LAUNCH("pack_records16_kernel");
  ctx->launches += 1;
  return 0;
}

int fv_scatter_records16(fv_ctx* ctx, fv_state* st, const int32_t* rec_dev, int64_t n, int W, int row0) {
  FV_REQUIRE(ctx && st && rec_dev, "null argument");
  FV_REQUIRE(st->W == W, "state film width %d != %d", st->W, W);
  FV_REQUIRE(row0 >= 0, "row offset must be >= 0");
  FV_TIMED(ctx, FV_KC_NETOPS, scatter_records16_kernel<<<grid_of(ctx, n), 256, 0, ctx->stream>>>(
                                  rec_dev, n, W, row0, st->H, st->x.p, st->Wp));
  FV_CHECK_LAUNCH("scatter_records16_kernel");
  ctx->launches += 1;
  return 0;
}

int fv_window_input(fv_ctx* ctx, fv_state* st, const uint8_t* bits_dev, int H_full, int W, int row0) {
  FV_REQUIRE(ctx && st && bits_dev, "null argument");
  FV_REQUIRE(st->W == W, "state film width %d != %d", st->W, W);
  FV_REQUIRE(row0 >= 0 && row0 < H_full + st->Hp, "row offset %d outside the film", row0);
  const int64_t n = (int64_t)st->H * W;
  FV_TIMED(ctx, FV_KC_MASK, window_input_kernel<<<grid_of(ctx, n), 256, 0, ctx->stream>>>(
                                bits_dev, H_full, W, row0, st->H, st->x.p, st->Wp));
  FV_CHECK_LAUNCH("window_input_kernel");
  ctx->launches += 1;
  return 0;
}

// The recurrent band [row0, row0 + rows) of a state (window-local L0 rows, multiples of the
// network divisor): the current decoder hidden tensors at their levels and the fp32 O_d, packed
// in that order. pack = 1: state -> buf; pack = 0: buf -> state, then the next input's O_d
// feedback channels for those rows. buf = null: only *bytes.
int fv_state_band(fv_ctx* ctx, fv_state* st, int pack, int row0, int rows, void* buf_dev, int64_t* bytes) {
  FV_REQUIRE(ctx && st, "null argument");
  const fv_net* net = st->net;
  const int div = 1 << net->n_enc;
  FV_REQUIRE(row0 >= 0 && rows >= 0 && row0 + rows <= st->Hp && row0 % div == 0 && rows % div == 0,
             "band [%d, %d) must lie in the state's %d rows at multiples of %d", row0, row0 + rows, st->Hp, div);
  int64_t off = 0;
  uint8_t* b = reinterpret_cast<uint8_t*>(buf_dev);
  const std::vector<fv_act>& hid = st->hidden[st->parity];
  for (int j = 0; j < net->n_dec; ++j) {
    const fv_act& a = hid[j];
    const int L = net->n_enc - j;
    const int r0 = row0 >> L, nr = rows >> L;
    const size_t width = (size_t)nr * a.W * 16, pitch = (size_t)a.H * a.W * 16;
    const int groups = a.C / 8;
    if (b && width) {
      uint8_t* t = reinterpret_cast<uint8_t*>(a.p) + (size_t)r0 * a.W * 16;
      if (pack)
        FV_CUDA(cudaMemcpy2DAsync(b + off, width, t, pitch, width, groups, cudaMemcpyDeviceToDevice, ctx->stream));
      else
        FV_CUDA(cudaMemcpy2DAsync(t, pitch, b + off, width, width, groups, cudaMemcpyDeviceToDevice, ctx->stream));
    }
    off += (int64_t)width * groups;
  }
  {
    const size_t width = (size_t)rows * st->Wp * 4, pitch = (size_t)st->Hp * st->Wp * 4;
    if (b && width) {
      uint8_t* t = reinterpret_cast<uint8_t*>(st->od) + (size_t)row0 * st->Wp * 4;
      if (pack)
        FV_CUDA(cudaMemcpy2DAsync(b + off, width, t, pitch, width, 3, cudaMemcpyDeviceToDevice, ctx->stream));
      else
        FV_CUDA(cudaMemcpy2DAsync(t, pitch, b + off, width, width, 3, cudaMemcpyDeviceToDevice, ctx->stream));
    }
    off += (int64_t)width * 3;
  }
  if (b && !pack && rows && net->recurrent) {
    FV_TIMED(ctx, FV_KC_NETOPS, feedback_rows_kernel<<<grid_of(ctx, (int64_t)rows * st->Wp), 256, 0, ctx->stream>>>(
                                    st->od, feedback_plane(st->x), st->Hp, st->Wp, row0, rows));
    FV_CHECK_LAUNCH("feedback_rows_kernel");
    ctx->launches += 1;
  }
  if (bytes) *bytes = off;
  return 0;
}

}  // extern "C"
