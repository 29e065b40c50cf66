// 3x3 convolution (stride 1, zero padding 1) as a tcgen05 implicit GEMM.
//
// Reference: autograd.conv2d (autograd.py:238-276) -- cross-correlation, weight (oc, ic, 3, 3),
// im2col column order (c, ky, kx), + bias -- followed by relu (autograd.py:134-141) and, for
// encoder blocks, avg_pool2 (autograd.py:279-291); concat_channels (autograd.py:173-185) of the
// block inputs is folded into the operand loader.
//
// Layout. Activations live in HBM as "NC8HW8": C/8 planes of (H, W, 8) fp16, i.e. every 8-channel
// group is a dense NHWC8 image. A CTA tile is R output rows x 128 output columns. Per K-stage
// (4 channel groups = 32 channels) the producer warp bulk-copies the (R+2) x 130 halo of each
// channel group into shared memory as [group][halo_row][halo_col][8 ch]: consecutive pixels are
// 16 bytes apart, which is exactly the SWIZZLE_NONE K-major canonical UMMA layout with
// SBO = 128 B and LBO = one group plane. A 3x3 tap (dy, dx) of output row r is therefore just a
// shifted descriptor start address ((r+dy)*130 + dx)*16 -- the im2col matrix is never built and
// the halo is read from L2 once per stage instead of nine times. Zero padding at image borders
// and the zero channel group of the 8-channel input layer are written with st.shared.
//
// Roles (192 threads, one CTA per SM, persistent over tiles):
//   warp 0     producer: cp.async.bulk of A halo rows + the stage's B (weight) image
//   warp 1     MMA issuer: tcgen05.mma 128 x N x 16, accumulators in TMEM (R x N columns,
//              double-buffered across tiles), tcgen05.commit to release smem / publish TMEM
//   warps 2-9  epilogue (two per TMEM lane quarter): tcgen05.ld -> +bias, ReLU -> fp16 NC8HW8 store, fused 2x2 average pool,
//              or the D.head mode (fp32 O_d planes + the next frame's feedback channels)
#include <cstdio>
#include <cstdlib>

#include "internal.h"
#include "sm100.cuh"

namespace fv {

namespace {

constexpr int kTileW = 128;          // output columns per tile (= MMA M)
constexpr int kHaloW = kTileW + 2;   // 130
constexpr int kRowBytes = kHaloW * 16;
constexpr int kStageGroups = 2;      // channel groups (of 8) per K-stage = one MMA K of 16
constexpr int kBResStages = 4;       // resident-weight kernels hold up to 4 stages (cin <= 64)
constexpr int kEpiWarps = 8;      // two epilogue warps per TMEM lane quarter
constexpr int kThreads = 64 + 32 * kEpiWarps;

struct ConvArgs {
  const __half* src[3];
  int src_groups[3];
  int n_src;
  int groups;        // total input channel groups (may be odd: cin = 8)
  int n_kstages;
  int H, W;
  const __half* wimg;  // B images of all stages
  const float* bias;   // n_pad
  int cout;
  __half* dst;         // NC8HW8, cout channels (nullable in head mode)
  __half* pool_dst;    // nullable: 2x2 average pool of dst
  int relu;
  int head;            // 1: aux epilogue (D.head and/or K-stage logits)
  float* od;           // head: (3, H, W) fp32 (nullable)
  __half* feedback;    // head: the next input's feedback group (internal.h kInGroups), nullable
  kw_t* kw[2];         // K-stage filter weights (9, H, W) per K block (nullable)
  int kcol[2];         // first logit column of each K block
  const __half* lw;    // LG: the K-stage logits' 1x1 weight image [cout/8][32][8] fp16 (columns 9 s + j)
  const float* lb;     // LG: their bias (32)
  int lg;              // LG: K blocks at this level (1 or 2)
  int center_only;     // 1x1 conv: only the centre tap's MMAs are issued
  int tiles_x, tiles_y;
  double flops;        // host-side: algorithmic FLOPs of the launch (kernel timing)
  unsigned long long* prof;  // nullable (FV_CONV_PROF=1): per-CTA wait-cycle counters, kProfSlots each
};
#ifndef FV_CONV_PROFILE
#define FV_CONV_PROFILE 0
#endif
constexpr bool kProfileBuild = FV_CONV_PROFILE != 0;
constexpr int kProfSlots = 6;  // producer empty-wait, MMA full-wait, MMA tempty-wait, epilogue tfull-wait, MMA total, tiles

// mbarrier wait that adds the cycles spent to *acc when profiling
__device__ __forceinline__ void pwait(uint32_t bar, uint32_t parity, bool prof, unsigned long long& acc) {
  if (!prof) {
    sm100::mbar_wait(bar, parity);
    return;
  }
  const unsigned long long t0 = clock64();
  sm100::mbar_wait(bar, parity);
  acc += clock64() - t0;
}

// one pixel of the input's feedback group: [O_d (3), 0 x 5], a whole 16-byte store
__device__ __forceinline__ void feedback_store(__half* px, float o0, float o1, float o2) {
  uint4 v;
  __half2* h2 = reinterpret_cast<__half2*>(&v);
  h2[0] = __floats2half2_rn(o0, o1);
  h2[1] = __floats2half2_rn(o2, 0.f);
  v.z = 0u;
  v.w = 0u;
  *reinterpret_cast<uint4*>(px) = v;
}

// fv_frames hooks after a conv launch: the march-ahead fork event and the filter-chain callback
int conv_launched(fv_ctx* ctx) {
  if (!ctx->conv_fork_ev && !ctx->conv_hook) return 0;
  ++ctx->conv_count;
  if (ctx->conv_fork_ev && ctx->conv_count == ctx->conv_fork_at)
    FV_CUDA(cudaEventRecord(ctx->conv_fork_ev, ctx->stream));
  if (ctx->conv_hook && ctx->conv_count == ctx->conv_hook_at) {
    auto hook = ctx->conv_hook;
    ctx->conv_hook = nullptr;  // once per frame
    return hook(ctx, ctx->conv_hook_arg);
  }
  return 0;
}

// R output rows per tile, N output channels (MMA N), S pipeline stages; BRES: the whole weight
// image (<= kBResStages stages, i.e. cin <= 64) is loaded once per CTA and stays in smem, so
// only activations stream (the weights were ~40% of the L2->SM bytes of a 64->64 conv).
template <int R, int N, int S = 2, bool BRES = false, bool TAPN = false, bool LG = false>
struct Cfg {
  static constexpr int kABytes = kStageGroups * (R + 2) * kRowBytes;
  static constexpr int kBBytes = 9 * kStageGroups * N * 16;
  static constexpr int kPlaneBytes = (R + 2) * kRowBytes;
  // TAPN: one accumulator block of N columns per HALO row (R + 2 of them), single-buffered
  static constexpr int kAccCols = TAPN ? (R + 2) * N : R * N;
  static constexpr int kAcc = (2 * kAccCols <= 512) ? 2 : 1;
  static constexpr int kBSlots = BRES ? kBResStages : S;
  static constexpr int kBiasBytes = N * 4;  // the epilogue's bias copy
  static constexpr int kXchgBytes = TAPN ? 512 : 0;  // TAPN: cross-quarter partial sums
  // LG: the tile's output rows staged as the logits GEMM's A operand ([row][g][128 px][8] fp16) and
  // the logits' weight image, plus their bias
  static constexpr int kStgBytes = LG ? R * N * 256 : 0;
  static constexpr int kLWBytes = LG ? (N / 8) * 512 : 0;
  static constexpr int kLBiasBytes = LG ? 128 : 0;
  static constexpr int kSmem = S * kABytes + kBSlots * kBBytes + kStgBytes + kLWBytes + 1024 + 256 + kBiasBytes +
                               kXchgBytes + kLBiasBytes;
};

// TAPN (the K-stage level-0 conv): the nine 3x3 taps of D.head sit in N next to the two K blocks'
// 1x1 logits -- column (dy*3 + dx)*3 + c is D.head output c's tap (dy, dx), columns 27.. and 36..
// the logits -- so ONE 128 x 48 x 16 MMA per halo row and K-stage covers all of it (instead of 18
// row-fused 128 x 96 x 16 dispatches, which left the launch MMA-issue bound at ~1280 cycles per
// stage). Halo row h's accumulator holds, in TMEM lane m (input pixel x0 - 1 + m), the products of
// that pixel with every tap's weights; the epilogue sums output pixel j = m - 1 over the 3 x 3
// neighbourhood across halo rows (TMEM columns) and lanes (shuffles; smem across lane quarters).
// Tiles therefore advance by 126 columns (lanes 1..126 are the valid outputs).
constexpr int kTapnStride = kTileW - 2;
constexpr int kTapnLogit[2] = {27, 36};
__host__ __device__ constexpr int tapn_logit(int s) { return s == 0 ? 27 : 36; }

// All MMAs of one K-stage: R output rows x 9 taps x NK k-steps, offsets folded at compile time.
// kCenter: 1x1 convolution -- only tap 4 (dy = dx = 1) is issued.
template <int R, int N, int NK, bool kCenter = false>
__device__ __forceinline__ void issue_stage(uint64_t a0, uint64_t b0, uint32_t d_base, uint32_t idesc,
                                            bool first_stage) {
  using C = Cfg<R, N>;
#pragma unroll
  for (int r = 0; r < R; ++r) {
#pragma unroll
    for (int t = kCenter ? 4 : 0; t < (kCenter ? 5 : 9); ++t) {
#pragma unroll
      for (int k = 0; k < NK; ++k) {
        const uint64_t ad = a0 + (uint64_t)((2 * k * C::kPlaneBytes + ((r + t / 3) * kHaloW + t % 3) * 16) >> 4);
        const uint64_t bd = b0 + (uint64_t)(((t * NK + k) * N * 32) >> 4);
        const bool acc = !first_stage || (kCenter ? k != 0 : (t | k) != 0);
        sm100::mma_f16(d_base + (R - 1 - r) * N, ad, bd, idesc, acc ? 1u : 0u);
      }
    }
  }
}

// Row-fused issue (3N <= 256). Input (halo) row h feeds output rows h-dy for dy = 0..2 through
// the weights of tap (dy, dx). The B image stacks the three dy slices along N ([dx][kg][dy*N+n]),
// and accumulator row r sits at column (R-1-r)*N, so ONE MMA of width (#dy)*N covers every output
// row an (h, dx) pair feeds: the A tile (the shifted halo row) is read from shared memory once
// instead of three times -- at N = 64 the A reads alone otherwise saturate the SM's operand
// bandwidth (ncu: L1/TEX 86% busy, tensor pipe 57%). In the first K-stage the dy = 0 slice (the
// row's first contribution) is issued separately without accumulate.
// kPairWait (single accumulator): before the first write of output rows (2p, 2p+1) in a tile's first
// K-stage, wait until the epilogue has drained that row pair of the previous tile (bar_pair + 8p,
// parity pair_par), so the next tile's MMAs start while the epilogue is still draining.
template <int R, int N, bool kDxOuter, bool kPairWait = false>
__device__ __forceinline__ void issue_stage_rows(uint64_t a0, uint64_t b0, uint32_t d_base, bool first_stage,
                                                 uint32_t bar_pair = 0, uint32_t pair_par = 0) {
  using C = Cfg<R, N>;
#pragma unroll
  for (int it = 0; it < 3 * (R + 2); ++it) {
    // kDxOuter: dx-major order (consecutive MMAs hit different accumulator rows); else h-major.
    // Either way row r is first written by (h = r, dx = 0, dy = 0) before any other MMA touches it.
    const int h = kDxOuter ? it % (R + 2) : it / 3;
    const int dx = kDxOuter ? it / (R + 2) : it % 3;
    if (kPairWait && first_stage && dx == 0 && (h & 1) == 0 && h < R) {
      sm100::mbar_wait(bar_pair + 8 * (h >> 1), pair_par);
      sm100::tc_fence_after();
    }
    const int dy_lo = h - R + 1 > 0 ? h - R + 1 : 0;
    const int dy_hi = h < 2 ? h : 2;
    const int r_first = h - dy_lo;
    {
      const uint64_t ad = a0 + (uint64_t)(((h * kHaloW + dx) * 16) >> 4);
      const uint64_t bdx = b0 + (uint64_t)((dx * 2 * 3 * N * 16) >> 4);
      const uint32_t d0 = d_base + (R - 1 - r_first) * N;
      if (first_stage && dx == 0 && dy_lo == 0) {
        // row h's first contribution (dy = 0): overwrite; the older rows accumulate
        sm100::mma_f16(d0, ad, bdx, sm100::idesc_f16(128, N), 0u);
        if (dy_hi >= 1)
          sm100::mma_f16(d0 + N, ad, bdx + (uint64_t)((N * 16) >> 4), sm100::idesc_f16(128, dy_hi * N), 1u);
      } else {
        sm100::mma_f16(d0, ad, bdx + (uint64_t)((dy_lo * N * 16) >> 4),
                       sm100::idesc_f16(128, (dy_hi - dy_lo + 1) * N), 1u);
      }
    }
  }
}

template <int R, int N, int kStages, bool BRES, bool FUSED, bool CO = false, bool TAPN = false, bool LG = false>
__global__ void __launch_bounds__(kThreads, 1) conv3x3_tc_kernel(ConvArgs a) {
  using C = Cfg<R, N, kStages, BRES, TAPN, LG>;
  constexpr int kStride = TAPN ? kTapnStride : kTileW;  // columns a tile advances by
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + kStages * C::kABytes;
  uint8_t* sStg = sB + C::kBSlots * C::kBBytes;  // LG: staged output rows
  uint8_t* sLW = sStg + C::kStgBytes;            // LG: logits weight image
  uint64_t* bars = reinterpret_cast<uint64_t*>(sLW + C::kLWBytes);
  // bars: full[kStages], empty[kStages], tfull[2], tempty[2], weights-resident, row-pair free[R/2],
  // LG: logits-done[R/2]
  constexpr bool kPairs = C::kAcc == 1 && FUSED;  // single accumulator: release it row pair by row pair
  static_assert(!(LG && (kPairs || TAPN || C::kAcc != 2)), "LG: double-buffered plain accumulators");
  uint32_t* tmem_slot =
      reinterpret_cast<uint32_t*>(bars + 2 * kStages + 5 + (kPairs ? R / 2 : 0) + (LG ? R / 2 : 0));
  float* s_bias = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(bars) + 256);  // N floats
  float* s_xchg = s_bias + N;  // TAPN: [half][quarter][left 3 | right 3]
  float* s_lbias = s_bias + N;  // LG: the logits' bias (32)
  const uint32_t bar_full = sm100::smem_u32(bars);
  const uint32_t bar_empty = bar_full + 8 * kStages;
  const uint32_t bar_tfull = bar_empty + 8 * kStages;
  const uint32_t bar_tempty = bar_tfull + 16;
  const uint32_t bar_bres = bar_tempty + 16;
  const uint32_t bar_pair = bar_bres + 8;
  const uint32_t bar_lfull = bar_pair + 8 * (kPairs ? R / 2 : 0);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      sm100::mbar_init(bar_full + 8 * s, 2);
      sm100::mbar_init(bar_empty + 8 * s, 1);
    }
    for (int s = 0; s < 2; ++s) {
      sm100::mbar_init(bar_tfull + 8 * s, 1);
      sm100::mbar_init(bar_tempty + 8 * s, kEpiWarps);
    }
    sm100::mbar_init(bar_bres, 1);
    if (kPairs)
      for (int p = 0; p < R / 2; ++p) sm100::mbar_init(bar_pair + 8 * p, kEpiWarps);
    if (LG)
      for (int p = 0; p < R / 2; ++p) sm100::mbar_init(bar_lfull + 8 * p, 1);
    sm100::fence_mbar_init();
    if (BRES || LG) {
      // resident weights (and the logits' weights): constant for the whole graph, so copied before
      // the dependency wait
      const uint32_t wb = BRES ? (uint32_t)(a.n_kstages * C::kBBytes) : 0u;
      sm100::mbar_arrive_expect_tx(bar_bres, wb + (uint32_t)C::kLWBytes);
      if (BRES) sm100::bulk_g2s(sm100::smem_u32(sB), a.wimg, wb, bar_bres);
      if (LG) sm100::bulk_g2s(sm100::smem_u32(sLW), a.lw, (uint32_t)C::kLWBytes, bar_bres);
    }
  }
  if (warp == 1) sm100::tmem_alloc<512>(sm100::smem_u32(tmem_slot));
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // PDL: everything above overlapped the previous kernel's tail; activations only after it is done
  fv::pdl_wait();

  const int n_tiles = a.tiles_x * a.tiles_y;
  // wait-cycle counters only in a profiling build (make EXTRA=-DFV_CONV_PROFILE=1, then
  // FV_CONV_PROF=1): every wait sits on a role's critical path, so the default build has none
  const bool prof = kProfileBuild && a.prof != nullptr;
  unsigned long long w_empty = 0, w_full = 0, w_tempty = 0, w_tfull = 0;
  const unsigned long long t_start = prof ? clock64() : 0ull;
  int n_my_tiles = 0;

  if (warp == 0) {
    // ---------------- producer ----------------
    int it = 0;
    for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
      const int x0 = (tile % a.tiles_x) * kStride;
      const int y0 = (tile / a.tiles_x) * R;
      uint32_t tile_bytes_per_group;
      {
        const int r_lo = CO ? 1 : 0, r_hi = CO ? R : R + 1;  // halo rows loaded
        const int rows_in = max(0, min(r_hi, a.H - y0) - max(r_lo, 1 - y0) + 1);
        const int lo = max(x0 - 1 + (CO ? 1 : 0), 0), hi = min(x0 + kTileW + 1 - (CO ? 1 : 0), a.W);
        tile_bytes_per_group = hi > lo ? (uint32_t)(rows_in * (hi - lo) * 16) : 0u;
      }
      for (int ks = 0; ks < a.n_kstages; ++ks, ++it) {
        const int st = it % kStages;
        const uint32_t round = it / kStages;
        pwait(bar_empty + 8 * st, (round & 1) ^ 1, prof, w_empty);
        const int g0 = ks * kStageGroups;
        int gs = a.groups - g0;
        if (gs > kStageGroups) gs = kStageGroups;
        const int gs_fill = (gs + 1) & ~1;  // odd group count: one zero group
        const int n_items = gs_fill * (R + 2);
        // CO (1x1 convs): only halo rows 1..R and columns 1..128 are read (the centre tap), so the
        // rest of the halo is neither loaded nor zero-filled
        constexpr int co = CO ? 1 : 0;
        // bytes the stage's bulk copies deliver: every real group copies the same in-image rows and
        // column span of the tile (no per-item pass and warp reduction on the producer's path)
        const uint32_t tot = (uint32_t)gs * tile_bytes_per_group;
        const uint32_t b_bytes = BRES ? 0u : (uint32_t)(9 * gs_fill * N * 16);
        // (no warp sync before the copies: a copy completing ahead of the expect-tx only takes the
        // barrier's tx-count below zero for a while; the phase still needs the final arrival below)
        if (lane == 0) sm100::mbar_arrive_expect_tx(bar_full + 8 * st, tot + b_bytes);
        const uint32_t a_st = sm100::smem_u32(sA + st * C::kABytes);
        if (!BRES && lane == 0)
          sm100::bulk_g2s(sm100::smem_u32(sB + st * C::kBBytes),
                          reinterpret_cast<const uint8_t*>(a.wimg) + (int64_t)ks * C::kBBytes,
                          b_bytes, bar_full + 8 * st);
        for (int item = lane; item < n_items; item += 32) {
          const int g = item / (R + 2), row = item % (R + 2);
          const int y = y0 - 1 + row;
          const uint32_t row_addr = a_st + g * C::kPlaneBytes + row * kRowBytes;
          const int gg = g0 + g;
          if (CO && (row == 0 || row == R + 1)) continue;
          if (gg < a.groups && y >= 0 && y < a.H) {
            const int lo = max(x0 - 1 + co, 0), hi = min(x0 + kTileW + 1 - co, a.W);
            // locate the source tensor of this channel group (concat folded into the loader)
            int s = 0, gl = gg;
            while (s + 1 < a.n_src && gl >= a.src_groups[s]) { gl -= a.src_groups[s]; ++s; }
            const __half* plane = a.src[s] + (int64_t)gl * a.H * a.W * 8;
            const int c_lo = lo - (x0 - 1), c_hi = hi - (x0 - 1);
            if (hi > lo)
              sm100::bulk_g2s(row_addr + c_lo * 16, plane + ((int64_t)y * a.W + lo) * 8,
                              (uint32_t)(hi - lo) * 16u, bar_full + 8 * st);
            for (int c = co; c < c_lo; ++c) sm100::st_shared_zero16(row_addr + c * 16);
            for (int c = max(c_hi, 0); c < kHaloW - co; ++c) sm100::st_shared_zero16(row_addr + c * 16);
          } else {
            for (int c = co; c < kHaloW - co; ++c) sm100::st_shared_zero16(row_addr + c * 16);
          }
        }
        sm100::fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) sm100::mbar_arrive(bar_full + 8 * st);
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    constexpr uint32_t idesc = sm100::idesc_f16(128, N);
    if (BRES) sm100::mbar_wait(bar_bres, 0);
    int it = 0, lt = 0;
    for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++lt) {
      ++n_my_tiles;
      const int acc = lt % C::kAcc;
      const uint32_t acc_round = lt / C::kAcc;
      if (!kPairs) pwait(bar_tempty + 8 * acc, (acc_round & 1) ^ 1, prof, w_tempty);
      sm100::tc_fence_after();
      const uint32_t d_base = tmem_base + acc * C::kAccCols;
      for (int ks = 0; ks < a.n_kstages; ++ks, ++it) {
        const int st = it % kStages;
        const uint32_t round = it / kStages;
        pwait(bar_full + 8 * st, round & 1, prof, w_full);
        sm100::tc_fence_after();
        int gs = a.groups - ks * kStageGroups;
        if (gs > kStageGroups) gs = kStageGroups;
        const int nk = (gs + 1) >> 1;
        // The whole warp walks the (warp-uniform) tap loop so descriptors stay in uniform
        // registers; elect.sync picks the one thread that issues each tcgen05.mma. Descriptors are
        // a base plus a 16-byte-unit offset in the start-address field.
        const uint64_t a0 = sm100::smem_desc(sm100::smem_u32(sA + st * C::kABytes), C::kPlaneBytes, 128);
        const uint64_t b0 = sm100::smem_desc(sm100::smem_u32(sB + (BRES ? ks : st) * C::kBBytes),
                                             (FUSED ? 3 : 1) * N * 16, 128);
        (void)nk;  // one 16-channel MMA K-step per stage
        const bool leader = sm100::elect_one();
        // (the dispatch-cost probe of round 1 -- the same MMA work per stage as 9 x N256, 18 x N128 or
        // 36 x N64 dispatches: 1054 / 1398 / 2085 cycles -- is summarised in profiles/r01_summary.md)
        // (row-fused weight images exist only for 3x3 convs: FUSED implies not centre-only)
        if (leader) {
          if constexpr (TAPN) {
            // one dispatch per halo row: A = the row from halo column 0 (pixel x0 - 1), all taps in N
#pragma unroll
            for (int h = 0; h < R + 2; ++h)
              sm100::mma_f16(d_base + h * N, a0 + (uint64_t)((h * kRowBytes) >> 4), b0, idesc, ks == 0 ? 0u : 1u);
          } else if constexpr (FUSED)
            issue_stage_rows<R, N, true, kPairs>(a0, b0, d_base, ks == 0, bar_pair, (acc_round & 1) ^ 1);
          else if (CO || a.center_only)
            issue_stage<R, N, 1, true>(a0, b0, d_base, idesc, ks == 0);
          else
            issue_stage<R, N, 1>(a0, b0, d_base, idesc, ks == 0);
        }
        __syncwarp();
        sm100::mma_commit_elect(bar_empty + 8 * st);
        __syncwarp();
      }
      sm100::mma_commit_elect(bar_tfull + 8 * acc);
      __syncwarp();
    }
  } else {
    // ---------------- epilogue ----------------
    // bias once per CTA into smem (broadcast reads, off the per-item dependency chain)
    for (int i = threadIdx.x - 64; i < N; i += kEpiWarps * 32) s_bias[i] = __ldg(a.bias + i);
    if (LG && threadIdx.x - 64 < 32) s_lbias[threadIdx.x - 64] = __ldg(a.lb + threadIdx.x - 64);
    sm100::named_bar_sync(1, kEpiWarps * 32);
    const int q = warp & 3;  // TMEM lane quarter accessible to this warp
    const int half = (warp - 2) >> 2;  // the two warps of a quarter split the tile's rows/columns
    int lt = 0;
    const int64_t plane = (int64_t)a.H * a.W * 8;
    const int Hp = a.H >> 1, Wp = a.W >> 1;
    const int64_t pplane = (int64_t)Hp * Wp * 8;
    for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++lt) {
      const int acc = lt % C::kAcc;
      const uint32_t acc_round = lt / C::kAcc;
      const int x0 = (tile % a.tiles_x) * kStride;
      const int y0 = (tile / a.tiles_x) * R;
      pwait(bar_tfull + 8 * acc, acc_round & 1, prof, w_tfull);
      sm100::tc_fence_after();
      const int x = x0 + 32 * q + lane;
      const bool xin = x < a.W;
      const uint32_t t_row0 = tmem_base + ((uint32_t)(32 * q) << 16) + acc * C::kAccCols;
      if constexpr (TAPN) {
        // output pixel j = m - 1 (m = this thread's TMEM lane in the tile): D.head = sum over dy of
        // L(m - 1) + M(m) + R(m + 1), L/M/R = the dx = 0/1/2 tap products of halo row r + dy in lane
        // m; the logits are the centre row's columns in lane m itself. The two warps of a lane
        // quarter take output rows {0, 1} and {2, 3}: each streams its four halo rows from TMEM once.
        const int m = 32 * q + lane, xo = x0 + m - 1;
        const bool valid = m >= 1 && m <= kTileW - 2 && xo < a.W;
        const int64_t hw = (int64_t)a.H * a.W;
        const int r0 = 2 * half;
        float Ls[2][3] = {}, Ms[2][3] = {}, Rs[2][3] = {};
#pragma unroll
        for (int hh = 0; hh < 4; ++hh) {
          uint32_t u0[16], u1[16];
          const uint32_t ta = t_row0 + (uint32_t)((r0 + hh) * N);
          sm100::tmem_ld16_nowait(ta, u0);
          sm100::tmem_ld16_nowait(ta + 16, u1);
          sm100::tmem_wait_ld_regs(u0, u1);
          float v[32];
#pragma unroll
          for (int i = 0; i < 16; ++i) { v[i] = __uint_as_float(u0[i]); v[16 + i] = __uint_as_float(u1[i]); }
#pragma unroll
          for (int o = 0; o < 2; ++o) {
            const int dy = hh - o;
            if (dy < 0 || dy > 2) continue;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
              Ls[o][c] += v[(dy * 3 + 0) * 3 + c];
              Ms[o][c] += v[(dy * 3 + 1) * 3 + c];
              Rs[o][c] += v[(dy * 3 + 2) * 3 + c];
            }
          }
          if (N >= 48 && (hh == 1 || hh == 2)) {
            // the centre row of output row r0 + hh - 1: its logits -> softmax -> filter weights
            uint32_t u2[16];
            sm100::tmem_ld16_nowait(ta + 32, u2);
            sm100::tmem_wait_ld();
            float lg[18];
#pragma unroll
            for (int i = 0; i < 5; ++i) lg[i] = v[27 + i];
#pragma unroll
            for (int i = 0; i < 13; ++i) lg[5 + i] = __uint_as_float(u2[i]);
            const int y = y0 + r0 + hh - 1;
            if (valid && y < a.H) {
              const int64_t pix = (int64_t)y * a.W + xo;
#pragma unroll
              for (int s_ = 0; s_ < 2; ++s_) {
                if (!a.kw[s_]) continue;
                float l[9], mx = -INFINITY;
#pragma unroll
                for (int j = 0; j < 9; ++j) {
                  l[j] = lg[9 * s_ + j] + s_bias[logit_col(s_) + j];
                  mx = fmaxf(mx, l[j]);
                }
                float sum = 0.f;
#pragma unroll
                for (int j = 0; j < 9; ++j) {
                  l[j] = __expf(l[j] - mx);  // arguments <= 0: ex2.approx, rel. error ~1e-7
                  sum += l[j];
                }
                const float inv = __frcp_rn(sum);
#pragma unroll
                for (int j = 0; j < 9; ++j) a.kw[s_][j * hw + pix] = l[j] * inv;
              }
            }
          }
        }
        // neighbours' partial sums: inside the quarter by shuffles, across quarters through smem
        float* xs = s_xchg + (half * 4 + q) * 12;
#pragma unroll
        for (int o = 0; o < 2; ++o) {
          if (lane == 31) { xs[6 * o] = Ls[o][0]; xs[6 * o + 1] = Ls[o][1]; xs[6 * o + 2] = Ls[o][2]; }
          if (lane == 0) { xs[6 * o + 3] = Rs[o][0]; xs[6 * o + 4] = Rs[o][1]; xs[6 * o + 5] = Rs[o][2]; }
        }
        sm100::named_bar_sync(2 + half, 128);
#pragma unroll
        for (int o = 0; o < 2; ++o) {
          float od[3];
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            float left = __shfl_up_sync(0xffffffffu, Ls[o][c], 1);
            float right = __shfl_down_sync(0xffffffffu, Rs[o][c], 1);
            if (lane == 0) left = q > 0 ? s_xchg[(half * 4 + q - 1) * 12 + 6 * o + c] : 0.f;
            if (lane == 31) right = q < 3 ? s_xchg[(half * 4 + q + 1) * 12 + 6 * o + 3 + c] : 0.f;
            od[c] = ((left + Ms[o][c]) + right) + s_bias[c];
          }
          const int y = y0 + r0 + o;
          if (valid && y < a.H && a.od) {
            const int64_t pix = (int64_t)y * a.W + xo;
#pragma unroll
            for (int c = 0; c < 3; ++c) a.od[c * hw + pix] = od[c];
            if (a.feedback) feedback_store(a.feedback + pix * 8, od[0], od[1], od[2]);
          }
        }
        sm100::named_bar_sync(2 + half, 128);  // the slots are rewritten by the next tile
      } else if (a.head) {
        // D.head (cols 0..2) and/or K-stage logits (9 cols per K block): O_d in fp32 planes +
        // next frame's feedback channels; logits -> max-subtracted softmax (autograd.py:188-199)
        // -> 9 fp32 filter-weight planes per K block.
        const int64_t hw = (int64_t)a.H * a.W;
        for (int r = half; r < R; r += 2) {
          float v[N >= 32 ? 32 : 16];
          if constexpr (N >= 32) {
            uint32_t r0[16], r1[16];
            sm100::tmem_ld16_nowait(t_row0 + (R - 1 - r) * N, r0);
            sm100::tmem_ld16_nowait(t_row0 + (R - 1 - r) * N + 16, r1);
            sm100::tmem_wait_ld_regs(r0, r1);
#pragma unroll
            for (int j = 0; j < 16; ++j) { v[j] = __uint_as_float(r0[j]); v[16 + j] = __uint_as_float(r1[j]); }
          } else {
            sm100::tmem_ld16(t_row0 + (R - 1 - r) * N, *reinterpret_cast<float(*)[16]>(v));
          }
          const int y = y0 + r;
          if (xin && y < a.H) {
            const int64_t pix = (int64_t)y * a.W + x;
            if (a.od) {
              float o[3];
#pragma unroll
              for (int c = 0; c < 3; ++c) {
                o[c] = v[c] + s_bias[c];
                a.od[c * hw + pix] = o[c];
              }
              if (a.feedback) feedback_store(a.feedback + pix * 8, o[0], o[1], o[2]);
            }
            if constexpr (N >= 32) {
#pragma unroll
              for (int s = 0; s < 2; ++s) {
                if (!a.kw[s]) continue;
                const int c0 = logit_col(s);  // compile-time: keeps v[] in registers
                float l[9], m = -INFINITY;
#pragma unroll
                for (int j = 0; j < 9; ++j) {
                  l[j] = v[c0 + j] + s_bias[c0 + j];
                  m = fmaxf(m, l[j]);
                }
                float sum = 0.f;
#pragma unroll
                for (int j = 0; j < 9; ++j) {
                  l[j] = __expf(l[j] - m);  // arguments <= 0: ex2.approx, rel. error ~1e-7
                  sum += l[j];
                }
                const float inv = __frcp_rn(sum);
#pragma unroll
                for (int j = 0; j < 9; ++j) a.kw[s][j * hw + pix] = l[j] * inv;
              }
            }
          }
        }
      } else if constexpr (LG) {
        // Decoder conv2 with the K stage's logits fused (network.py:268-277): per row pair, the
        // output rows go to HBM (the hidden state) AND, as fp16, to the staged A operand; then one
        // elected epilogue thread runs the 1x1 logits GEMM (128 x 32 x cout) into the drained
        // accumulator columns of those rows, and after the last row pair the epilogue turns them
        // into the softmax filter weights (the separate level-L logits conv of the K stage).
        constexpr int kCb = N / 16;
        const int m = 32 * q + lane;  // TMEM lane = pixel of the tile
#pragma unroll 1
        for (int p = 0; p < R / 2; ++p) {
          const int r = 2 * p;
          const int y = y0 + r;
#pragma unroll 1
          for (int item = p * kCb + half; item < (p + 1) * kCb; item += 2) {
            const int cb = 16 * (item - p * kCb);
            float v0[16], v1[16];
            {
              uint32_t r0[16], r1[16];
              sm100::tmem_ld16_nowait(t_row0 + (R - 1 - r) * N + cb, r0);
              sm100::tmem_ld16_nowait(t_row0 + (R - 2 - r) * N + cb, r1);
              sm100::tmem_wait_ld_regs(r0, r1);
#pragma unroll
              for (int j = 0; j < 16; ++j) { v0[j] = __uint_as_float(r0[j]); v1[j] = __uint_as_float(r1[j]); }
            }
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const float b = s_bias[cb + j];
              v0[j] += b;
              v1[j] += b;
              if (a.relu) { v0[j] = fmaxf(v0[j], 0.f); v1[j] = fmaxf(v1[j], 0.f); }
            }
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int g = (cb >> 3) + h;
              uint4 pk0, pk1;
              __half2* p0 = reinterpret_cast<__half2*>(&pk0);
              __half2* p1 = reinterpret_cast<__half2*>(&pk1);
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                p0[j] = __floats2half2_rn(v0[8 * h + 2 * j], v0[8 * h + 2 * j + 1]);
                p1[j] = __floats2half2_rn(v1[8 * h + 2 * j], v1[8 * h + 2 * j + 1]);
              }
              *reinterpret_cast<uint4*>(sStg + (((int64_t)r * (N / 8) + g) * 128 + m) * 16) = pk0;
              *reinterpret_cast<uint4*>(sStg + (((int64_t)(r + 1) * (N / 8) + g) * 128 + m) * 16) = pk1;
              if (xin && 8 * g < a.cout) {
                if (y < a.H) *reinterpret_cast<uint4*>(a.dst + g * plane + ((int64_t)y * a.W + x) * 8) = pk0;
                if (y + 1 < a.H) *reinterpret_cast<uint4*>(a.dst + g * plane + ((int64_t)(y + 1) * a.W + x) * 8) = pk1;
              }
            }
          }
          // rows r, r + 1 staged and their accumulator columns read: the logits GEMM may overwrite them
          sm100::fence_proxy_async_smem();
          sm100::tc_fence_before();
          sm100::named_bar_sync(1, kEpiWarps * 32);
          if (threadIdx.x == 64) {
            if (lt == 0 && p == 0) sm100::mbar_wait(bar_bres, 0);  // the logits' weight image
            sm100::tc_fence_after();
            constexpr uint32_t lidesc = sm100::idesc_f16(128, 32);
#pragma unroll
            for (int rr = r; rr < r + 2; ++rr)
#pragma unroll
              for (int k = 0; k < N / 16; ++k) {
                const uint64_t ad = sm100::smem_desc(sm100::smem_u32(sStg + (rr * (N / 8) + 2 * k) * 2048), 2048, 128);
                const uint64_t bd = sm100::smem_desc(sm100::smem_u32(sLW + 2 * k * 512), 512, 128);
                sm100::mma_f16(tmem_base + acc * C::kAccCols + (R - 1 - rr) * N, ad, bd, lidesc, k ? 1u : 0u);
              }
            sm100::mma_commit(bar_lfull + 8 * p);
          }
        }
        const int64_t hw = (int64_t)a.H * a.W;
#pragma unroll 1
        for (int p = 0; p < R / 2; ++p) {
          sm100::mbar_wait(bar_lfull + 8 * p, lt & 1);  // completes once per tile
          sm100::tc_fence_after();
          const int rr = 2 * p + half;
          uint32_t u0[16], u1[16];
          sm100::tmem_ld16_nowait(t_row0 + (R - 1 - rr) * N, u0);
          sm100::tmem_ld16_nowait(t_row0 + (R - 1 - rr) * N + 16, u1);
          sm100::tmem_wait_ld_regs(u0, u1);
          const int y = y0 + rr;
          if (xin && y < a.H) {
            const int64_t pix = (int64_t)y * a.W + x;
#pragma unroll
            for (int s_ = 0; s_ < 2; ++s_) {
              if (s_ >= a.lg) break;
              float l[9], mx = -INFINITY;
#pragma unroll
              for (int j = 0; j < 9; ++j) {
                const int c = 9 * s_ + j;
                l[j] = __uint_as_float(c < 16 ? u0[c] : u1[c - 16]) + s_lbias[c];
                mx = fmaxf(mx, l[j]);
              }
              float sum = 0.f;
#pragma unroll
              for (int j = 0; j < 9; ++j) {
                l[j] = __expf(l[j] - mx);  // arguments <= 0: ex2.approx, rel. error ~1e-7
                sum += l[j];
              }
              const float inv = __frcp_rn(sum);
#pragma unroll
              for (int j = 0; j < 9; ++j) a.kw[s_][j * hw + pix] = l[j] * inv;
            }
          }
        }
      } else {
        constexpr int kCb = N / 16;
#pragma unroll 1
        for (int item = half; item < (R / 2) * kCb; item += 2) {
          const int r = 2 * (item / kCb);
          const int cb = 16 * (item % kCb);
          const int y = y0 + r;
          {
            float v0[16], v1[16];
            {
              uint32_t r0[16], r1[16];
              sm100::tmem_ld16_nowait(t_row0 + (R - 1 - r) * N + cb, r0);
              sm100::tmem_ld16_nowait(t_row0 + (R - 2 - r) * N + cb, r1);
              sm100::tmem_wait_ld_regs(r0, r1);
#pragma unroll
              for (int j = 0; j < 16; ++j) { v0[j] = __uint_as_float(r0[j]); v1[j] = __uint_as_float(r1[j]); }
            }
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const float b = s_bias[cb + j];
              v0[j] += b;
              v1[j] += b;
              if (a.relu) { v0[j] = fmaxf(v0[j], 0.f); v1[j] = fmaxf(v1[j], 0.f); }
            }
            if (xin) {
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const int g = (cb >> 3) + h;
                if (8 * g >= a.cout) continue;
                if (y < a.H) {
                  uint4 pk;
                  __half2* p2 = reinterpret_cast<__half2*>(&pk);
#pragma unroll
                  for (int j = 0; j < 4; ++j) p2[j] = __floats2half2_rn(v0[8 * h + 2 * j], v0[8 * h + 2 * j + 1]);
                  *reinterpret_cast<uint4*>(a.dst + g * plane + ((int64_t)y * a.W + x) * 8) = pk;
                }
                if (y + 1 < a.H) {
                  uint4 pk;
                  __half2* p2 = reinterpret_cast<__half2*>(&pk);
#pragma unroll
                  for (int j = 0; j < 4; ++j) p2[j] = __floats2half2_rn(v1[8 * h + 2 * j], v1[8 * h + 2 * j + 1]);
                  *reinterpret_cast<uint4*>(a.dst + g * plane + ((int64_t)(y + 1) * a.W + x) * 8) = pk;
                }
              }
            }
            if (a.pool_dst) {
              // avg_pool2: 0.25 * (p00 + p10 + p01 + p11) (autograd.py:285-286), x-pairs are lanes
              float pv[16];
#pragma unroll
              for (int j = 0; j < 16; ++j) {
                const float nb0 = __shfl_xor_sync(0xffffffffu, v0[j], 1);
                const float nb1 = __shfl_xor_sync(0xffffffffu, v1[j], 1);
                pv[j] = 0.25f * (((v0[j] + v1[j]) + nb0) + nb1);
              }
              if (((lane & 1) == 0) && xin && y < a.H) {
                const int px = x >> 1, py = y >> 1;
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                  if (cb + 8 * h >= a.cout) continue;
                  uint4 pk;
                  __half2* p2 = reinterpret_cast<__half2*>(&pk);
#pragma unroll
                  for (int j = 0; j < 4; ++j) p2[j] = __floats2half2_rn(pv[8 * h + 2 * j], pv[8 * h + 2 * j + 1]);
                  *reinterpret_cast<uint4*>(a.pool_dst + ((cb >> 3) + h) * pplane + ((int64_t)py * Wp + px) * 8) = pk;
                }
              }
            }
          }
          if constexpr (kPairs) {
            // last item of this row pair for this warp: release the pair to the next tile's MMAs
            if (item + 2 >= (R / 2) * kCb || (item + 2) / kCb != item / kCb) {
              sm100::tc_fence_before();
              __syncwarp();
              if (lane == 0) sm100::mbar_arrive(bar_pair + 8 * (item / kCb));
            }
          }
        }
      }
      sm100::tc_fence_before();
      __syncwarp();
      if (!kPairs && lane == 0) sm100::mbar_arrive(bar_tempty + 8 * acc);
    }
  }
  if (prof && lane == 0) {
    unsigned long long* o = a.prof + (int64_t)blockIdx.x * kProfSlots;
    if (warp == 0) atomicAdd(o + 0, w_empty);
    if (warp == 1) {
      atomicAdd(o + 1, w_full);
      atomicAdd(o + 2, w_tempty);
      atomicAdd(o + 4, clock64() - t_start);
      atomicAdd(o + 5, (unsigned long long)n_my_tiles);
    }
    if (warp >= 2) atomicAdd(o + 3, w_tfull / kEpiWarps);
  }
  __syncthreads();
  if (warp == 1) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc<512>(tmem_base);
  }
}

// ---- CTA pairs (cta_group::2) for the cout = 64 row-fused convs -----------------------------------
// A 2-CTA cluster runs one 128 x (2 x 4)-pixel tile pair: CTA c holds output rows [4c, 4c + 4) of the
// pair's eight and its own A halo; the leader's elected thread issues tcgen05.mma.cta_group::2 with
// M = 256 (each CTA's 128 pixels), and B's N columns are split between the two CTAs' shared memory.
// Each CTA therefore streams HALF of the weight operand per MMA: the per-SM operand reads of a
// K-stage drop from 72 KB A + 72 KB B to 72 KB + 36 KB (the single-CTA engine is bound by exactly
// these reads at ~107 B/cycle). The row-fused windows ([dy_lo, dy_hi] x 64 columns) are the same in
// both CTAs (the same relative halo row), so each CTA keeps, per dx, its half of each of the six
// window types as a contiguous block ([n/8][k-half][8][8] fp16: LBO 128 B, SBO 256 B).
// Synchronisation: each CTA's copies complete on its own full barrier; the peer's (idle) MMA warp
// forwards its full / resident-weight phases to the leader with remote mbarrier arrivals; the
// leader's commits multicast to both CTAs' empty and accumulator-full barriers; both CTAs'
// epilogue warps release the accumulator on the leader's barrier.
constexpr int kPairWinCols[6] = {32, 32, 32, 64, 64, 96};  // half-window widths: [0] [1] [2] [01] [12] [012]
constexpr int kPairWinOff[6] = {0, 32, 64, 96, 160, 224};
__host__ __device__ constexpr int pair_win_off(int wt) {
  return wt == 0 ? 0 : wt == 1 ? 32 : wt == 2 ? 64 : wt == 3 ? 96 : wt == 4 ? 160 : 224;
}
constexpr int kPairDxCols = 320;
constexpr int kPairStageBytes = 3 * kPairDxCols * 32;  // per CTA per K-stage: 30 KB
__host__ __device__ constexpr int pair_win(int lo, int hi) {
  return lo == hi ? lo : (hi - lo == 1 ? 3 + lo : 5);
}

template <int S, bool BRES>
struct PairCfg {
  static constexpr int R = 4, N = 64;
  static constexpr int kABytes = kStageGroups * (R + 2) * kRowBytes;
  static constexpr int kPlaneBytes = (R + 2) * kRowBytes;
  static constexpr int kBSlots = BRES ? kBResStages : S;
  static constexpr int kSmem = S * kABytes + kBSlots * kPairStageBytes + 1024 + 256 + N * 4;
};

template <int S, bool BRES>
__global__ void __launch_bounds__(kThreads, 1) conv3x3_pair_kernel(ConvArgs a) {
  using C = PairCfg<S, BRES>;
  constexpr int R = 4, N = 64;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + S * C::kABytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sB + C::kBSlots * kPairStageBytes);
  // bars: full[S], empty[S], pairfull[S], tfull[2], tempty[2], bres, pairbres
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * S + 6);
  float* s_bias = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(bars) + 256);
  const uint32_t bar_full = sm100::smem_u32(bars);
  const uint32_t bar_empty = bar_full + 8 * S;
  const uint32_t bar_pfull = bar_empty + 8 * S;
  const uint32_t bar_tfull = bar_pfull + 8 * S;
  const uint32_t bar_tempty = bar_tfull + 16;
  const uint32_t bar_bres = bar_tempty + 16;
  const uint32_t bar_pbres = bar_bres + 8;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = sm100::cluster_ctarank();
  const bool leader = rank == 0;

  if (threadIdx.x == 0) {
    for (int s_ = 0; s_ < S; ++s_) {
      sm100::mbar_init(bar_full + 8 * s_, 2);
      sm100::mbar_init(bar_empty + 8 * s_, 1);
      sm100::mbar_init(bar_pfull + 8 * s_, 1);
    }
    for (int s_ = 0; s_ < 2; ++s_) {
      sm100::mbar_init(bar_tfull + 8 * s_, 1);
      sm100::mbar_init(bar_tempty + 8 * s_, 2 * kEpiWarps);
    }
    sm100::mbar_init(bar_bres, 1);
    sm100::mbar_init(bar_pbres, 1);
    sm100::fence_mbar_init();
    if (BRES) {
      const uint32_t wb = (uint32_t)(a.n_kstages * kPairStageBytes);
      sm100::mbar_arrive_expect_tx(bar_bres, wb);
      // this CTA's halves: stage s at image offset (2 s + rank) * kPairStageBytes
      for (int s_ = 0; s_ < a.n_kstages; ++s_)
        sm100::bulk_g2s(sm100::smem_u32(sB + s_ * kPairStageBytes),
                        reinterpret_cast<const uint8_t*>(a.wimg) + (int64_t)(2 * s_ + rank) * kPairStageBytes,
                        kPairStageBytes, bar_bres);
    }
  }
  if (warp == 1) sm100::tmem_alloc_pair<512>(sm100::smem_u32(tmem_slot));
  sm100::tc_fence_before();
  sm100::cluster_sync();  // both CTAs' barriers initialised before any remote arrival
  sm100::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  fv::pdl_wait();

  const int pair_rows = 2 * R;
  const int tiles_py = (a.H + pair_rows - 1) / pair_rows;
  const int n_tiles = a.tiles_x * tiles_py;
  const int cluster = blockIdx.x >> 1, n_clusters = gridDim.x >> 1;

  if (warp == 0) {
    // ---------------- producer (both CTAs): this CTA's halo rows + (streamed) its B halves ----------------
    int it = 0;
    for (int tile = cluster; tile < n_tiles; tile += n_clusters) {
      const int x0 = (tile % a.tiles_x) * kTileW;
      const int y0 = (tile / a.tiles_x) * pair_rows + (int)rank * R;
      const int rows_in = max(0, min(R + 1, a.H - y0) - max(0, 1 - y0) + 1);
      const int lo = max(x0 - 1, 0), hi = min(x0 + kTileW + 1, a.W);
      const uint32_t tile_bytes_per_group = hi > lo ? (uint32_t)(rows_in * (hi - lo) * 16) : 0u;
      for (int ks = 0; ks < a.n_kstages; ++ks, ++it) {
        const int st = it % S;
        const uint32_t round = it / S;
        sm100::mbar_wait_cluster(bar_empty + 8 * st, (round & 1) ^ 1);  // released by the leader's commit
        const int g0 = ks * kStageGroups;
        int gs = a.groups - g0;
        if (gs > kStageGroups) gs = kStageGroups;
        const int gs_fill = (gs + 1) & ~1;
        const int n_items = gs_fill * (R + 2);
        const uint32_t tot = (uint32_t)gs * tile_bytes_per_group;
        const uint32_t b_bytes = BRES ? 0u : (uint32_t)kPairStageBytes;
        if (lane == 0) sm100::mbar_arrive_expect_tx(bar_full + 8 * st, tot + b_bytes);
        const uint32_t a_st = sm100::smem_u32(sA + st * C::kABytes);
        if (!BRES && lane == 0)
          sm100::bulk_g2s(sm100::smem_u32(sB + st * kPairStageBytes),
                          reinterpret_cast<const uint8_t*>(a.wimg) + (int64_t)(2 * ks + rank) * kPairStageBytes,
                          b_bytes, bar_full + 8 * st);
        for (int item = lane; item < n_items; item += 32) {
          const int g = item / (R + 2), row = item % (R + 2);
          const int y = y0 - 1 + row;
          const uint32_t row_addr = a_st + g * C::kPlaneBytes + row * kRowBytes;
          const int gg = g0 + g;
          if (gg < a.groups && y >= 0 && y < a.H) {
            int s_ = 0, gl = gg;
            while (s_ + 1 < a.n_src && gl >= a.src_groups[s_]) { gl -= a.src_groups[s_]; ++s_; }
            const __half* plane = a.src[s_] + (int64_t)gl * a.H * a.W * 8;
            const int c_lo = lo - (x0 - 1), c_hi = hi - (x0 - 1);
            if (hi > lo)
              sm100::bulk_g2s(row_addr + c_lo * 16, plane + ((int64_t)y * a.W + lo) * 8, (uint32_t)(hi - lo) * 16u,
                              bar_full + 8 * st);
            for (int c = 0; c < c_lo; ++c) sm100::st_shared_zero16(row_addr + c * 16);
            for (int c = max(c_hi, 0); c < kHaloW; ++c) sm100::st_shared_zero16(row_addr + c * 16);
          } else {
            for (int c = 0; c < kHaloW; ++c) sm100::st_shared_zero16(row_addr + c * 16);
          }
        }
        sm100::fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) sm100::mbar_arrive(bar_full + 8 * st);
      }
    }
  } else if (warp == 1 && !leader) {
    // ---------------- peer: forward this CTA's operand phases to the leader ----------------
    if (BRES) {
      sm100::mbar_wait(bar_bres, 0);
      if (lane == 0) sm100::mbar_arrive_cluster(sm100::mapa_shared(bar_pbres, 0));
    }
    int it = 0;
    for (int tile = cluster; tile < n_tiles; tile += n_clusters)
      for (int ks = 0; ks < a.n_kstages; ++ks, ++it) {
        const int st = it % S;
        sm100::mbar_wait(bar_full + 8 * st, (it / S) & 1);
        if (lane == 0) sm100::mbar_arrive_cluster(sm100::mapa_shared(bar_pfull + 8 * st, 0));
      }
  } else if (warp == 1) {
    // ---------------- leader: MMA issue for the pair ----------------
    const bool prof = kProfileBuild && a.prof != nullptr;
    unsigned long long w_full = 0, w_pfull = 0, w_tempty = 0;
    const unsigned long long t_start = prof ? clock64() : 0ull;
    if (BRES) {
      sm100::mbar_wait(bar_bres, 0);
      sm100::mbar_wait_cluster(bar_pbres, 0);
    }
    int it = 0, lt = 0;
    for (int tile = cluster; tile < n_tiles; tile += n_clusters, ++lt) {
      const int acc = lt & 1;
      {
        const unsigned long long t0 = prof ? clock64() : 0ull;
        sm100::mbar_wait_cluster(bar_tempty + 8 * acc, ((lt >> 1) & 1) ^ 1);
        if (prof) w_tempty += clock64() - t0;
      }
      sm100::tc_fence_after();
      const uint32_t d_base = tmem_base + acc * R * N;
      for (int ks = 0; ks < a.n_kstages; ++ks, ++it) {
        const int st = it % S;
        const uint32_t par = (it / S) & 1;
        pwait(bar_full + 8 * st, par, prof, w_full);
        {
          const unsigned long long t0 = prof ? clock64() : 0ull;
          sm100::mbar_wait_cluster(bar_pfull + 8 * st, par);
          if (prof) w_pfull += clock64() - t0;
        }
        sm100::tc_fence_after();
        const uint64_t a0 = sm100::smem_desc(sm100::smem_u32(sA + st * C::kABytes), C::kPlaneBytes, 128);
        const uint32_t b_stage = sm100::smem_u32(sB + (BRES ? ks : st) * kPairStageBytes);
        if (sm100::elect_one()) {
#pragma unroll
          for (int it2 = 0; it2 < 3 * (R + 2); ++it2) {
            const int h = it2 % (R + 2), dx = it2 / (R + 2);
            const int dy_lo = h - R + 1 > 0 ? h - R + 1 : 0;
            const int dy_hi = h < 2 ? h : 2;
            const int r_first = h - dy_lo;
            const uint64_t ad = a0 + (uint64_t)(((h * kHaloW + dx) * 16) >> 4);
            const uint32_t d0 = d_base + (R - 1 - r_first) * N;
            const uint32_t bdx = b_stage + dx * kPairDxCols * 32;
            if (ks == 0 && dx == 0 && dy_lo == 0) {
              // row h's first contribution (dy = 0) overwrites; the older rows accumulate
              sm100::mma_f16_pair(d0, ad, sm100::smem_desc(bdx + pair_win_off(0) * 32, 128, 256),
                                  sm100::idesc_f16(256, N), 0u);
              if (dy_hi >= 1)
                sm100::mma_f16_pair(d0 + N, ad,
                                    sm100::smem_desc(bdx + pair_win_off(pair_win(1, dy_hi)) * 32, 128, 256),
                                    sm100::idesc_f16(256, dy_hi * N), 1u);
            } else {
              sm100::mma_f16_pair(d0, ad, sm100::smem_desc(bdx + pair_win_off(pair_win(dy_lo, dy_hi)) * 32, 128, 256),
                                  sm100::idesc_f16(256, (dy_hi - dy_lo + 1) * N), 1u);
            }
          }
        }
        __syncwarp();
        sm100::mma_commit_pair_elect(bar_empty + 8 * st);
        __syncwarp();
      }
      sm100::mma_commit_pair_elect(bar_tfull + 8 * acc);
      __syncwarp();
    }
    if (prof && lane == 0) {
      unsigned long long* o = a.prof + (int64_t)blockIdx.x * kProfSlots;
      atomicAdd(o + 1, w_full);
      atomicAdd(o + 0, w_pfull);  // (slot 0 = the peer-forward wait in the pair kernel)
      atomicAdd(o + 2, w_tempty);
      atomicAdd(o + 4, clock64() - t_start);
      atomicAdd(o + 5, (unsigned long long)lt);
    }
  } else if (warp >= 2) {
    // ---------------- epilogue (both CTAs): this CTA's 4 rows of the pair ----------------
    for (int i = threadIdx.x - 64; i < N; i += kEpiWarps * 32) s_bias[i] = __ldg(a.bias + i);
    sm100::named_bar_sync(1, kEpiWarps * 32);
    const int q = warp & 3;
    const int half = (warp - 2) >> 2;
    const int64_t plane = (int64_t)a.H * a.W * 8;
    const int Hp = a.H >> 1, Wp = a.W >> 1;
    const int64_t pplane = (int64_t)Hp * Wp * 8;
    const uint32_t tempty_leader = sm100::mapa_shared(bar_tempty, 0);
    int lt = 0;
    for (int tile = cluster; tile < n_tiles; tile += n_clusters, ++lt) {
      const int acc = lt & 1;
      const int x0 = (tile % a.tiles_x) * kTileW;
      const int y0 = (tile / a.tiles_x) * pair_rows + (int)rank * R;
      sm100::mbar_wait_cluster(bar_tfull + 8 * acc, (lt >> 1) & 1);  // the leader's commit
      sm100::tc_fence_after();
      const int x = x0 + 32 * q + lane;
      const bool xin = x < a.W;
      const uint32_t t_row0 = tmem_base + ((uint32_t)(32 * q) << 16) + acc * R * N;
      constexpr int kCb = N / 16;
#pragma unroll 1
      for (int item = half; item < (R / 2) * kCb; item += 2) {
        const int r = 2 * (item / kCb);
        const int cb = 16 * (item % kCb);
        const int y = y0 + r;
        float v0[16], v1[16];
        {
          uint32_t r0[16], r1[16];
          sm100::tmem_ld16_nowait(t_row0 + (R - 1 - r) * N + cb, r0);
          sm100::tmem_ld16_nowait(t_row0 + (R - 2 - r) * N + cb, r1);
          sm100::tmem_wait_ld_regs(r0, r1);
#pragma unroll
          for (int j = 0; j < 16; ++j) { v0[j] = __uint_as_float(r0[j]); v1[j] = __uint_as_float(r1[j]); }
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const float b = s_bias[cb + j];
          v0[j] += b;
          v1[j] += b;
          if (a.relu) { v0[j] = fmaxf(v0[j], 0.f); v1[j] = fmaxf(v1[j], 0.f); }
        }
        if (xin) {
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const int g = (cb >> 3) + hh;
            if (8 * g >= a.cout) continue;
            if (y < a.H) {
              uint4 pk;
              __half2* p2 = reinterpret_cast<__half2*>(&pk);
#pragma unroll
              for (int j = 0; j < 4; ++j) p2[j] = __floats2half2_rn(v0[8 * hh + 2 * j], v0[8 * hh + 2 * j + 1]);
              *reinterpret_cast<uint4*>(a.dst + g * plane + ((int64_t)y * a.W + x) * 8) = pk;
            }
            if (y + 1 < a.H) {
              uint4 pk;
              __half2* p2 = reinterpret_cast<__half2*>(&pk);
#pragma unroll
              for (int j = 0; j < 4; ++j) p2[j] = __floats2half2_rn(v1[8 * hh + 2 * j], v1[8 * hh + 2 * j + 1]);
              *reinterpret_cast<uint4*>(a.dst + g * plane + ((int64_t)(y + 1) * a.W + x) * 8) = pk;
            }
          }
        }
        if (a.pool_dst) {
          float pv[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const float nb0 = __shfl_xor_sync(0xffffffffu, v0[j], 1);
            const float nb1 = __shfl_xor_sync(0xffffffffu, v1[j], 1);
            pv[j] = 0.25f * (((v0[j] + v1[j]) + nb0) + nb1);
          }
          if (((lane & 1) == 0) && xin && y < a.H) {
            const int px = x >> 1, py = y >> 1;
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
              if (cb + 8 * hh >= a.cout) continue;
              uint4 pk;
              __half2* p2 = reinterpret_cast<__half2*>(&pk);
#pragma unroll
              for (int j = 0; j < 4; ++j) p2[j] = __floats2half2_rn(pv[8 * hh + 2 * j], pv[8 * hh + 2 * j + 1]);
              *reinterpret_cast<uint4*>(a.pool_dst + ((cb >> 3) + hh) * pplane + ((int64_t)py * Wp + px) * 8) = pk;
            }
          }
        }
      }
      sm100::tc_fence_before();
      __syncwarp();
      if (lane == 0) sm100::mbar_arrive_cluster(tempty_leader + 8 * acc);
    }
  }
  sm100::tc_fence_before();
  sm100::cluster_sync();  // the pair's MMAs and both epilogues are done before the TMEM is freed
  if (warp == 1) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc_pair<512>(tmem_base);
  }
}

template <int S, bool BRES>
int launch_pair(fv_ctx* ctx, const ConvArgs& args) {
  using C = PairCfg<S, BRES>;
  static_assert(C::kSmem <= 227 * 1024, "pair conv configuration exceeds shared memory");
  static bool attr_set = false;
  if (!attr_set) {
    FV_CUDA(cudaFuncSetAttribute(conv3x3_pair_kernel<S, BRES>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem));
    attr_set = true;
  }
  ConvArgs a = args;
  a.tiles_x = (a.W + kTileW - 1) / kTileW;
  a.tiles_y = (a.H + 7) / 8;
  const int n_pairs = a.tiles_x * a.tiles_y;
  const int clusters = std::min(n_pairs, ctx->num_sms / 2);
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = fv::pdl_enabled() ? 1 : 0;
  at[1].id = cudaLaunchAttributeClusterDimension;
  at[1].val.clusterDim.x = 2;
  at[1].val.clusterDim.y = 1;
  at[1].val.clusterDim.z = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * clusters);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = C::kSmem;
  cfg.stream = ctx->stream;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  ktime_begin(ctx);
  FV_CUDA(cudaLaunchKernelEx(&cfg, conv3x3_pair_kernel<S, BRES>, a));
  ktime_end(ctx, FV_KC_CONV, a.flops);
  if (a.prof) {
    const int grid = 2 * clusters;
    std::vector<unsigned long long> h((size_t)grid * kProfSlots);
    FV_CUDA(cudaMemcpyAsync(h.data(), a.prof, h.size() * 8, cudaMemcpyDeviceToHost, ctx->stream));
    FV_CUDA(cudaStreamSynchronize(ctx->stream));
    double sm[kProfSlots] = {};
    for (int b = 0; b < grid; b += 2)
      for (int k = 0; k < kProfSlots; ++k) sm[k] += (double)h[(size_t)b * kProfSlots + k] / clusters;
    fprintf(stderr, "[pair prof] %dx%d groups=%d: per leader %.1f tiles, total %.0f cyc; waits full %.0f peer %.0f tempty %.0f\n",
            a.H, a.W, a.groups, sm[5], sm[4], sm[1], sm[0], sm[2]);
  }
  {
    const int hrc = conv_launched(ctx);
    if (hrc) return hrc;
  }
  FV_CHECK_LAUNCH("conv3x3_pair_kernel");
  ctx->launches += 1;
  return 0;
}

template <int R, int N, int S, bool BRES, bool FUSED, bool CO = false, bool TAPN = false, bool LG = false>
int launch(fv_ctx* ctx, const ConvArgs& args) {
  using C = Cfg<R, N, S, BRES, TAPN, LG>;
  static_assert(C::kSmem <= 227 * 1024, "conv tile configuration exceeds shared memory");
  static_assert(!TAPN || (R == 4 && N >= 32 && !FUSED && !CO), "TAPN: 4-row tiles, >= 32 columns, plain issue");
  static bool attr_set = false;
  if (!attr_set) {
    FV_CUDA(cudaFuncSetAttribute(conv3x3_tc_kernel<R, N, S, BRES, FUSED, CO, TAPN, LG>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem));
    attr_set = true;
  }
  ConvArgs a = args;
  constexpr int kStride = TAPN ? kTapnStride : kTileW;
  a.tiles_x = (a.W + kStride - 1) / kStride;
  a.tiles_y = (a.H + R - 1) / R;
  const int n_tiles = a.tiles_x * a.tiles_y;
  const int grid = n_tiles < ctx->num_sms ? n_tiles : ctx->num_sms;
  ktime_begin(ctx);
  fv::launch_pdl(conv3x3_tc_kernel<R, N, S, BRES, FUSED, CO, TAPN, LG>, grid, kThreads, C::kSmem, ctx->stream, a);
  ktime_end(ctx, FV_KC_CONV, a.flops);
  {
    const int hrc = conv_launched(ctx);
    if (hrc) return hrc;
  }
  if (a.prof) {
    std::vector<unsigned long long> h((size_t)grid * kProfSlots);
    FV_CUDA(cudaMemcpyAsync(h.data(), a.prof, h.size() * 8, cudaMemcpyDeviceToHost, ctx->stream));
    FV_CUDA(cudaStreamSynchronize(ctx->stream));
    double s[kProfSlots] = {};
    for (int b = 0; b < grid; ++b)
      for (int k = 0; k < kProfSlots; ++k) s[k] += (double)h[(size_t)b * kProfSlots + k] / grid;
    fprintf(stderr,
            "[conv prof] R=%d N=%d S=%d bres=%d fused=%d %dx%d groups=%d: per CTA %.1f tiles, total %.0f cyc; "
            "MMA waits full %.0f tempty %.0f; producer empty-wait %.0f; epilogue tfull-wait %.0f\n",
            R, N, S, (int)BRES, (int)FUSED, a.H, a.W, a.groups, s[5], s[4], s[1], s[2], s[0], s[3]);
  }
  FV_CHECK_LAUNCH("conv3x3_tc_kernel");
  ctx->launches += 1;
  return 0;
}

}  // namespace

// B image of stage s (channels c = (2s + kg)*8 + e): [tap t (9)][kg (2)][n (N)][8] fp16, or for
// row-fused convs [dx (3)][kg (2)][dy*N + n][8] (see issue_stage_rows).
int conv_prepare(fv_ctx* ctx, ConvParam& cp) {
  const int groups = (cp.cin + 7) / 8;
  const int N = cp.n_pad;
  static const bool no_fuse = getenv("FV_CONV_FUSE") && atoi(getenv("FV_CONV_FUSE")) == 0;  // A/B runs
  cp.row_fused = !no_fuse && !cp.center_only && !cp.tapn && 3 * N <= 256;
  // CTA pairs for the row-fused cout = 64 convs: opt-in FV_CONV_PAIR=1 (see conv3x3_pair_kernel)
  static const bool pair_on = getenv("FV_CONV_PAIR") && atoi(getenv("FV_CONV_PAIR")) == 1;
  cp.pair = pair_on && cp.row_fused && N == 64 && !cp.head_conv;
  cp.n_stages = (groups + kStageGroups - 1) / kStageGroups;
  cp.stage_groups.clear();
  cp.stage_off.clear();
  int64_t off = 0;
  for (int s = 0; s < cp.n_stages; ++s) {
    int gs = groups - s * kStageGroups;
    if (gs > kStageGroups) gs = kStageGroups;
    gs = (gs + 1) & ~1;
    cp.stage_groups.push_back(gs);
    cp.stage_off.push_back(off);
    off += (int64_t)9 * kStageGroups * N * 16;  // stages strided at the full-stage size
  }
  if (cp.pair) off = (int64_t)cp.n_stages * 2 * kPairStageBytes;  // [stage][rank][dx][320 cols][32 B]
  cp.wbytes = off;
  std::vector<__half> img(off / 2, __float2half(0.f));
  for (int s = 0; s < cp.n_stages && cp.pair; ++s)
    for (int rk = 0; rk < 2; ++rk)
      for (int dx = 0; dx < 3; ++dx)
        for (int wt = 0; wt < 6; ++wt) {
          const int lo = wt < 3 ? wt : (wt == 3 ? 0 : (wt == 4 ? 1 : 0));
          const int half_w = kPairWinCols[wt];
          __half* base = img.data() + (((int64_t)(2 * s + rk) * 3 + dx) * kPairDxCols + kPairWinOff[wt]) * 16;
          for (int j = 0; j < half_w; ++j) {
            const int wj = rk * half_w + j;  // column of the full window
            const int dy = lo + wj / 64, n = wj % 64;
            const int t = dy * 3 + dx;
            for (int kg = 0; kg < 2; ++kg)
              for (int e = 0; e < 8; ++e) {
                const int c = (s * kStageGroups + kg) * 8 + e;
                const float w = (n < cp.cout && c < cp.cin) ? cp.w_host[((int64_t)n * cp.cin + c) * 9 + t] : 0.f;
                // [n/8][kg][8 rows][8 elements]
                base[((int64_t)(j / 8) * 2 + kg) * 64 + (j % 8) * 8 + e] = __float2half(w);
              }
          }
        }
  for (int s = 0; s < cp.n_stages && cp.tapn; ++s) {
    // TAPN: [kg][n][8] per stage; column n -> (output o, tap t) of the K-stage layout (D.head
    // outputs 0..2 with their nine taps, the logits of the two K blocks at the centre tap)
    __half* base = img.data() + cp.stage_off[s] / 2;
    for (int kg = 0; kg < 2; ++kg)
      for (int n = 0; n < N; ++n) {
        int o = -1, t = 4;
        if (n < 27) { o = n % 3; t = n / 3; }
        else if (n < 36) o = kLogitCol[0] + (n - 27);
        else if (n < 45) o = kLogitCol[1] + (n - 36);
        for (int e = 0; e < 8; ++e) {
          const int c = (s * kStageGroups + kg) * 8 + e;
          const float w = (o >= 0 && o < cp.cout && c < cp.cin) ? cp.w_host[((int64_t)o * cp.cin + c) * 9 + t] : 0.f;
          base[((int64_t)kg * N + n) * 8 + e] = __float2half(w);
        }
      }
  }
  for (int s = 0; s < cp.n_stages && !cp.tapn && !cp.pair; ++s) {
    const int gs = cp.stage_groups[s];
    const int nk = gs / 2;
    __half* base = img.data() + cp.stage_off[s] / 2;
    for (int t = 0; t < 9; ++t)
      for (int k = 0; k < nk; ++k)
        for (int kg = 0; kg < 2; ++kg)
          for (int n = 0; n < N; ++n)
            for (int e = 0; e < 8; ++e) {
              const int c = (s * kStageGroups + 2 * k + kg) * 8 + e;
              float w = 0.f;
              if (n < cp.cout && c < cp.cin) w = cp.w_host[((int64_t)n * cp.cin + c) * 9 + t];
              if (cp.row_fused)  // nk == 1
                base[(((int64_t)(t % 3) * 2 + kg) * 3 * N + (t / 3) * N + n) * 8 + e] = __float2half(w);
              else
                base[((((int64_t)t * nk + k) * 2 + kg) * N + n) * 8 + e] = __float2half(w);
            }
  }
  if (cp.w_dev) cudaFree(cp.w_dev);
  if (cp.b_dev) cudaFree(cp.b_dev);
  cp.w_dev = nullptr;
  cp.b_dev = nullptr;
  FV_CUDA(cudaMalloc(&cp.w_dev, cp.wbytes));
  FV_CUDA(cudaMemcpy(cp.w_dev, img.data(), cp.wbytes, cudaMemcpyHostToDevice));
  std::vector<float> b(N, 0.f);
  for (int n = 0; n < cp.cout; ++n) b[n] = cp.b_host[n];
  FV_CUDA(cudaMalloc(&cp.b_dev, sizeof(float) * N));
  FV_CUDA(cudaMemcpy(cp.b_dev, b.data(), sizeof(float) * N, cudaMemcpyHostToDevice));
  (void)ctx;
  return 0;
}

// 4-row tiles (single accumulator, row-pair release) for the row-fused 80-column convs
// (FV_N80_R=4 measured: D4.conv1 256 -> 80 at 270 x 480 66 -> 53 us, frame conv 1133 -> 1117 us;
// 4-row tiles halve the streamed weight bytes per output pixel). FV_N80_R=2 keeps 2-row tiles.
static bool n80_r4() {
  static const bool on = !(getenv("FV_N80_R") && atoi(getenv("FV_N80_R")) == 2);
  return on;
}


// Whether conv3x3 has a fused-logits (LG) variant for this conv's shape (see its dispatch)
bool logits_fusable(const ConvParam& cp) {
  const bool res = cp.n_stages <= kBResStages;
  return (cp.n_pad == 64 && res && cp.row_fused) || (cp.n_pad == 80 && !res && cp.row_fused) ||
         (cp.n_pad == 96 && !res && !cp.row_fused);
}

// The K stage's level logits as the LG epilogue's 1x1 GEMM B operand: w_host (cout = 9 x blocks,
// cin) row-major -> [cin/8][32][8] fp16 (K-major, LBO 512 B, SBO 128 B), bias padded to 32.
int logits_prepare(fv_ctx* ctx, ConvParam& cp) {
  FV_REQUIRE(cp.cin % 8 == 0 && cp.cout <= 32, "logits %s: cin %d / cout %d", cp.name.c_str(), cp.cin, cp.cout);
  cp.wbytes = (int64_t)(cp.cin / 8) * 512;
  std::vector<__half> img(cp.wbytes / 2, __float2half(0.f));
  for (int o = 0; o < cp.cout; ++o)
    for (int c = 0; c < cp.cin; ++c)
      img[((size_t)(c / 8) * 32 + o) * 8 + (c % 8)] = __float2half(cp.w_host[(size_t)o * cp.cin + c]);
  if (cp.w_dev) cudaFree(cp.w_dev);
  if (cp.b_dev) cudaFree(cp.b_dev);
  cp.w_dev = nullptr;
  cp.b_dev = nullptr;
  FV_CUDA(cudaMalloc(&cp.w_dev, cp.wbytes));
  FV_CUDA(cudaMemcpy(cp.w_dev, img.data(), cp.wbytes, cudaMemcpyHostToDevice));
  std::vector<float> b(32, 0.f);
  for (int n = 0; n < cp.cout; ++n) b[n] = cp.b_host[n];
  FV_CUDA(cudaMalloc(&cp.b_dev, sizeof(float) * 32));
  FV_CUDA(cudaMemcpy(cp.b_dev, b.data(), sizeof(float) * 32, cudaMemcpyHostToDevice));
  (void)ctx;
  return 0;
}

// Public-internal entry: run one 3x3 conv. srcs: up to 3 NC8HW8 tensors at the same level.
int conv3x3(fv_ctx* ctx, const ConvParam& cp, const fv_act* srcs, int n_src, fv_act* dst,
            fv_act* pool_dst, bool relu, const ConvAux* aux) {
  ConvArgs a{};
  a.n_src = n_src;
  int groups = 0;
  for (int i = 0; i < n_src; ++i) {
    a.src[i] = srcs[i].p;
    a.src_groups[i] = srcs[i].C / 8;
    groups += srcs[i].C / 8;
  }
  FV_REQUIRE(groups * 8 == cp.cin,
             "conv %s: input has %d channels, weight expects %d", cp.name.c_str(), groups * 8, cp.cin);
  a.groups = groups;
  a.n_kstages = cp.n_stages;
  a.H = srcs[0].H;
  a.W = srcs[0].W;
  a.wimg = cp.w_dev;
  a.bias = cp.b_dev;
  a.cout = cp.cout;
  a.dst = dst ? dst->p : nullptr;
  a.pool_dst = pool_dst ? pool_dst->p : nullptr;
  a.relu = relu ? 1 : 0;
  static unsigned long long* prof_buf = nullptr;
  static const bool want_prof = kProfileBuild && getenv("FV_CONV_PROF") != nullptr;
  if (want_prof) {
    if (!prof_buf) FV_CUDA(cudaMalloc(&prof_buf, sizeof(unsigned long long) * kProfSlots * 1024));
    FV_CUDA(cudaMemsetAsync(prof_buf, 0, sizeof(unsigned long long) * kProfSlots * 1024, ctx->stream));
    a.prof = prof_buf;
  }
  a.flops = 2.0 * a.H * a.W *
            (cp.macs_per_px > 0 ? cp.macs_per_px : (double)cp.cin * cp.cout * cp.ksize * cp.ksize);
  if (aux && aux->logits) {
    // decoder conv2 with the K stage's level logits fused into its epilogue (LG)
    const ConvParam& lp = *aux->logits;
    FV_REQUIRE(!pool_dst && dst && lp.w_dev && lp.cin == cp.cout && (aux->kw[0] || aux->kw[1]),
               "conv %s: fused logits need a plain output and the level's weight planes", cp.name.c_str());
    a.lw = lp.w_dev;
    a.lb = lp.b_dev;
    a.lg = aux->kw[1] ? 2 : 1;
    a.kw[0] = aux->kw[0];
    a.kw[1] = aux->kw[1];
    a.flops += 2.0 * a.H * a.W * (double)lp.cin * 9 * a.lg;
    const bool res = cp.n_stages <= kBResStages;
    switch (cp.n_pad) {
      case 64:
        if (res && cp.row_fused) return launch<4, 64, 3, true, true, false, false, true>(ctx, a);
        break;
      case 80:
        if (!res && cp.row_fused) return launch<2, 80, 4, false, true, false, false, true>(ctx, a);
        break;
      case 96:
        if (!res && !cp.row_fused) return launch<2, 96, 3, false, false, false, false, true>(ctx, a);
        break;
    }
    set_error("conv %s: no fused-logits variant for %d columns", cp.name.c_str(), cp.n_pad);
    return FV_E_UNSUPPORTED;
  }
  if (aux) {
    a.head = 1;
    a.od = aux->od;
    a.feedback = aux->feedback;
    for (int s = 0; s < 2; ++s) {
      a.kw[s] = aux->kw[s];
      a.kcol[s] = aux->kcol[s];
    }
    a.center_only = aux->center_only ? 1 : 0;
    FV_REQUIRE((!aux->kw[0] || aux->kcol[0] == kLogitCol[0]) && (!aux->kw[1] || aux->kcol[1] == kLogitCol[1]),
               "conv %s: K-stage logits must sit at columns %d and %d", cp.name.c_str(), kLogitCol[0], kLogitCol[1]);
    FV_REQUIRE(aux->center_only == cp.center_only, "conv %s: 1x1 use needs a center-only weight image",
               cp.name.c_str());
    FV_REQUIRE(!(aux->kw[0] || aux->kw[1]) || cp.n_pad >= 32, "conv %s: logits need N >= 32", cp.name.c_str());
  }
  // stage = 16 input channels; weights resident when they fit (<= 4 stages, i.e. cin <= 64);
  // row-fused MMAs whenever 3N <= 256 (the B image was laid out for it in conv_prepare)
  const bool res = cp.n_stages <= kBResStages;
  const bool fu = cp.row_fused;
  if (cp.tapn) {
    // 48 columns: D.head's 27 tap columns + the level-0 logits; 32: D.head alone (the fused K stage)
    FV_REQUIRE(res && (cp.n_pad == 48 || (cp.n_pad == 32 && !aux->kw[0] && !aux->kw[1])) && aux,
               "conv %s: the taps-in-N K-stage conv needs cin <= 64 and 48 (32 without logits) columns",
               cp.name.c_str());
    return cp.n_pad == 48 ? launch<4, 48, 5, true, false, false, true>(ctx, a)
                          : launch<4, 32, 6, true, false, false, true>(ctx, a);
  }
#define FV_LAUNCH(R_, N_, S_) \
  (res ? (fu ? launch<R_, N_, S_, true, true>(ctx, a) : launch<R_, N_, S_, true, false>(ctx, a)) \
       : (fu ? launch<R_, N_, S_, false, true>(ctx, a) : launch<R_, N_, S_, false, false>(ctx, a)))
  if (a.center_only && cp.n_pad == 32 && !fu)  // (2-row tiles on the small levels: L2 16.9 -> 21.2 us, measured)
    return res ? launch<4, 32, 5, true, false, true>(ctx, a) : launch<4, 32, 5, false, false, true>(ctx, a);
  if (cp.pair && !aux)
    return res ? launch_pair<4, true>(ctx, a) : launch_pair<4, false>(ctx, a);
  // D.head alone (the fused K stage's level-0 conv): 8-row tiles -- 30 row-fused dispatches per
  // 8 output rows instead of 18 per 4 (the launch is bound by those A-operand reads); FV_KHEAD_R=4 A/B
  static const int khead_r = getenv("FV_KHEAD_R") ? atoi(getenv("FV_KHEAD_R")) : 8;
  if (cp.n_pad == 16 && cp.head_conv && fu && res && khead_r == 8) return launch<8, 16, 4, true, true>(ctx, a);
  switch (cp.n_pad) {
    case 16: return FV_LAUNCH(4, 16, 6);
    case 32: return FV_LAUNCH(4, 32, 5);
    case 48: return FV_LAUNCH(4, 48, 4);
    case 64:
      // (8-row tiles here -- single accumulator, 3 stages -- measured slower: E0.conv2 117 -> 171 us)
      // (8-row tiles for the streamed-weight ones measured flat / slower: D5.conv1 119 -> 118 us,
      // D6.conv1 346 -> 359 us)
      return res ? (fu ? launch<4, 64, 5, true, true>(ctx, a) : launch<4, 64, 5, true, false>(ctx, a))
                        : (fu ? launch<4, 64, 4, false, true>(ctx, a) : launch<4, 64, 4, false, false>(ctx, a));
    case 80:
      if (fu && n80_r4()) return res ? launch<4, 80, 4, true, true>(ctx, a) : launch<4, 80, 4, false, true>(ctx, a);
      return res ? (fu ? launch<2, 80, 5, true, true>(ctx, a) : launch<2, 80, 5, true, false>(ctx, a))
                        : (fu ? launch<2, 80, 4, false, true>(ctx, a) : launch<2, 80, 4, false, false>(ctx, a));
    case 96: return res ? launch<2, 96, 5, true, false>(ctx, a) : launch<2, 96, 4, false, false>(ctx, a);
    case 128: return res ? launch<2, 128, 4, true, false>(ctx, a) : launch<2, 128, 4, false, false>(ctx, a);
#undef FV_LAUNCH
    default:
      set_error("conv %s: unsupported output width %d", cp.name.c_str(), cp.cout);
      return FV_E_UNSUPPORTED;
  }
}

}  // namespace fv

extern "C" {

// Diagnostic entry: one conv over caller device buffers (NC8HW8 fp16), weights in the reference
// (oc, ic, 3, 3) float32 layout on the host. Used by the layer-level parity tests.
int fv_debug_conv3x3(fv_ctx* ctx, int cin, int cout, int H, int W, const void* x_nc8,
                     const float* w_host, const float* b_host, void* y_nc8, void* pool_nc8, int relu) {
  FV_REQUIRE(ctx && x_nc8 && w_host && b_host, "null argument");
  FV_REQUIRE(cin % 8 == 0 && cin > 0, "cin must be a positive multiple of 8");
  fv::ConvParam cp;
  cp.name = "debug";
  cp.cin = cin;
  cp.cout = cout;
  cp.n_pad = (cout + 15) / 16 * 16;
  cp.w_host.assign(w_host, w_host + (size_t)cout * cin * 9);
  cp.b_host.assign(b_host, b_host + cout);
  int rc = fv::conv_prepare(ctx, cp);
  if (rc) return rc;
  fv_act src;
  src.p = (__half*)x_nc8;
  src.C = cin;
  src.H = H;
  src.W = W;
  fv_act dst = src, pool = src;
  dst.p = (__half*)y_nc8;
  dst.C = cout;
  pool.p = (__half*)pool_nc8;
  pool.C = cout;
  pool.H = H / 2;
  pool.W = W / 2;
  rc = fv::conv3x3(ctx, cp, &src, 1, &dst, pool_nc8 ? &pool : nullptr, relu != 0, nullptr);
  cudaStreamSynchronize(ctx->stream);
  cudaFree(cp.w_dev);
  cudaFree(cp.b_dev);
  return rc;
}

}  // extern "C"
