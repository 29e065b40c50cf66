// Internal structures shared by the libfovnet translation units.
#pragma once

#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <stdint.h>
#include <string>
#include <utility>
#include <vector>

#include "../../include/fovnet.h"

namespace fv {

void set_error(const char* fmt, ...);
int cuda_fail(cudaError_t e, const char* what);

#define FV_CUDA(expr)                                   \
  do {                                                  \
    cudaError_t _e = (expr);                            \
    if (_e != cudaSuccess) return fv::cuda_fail(_e, #expr); \
  } while (0)

#define FV_CHECK_LAUNCH(what)                           \
  do {                                                  \
    cudaError_t _e = cudaGetLastError();                \
    if (_e != cudaSuccess) return fv::cuda_fail(_e, what); \
  } while (0)

#define FV_REQUIRE(cond, ...)                           \
  do {                                                  \
    if (!(cond)) { fv::set_error(__VA_ARGS__); return FV_E_INVALID; } \
  } while (0)

// Programmatic dependent launch (PDL) for the reconstruction's launch chain: a kernel launched
// with launch_pdl may start (prologue: barrier init, TMEM alloc, resident-weight copies) while the
// previous kernel on the stream drains; its pdl_wait() (griddepcontrol.wait) holds every access to
// activations until that kernel has completed and flushed, so the order of reads and writes is
// the plain stream order. No kernel triggers its dependents early (griddepcontrol.launch_dependents
// at block start measured -0.6% frames/s: the waiting blocks of the next kernel crowd the SMs);
// they launch as the blocks exit. FV_PDL=0 launches without the attribute (pdl_wait is a no-op).
bool pdl_enabled();
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args... args) {
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}
#ifdef __CUDACC__
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
#endif

// One stage of the fused K-stage chain (netops.cu kchain_kernel): op 0 = filter + 2x2 pool
// (encoder block), 1 = filter, 2 = 3-channel 2x upsample; h, w = the stage's input dims.
struct KChainStage {
  int op;
  int h, w;
  const float* kw;
  const float* in;
  float* out;
};
struct KChain {
  int n = 0;
  KChainStage s[16];
};

// Device-side counters (one cache line each to avoid false sharing).
struct DevCounters {
  unsigned long long rays;
  unsigned long long hit_rays;
  unsigned long long samples_main;
  unsigned long long samples_shadow;
  unsigned int scan_tile;  // dynamic tile counter of the mask scan
  unsigned int ray_next;   // work counter of the persistent marcher
  unsigned int wave_rec;   // wavefront marcher: records allocated
  unsigned int wave_next;  // wavefront marcher: shadow-pass work counter
  unsigned int wave_ord;   // wavefront marcher: chunks listed in ray order
  unsigned int hit_count;  // wavefront marcher: hitting rays listed by the setup pass
  unsigned int hit_next;   // wavefront marcher: work counter of the main pass over that list
  unsigned int ovf_count;  // wavefront marcher: rays that found the record buffer full
};

// Per-launch timing spans (fv_ctx_set_kernel_timing).
struct KSpan {
  cudaEvent_t a, b;
  int cls;
  double work;
};
void ktime_begin(fv_ctx* ctx);
void ktime_end(fv_ctx* ctx, int cls, double work = 0.0);
// Launch statement bracketed by the context's kernel-timing events (no-ops unless enabled).
#define FV_TIMED(ctx_, cls_, ...)     \
  do {                                \
    fv::ktime_begin(ctx_);            \
    __VA_ARGS__;                      \
    fv::ktime_end(ctx_, cls_);        \
  } while (0)

}  // namespace fv

namespace fv {
// The per-frame inputs of the mask and the marcher, read by the kernels from device memory when a
// frame is replayed as a CUDA graph (fv_frames): the camera basis of the frame being rendered and
// the fovea / noise frame / scan epoch of the mask computed next to its network. Host-filled per
// frame, copied to the device ahead of the graph launch.
struct FrameDyn {
  double pos[3], right[3], up[3], fwd[3];
  double tan_half, aspect;
  double fx, fy, sigma, pb, scale;
  int frame;
  unsigned int epoch;
};
int fill_camera_dyn(const fv_camera* cam, FrameDyn* d);
}  // namespace fv

struct fv_ctx {
  int device = 0;
  int num_sms = 148;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  // noise stack (T,H,W) float32
  float* noise = nullptr;
  int noise_T = 0, noise_H = 0, noise_W = 0;
  // mask scan tile status words (epoch-tagged), sized for the largest film seen
  unsigned long long* scan_status = nullptr;
  int scan_tiles_cap = 0;
  void* scan_aux = nullptr;  // two-pass mask: per-thread bit bytes + per-tile counts
  int64_t scan_aux_cap = 0;
  unsigned int epoch = 0;
  fv::DevCounters* counters = nullptr;  // device
  int32_t* k_scratch = nullptr;          // device int32 for fv_frame
  int32_t* idx_scratch = nullptr;        // device, capacity idx_cap
  int64_t idx_cap = 0;
  float* rgb_scratch = nullptr;          // device (H,W,3) for fv_frame
  int64_t rgb_cap = 0;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  // wavefront marcher workspace
  void* wave_rec = nullptr;   // 2 x cap float4 records
  int64_t wave_cap = 0;
  void* wave_ray = nullptr;   // int4 per compacted ray
  int64_t wave_ray_cap = 0;
  void* wave_hits = nullptr;  // 3 float4 per hitting ray (setup pass -> main pass)
  int64_t wave_hits_cap = 0;
  void* wave_ovf = nullptr;   // int per compacted ray: the record-overflow list
  int64_t wave_ovf_cap = 0;
  // previous render's record usage, read back asynchronously into pinned memory: [0] = compacted
  // rays k, [1..7] = DevCounters ray_next..ovf_count (see march.cu, record buffer sizing)
  unsigned int* wave_fb = nullptr;
  cudaEvent_t wave_fb_ev = nullptr;
  bool wave_fb_pending = false;
  unsigned long long launches = 0;
  // fv_frames whole-frame graphs: the device FrameDyn the captured kernels read (dyn_active is
  // set while a frame's launches are enqueued or captured), a pinned ring of host copies
  fv::FrameDyn* dyn_dev = nullptr;
  const fv::FrameDyn* dyn_active = nullptr;
  fv::FrameDyn* dyn_host = nullptr;  // kDynRing slots
  cudaEvent_t dyn_ev[8] = {};
  uint64_t wave_version = 0;  // bumped when the marcher record buffer is reallocated
  // march-ahead frames (fv_frames, FV_MARCH_AHEAD=k): record conv_fork_ev after the k-th conv launch
  cudaEvent_t conv_fork_ev = nullptr;
  int conv_fork_at = 0, conv_count = 0;
  // fv_frames graph path: the network's launches stop after D.head (kchain_split); the filter chain
  // + output stage run as their own graph on kstream, and the next network waits for kw_wait_ev
  // (the chain's completion) before it rewrites the weight planes / O_d
  bool kchain_split = false;
  cudaEvent_t kw_wait_ev = nullptr;
  bool kw_wait_external = false;  // kw_wait_ev recorded outside the capture (an external wait node)
  // called after the conv_hook_at-th conv launch of a frame (fv_frames: forks the previous frame's
  // filter chain off the network; counted with conv_fork_ev's counter)
  int (*conv_hook)(fv_ctx*, void*) = nullptr;
  void* conv_hook_arg = nullptr;
  int conv_hook_at = 0;
  cudaStream_t kstream = nullptr;
  cudaEvent_t kev[3] = {};  // chain done (per output buffer) [2], chain done (latest) [1]
  cudaEvent_t kdone[2] = {};  // folded chain of the frame writing image b complete (an external record node)
  // fv_frames: render / network / copy streams and their event rings (created on first use)
  cudaStream_t fstream[4] = {nullptr, nullptr, nullptr, nullptr};
  cudaEvent_t fev[10] = {};
  // kernel timing (off by default)
  bool ktiming = false;
  cudaEvent_t kopen = nullptr;
  std::vector<cudaEvent_t> kpool;
  std::vector<fv::KSpan> kspans;
  double k_ms[FV_KC_COUNT] = {}, k_work[FV_KC_COUNT] = {};
  uint64_t k_n[FV_KC_COUNT] = {};
};

struct fv_volume {
  int nx = 0, ny = 0, nz = 0;
  double spacing[3] = {1, 1, 1};
  float* data = nullptr;  // (nz,ny,nx)
  bool owns_data = true;
  float* lut_dev = nullptr;  // (K,4) float32, K <= 256
  float* bricks = nullptr;   // 8^3-bricked copy used by the fp32 marcher
  uint64_t version = 1, bricks_version = 0;
  // the same quads as a point-sampled 3D texture (block-linear layout; FV_VOL_TEX=1, A/B)
  cudaArray_t qarr = nullptr;
  unsigned long long qtex = 0;  // cudaTextureObject_t
  uint64_t tex_version = 0;
  // the voxels as a hardware-filtered (trilinear, 8-bit fractional weights) float texture: the
  // shadow pass's fast-tier sample source (one 4-byte return per sample instead of two quads)
  cudaArray_t larr = nullptr;
  unsigned long long ltex = 0;
  uint64_t ltex_version = 0;
  int ltex_bits = 0;  // texel format of larr: 16 (unorm16, voxels in [0, 1]) or 32 (float)
  int K = 0;
  double value_range[2] = {0, 0};
};

namespace fv {

// One 3x3 (or 1x1) convolution of the W-Net as stored on the device.
struct ConvParam {
  std::string name;
  int cin = 0, cout = 0, ksize = 3;
  int n_pad = 0;           // cout padded to a multiple of 16 (MMA N)
  int n_stages = 0;        // ceil(cgroups / 4)
  std::vector<int> stage_groups;   // cgroups per stage (even)
  std::vector<int64_t> stage_off;  // byte offset of each stage's B image
  int64_t wbytes = 0;
  __half* w_dev = nullptr;  // implicit-GEMM B image (see conv_tc.cu)
  float* b_dev = nullptr;   // bias (n_pad) fp32
  bool center_only = false;   // used as a 1x1 conv (K-stage logits at levels > 0)
  bool row_fused = false;     // B image stacked by dy for row-fused MMAs (conv_tc.cu)
  bool tapn = false;          // K-stage level 0: 3x3 taps of D.head in N, one MMA per halo row
  bool pair = false;          // run as 2-CTA clusters with tcgen05 cta_group::2 (conv_tc.cu)
  bool head_conv = false;     // a K-stage conv (auxiliary epilogue): never paired
  double macs_per_px = 0;     // algorithmic MACs per output pixel (0: cin * cout * ksize^2)
  std::vector<float> w_host;  // reference layout (oc,ic,kh,kw), fp16-rounded values
  std::vector<float> b_host;
  bool w_set = false, b_set = false;
};

}  // namespace fv

namespace fv {
// Auxiliary epilogue of a conv: D.head outputs and/or K-stage logits -> softmax filter weights.
// Storage type of the K-stage softmax filter weights (written by the K conv epilogue, read by the
// filter pass). fp32: measured A/B with fp16 storage saved only ~8 us per 1080p frame (the filter
// pass is not bound by these bytes) for a 100 -> 91 dB PSNR drop against the reference.
using kw_t = float;
__device__ __forceinline__ float kw_load(const kw_t* p) { return __ldg(p); }

// First logit column of the s-th K block in a K-stage conv (columns 0..2 = D.head); the conv
// epilogue indexes its TMEM registers with these, so they are compile-time constants.
constexpr int kLogitCol[2] = {4, 13};
__host__ __device__ constexpr int logit_col(int s) { return s == 0 ? 4 : 13; }
struct ConvAux {
  float* od = nullptr;         // (3,H,W) fp32, columns 0..2
  __half* feedback = nullptr;  // the next input's feedback group (kInGroups)
  const ConvParam* logits = nullptr;  // non-null: a decoder conv2 with its level's K logits fused (LG)
  kw_t* kw[2] = {nullptr, nullptr};  // (9,H,W) per K block
  int kcol[2] = {0, 0};
  bool center_only = false;    // 1x1 conv (logits only)
};
}  // namespace fv

struct fv_net {
  std::vector<std::pair<char, int>> blocks;
  int n_enc = 0, n_dec = 0;
  int in_channels = 8;
  int predicted_kernel = 3;
  bool recurrent = true;
  bool include_mask = true;
  std::vector<fv::ConvParam> convs;  // D.block{i}.conv{1,2} (2 per block), D.head, K.block{i}
  int head_index = -1;
  int k_index0 = -1;  // first K conv
  // K stage as tcgen05 convs, one per level: D.head (level 0) + the logits of the K blocks there
  std::vector<fv::ConvParam> kconv;
  // fused K stage (FV_KFUSE, default on): D.head alone as the level-0 conv, and per level L the K
  // blocks' 1x1 logits as a [cin/8][32][8] image for the decoder conv2 epilogue (conv_tc.cu LG)
  fv::ConvParam khead;
  std::vector<fv::ConvParam> klog;
  bool kstage_dirty = true;
  uint64_t version = 1;  // bumped by every parameter change (captured frame graphs key on it)
};

// Activation tensor in "NC8HW8" layout: C/8 planes of (H, W, 8) fp16.
struct fv_act {
  __half* p = nullptr;
  int C = 0, H = 0, W = 0;
  int64_t plane() const { return (int64_t)H * W * 8; }
};

// The network input x (NC8HW8, two channel groups): group 0 = [r*m, g*m, b*m, a*m, m, 0, 0, 0]
// (written whole by the mask, the march's records fill channels 0..3 of active pixels), group 1 =
// [O_d feedback (3), 0 x 5] (written whole by the K-stage level-0 conv of the previous frame).
// Separate groups keep every writer's stores full 16-byte pixels with no shared bytes, so the
// next frame's mask and this frame's D.head can run concurrently on one buffer.
// FV_MARCH_CARVEOUT (A/B knob): preferred shared-memory carveout (percent) of the render branch's
// kernels, set once per kernel; FV_MARCH_OCC (percent): the persistent march passes' blocks per SM
template <typename K>
inline void render_carveout(K kernel) {
  static const int pc = getenv("FV_MARCH_CARVEOUT") ? atoi(getenv("FV_MARCH_CARVEOUT")) : -1;
  if (pc >= 0) cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, pc);
}
inline int render_occ(int per_sm) {
  static const int occ = getenv("FV_MARCH_OCC") ? atoi(getenv("FV_MARCH_OCC")) : 100;
  return per_sm * occ / 100 > 1 ? per_sm * occ / 100 : 1;
}
constexpr int kInGroups = 2;
inline __half* feedback_plane(const fv_act& x) { return x.p + x.plane(); }

struct fv_state {
  const fv_net* net = nullptr;
  int H = 0, W = 0, Hp = 0, Wp = 0;
  int parity = 0;  // which hidden buffer holds the carried state
  bool fresh = true;
  fv_act x;                         // 8-ch input the next reconstruct reads (render writes it)
  fv_act xalt;                      // the other input buffer: receives O_d feedback, then swaps
  std::vector<fv_act> enc_a;        // conv1 outputs per encoder block
  std::vector<fv_act> skips;        // conv2 outputs (skip) per encoder block
  std::vector<fv_act> pooled;       // pooled skip per encoder block
  std::vector<fv_act> dec_a;        // conv1 outputs per decoder block
  std::vector<fv_act> ups;          // upsampled previous decoder output (j>0)
  std::vector<fv_act> hidden[2];    // ping-pong Hd per decoder block
  fv_act zero8;                     // unused
  float* od = nullptr;              // (3,Hp,Wp) fp32 O_d (padded): the current frame's, od_buf[parity]
  float* od_buf[2] = {nullptr, nullptr};  // per hidden parity, so frame t's filter chain can run next
                                          // to frame t+1's network (fv_frames)
  std::vector<float*> img;          // K-stage ping buffers per level (3,HL,WL) fp32
  std::vector<float*> img2;
  std::vector<fv::kw_t*> kw;        // per K block: softmax filter weights (9,HL,WL): kw_buf[parity]
  std::vector<fv::kw_t*> kw_buf[2];
  void* arena = nullptr;
  int64_t arena_bytes = 0;
  // reconstruct() as captured CUDA graphs, one per launch configuration (the two input / hidden
  // buffer parities, output pointers, network version); captured on the configuration's second use
  struct Graph {
    const fv_net* net = nullptr;
    uint64_t version = 0;
    const void* x = nullptr;
    int parity = 0, use_k = 0;
    const float *rgb = nullptr, *o = nullptr, *od = nullptr;
    int uses = 0;
    unsigned long long n_launches = 0;  // kernels in the graph (ctx->launches accounting)
    cudaGraphExec_t exec = nullptr;
  };
  std::vector<Graph> graphs;
  cudaStream_t capture_stream = nullptr;
  int capture_prio = 0;
  // fv_frames: one whole frame (march of frame t, then its network next to the mask of frame t+1)
  // as a captured CUDA graph per launch configuration; the per-frame camera / fovea / noise frame
  // come from the context's FrameDyn block
  struct FrameGraph {
    const void* vol = nullptr;
    const fv_net* net = nullptr;
    uint64_t version = 0, wave_version = 0;
    const void* x = nullptr;
    int parity = 0, ahead = 0;
    const float* img = nullptr;
    const float* prev_img = nullptr;  // the previous frame's filter chain folded in (FV_KCHAIN_SPLIT=2)
    fv_light light{};
    int has_light = 0;
    fv_settings settings{};
    int uses = 0;
    unsigned long long n_launches = 0;
    cudaGraphExec_t exec = nullptr;
  };
  std::vector<FrameGraph> fgraphs;
  // fv_frames: the K filter chain + output stage of a frame into image `img`, per image buffer
  struct ChainGraph {
    const fv_net* net = nullptr;
    uint64_t version = 0;
    const float* img = nullptr;
    const float* od = nullptr;  // the parity's O_d / weight planes the chain reads
    int uses = 0;
    unsigned long long n_launches = 0;
    cudaGraphExec_t exec = nullptr;
  };
  std::vector<ChainGraph> cgraphs;
  cudaStream_t fcap[3] = {nullptr, nullptr, nullptr};
  cudaEvent_t fcap_ev[4] = {nullptr, nullptr, nullptr, nullptr};
};

namespace fv {
// The host-side state change of one reconstruction (after its launches, whether eager, captured or a
// replayed graph): the input buffers swap, the hidden parity flips, and the O_d / K weight-plane
// views follow the parity the frame wrote.
inline void state_views(fv_state* st) {
  st->od = st->od_buf[st->parity];
  st->kw = st->kw_buf[st->parity];
}
inline void state_advance(fv_state* st) {
  std::swap(st->x, st->xalt);
  st->parity ^= 1;
  st->fresh = false;
  state_views(st);
}
int prepare_net(fv_ctx* ctx, const fv_net* net);
int reconstruct_launches(fv_ctx* ctx, fv_net* net, fv_state* st, int use_k, float* out_rgb, float* out_o,
                         float* out_od);
int kfilter_launches(fv_ctx* ctx, fv_net* net, fv_state* st, int use_k, const float* od, float* out_rgb,
                     float* out_o, float* out_od, const std::vector<kw_t*>* kw = nullptr);
// launchers (return 0 / negative)
int launch_mask_compact(fv_ctx* ctx, int frame, int H, int W, const fv_fovea* f,
                        const double* pb_map, uint8_t* bits, int32_t* idx, int32_t* k,
                        __half* net_in, int net_wp, const double* tau_map = nullptr);
int launch_direct_draws(fv_ctx* ctx, int H, int W, const fv_fovea* f, const double* pb_map, const double* tau_map,
                        const double* r, int64_t count, int32_t* idx);
int launch_tau_sum(fv_ctx* ctx, int H, int W, const fv_fovea* f, const double* pb_map, const double* tau_map,
                   double* sum_dev);
int launch_foveal_density(fv_ctx* ctx, const double* ox, const double* oy, int64_t n, double sigma, double scale,
                          double* out);
int launch_tau_map(fv_ctx* ctx, int H, int W, const fv_fovea* f, const double* pb_map,
                   double* tau);
int launch_render(fv_ctx* ctx, const fv_volume* vol, const fv_camera* cam, const fv_light* light,
                  const fv_settings* settings, const int32_t* idx, const int32_t* k, int k_max,
                  float* rgba, float* depth, __half* net_in, int net_wp, int force_variant = -1);
// naive renderer's lane list: every pixel of each occupied kChunkNaive-pixel chunk, idle lanes as
// -(pix+1); returns the entry count in *k_dev
constexpr int kChunkNaive = 64;  // WARP_CHUNK (renderer.py:34)
int launch_naive_list(fv_ctx* ctx, const uint8_t* bits, int H, int W, int32_t* idx, int32_t* k_dev);
int launch_volume_procedural(fv_ctx* ctx, fv_volume* vol, int kind, double* range);
int launch_volume_from_raw(fv_ctx* ctx, fv_volume* vol, const void* raw, int dtype, double* range_out,
                           int64_t* first_nan_out);
int reconstruct(fv_ctx* ctx, const fv_net* net, fv_state* st, int use_k, float* out_rgb,
                float* out_o, float* out_od);
int conv_prepare(fv_ctx* ctx, ConvParam& cp);
int logits_prepare(fv_ctx* ctx, ConvParam& cp);
bool logits_fusable(const ConvParam& cp);
}  // namespace fv
