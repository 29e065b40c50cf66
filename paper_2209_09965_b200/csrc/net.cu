// W-Net reconstruction: parameter store, recurrent state and the per-frame forward.
//
// Reference (pkg/src/fovray/network.py):
//   NetConfig / _conv_channels / _block_levels   :37-91, :128-159
//   init_network / load_network (param names)     :162-180, :342-357
//   reset_state / RecurrentState                  :103-119
//   forward_D (encoder, decoder, head)            :203-254
//   forward_K (per-scale predicted kernels)       :280-293
//   forward_full (pad to /divisor, crop)          :296-323
// The recurrent hidden states are ping-ponged between two device buffers, so carrying the state
// into the next frame costs no copy; O_d is written by the head conv straight into channels 5..7
// of the next frame's input tensor.
#include <cmath>
#include <cstring>
#include <string>
#include <utility>

#include "internal.h"

namespace fv {
int conv3x3(fv_ctx* ctx, const ConvParam& cp, const fv_act* srcs, int n_src, fv_act* dst,
            fv_act* pool_dst, bool relu, const ConvAux* aux);
int upsample2_nc8(fv_ctx* ctx, const fv_act& in, fv_act& out);
int kapply(fv_ctx* ctx, const kw_t* kw, const float* img, float* out, int h, int w);
int pool3(fv_ctx* ctx, const float* in, float* out, int h_out, int w_out);
int up3(fv_ctx* ctx, const float* in, float* out, int h_in, int w_in);
int finalize(fv_ctx* ctx, fv_state* st, const float* img, float* rgb, float* o_raw, float* od_raw);
int kapply_pool(fv_ctx* ctx, const kw_t* kw, const float* img, float* out, int h, int w);
int kchain(fv_ctx* ctx, const KChain& ch);
bool kchain_enabled();
int kapply_final(fv_ctx* ctx, fv_state* st, const kw_t* kw, const float* img, float* rgb, float* o_raw,
                 float* od_raw);
int nc8_to_nchw(fv_ctx* ctx, const fv_act& a, float* out);
int nchw_to_nc8(fv_ctx* ctx, const float* in, fv_act& a);
int od_to_feedback(fv_ctx* ctx, fv_state* st);
int kfield_logits(fv_ctx* ctx, const float* w_host, const float* b_host, const float* hd, int C, int h, int w,
                  int normalize, float* out);
int set_input(fv_ctx* ctx, fv_state* st, const float* xin, int C);

namespace {

float truncate_fp16(float v) {
  // autograd.truncate_fp16 (autograd.py:499-503): clip to +-65504, round through binary16
  if (v > 65504.f) v = 65504.f;
  if (v < -65504.f) v = -65504.f;
  return __half2float(__float2half_rn(v));
}

int parse_blocks(const char* s, std::vector<std::pair<char, int>>& out) {
  out.clear();
  std::string str(s ? s : "");
  size_t pos = 0;
  while (pos <= str.size()) {
    size_t e = str.find('-', pos);
    if (e == std::string::npos) e = str.size();
    std::string tok = str.substr(pos, e - pos);
    if (tok.size() < 2 || (tok[0] != 'e' && tok[0] != 'd')) {
      set_error("bad block token '%s'", tok.c_str());
      return FV_E_INVALID;
    }
    char* endp = nullptr;
    long ch = strtol(tok.c_str() + 1, &endp, 10);
    if (*endp != 0 || ch <= 0) {
      set_error("bad block token '%s'", tok.c_str());
      return FV_E_INVALID;
    }
    out.push_back({tok[0], (int)ch});
    pos = e + 1;
  }
  return 0;
}

std::vector<int> block_levels(const fv_net* net) {
  std::vector<int> lv;
  for (int i = 0; i < net->n_enc; ++i) lv.push_back(i);
  for (int j = 0; j < net->n_dec; ++j) lv.push_back(net->n_enc - j);
  return lv;
}

int64_t align_up(int64_t v, int64_t a) { return (v + a - 1) / a * a; }

}  // namespace

// Build the level convs of the K stage from D.head + K.block{i} parameters: conv L reads the
// decoder hidden state at level L; columns 0..2 = D.head (level 0 only, all 9 taps), columns
// kLogitCol[s].. = the 9 logits of the s-th K block at that level (1x1 = centre tap).
static void free_conv_dev(ConvParam& cp) {
  if (cp.w_dev) cudaFree(cp.w_dev);
  if (cp.b_dev) cudaFree(cp.b_dev);
  cp.w_dev = nullptr;
  cp.b_dev = nullptr;
}

int build_kstage(fv_ctx* ctx, fv_net* net) {
  const int ne = net->n_enc;
  for (auto& cp : net->kconv) free_conv_dev(cp);
  for (auto& cp : net->klog) free_conv_dev(cp);
  free_conv_dev(net->khead);
  const std::vector<int> lv = block_levels(net);
  const ConvParam& head = net->convs[net->head_index];
  net->kconv.assign(ne + 1, ConvParam());
  for (int L = 0; L <= ne; ++L) {
    ConvParam& cp = net->kconv[L];
    const int cin = net->blocks[ne + (ne - L)].second;  // decoder block at level L
    cp.name = "K.level" + std::to_string(L);
    cp.cin = cin;
    cp.cout = 32;
    cp.n_pad = 32;
    cp.w_host.assign((size_t)32 * cin * 9, 0.f);
    cp.b_host.assign(32, 0.f);
    if (L == 0) {
      for (size_t i = 0; i < (size_t)3 * cin * 9; ++i) cp.w_host[i] = head.w_host[i];
      for (int o = 0; o < 3; ++o) cp.b_host[o] = head.b_host[o];
    }
    int s = 0;
    for (size_t i = 0; i < lv.size(); ++i) {
      if (lv[i] != L || s >= 2) continue;
      const ConvParam& kp = net->convs[net->k_index0 + i];  // (9, cin, 1, 1)
      for (int j = 0; j < 9; ++j) {
        for (int c = 0; c < cin; ++c)
          cp.w_host[((size_t)(kLogitCol[s] + j) * cin + c) * 9 + 4] = kp.w_host[(size_t)j * cin + c];
        cp.b_host[kLogitCol[s] + j] = kp.b_host[j];
      }
      ++s;
    }
    cp.w_set = cp.b_set = true;
    cp.center_only = L > 0;
    cp.head_conv = true;
    // FV_K0_TAPN=1: level 0 with D.head's nine taps in N next to the logits (conv_tc.cu, TAPN).
    // Measured at C3 (per-launch CUDA events, 8 frames): 124.3 us against 100.7 us for the default
    // row-fused 32-column conv -- the MMA work drops ~4x but the launch is bound by its epilogue
    // (three TMEM rows read per output row, 21 scattered stores per pixel) and the single-buffered
    // 288-column accumulator; kept opt-in as the measured alternative.
    static const bool tapn = getenv("FV_K0_TAPN") && atoi(getenv("FV_K0_TAPN")) == 1;
    cp.tapn = L == 0 && tapn && cin <= 64;
    if (cp.tapn) {
      cp.n_pad = 48;
      cp.b_host.resize(48, 0.f);
    }
    cp.macs_per_px = (L == 0 ? 27.0 * cin : 0.0) + 9.0 * cin * s;  // D.head 3x3 + s 1x1 logit convs
    const int rc = conv_prepare(ctx, cp);
    if (rc) return rc;
  }
  // the fused K stage: D.head alone (3 of 16 columns) and the per-level logits images
  {
    ConvParam& cp = net->khead;
    cp = ConvParam();
    cp.name = "K.head";
    cp.cin = head.cin;
    cp.cout = 3;
    // FV_KHEAD_TAPN=1: the nine taps of D.head in N (27 of 32 columns, one MMA per halo row and
    // K-stage; conv_tc.cu TAPN). Measured at C3 on the frame timeline: 108.5 us against 85.3 us for
    // the row-fused 16-column form (bound by its 18 A-operand reads per stage, ncu tensor pipe 69%;
    // TAPN trades them for its three-row, cross-lane epilogue), so opt-in.
    static const bool tapn = getenv("FV_KHEAD_TAPN") && atoi(getenv("FV_KHEAD_TAPN")) == 1;
    cp.tapn = tapn && cp.cin <= 64;
    cp.n_pad = cp.tapn ? 32 : 16;
    cp.w_host = head.w_host;
    cp.b_host = head.b_host;
    cp.w_set = cp.b_set = true;
    cp.head_conv = true;
    cp.macs_per_px = 27.0 * cp.cin;
    const int rc = conv_prepare(ctx, cp);
    if (rc) return rc;
  }
  net->klog.assign(ne + 1, ConvParam());
  for (int L = 0; L <= ne; ++L) {
    ConvParam& cp = net->klog[L];
    const int cin = net->blocks[ne + (ne - L)].second;
    cp.name = "K.logits" + std::to_string(L);
    cp.cin = cin;
    cp.ksize = 1;
    int s = 0;
    for (size_t i = 0; i < lv.size(); ++i) {
      if (lv[i] != L || s >= 2) continue;
      const ConvParam& kp = net->convs[net->k_index0 + i];  // (9, cin, 1, 1)
      for (int j = 0; j < 9; ++j) {
        for (int c = 0; c < cin; ++c) cp.w_host.push_back(kp.w_host[(size_t)j * cin + c]);
        cp.b_host.push_back(kp.b_host[j]);
      }
      ++s;
    }
    cp.cout = 9 * s;
    cp.w_set = cp.b_set = true;
    if (s == 0) continue;
    const int rc = logits_prepare(ctx, cp);
    if (rc) return rc;
  }
  net->kstage_dirty = false;
  return 0;
}

// FV_KFUSE (default 1): the K stage's logits in the decoder conv2 epilogues, when every decoder
// conv2 has a fused variant (conv_tc.cu LG); 0 = the separate level convs (A/B, and forward_K)
static bool kfuse(const fv_net* net) {
  static const bool off = getenv("FV_KFUSE") && atoi(getenv("FV_KFUSE")) == 0;
  if (off) return false;
  const std::vector<int> lv = block_levels(net);
  for (int j = 0; j < net->n_dec; ++j) {
    const int L = net->n_enc - j;
    if (net->klog.size() <= (size_t)L || !net->klog[L].w_dev) return false;
    if (!logits_fusable(net->convs[2 * (net->n_enc + j) + 1])) return false;
  }
  return true;
}

// The K stage (network.py:268-293) plus D.head over the decoder hidden states hidden[hp]: the
// level-0 conv writes D.head's O_d to od_out (and the next frame's feedback channels when feedback
// is set), the filter chain starts from od_in (forward_K's given O_d) or, when null, from od_out.
static int kstage_launches(fv_ctx* ctx, fv_net* net, fv_state* st, int hp, float* od_out, __half* feedback,
                           int use_k, const float* od_in, float* out_rgb, float* out_o, float* out_od,
                           bool fused = false) {
  const int ne = net->n_enc;
  int rc;
  // Level 0: one tcgen05 conv over Hd3 computes D.head (3x3, columns 0..2) AND the logits of
  // the two K blocks at level 0 (1x1, centre tap only, columns 4.. and 13..); its epilogue writes
  // O_d, the NEXT frame's feedback channels 5..7 (the two input buffers alternate, so the next
  // frame's mask + march may already write channels 0..4 of it on another stream) and the
  // softmax-normalised 3x3 filter weights of both K blocks. Levels > 0: a 1x1 logits conv each.
  const std::vector<int> lv = block_levels(net);
  const int nb = (int)lv.size();
  if (fused) {
    // the logits came with the decoder conv2s (conv_tc.cu LG): only D.head here
    ConvAux aux;
    aux.od = od_out;
    aux.feedback = feedback;
    rc = conv3x3(ctx, net->khead, &st->hidden[hp][ne], 1, nullptr, nullptr, false, &aux);
    if (rc) return rc;
  }
  for (int L = 0; L <= ne && !fused; ++L) {
    if (L > 0 && !use_k) break;
    ConvAux aux;
    if (L == 0) {
      aux.od = od_out;
      aux.feedback = feedback;
    } else {
      aux.center_only = true;
    }
    int s = 0;
    for (int i = 0; i < nb; ++i)
      if (lv[i] == L && s < 2) {
        aux.kw[s] = st->kw[i];
        aux.kcol[s] = kLogitCol[s];
        ++s;
      }
    rc = conv3x3(ctx, net->kconv[L], &st->hidden[hp][ne - L], 1, nullptr, nullptr, false, &aux);
    if (rc) return rc;
  }
  if (ctx->kchain_split && !od_in) return 0;  // the filter chain follows as its own graph (fv_frames)
  return kfilter_launches(ctx, net, st, use_k, od_in ? od_in : od_out, out_rgb, out_o, out_od);
}

// The K stage's filter chain (forward_K, network.py:280-293) from O_d `od` and the weight planes
// st->kw, then the output stage; use_k = 0: the output stage on O_d alone (forward_D's ablation).
int kfilter_launches(fv_ctx* ctx, fv_net* net, fv_state* st, int use_k, const float* od, float* out_rgb,
                     float* out_o, float* out_od, const std::vector<kw_t*>* kwv) {
  int rc;
  const std::vector<kw_t*>& kwp = kwv ? *kwv : st->kw;
  const std::vector<int> lv = block_levels(net);
  const int nb = (int)lv.size();
  if (use_k) {
    // forward_K (network.py:280-293): encoder levels fuse the filter with the following pool, the
    // last block (level 0) with the output stage
    const float* img = od;
    // blocks 1 .. nb-2 (the small levels) as one cooperative launch when every encoder level there
    // has even width (the paired-pixel filter + pool)
    KChain ch;
    bool chain = kchain_enabled() && nb >= 3 && nb - 2 <= 8 && net->blocks[0].first == 'e';
    for (int i = 1; chain && i < nb - 1; ++i)
      if (net->blocks[i].first == 'e' && (((st->Wp >> lv[i]) & 1) || ((st->Hp >> lv[i]) & 1))) chain = false;
    for (int i = 0; i < nb; ++i) {
      const int L = lv[i];
      if (chain && i >= 1 && i < nb - 1) {
        const int h = st->Hp >> L, w = st->Wp >> L;
        if (net->blocks[i].first == 'e') {
          ch.s[ch.n++] = {0, h, w, kwp[i], img, st->img[L + 1]};
          img = st->img[L + 1];
        } else {
          ch.s[ch.n++] = {1, h, w, kwp[i], img, st->img2[L]};
          ch.s[ch.n++] = {2, h, w, nullptr, st->img2[L], st->img[L - 1]};
          img = st->img[L - 1];
        }
        if (i == nb - 2) {
          rc = kchain(ctx, ch);
          if (rc) return rc;
        }
        continue;
      }
      if (net->blocks[i].first == 'e') {
        rc = kapply_pool(ctx, kwp[i], img, st->img[L + 1], st->Hp >> L, st->Wp >> L);
        if (rc) return rc;
        img = st->img[L + 1];
      } else if (i < nb - 1) {
        float* out = st->img2[L];
        rc = kapply(ctx, kwp[i], img, out, st->Hp >> L, st->Wp >> L);
        if (rc) return rc;
        rc = up3(ctx, out, st->img[L - 1], st->Hp >> L, st->Wp >> L);
        if (rc) return rc;
        img = st->img[L - 1];
      } else if (L == 0) {
        rc = kapply_final(ctx, st, kwp[i], img, out_rgb, out_o, out_od);
        if (rc) return rc;
        img = nullptr;
      } else {
        set_error("the last K block must be at level 0 (got level %d)", L);
        return FV_E_INVALID;
      }
    }
  } else {
    rc = finalize(ctx, st, od, out_rgb, out_o, out_od);
    if (rc) return rc;
  }
  return 0;
}


// The launches of one reconstruction (no host-side state change: see reconstruct()).
int reconstruct_launches(fv_ctx* ctx, fv_net* net, fv_state* st, int use_k, float* out_rgb,
                                float* out_o, float* out_od) {
  const int ne = net->n_enc, nd = net->n_dec;
  int rc;
  const fv_act* cur = &st->x;
  for (int i = 0; i < ne; ++i) {
    rc = conv3x3(ctx, net->convs[2 * i], cur, 1, &st->enc_a[i], nullptr, true, nullptr);
    if (rc) return rc;
    rc = conv3x3(ctx, net->convs[2 * i + 1], &st->enc_a[i], 1, &st->skips[i], &st->pooled[i], true,
                 nullptr);
    if (rc) return rc;
    cur = &st->pooled[i];
  }
  const int oldp = st->parity, newp = st->parity ^ 1;
  // this frame's O_d and K weight planes (the previous frame's stay intact for its filter chain)
  st->od = st->od_buf[newp];
  st->kw = st->kw_buf[newp];
  const bool fused = use_k && kfuse(net);
  const std::vector<int> lv = block_levels(net);
  for (int j = 0; j < nd; ++j) {
    fv_act srcs[3];
    int n = 0;
    if (j > 0) {
      rc = upsample2_nc8(ctx, st->hidden[newp][j - 1], st->ups[j]);
      if (rc) return rc;
      srcs[n++] = st->ups[j];
      srcs[n++] = st->skips[ne - j];
    } else {
      srcs[n++] = *cur;
    }
    if (net->recurrent) srcs[n++] = st->hidden[oldp][j];
    const int b = ne + j;
    rc = conv3x3(ctx, net->convs[2 * b], srcs, n, &st->dec_a[j], nullptr, true, nullptr);
    if (rc) return rc;
    if (j == 0 && ctx->kw_wait_ev) {
      // fv_frames with the filter chain split off: the previous frame's chain (another stream)
      // still reads the weight planes and O_d this conv2 and the K stage are about to rewrite
      cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
      FV_CUDA(cudaStreamIsCapturing(ctx->stream, &cs));
      FV_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->kw_wait_ev,
                                  cs == cudaStreamCaptureStatusActive && ctx->kw_wait_external
                                      ? cudaEventWaitExternal : 0));
    }
    ConvAux laux;
    if (fused) {
      const int L = ne - j;
      laux.logits = &net->klog[L];
      int s = 0;
      for (size_t i = 0; i < lv.size(); ++i)
        if (lv[i] == L && s < 2) laux.kw[s++] = st->kw[i];
    }
    rc = conv3x3(ctx, net->convs[2 * b + 1], &st->dec_a[j], 1, &st->hidden[newp][j], nullptr, true,
                 fused ? &laux : nullptr);
    if (rc) return rc;
  }
  return kstage_launches(ctx, net, st, newp, st->od, net->recurrent ? feedback_plane(st->xalt) : nullptr, use_k, nullptr,
                         out_rgb, out_o, out_od, fused);
}

static bool graphs_enabled(const fv_ctx* ctx) {
  static const bool off = (getenv("FV_GRAPH") && atoi(getenv("FV_GRAPH")) == 0) || getenv("FV_CONV_PROF");
  return !off && !ctx->ktiming;
}

// Parameters complete and the fused K-stage convs built (before any launch or capture).
int prepare_net(fv_ctx* ctx, const fv_net* cnet) {
  fv_net* net = const_cast<fv_net*>(cnet);  // the fused K-stage convs are a cache of the params
  for (const auto& cp : net->convs)
    if (!(cp.w_set && cp.b_set)) {
      set_error("network parameter %s not set", cp.name.c_str());
      return FV_E_INVALID;
    }
  if (net->kstage_dirty) return build_kstage(ctx, net);
  return 0;
}

// One frame of the W-Net. A configuration's first run is eager (it sets kernel attributes and
// allocates lazily); from its second run on the ~31 launches are replayed as one CUDA graph.
int reconstruct(fv_ctx* ctx, const fv_net* cnet, fv_state* st, int use_k, float* out_rgb,
                float* out_o, float* out_od) {
  fv_net* net = const_cast<fv_net*>(cnet);
  {
    const int rc0 = prepare_net(ctx, net);
    if (rc0) return rc0;
  }
  int rc = 0;
  fv_state::Graph* g = nullptr;
  if (graphs_enabled(ctx)) {
    for (auto& e : st->graphs)
      if (e.net == net && e.version == net->version && e.x == st->x.p && e.parity == st->parity &&
          e.use_k == use_k && e.rgb == out_rgb && e.o == out_o && e.od == out_od) {
        g = &e;
        break;
      }
    if (!g) {
      if (st->graphs.size() >= 8) {  // configurations changed (new outputs / weights): start over
        for (auto& e : st->graphs)
          if (e.exec) cudaGraphExecDestroy(e.exec);
        st->graphs.clear();
      }
      fv_state::Graph e;
      e.net = net; e.version = net->version; e.x = st->x.p; e.parity = st->parity; e.use_k = use_k;
      e.rgb = out_rgb; e.o = out_o; e.od = out_od;
      st->graphs.push_back(e);
      g = &st->graphs.back();
    }
  }
  if (g && g->uses >= 1 && !g->exec) {
    // record on a private stream (the context's may be the legacy default stream, which cannot
    // capture); the graph is then launched on the context's stream
    // (with the context stream's priority: captured kernel nodes keep the capturing stream's
    // priority, and the network's high priority is what lets it win SMs over the marcher)
    int prio = 0;
    if (ctx->stream) FV_CUDA(cudaStreamGetPriority(ctx->stream, &prio));
    if (st->capture_stream && st->capture_prio != prio) {
      cudaStreamDestroy(st->capture_stream);
      st->capture_stream = nullptr;
    }
    if (!st->capture_stream) {
      FV_CUDA(cudaStreamCreateWithPriority(&st->capture_stream, cudaStreamNonBlocking, prio));
      st->capture_prio = prio;
    }
    cudaGraph_t graph = nullptr;
    const cudaStream_t own = ctx->stream;
    ctx->stream = st->capture_stream;
    cudaError_t e0 = cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal);
    if (e0 != cudaSuccess) { ctx->stream = own; return cuda_fail(e0, "cudaStreamBeginCapture (reconstruct)"); }
    rc = reconstruct_launches(ctx, net, st, use_k, out_rgb, out_o, out_od);
    const cudaError_t e1 = cudaStreamEndCapture(ctx->stream, &graph);
    ctx->stream = own;
    if (rc) { if (graph) cudaGraphDestroy(graph); return rc; }
    if (e1 != cudaSuccess) return cuda_fail(e1, "cudaStreamEndCapture (reconstruct)");
    const cudaError_t e2 = cudaGraphInstantiate(&g->exec, graph, 0);
    cudaGraphDestroy(graph);
    if (e2 != cudaSuccess) { g->exec = nullptr; return cuda_fail(e2, "cudaGraphInstantiate (reconstruct)"); }
  }
  if (g && g->exec) {
    FV_CUDA(cudaGraphLaunch(g->exec, ctx->stream));
    ctx->launches += g->n_launches;
  } else {
    const unsigned long long before = ctx->launches;
    rc = reconstruct_launches(ctx, net, st, use_k, out_rgb, out_o, out_od);
    if (rc) return rc;
    if (g) g->n_launches = ctx->launches - before;
  }
  if (g) ++g->uses;
  state_advance(st);
  return 0;
}

}  // namespace fv

using namespace fv;

extern "C" {

int fv_net_create(fv_ctx* ctx, const char* blocks, int predicted_kernel, int recurrent,
                  int include_mask_channel, fv_net** out) {
  FV_REQUIRE(ctx && out, "null argument");
  auto* net = new fv_net();
  int rc = parse_blocks(blocks, net->blocks);
  if (rc) { delete net; return rc; }
  int ne = 0, nd = 0;
  bool seen_d = false;
  for (auto& b : net->blocks) {
    if (b.first == 'e') {
      if (seen_d) { delete net; set_error("block config must list e-blocks then d-blocks"); return FV_E_INVALID; }
      ++ne;
    } else { seen_d = true; ++nd; }
  }
  if (ne != nd - 1) {
    delete net;
    set_error("structural encoder count (e-blocks + bottleneck = %d) must be one more than decoder count (%d); got %d e and %d d blocks",
              ne + 1, nd - 1, ne, nd);
    return FV_E_INVALID;
  }
  if (predicted_kernel != 3) { delete net; set_error("only predicted_kernel = 3 is supported"); return FV_E_UNSUPPORTED; }
  net->n_enc = ne;
  net->n_dec = nd;
  net->predicted_kernel = predicted_kernel;
  net->recurrent = recurrent != 0;
  net->include_mask = include_mask_channel != 0;
  net->in_channels = 4 + (net->include_mask ? 1 : 0) + (net->recurrent ? 3 : 0);
  std::vector<int> ch;
  for (auto& b : net->blocks) ch.push_back(b.second);
  for (int c : ch)
    if (c % 8 != 0) { delete net; set_error("block widths must be multiples of 8 (got %d)", c); return FV_E_UNSUPPORTED; }
  std::vector<int> d_ch(ch.begin() + ne, ch.end());
  // _conv_channels (network.py:128-149)
  std::vector<std::pair<int, int>> io;
  // block0 input: 16 slots in two channel groups [rgba, m, 0 x 3 | prev(3), 0 x 5] (internal.h)
  for (int i = 0; i < ne; ++i) io.push_back({i == 0 ? 8 * kInGroups : ch[i - 1], ch[i]});
  for (int j = 0; j < nd; ++j) {
    int inc = j == 0 ? ch[ne - 1] : d_ch[j - 1] + ch[ne - j];
    if (net->recurrent) inc += d_ch[j];
    io.push_back({inc, d_ch[j]});
  }
  for (size_t i = 0; i < io.size(); ++i) {
    for (int c = 1; c <= 2; ++c) {
      ConvParam cp;
      cp.name = "D.block" + std::to_string(i) + ".conv" + std::to_string(c);
      cp.cin = c == 1 ? io[i].first : io[i].second;
      cp.cout = io[i].second;
      cp.n_pad = (cp.cout + 15) / 16 * 16;
      // algorithmic MACs of block0.conv1: the reference's in_channels, not the padded slots
      if (i == 0 && c == 1) cp.macs_per_px = (double)net->in_channels * cp.cout * 9;
      net->convs.push_back(cp);
    }
  }
  {
    ConvParam cp;
    cp.name = "D.head";
    cp.cin = d_ch.back();
    cp.cout = 3;
    cp.n_pad = 16;
    net->head_index = (int)net->convs.size();
    net->convs.push_back(cp);
  }
  net->k_index0 = (int)net->convs.size();
  const std::vector<int> lv = block_levels(net);
  for (size_t i = 0; i < lv.size(); ++i) {
    ConvParam cp;
    cp.name = "K.block" + std::to_string(i);
    cp.cin = d_ch[ne - lv[i]];
    cp.cout = 9;
    cp.ksize = 1;
    net->convs.push_back(cp);
  }
  *out = net;
  return 0;
}

int fv_net_destroy(fv_net* net) {
  if (!net) return 0;
  for (auto* v : {&net->convs, &net->kconv, &net->klog})
    for (auto& cp : *v) free_conv_dev(cp);
  free_conv_dev(net->khead);
  delete net;
  return 0;
}

int fv_net_set_param(fv_ctx* ctx, fv_net* net, const char* name, const float* host, int64_t count) {
  FV_REQUIRE(ctx && net && name && host, "null argument");
  std::string n(name);
  const bool is_w = n.size() > 2 && n.compare(n.size() - 2, 2, ".w") == 0;
  const bool is_b = n.size() > 2 && n.compare(n.size() - 2, 2, ".b") == 0;
  FV_REQUIRE(is_w || is_b, "checkpoint parameter '%s' not in network", name);
  const std::string base = n.substr(0, n.size() - 2);
  int idx = -1;
  for (size_t i = 0; i < net->convs.size(); ++i)
    if (net->convs[i].name == base) idx = (int)i;
  FV_REQUIRE(idx >= 0, "checkpoint parameter '%s' not in network", name);
  ConvParam& cp = net->convs[idx];
  const int ks = cp.ksize;
  // reference cin of block0.conv1 is in_channels; device layout uses 16 slots [rgba, m, 0 x 3 | prev, 0 x 5]
  const bool first = base == "D.block0.conv1";
  const int ref_cin = first ? net->in_channels : cp.cin;
  const int64_t expect = is_w ? (int64_t)cp.cout * ref_cin * ks * ks : cp.cout;
  FV_REQUIRE(count == expect, "checkpoint shape mismatch for '%s' (%lld values, expected %lld)", name,
             (long long)count, (long long)expect);
  for (int64_t i = 0; i < count; ++i)
    FV_REQUIRE(std::isfinite(host[i]), "parameter '%s' has a non-finite value", name);
  if (is_w) {
    cp.w_host.assign((size_t)cp.cout * cp.cin * ks * ks, 0.f);
    for (int o = 0; o < cp.cout; ++o)
      for (int c = 0; c < ref_cin; ++c) {
        int slot = c;
        if (first) {
          // reference order: rgba(4), [mask], [prev(3)]
          if (c < 4) slot = c;
          else if (net->include_mask && c == 4) slot = 4;
          else slot = 8 + (c - 4 - (net->include_mask ? 1 : 0));
        }
        for (int t = 0; t < ks * ks; ++t)
          cp.w_host[((size_t)o * cp.cin + slot) * ks * ks + t] =
              truncate_fp16(host[((size_t)o * ref_cin + c) * ks * ks + t]);
      }
    cp.w_set = true;
  } else {
    cp.b_host.assign(host, host + count);
    cp.b_set = true;
  }
  ++net->version;
  if (idx == net->head_index || cp.ksize == 1) net->kstage_dirty = true;  // folded into kconv
  if (!(cp.w_set && cp.b_set) || cp.ksize == 1 || idx == net->head_index) return 0;
  return conv_prepare(ctx, cp);
}

int fv_state_create(fv_ctx* ctx, const fv_net* net, int H, int W, fv_state** out) {
  FV_REQUIRE(ctx && net && out, "null argument");
  FV_REQUIRE(H >= 1 && W >= 1, "dims must be positive, got (%d, %d)", H, W);
  const int div = 1 << net->n_enc;
  auto* st = new fv_state();
  st->net = net;
  st->H = H;
  st->W = W;
  st->Hp = (H + div - 1) / div * div;
  st->Wp = (W + div - 1) / div * div;
  const int ne = net->n_enc, nd = net->n_dec;
  std::vector<int> ch;
  for (auto& b : net->blocks) ch.push_back(b.second);
  std::vector<int> d_ch(ch.begin() + ne, ch.end());
  // plan the arena
  struct Req { fv_act* a; int C, L; };
  std::vector<Req> reqs;
  st->enc_a.resize(ne); st->skips.resize(ne); st->pooled.resize(ne);
  st->dec_a.resize(nd); st->ups.resize(nd); st->hidden[0].resize(nd); st->hidden[1].resize(nd);
  reqs.push_back({&st->x, 8 * kInGroups, 0});
  reqs.push_back({&st->xalt, 8 * kInGroups, 0});
  for (int i = 0; i < ne; ++i) {
    reqs.push_back({&st->enc_a[i], ch[i], i});
    reqs.push_back({&st->skips[i], ch[i], i});
    reqs.push_back({&st->pooled[i], ch[i], i + 1});
  }
  for (int j = 0; j < nd; ++j) {
    const int L = ne - j;
    reqs.push_back({&st->dec_a[j], d_ch[j], L});
    if (j > 0) reqs.push_back({&st->ups[j], d_ch[j - 1], L});
    reqs.push_back({&st->hidden[0][j], d_ch[j], L});
    reqs.push_back({&st->hidden[1][j], d_ch[j], L});
  }
  int64_t bytes = 0;
  std::vector<int64_t> offs;
  for (auto& r : reqs) {
    offs.push_back(bytes);
    const int64_t h = st->Hp >> r.L, w = st->Wp >> r.L;
    bytes += align_up((int64_t)r.C * h * w * 2, 256);
  }
  int64_t od_off[2];
  for (int p = 0; p < 2; ++p) {
    od_off[p] = bytes;
    bytes += align_up((int64_t)3 * st->Hp * st->Wp * 4, 256);
  }
  std::vector<int64_t> img_off, img2_off;
  for (int L = 0; L <= ne; ++L) {
    img_off.push_back(bytes);
    bytes += align_up((int64_t)3 * (st->Hp >> L) * (st->Wp >> L) * 4, 256);
    img2_off.push_back(bytes);
    bytes += align_up((int64_t)3 * (st->Hp >> L) * (st->Wp >> L) * 4, 256);
  }
  const std::vector<int> lv = block_levels(net);
  std::vector<int64_t> kw_off[2];
  for (int p = 0; p < 2; ++p)
    for (int L : lv) {
      kw_off[p].push_back(bytes);
      bytes += align_up((int64_t)9 * (st->Hp >> L) * (st->Wp >> L) * (int64_t)sizeof(kw_t), 256);
    }
  if (cudaMalloc(&st->arena, bytes) != cudaSuccess) {
    delete st;
    set_error("cudaMalloc of %lld bytes for the state failed", (long long)bytes);
    return FV_E_NOMEM;
  }
  st->arena_bytes = bytes;
  uint8_t* base = reinterpret_cast<uint8_t*>(st->arena);
  for (size_t i = 0; i < reqs.size(); ++i) {
    reqs[i].a->p = reinterpret_cast<__half*>(base + offs[i]);
    reqs[i].a->C = reqs[i].C;
    reqs[i].a->H = st->Hp >> reqs[i].L;
    reqs[i].a->W = st->Wp >> reqs[i].L;
  }
  for (int p = 0; p < 2; ++p) st->od_buf[p] = reinterpret_cast<float*>(base + od_off[p]);
  st->od = st->od_buf[st->parity];
  for (int L = 0; L <= ne; ++L) {
    st->img.push_back(reinterpret_cast<float*>(base + img_off[L]));
    st->img2.push_back(reinterpret_cast<float*>(base + img2_off[L]));
  }
  for (int p = 0; p < 2; ++p)
    for (int64_t o : kw_off[p]) st->kw_buf[p].push_back(reinterpret_cast<kw_t*>(base + o));
  st->kw = st->kw_buf[st->parity];
  if (cudaMemsetAsync(st->arena, 0, bytes, ctx->stream) != cudaSuccess) {
    cudaFree(st->arena);
    delete st;
    set_error("cudaMemset of the state failed");
    return FV_E_CUDA;
  }
  *out = st;
  return 0;
}

int fv_state_reset(fv_ctx* ctx, fv_state* st) {
  FV_REQUIRE(ctx && st, "null argument");
  FV_CUDA(cudaMemsetAsync(st->arena, 0, st->arena_bytes, ctx->stream));
  st->parity = 0;
  st->fresh = true;
  state_views(st);
  return 0;
}

int fv_state_destroy(fv_state* st) {
  if (!st) return 0;
  for (auto& e : st->graphs)
    if (e.exec) cudaGraphExecDestroy(e.exec);
  for (auto& e : st->fgraphs)
    if (e.exec) cudaGraphExecDestroy(e.exec);
  for (auto& e : st->cgraphs)
    if (e.exec) cudaGraphExecDestroy(e.exec);
  for (auto& s_ : st->fcap)
    if (s_) cudaStreamDestroy(s_);
  for (auto& e : st->fcap_ev)
    if (e) cudaEventDestroy(e);
  if (st->capture_stream) cudaStreamDestroy(st->capture_stream);
  if (st->arena) cudaFree(st->arena);
  delete st;
  return 0;
}

void* fv_state_net_input(fv_state* st) { return st ? st->x.p : nullptr; }

int fv_state_dims(const fv_state* st, int* H, int* W, int* Hp, int* Wp) {
  FV_REQUIRE(st, "null state");
  if (H) *H = st->H;
  if (W) *W = st->W;
  if (Hp) *Hp = st->Hp;
  if (Wp) *Wp = st->Wp;
  return 0;
}

int fv_reconstruct(fv_ctx* ctx, const fv_net* net, fv_state* st, int use_kernel_stage,
                   float* out_rgb_dev, float* out_o_dev, float* out_od_dev) {
  FV_REQUIRE(ctx && net && st, "null argument");
  if (st->net != net) {
    set_error("carried state belongs to a different network; reset the state");
    return FV_E_STATE;
  }
  return reconstruct(ctx, net, st, use_kernel_stage, out_rgb_dev, out_o_dev, out_od_dev);
}

// forward_K (network.py:280-293) on the decoder hidden states the state currently holds (written
// with fv_state_write, or left by the last fv_reconstruct) and a given O_d (3, Hp, Wp) fp32 on
// the device; writes the filtered image (3, H, W) to out_dev. The state's recurrent buffers and
// its O_d are not modified.
int fv_forward_k(fv_ctx* ctx, const fv_net* cnet, fv_state* st, const float* od_dev, float* out_dev) {
  FV_REQUIRE(ctx && cnet && st && od_dev && out_dev, "null argument");
  FV_REQUIRE(st->net == cnet, "carried state belongs to a different network; reset the state");
  fv_net* net = const_cast<fv_net*>(cnet);
  for (const auto& cp : net->convs)
    FV_REQUIRE(cp.w_set && cp.b_set, "network parameter %s not set", cp.name.c_str());
  if (net->kstage_dirty) {
    const int rc0 = build_kstage(ctx, net);
    if (rc0) return rc0;
  }
  // the level-0 conv's D.head output goes to the level-0 scratch image (unused by the chain)
  return kstage_launches(ctx, net, st, st->parity, st->img2[0], nullptr, 1, od_dev, nullptr, out_dev, nullptr);
}

// predict_kernel_fields (network.py:268-277) for one K block: the 9 logits of the 1x1 conv over
// a decoder hidden state hd (C, h, w) fp32 (device), in fp32; normalize = 1 applies the softmax
// over the taps (KernelField.normalized).
int fv_kfield_logits(fv_ctx* ctx, const fv_net* net, int block, const float* hd_dev, int C, int h, int w,
                     int normalize, float* logits_dev) {
  FV_REQUIRE(ctx && net && hd_dev && logits_dev, "null argument");
  FV_REQUIRE(block >= 0 && block < (int)net->convs.size() - net->k_index0, "K block %d out of range", block);
  const ConvParam& kp = net->convs[net->k_index0 + block];
  FV_REQUIRE(kp.w_set && kp.b_set, "network parameter %s not set", kp.name.c_str());
  FV_REQUIRE(C == kp.cin, "K.block%d expects %d channels, got %d", block, kp.cin, C);
  FV_REQUIRE(h >= 1 && w >= 1, "dims must be positive, got (%d, %d)", h, w);
  return kfield_logits(ctx, kp.w_host.data(), kp.b_host.data(), hd_dev, C, h, w, normalize, logits_dev);
}

int fv_state_read(fv_ctx* ctx, const fv_state* st, int which, float* host, int64_t cap,
                  int64_t* count) {
  FV_REQUIRE(ctx && st, "null argument");
  const fv_net* net = st->net;
  int64_t n;
  float* tmp = nullptr;
  if (which == -1) {
    n = (int64_t)3 * st->Hp * st->Wp;
    if (count) *count = n;
    if (!host) return 0;
    FV_REQUIRE(cap >= n, "buffer too small (%lld < %lld)", (long long)cap, (long long)n);
    FV_CUDA(cudaMemcpyAsync(host, st->od, n * 4, cudaMemcpyDeviceToHost, ctx->stream));
    FV_CUDA(cudaStreamSynchronize(ctx->stream));
    return 0;
  }
  FV_REQUIRE(which >= 0 && which < net->n_dec, "hidden index %d out of range", which);
  const fv_act& a = st->hidden[st->parity][which];
  n = (int64_t)a.C * a.H * a.W;
  if (count) *count = n;
  if (!host) return 0;
  FV_REQUIRE(cap >= n, "buffer too small (%lld < %lld)", (long long)cap, (long long)n);
  FV_CUDA(cudaMallocAsync(&tmp, n * 4, ctx->stream));
  int rc = nc8_to_nchw(ctx, a, tmp);
  if (rc) return rc;
  FV_CUDA(cudaMemcpyAsync(host, tmp, n * 4, cudaMemcpyDeviceToHost, ctx->stream));
  FV_CUDA(cudaFreeAsync(tmp, ctx->stream));
  FV_CUDA(cudaStreamSynchronize(ctx->stream));
  return 0;
}

int fv_state_set_input(fv_ctx* ctx, fv_state* st, const float* x_dev, int channels) {
  FV_REQUIRE(ctx && st && x_dev, "null argument");
  const int expect = 4 + (st->net->include_mask ? 1 : 0);
  FV_REQUIRE(channels == expect, "input has %d channels, expected %d", channels, expect);
  return set_input(ctx, st, x_dev, channels);
}

int fv_state_write(fv_ctx* ctx, fv_state* st, int which, const float* host, int64_t count) {
  FV_REQUIRE(ctx && st && host, "null argument");
  const fv_net* net = st->net;
  float* tmp = nullptr;
  if (which == -1) {
    const int64_t n = (int64_t)3 * st->Hp * st->Wp;
    FV_REQUIRE(count == n, "prev_output must have %lld values (3 x padded film), got %lld", (long long)n,
               (long long)count);
    FV_CUDA(cudaMemcpyAsync(st->od, host, n * 4, cudaMemcpyHostToDevice, ctx->stream));
    int rc = od_to_feedback(ctx, st);
    if (rc) return rc;
    FV_CUDA(cudaStreamSynchronize(ctx->stream));
    st->fresh = false;
    return 0;
  }
  FV_REQUIRE(which >= 0 && which < net->n_dec, "hidden index %d out of range", which);
  fv_act& a = st->hidden[st->parity][which];
  const int64_t n = (int64_t)a.C * a.H * a.W;
  FV_REQUIRE(count == n, "hidden[%d] must have %lld values, got %lld", which, (long long)n, (long long)count);
  FV_CUDA(cudaMallocAsync(&tmp, n * 4, ctx->stream));
  FV_CUDA(cudaMemcpyAsync(tmp, host, n * 4, cudaMemcpyHostToDevice, ctx->stream));
  int rc = nchw_to_nc8(ctx, tmp, a);
  if (rc) return rc;
  FV_CUDA(cudaFreeAsync(tmp, ctx->stream));
  FV_CUDA(cudaStreamSynchronize(ctx->stream));
  st->fresh = false;
  return 0;
}

}  // extern "C"
