// api.cu -- the C-ABI (include/nf.h) and the host runtime behind it: parameter
// arena, activation/derivative stash, host<->device staging, and the launch
// sequences of one SGD step.  Every arithmetic step of the method runs in this
// library's CUDA kernels; there is no CPU fallback (NF_ENODEV without a GPU).
#include <cmath>
#include <cstdlib>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/nf.h"
#include "deep_mk.cuh"
#include "fp64.cuh"
#include "fused_small.cuh"
#include "infer_small.cuh"
#include "infer_tc.cuh"
#include "single_cta.cuh"
#include "kernels.cuh"

using namespace nf;

namespace {

thread_local std::string g_err;

int fail(int code, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define NF_CUDA(expr)                                                                  \
  do {                                                                                 \
    cudaError_t e_ = (expr);                                                           \
    if (e_ != cudaSuccess)                                                             \
      return fail(e_ == cudaErrorMemoryAllocation ? NF_ENOMEM : NF_ECUDA, "%s: %s (%s:%d)", \
                  #expr, cudaGetErrorString(e_), __FILE__, __LINE__);                  \
  } while (0)

struct DevBuf {
  void *p = nullptr;
  size_t cap = 0;
  cudaError_t ensure(size_t bytes) {
    if (bytes <= cap) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e == cudaSuccess) cap = bytes;
    return e;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
  template <class T> T *as() const { return static_cast<T *>(p); }
};

int parse_act(const std::string &s) {
  static const char *names[] = {"sigmoid", "tanh", "relu", "gaussian", "step"};
  for (int i = 0; i < 5; ++i)
    if (s == names[i]) return i;
  return -1;
}

bool is_device_ptr(const void *p) {
  // Small per-thread cache of the last answers (a call passes the same X, Y and step_loss every
  // step; cudaPointerGetAttributes costs ~1 us).  Sound under unified addressing: an address the
  // driver reports as device memory stays in its reserved device VA range, and host addresses never
  // enter it, so a cached answer for an address cannot flip.
  constexpr int kCache = 8;
  static thread_local const void *ck[kCache] = {};
  static thread_local bool cv[kCache] = {};
  static thread_local int cn = 0;
  if (!p) return false;
  for (int i = 0; i < kCache; ++i)
    if (ck[i] == p) return cv[i];
  cudaPointerAttributes at;
  bool dev;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    dev = false;
  } else {
    dev = at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
  }
  // only device answers are cached: a host address can later become registered / mapped memory
  if (dev) {
    ck[cn] = p;
    cv[cn] = dev;
    cn = (cn + 1) % kCache;
  }
  return dev;
}

// splitmix64 + Box-Muller: the documented host stream of nf_net_create.
struct HostRng {
  uint64_t s;
  uint64_t next() {
    uint64_t z = (s += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
  double uniform() { return ((next() >> 11) + 0.5) * (1.0 / 9007199254740992.0); }
  double normal() {
    const double u1 = uniform(), u2 = uniform();
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2);
  }
};

}  // namespace

struct nf_net {
  std::vector<int> dims;
  int L = 0;
  std::vector<int> acts;                 // activation kind of layer l = acts[l], l = 1..L
  std::string act_spec;                  // the spec it was created with (nf_save)
  int act_h = 0, act_o = 0;              // acts[1] and acts[L]
  int math = NF_MATH_FP32;
  cudaStream_t stream = nullptr;
  int64_t nparams = 0;
  float *params = nullptr;               // device, flat layout of nf.h
  // NF_MATH_TF32: the TF32-rounded shadow of the parameters (same layout; only the W blocks are
  // read), the tensor-core operand in place of W.  Kept current by the SGD epilogues of the
  // TF32 step; re-rounded from params when shadow_ok is false (any other writer of params).
  float *params_t = nullptr;
  bool shadow_ok = false;
  // NF_MATH_FP32 with pre-split 3xTF32 (NF_PRESPLIT, default on): tf32_lo of every tensor-core
  // operand, written by its producer -- the weights' lo shadow (kept by the SGD epilogue like
  // params_t), the hidden activations' and deltas' lo arrays (stash_lo), the input rows' (xlo)
  float *params_lo = nullptr;             // (with params_t = tf32_rn(W) as the weights' hi)
  bool lo_ok = false;
  DevBuf stash_lo, xlo;
  std::vector<float *> Ahi, Alo, Dlo;     // index 0: the input rows
  int64_t lo_rows = 0;
  std::vector<int64_t> offW, offB;       // index 1..L
  // stash: A_l (activations) and S_l (sigma'(Z_l), overwritten by delta_l), l = 1..L
  int64_t ws_rows = 0;
  std::vector<float *> A, S;
  DevBuf stash;
  // transposed copies for the weight-gradient contractions that read them K-major:
  // tpose[l] -> DT[l] = delta_l^T [n_l][rows] and (l >= 2) AT[l-1] = A_{l-1}^T [n_{l-1}][rows]
  std::vector<char> tpose;
  std::vector<float *> AT, DT;
  DevBuf tstash;
  int64_t t_rows = 0;
  std::vector<char> t_key;
  bool red_round = false;                // a TF32 step reduced split-K terms into W: re-round shadow
  Workspace ws;
  DevBuf partial;
  // backward: the weight-gradient GEMMs (K4 + bias) of layer l run on a side stream,
  // concurrently with the delta GEMM (K3) of layer l-1 on the main stream
  cudaStream_t side = nullptr;
  std::vector<cudaEvent_t> ev;           // fork, per-layer K3-done, join
  Workspace ws2;                         // the side stream's own split-K / column-sum scratch
  DevBuf partial2;
  DevBuf red;                            // loss/acc partials + results
  DevBuf part_out;                       // partial tendencies of the fused narrow output layer
  bool out_fused = false;                // forward fused K1/K2(L) + K3(L-1): backward skips them
  DevBuf stage_x, stage_y, stage_o, stage_g;  // host-pointer staging
  DevBuf d_starts;
  FusedSmall fused;                      // persistent small-net kernel state
  DeepMK deep;                           // deep narrow-net task megakernel state (deep_mk.cu)
  // CUDA graph of the generic multi-step sequence (nf_train_steps): replayed when a call
  // repeats the same arguments, rebuilt otherwise
  cudaGraphExec_t graph = nullptr;
  std::vector<int64_t> graph_key;
  int64_t graph_kernels = 0;             // kernels in the graph (nf_launch_count on replay)
  cudaStream_t h2d = nullptr, h2d_y = nullptr;  // copy streams of the host-dataset path
  cudaEvent_t h2d_ev[6] = {};            // x slot 0/1 filled, slot 0/1 consumed, y slot 0/1 filled
  cudaStream_t cap_stream = nullptr;     // private stream the graph is captured on (the
                                         // caller's stream may be the legacy default stream)

  // NF_MATH_FP64: double parameters (authoritative while the mode is set), stash and scratch
  double *params64 = nullptr;
  int64_t ws64_rows = 0;
  std::vector<double *> A64, S64;
  DevBuf stash64, partial64, grad64;

  float *W(int l) const { return params + offW[l]; }
  float *Wt(int l) const { return params_t + offW[l]; }
  float *Wlo(int l) const { return params_lo + offW[l]; }
  bool tf32() const { return math == NF_MATH_TF32; }
  bool presplit() const {
    static const bool on = getenv("NF_PRESPLIT") == nullptr || atoi(getenv("NF_PRESPLIT")) != 0;
    return on && math == NF_MATH_FP32;
  }
  double *W64(int l) const { return params64 + offW[l]; }
  double *b64(int l) const { return params64 + offB[l]; }
  float *b(int l) const { return params + offB[l]; }
  int act(int l) const { return acts[l]; }
};

namespace {

constexpr int64_t kEvalChunk = 32768;    // rows per forward chunk for eval calls

void drop_graph(nf_net *net) {
  if (net->graph) cudaGraphExecDestroy(net->graph);
  net->graph = nullptr;
  net->graph_key.clear();
}

int ensure_ws(nf_net *net, int64_t rows) {
  if (rows <= net->ws_rows) return NF_OK;
  int64_t per_row = 0;
  for (int l = 1; l <= net->L; ++l) per_row += 2 * (int64_t)net->dims[l];
  NF_CUDA(cudaStreamSynchronize(net->stream));
  drop_graph(net);
  NF_CUDA(net->stash.ensure((size_t)(per_row * rows) * sizeof(float)));
  if (net->L >= 2)
    NF_CUDA(net->part_out.ensure((size_t)out_layer_blocks((int)rows, net->dims[net->L - 1]) *
                                 (net->dims[net->L] * (net->dims[net->L - 1] + 1) + 1) * sizeof(float)));
  float *p = net->stash.as<float>();
  net->A.assign(net->L + 1, nullptr);
  net->S.assign(net->L + 1, nullptr);
  for (int l = 1; l <= net->L; ++l) {
    net->A[l] = p; p += rows * net->dims[l];
    net->S[l] = p; p += rows * net->dims[l];
  }
  net->ws_rows = rows;
  return NF_OK;
}

// Which weight-gradient contractions read transposed (K-major) copies of their operands, written
// by the producing epilogues: the big tensor-core ones (a wave of 128 x 256 tiles or more: config
// 5's), whose MN-major smem operands cost ~16 % of the tensor rate.
// Off by default since the tensor-core instructions are issued warp-uniformly (the MN/MN kernel no
// longer pays the per-instruction issue overhead and the transposed copies' extra HBM writes cost
// more than they save: config 5 TF32 7.73 -> 7.36 ms per step, profiles/r02_uniform_issue.txt);
// NF_TPOSE=1 turns it on for NF_MATH_TF32, NF_TPOSE=2 also in the 3xTF32 fp32 mode.
int ensure_tpose(nf_net *net, const float *x, int64_t n) {
  const int mode = getenv("NF_TPOSE") ? atoi(getenv("NF_TPOSE")) : 0;  // (read per call: tests toggle it)
  const int L = net->L;
  std::vector<char> tp(L + 1, 0);
  const bool on = mode == 2 ? net->math != NF_MATH_FP64 : (mode == 1 && net->math == NF_MATH_TF32);
  if (on && n >= 1024) {
    for (int l = 1; l <= L; ++l) {
      const int M = net->dims[l], N = net->dims[l - 1];
      const int64_t tiles = (int64_t)((M + 127) / 128) * ((N + 255) / 256);
      // (one wave of 128 x 256 tiles or more: config 5's 4096-wide layers and its 1024-wide output layer)
      if (N <= 128 || tiles < 148 * 4 / 5 || !gemm_grad_tc(M, N, (int)n, net->S[l], l > 1 ? net->A[l - 1] : x)) continue;
      // the producers must be tensor-core epilogues (they write the copies)
      const bool d_ok = l == L ? gemm_fwd_tc((int)n, M, N, l > 1 ? net->A[l - 1] : x, net->W(l))
                               : gemm_bwd_tc((int)n, M, net->dims[l + 1], net->S[l + 1], net->W(l + 1));
      const bool a_ok = l == 1 || gemm_fwd_tc((int)n, N, net->dims[l - 2], l > 2 ? net->A[l - 2] : x, net->W(l - 1));
      tp[l] = d_ok && a_ok;
    }
  }
  net->tpose = tp;
  int64_t need = 0;
  for (int l = 1; l <= L; ++l)
    if (tp[l]) need += (int64_t)net->dims[l] + (l > 1 ? net->dims[l - 1] : 0);
  if (need == 0) return NF_OK;
  if (tp == net->t_key && n <= net->t_rows) return NF_OK;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(net->stream, &cs);
  if (cs != cudaStreamCaptureStatusNone) {  // no allocation inside a graph capture: MN-major operands
    net->tpose.assign(L + 1, 0);
    return NF_OK;
  }
  NF_CUDA(cudaStreamSynchronize(net->stream));
  drop_graph(net);
  NF_CUDA(net->tstash.ensure((size_t)(need * n) * sizeof(float)));
  net->AT.assign(L + 1, nullptr);
  net->DT.assign(L + 1, nullptr);
  float *p = net->tstash.as<float>();
  for (int l = 1; l <= L; ++l)
    if (tp[l]) {
      net->DT[l] = p; p += (int64_t)net->dims[l] * n;
      if (l > 1) { net->AT[l - 1] = p; p += (int64_t)net->dims[l - 1] * n; }
    }
  net->t_key = tp;
  net->t_rows = n;
  return NF_OK;
}

bool tposed(const nf_net *net, int l) { return l >= 1 && l < (int)net->tpose.size() && net->tpose[l]; }

// NF_MATH_TF32: make the weight shadow current (one rounding pass after any write of params
// other than a TF32 step's own epilogues)
int ensure_shadow(nf_net *net) {
  if (!net->tf32() || net->shadow_ok) return NF_OK;
  if (!net->params_t) NF_CUDA(cudaMalloc(&net->params_t, net->nparams * sizeof(float)));
  NF_CUDA(round_tf32(net->stream, net->params, net->params_t, net->nparams));
  net->shadow_ok = true;
  return NF_OK;
}

// The weights' RN split (hi in params_t, lo in params_lo) for the tensor-core inference kernel,
// in either fp32 or TF32 mode (the TF32 shadow is the same hi: cvt.rna of params)
int ensure_wsplit(nf_net *net) {
  if (!net->params_lo) NF_CUDA(cudaMalloc(&net->params_lo, net->nparams * sizeof(float)));
  if (!net->params_t) NF_CUDA(cudaMalloc(&net->params_t, net->nparams * sizeof(float)));
  if (!net->lo_ok) {
    NF_CUDA(split_rn(net->stream, net->params, net->params_t, net->params_lo, net->nparams));
    net->lo_ok = true;
    net->shadow_ok = true;
  }
  return NF_OK;
}

// fp32 mode: the lo shadow of the weights and the lo arrays of a training batch of `rows` rows
int ensure_lo(nf_net *net, int64_t rows) {
  if (!net->presplit()) return NF_OK;
  if (!net->params_lo) NF_CUDA(cudaMalloc(&net->params_lo, net->nparams * sizeof(float)));
  if (!net->params_t) NF_CUDA(cudaMalloc(&net->params_t, net->nparams * sizeof(float)));
  if (!net->lo_ok) {  // the weights' RN split: hi in params_t, lo in params_lo
    NF_CUDA(split_rn(net->stream, net->params, net->params_t, net->params_lo, net->nparams));
    net->lo_ok = true;
  }
  if (rows > net->lo_rows) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(net->stream, &cs);
    if (cs != cudaStreamCaptureStatusNone) return fail(NF_ECUDA, "lo arrays must be sized before a graph capture");
    auto blk = [&](int w) { return (rows * w + 31) / 32 * 32; };  // 128-B aligned arrays (TMA, float4)
    int64_t total = 2 * blk(net->dims[0]);
    for (int l = 1; l <= net->L; ++l) total += 3 * blk(net->dims[l]);
    NF_CUDA(cudaStreamSynchronize(net->stream));
    drop_graph(net);
    NF_CUDA(net->stash_lo.ensure((size_t)total * sizeof(float)));
    float *p = net->stash_lo.as<float>();
    net->Ahi.assign(net->L + 1, nullptr);
    net->Alo.assign(net->L + 1, nullptr);
    net->Dlo.assign(net->L + 1, nullptr);
    net->Ahi[0] = p; p += blk(net->dims[0]);  // the input rows' RN split
    net->Alo[0] = p; p += blk(net->dims[0]);
    for (int l = 1; l <= net->L; ++l) {
      net->Ahi[l] = p; p += blk(net->dims[l]);
      net->Alo[l] = p; p += blk(net->dims[l]);
      net->Dlo[l] = p; p += blk(net->dims[l]);
    }
    net->lo_rows = rows;
  }
  return NF_OK;
}

// fwdprop over a batch.  mode: 0 train (stash A, S; output layer
// S = delta_L), 2 inference (A only).  y only for mode 0.
int forward(nf_net *net, const float *x, const float *y, int64_t n, int mode) {
  const float *in = x;
  const int L = net->L;
  if (int rc = ensure_shadow(net)) return rc;
  const bool t = net->tf32();
  // fp32 training / tendencies: pre-split operands (the input rows' lo first)
  const bool lo = mode == 0 && net->presplit();
  if (lo) {
    if (int rc = ensure_lo(net, n)) return rc;
    NF_CUDA(split_rn(net->stream, x, net->Ahi[0], net->Alo[0], n * net->dims[0]));
  }
  net->out_fused = mode == 0 && L >= 2 &&
                   out_layer_fusable((int)n, net->dims[L - 1], net->dims[L], net->A[L - 1], net->S[L - 1], net->W(L));
  for (int l = 1; l <= net->L; ++l) {
    if (l == L && net->out_fused) {  // K1+K2 of the output layer, K3 of layer L-1, K4(L) partials
      NF_CUDA(out_layer_train_fused(net->stream, (int)n, net->dims[L - 1], net->dims[L], net->A[L - 1],
                                    net->S[L - 1], net->W(L), net->b(L), y, net->A[L], net->S[L], net->act_o,
                                    net->part_out.as<float>(), t ? 1 : 0, lo ? net->Dlo[L - 1] : nullptr));
      break;
    }
    const int lm = (mode == 2) ? 2 : (l < net->L ? 0 : 1);
    // TF32: a hidden layer's A and the output layer's delta_L are operands of later tensor-core
    // contractions -> stored RN-rounded (the net's output A_L never is)
    EpiFwd epi{net->b(l), net->A[l], net->S[l], y, net->dims[l], net->act(l), lm, (t && (lm == 1 || l < L)) ? 1 : 0};
    if (lm == 0 && tposed(net, l + 1)) { epi.T = net->AT[l]; epi.ldT = (int)n; }   // A_l^T for K4(l+1)
    if (lm == 1 && tposed(net, l)) { epi.T = net->DT[l]; epi.ldT = (int)n; }       // delta_L^T for K4(L)
    if (lo) {
      epi.lo = lm == 0 ? net->Alo[l] : net->Dlo[l];
      epi.hi = lm == 0 ? net->Ahi[l] : nullptr;
    }
    NF_CUDA(gemm_fwd(net->stream, (int)n, net->dims[l], net->dims[l - 1], in, net->W(l), epi, net->ws,
                     (t || lo) ? net->Wt(l) : nullptr, lo ? net->Alo[l - 1] : nullptr, lo ? net->Wlo(l) : nullptr,
                     lo ? net->Ahi[l - 1] : nullptr));
    in = net->A[l];
  }
  return NF_OK;
}

// backprop + batch sum + update.  With
// grad != nullptr the summed tendencies are stored there instead (nf_grad).
// Order per layer: the delta of layer l-1 (reads W_l) BEFORE W_l is updated.
int ensure_side(nf_net *net) {
  if (net->side) return NF_OK;
  NF_CUDA(cudaStreamCreateWithFlags(&net->side, cudaStreamNonBlocking));
  net->ev.assign(net->L + 2, nullptr);
  for (auto &e : net->ev) NF_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  NF_CUDA(net->partial2.ensure(size_t(16) << 20 << 2));
  net->ws2.partial = net->partial2.as<float>();
  net->ws2.partial_floats = size_t(16) << 20;
  return NF_OK;
}

// backprop + batch sum + update.  With grad != nullptr the
// summed tendencies are stored there instead (nf_grad).  Per layer l (L..1): K3(l) computes
// delta_{l-1} from delta_l and W_l on the main stream; K4(l) (tendencies of W_l, b_l and the
// update) runs on the side stream once K3(l) has read W_l, overlapping K3(l-1).
int backward(nf_net *net, const float *x, int64_t n, float eta, float *grad, float *step_loss = nullptr,
             cudaEvent_t const *layer_done = nullptr) {
  if (int rc = ensure_side(net)) return rc;
  net->ws2.math = net->ws.math;
  // The overlap only pays while the GEMMs are under one wave of 128x256 tiles (c3, c4): a
  // GEMM that fills the GPU (c5: 2048 tiles, the persistent kernel) would just contend for
  // the SMs with the other stream's GEMM, so those nets keep both on the main stream.
  int64_t max_tiles = 0;
  for (int l = 1; l <= net->L; ++l)
    max_tiles = std::max<int64_t>(max_tiles, ((n + 127) / 128) * ((net->dims[l - 1] + 255) / 256));
  static const bool force_overlap = getenv("NF_BWD_OVERLAP") != nullptr;
  const bool overlap = force_overlap || max_tiles <= 148;
  cudaStream_t main_st = net->stream, side = overlap ? net->side : net->stream;
  NF_CUDA(cudaEventRecord(net->ev[0], main_st));  // fork (delta_L and the stash are ready)
  NF_CUDA(cudaStreamWaitEvent(side, net->ev[0], 0));
  const float scale = (float)((double)eta / (double)n);
  std::vector<char> bias_done(net->L + 1, 0);  // layer's bias update applied by K3's epilogue
  // TF32 SGD: split-K terms reduced into W leave the shadow stale -> one rounding pass at the end
  // (fp32 with pre-split: the lo shadow, one split pass)
  const bool lo = net->presplit() && net->lo_rows >= n && !net->Alo.empty();
  net->red_round = false;
  net->ws.red_flag = net->ws2.red_flag = (!grad && (net->tf32() || lo)) ? &net->red_round : nullptr;
  for (int l = net->L; l >= 1; --l) {
    const int nl = net->dims[l], nk = net->dims[l - 1];
    const bool fused = l == net->L && net->out_fused;  // K3(L) ran inside the forward kernel
    const bool t = net->tf32();
    if (l > 1 && !fused) {
      EpiBwd eb{net->S[l - 1], nk};
      eb.rnd = t ? 1 : 0;
      if (tposed(net, l - 1)) { eb.T = net->DT[l - 1]; eb.ldT = (int)n; }  // delta_{l-1}^T for K4(l-1)
      if (lo) eb.lo = net->Dlo[l - 1];
      const float *aprev2 = l > 2 ? net->A[l - 2] : x;  // the operand of layer l-1's weight GEMM
      if (!grad && gemm_bwd_fuses_bias((int)n, nk, nl, net->S[l], net->W(l)) &&
          gemm_grad_tc(nk, net->dims[l - 2], (int)n, net->S[l - 1], aprev2)) {
        eb.bias = net->b(l - 1);  // b_{l-1} -= scale * column sums of delta_{l-1}, in the epilogue
        eb.bscale = scale;
        bias_done[l - 1] = 1;
      }
      NF_CUDA(gemm_bwd(main_st, (int)n, nk, nl, net->S[l], net->W(l), eb, net->ws, (t || lo) ? net->Wt(l) : nullptr,
                       lo ? net->Dlo[l] : nullptr, lo ? net->Wlo(l) : nullptr));
    }
    NF_CUDA(cudaEventRecord(net->ev[l], main_st));  // K3(l) done with W_l and delta_l is final
    NF_CUDA(cudaStreamWaitEvent(side, net->ev[l], 0));
    const float *aprev = l > 1 ? net->A[l - 1] : x;
    EpiGrad eg = grad ? EpiGrad{grad + net->offW[l], grad + net->offB[l], nk, nk, 0.0f, 1}
                      : EpiGrad{net->W(l), net->b(l), nk, nk, scale, 0};
    if (!grad && t) eg.Wt = net->Wt(l);  // the update also refreshes the TF32 shadow of W_l
    if (!grad && lo) {  // ... or the RN split of W_l (fp32 mode)
      eg.Wt = net->Wt(l);
      eg.Wlo = net->Wlo(l);
    }
    cudaStream_t kst = side;  // the stream layer l's tendencies are produced on
    if (fused) NF_CUDA(out_layer_grad_final(side, (int)n, nk, nl, net->part_out.as<float>(), eg, step_loss));
    else if (l == 1 && net->L > 1 && side != main_st && (net->math != NF_MATH_TF32 || n <= 2048)) {
      // the main stream is idle after the last K3: K4(1) there, concurrent with K4(2) on the side
      // stream (c4 134 -> 130 us, 3xTF32 c3 462 -> 445 us; c3's 1xTF32 pair contends: 154 -> 157)
      NF_CUDA(gemm_grad(main_st, nl, nk, (int)n, net->S[l], aprev, eg, net->ws, bias_done[l] != 0,
                        tposed(net, l) ? net->DT[l] : nullptr, tposed(net, l) && l > 1 ? net->AT[l - 1] : nullptr,
                        lo ? net->Dlo[l] : nullptr, lo ? net->Alo[l - 1] : nullptr, lo ? net->Ahi[l - 1] : nullptr));
      kst = main_st;
    } else NF_CUDA(gemm_grad(side, nl, nk, (int)n, net->S[l], aprev, eg, net->ws2, bias_done[l] != 0,
                             tposed(net, l) ? net->DT[l] : nullptr, tposed(net, l) && l > 1 ? net->AT[l - 1] : nullptr,
                             lo ? net->Dlo[l] : nullptr, lo ? net->Alo[l - 1] : nullptr, lo ? net->Ahi[l - 1] : nullptr));
    if (layer_done && layer_done[l - 1]) NF_CUDA(cudaEventRecord(layer_done[l - 1], kst));  // nf_grad_layers
  }
  NF_CUDA(cudaEventRecord(net->ev[net->L + 1], side));  // join
  NF_CUDA(cudaStreamWaitEvent(main_st, net->ev[net->L + 1], 0));
  net->ws.red_flag = net->ws2.red_flag = nullptr;
  if (net->red_round) {
    if (net->tf32()) NF_CUDA(round_tf32(main_st, net->params, net->params_t, net->nparams));
    else NF_CUDA(split_rn(main_st, net->params, net->params_t, net->params_lo, net->nparams));
  }
  return NF_OK;
}

// ---- NF_MATH_FP64: the same steps in double (fp64.cu), all on the net's stream -------------
constexpr size_t kPartial64 = size_t(8) << 20;  // split-K partials (doubles)

int ensure_ws64(nf_net *net, int64_t rows) {
  if (rows <= net->ws64_rows) return NF_OK;
  int64_t per_row = 0;
  for (int l = 1; l <= net->L; ++l) per_row += 2 * (int64_t)net->dims[l];
  NF_CUDA(cudaStreamSynchronize(net->stream));
  drop_graph(net);
  NF_CUDA(net->stash64.ensure((size_t)(per_row * rows) * sizeof(double)));
  double *p = net->stash64.as<double>();
  net->A64.assign(net->L + 1, nullptr);
  net->S64.assign(net->L + 1, nullptr);
  for (int l = 1; l <= net->L; ++l) {
    net->A64[l] = p; p += rows * net->dims[l];
    net->S64[l] = p; p += rows * net->dims[l];
  }
  net->ws64_rows = rows;
  return NF_OK;
}

int forward64(nf_net *net, const float *x, const float *y, int64_t n, int mode) {
  for (int l = 1; l <= net->L; ++l) {
    const int lm = (mode == 2) ? 2 : (l < net->L ? 0 : 1);
    Epi64Fwd epi{net->b64(l), net->A64[l], net->S64[l], y, net->dims[l], net->act(l), lm};
    NF_CUDA(gemm64_fwd(net->stream, (int)n, net->dims[l], net->dims[l - 1], l == 1 ? x : nullptr,
                       l == 1 ? nullptr : net->A64[l - 1], net->W64(l), epi, net->partial64.as<double>(),
                       kPartial64));
  }
  return NF_OK;
}

int backward64(nf_net *net, const float *x, int64_t n, double eta, double *grad) {
  for (int l = net->L; l >= 1; --l) {
    const int nl = net->dims[l], nk = net->dims[l - 1];
    if (l > 1) {
      Epi64Bwd eb{net->S64[l - 1], nk};
      NF_CUDA(gemm64_bwd(net->stream, (int)n, nk, nl, net->S64[l], net->W64(l), eb, net->partial64.as<double>(),
                         kPartial64));
    }
    Epi64Grad eg = grad ? Epi64Grad{grad + net->offW[l], grad + net->offB[l], nk, nk, 0.0, 1}
                        : Epi64Grad{net->W64(l), net->b64(l), nk, nk, eta / (double)n, 0};
    NF_CUDA(gemm64_grad(net->stream, nl, nk, (int)n, net->S64[l], l == 1 ? x : nullptr,
                        l == 1 ? nullptr : net->A64[l - 1], eg, net->partial64.as<double>(), kPartial64));
  }
  return NF_OK;
}

size_t red_bytes() {
  return sizeof(double2) * std::max<size_t>(loss_acc_parts(), loss_acc64_parts()) + 64;
}

int train_batch_dev(nf_net *net, const float *x, const float *y, int64_t n, float eta,
                    float *step_loss) {
  int rc;
  if (net->math == NF_MATH_FP64) {
    if ((rc = ensure_ws64(net, n))) return rc;
    if ((rc = forward64(net, x, y, n, 0))) return rc;
    if (step_loss) {
      NF_CUDA(net->red.ensure(red_bytes()));
      NF_CUDA(loss_acc64(net->stream, net->A64[net->L], y, n, net->dims[net->L], net->red.as<double2>(), nullptr,
                         step_loss));
    }
    return backward64(net, x, n, (double)eta, nullptr);
  }
  if ((rc = ensure_ws(net, n))) return rc;
  if ((rc = ensure_tpose(net, x, n))) return rc;
  if ((rc = forward(net, x, y, n, 0))) return rc;
  if (step_loss && !net->out_fused) {  // (the fused output layer computes the cost itself)
    NF_CUDA(net->red.ensure(red_bytes()));
    NF_CUDA(loss_acc(net->stream, net->A[net->L], y, n, net->dims[net->L], net->red.as<double2>(),
                     nullptr, step_loss));
  }
  return backward(net, x, n, eta, nullptr, net->out_fused ? step_loss : nullptr);
}

const float *stage_in(nf_net *net, const float *p, size_t count, DevBuf &buf, int *rc) {
  *rc = NF_OK;
  if (is_device_ptr(p)) return p;
  cudaError_t e = buf.ensure(count * sizeof(float));
  if (e == cudaSuccess) e = cudaMemcpyAsync(buf.p, p, count * sizeof(float), cudaMemcpyHostToDevice, net->stream);
  if (e != cudaSuccess) {
    *rc = fail(NF_ECUDA, "staging input: %s", cudaGetErrorString(e));
    return nullptr;
  }
  return buf.as<float>();
}

int check_net(const nf_net *net) { return net ? NF_OK : fail(NF_EINVAL, "null net"); }

int check_ptr(const void *p, const char *what) {
  if (!p) return fail(NF_EINVAL, "%s is NULL", what);
  if (reinterpret_cast<uintptr_t>(p) & 3) return fail(NF_EINVAL, "%s is not 4-byte aligned", what);
  return NF_OK;
}

}  // namespace

// ============================================================================ C-ABI
extern "C" {

const char *nf_last_error(void) { return g_err.c_str(); }

int64_t nf_launch_count(void) { return __atomic_load_n(&g_launches, __ATOMIC_RELAXED); }

int nf_net_create(const int32_t *dims, int32_t n_dims, const char *activation, uint64_t seed,
                  nf_net **out) {
  if (!out) return fail(NF_EINVAL, "out is NULL");
  *out = nullptr;
  if (!dims || n_dims < 2) return fail(NF_EINVAL, "need at least 2 dims (S:118-124)");
  for (int i = 0; i < n_dims; ++i)
    if (dims[i] < 1) return fail(NF_EINVAL, "dims[%d] = %d < 1", i, dims[i]);
  // activation spec: one name (every layer), "hidden,output" (R7), or one name per layer
  const std::string spec = activation ? activation : "sigmoid";
  std::vector<int> names;
  for (size_t b = 0;;) {
    const size_t e = spec.find(',', b);
    const int k = parse_act(spec.substr(b, e == std::string::npos ? std::string::npos : e - b));
    if (k < 0) return fail(NF_EINVAL, "unknown activation '%s' (S:32-33)", spec.c_str());
    names.push_back(k);
    if (e == std::string::npos) break;
    b = e + 1;
  }
  const int L_ = n_dims - 1;
  std::vector<int> acts(L_ + 1, 0);  // acts[l], l = 1..L
  if (names.size() == 1) {
    for (int l = 1; l <= L_; ++l) acts[l] = names[0];
  } else if (names.size() == 2) {
    for (int l = 1; l <= L_; ++l) acts[l] = l < L_ ? names[0] : names[1];
  } else if ((int)names.size() == L_) {
    for (int l = 1; l <= L_; ++l) acts[l] = names[l - 1];
  } else {
    return fail(NF_EINVAL, "activation spec '%s' needs 1, 2 or %d names", spec.c_str(), L_);
  }

  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return fail(NF_ENODEV, "no CUDA device: this library has no CPU fallback");
  }
  int dev = 0, major = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  if (major != 10) return fail(NF_ENODEV, "device %d is sm_%d0, this build targets sm_100a", dev, major);

  nf_net *net = new nf_net();
  net->dims.assign(dims, dims + n_dims);
  net->L = n_dims - 1;
  net->acts = acts;
  net->act_spec = spec;
  net->act_h = acts[1];       // the two-layer kernels (K6, infer_small, single-CTA for L = 2)
  net->act_o = acts[net->L];
  net->offW.assign(net->L + 1, 0);
  net->offB.assign(net->L + 1, 0);
  int64_t o_ = 0;
  for (int l = 1; l <= net->L; ++l) {
    net->offW[l] = o_; o_ += (int64_t)dims[l] * dims[l - 1];
    net->offB[l] = o_; o_ += dims[l];
  }
  net->nparams = o_;
  std::vector<float> host(o_);
  HostRng rng{seed};
  for (int l = 1; l <= net->L; ++l) {
    for (int64_t i = 0; i < (int64_t)dims[l] * dims[l - 1]; ++i)
      host[net->offW[l] + i] = (float)(rng.normal() / dims[l - 1]);
    for (int i = 0; i < dims[l]; ++i) host[net->offB[l] + i] = (float)rng.normal();
  }
  cudaError_t e = cudaMalloc(&net->params, o_ * sizeof(float));
  if (e == cudaSuccess) e = cudaMemcpy(net->params, host.data(), o_ * sizeof(float), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = net->partial.ensure(size_t(16) << 20 << 2);  // 16M floats
  if (e != cudaSuccess) {
    nf_net_destroy(net);
    return fail(NF_ECUDA, "nf_net_create: %s", cudaGetErrorString(e));
  }
  net->ws.partial = net->partial.as<float>();
  net->ws.partial_floats = size_t(16) << 20;
  *out = net;
  return NF_OK;
}

// ---- saving and loading networks (the paper's feature list; file format of this
// library, the paper does not give one).  Text:
//   "nf-b200-net 2" / n_dims / dims / activation spec / precision "fp32" | "fp64" /
//   the flat parameters (include/nf.h layout), one per line: %.9g for fp32 (exact), %.17g for
//   fp64 (exact).  Version 1 files (no precision line) are fp32.  The header is parsed and
//   validated before the payload; every kind of format error has its own code.
int nf_save(nf_net *net, const char *path) {
  if (int rc = check_net(net)) return rc;
  if (!path) return fail(NF_EINVAL, "path is NULL");
  const bool f64 = net->math == NF_MATH_FP64;
  std::vector<float> p;
  std::vector<double> p64;
  if (f64) {  // the double parameters themselves: never narrowed
    p64.resize(net->nparams);
    NF_CUDA(cudaMemcpyAsync(p64.data(), net->params64, net->nparams * sizeof(double), cudaMemcpyDeviceToHost,
                            net->stream));
    NF_CUDA(cudaStreamSynchronize(net->stream));
  } else {
    p.resize(net->nparams);
    if (int rc = nf_get_params(net, p.data(), net->nparams)) return rc;
  }
  FILE *f = fopen(path, "w");
  if (!f) return fail(NF_EIO, "cannot open '%s' for writing", path);
  fprintf(f, "nf-b200-net 2\n%d\n", (int)net->dims.size());
  for (size_t i = 0; i < net->dims.size(); ++i) fprintf(f, "%d%c", net->dims[i], i + 1 < net->dims.size() ? ' ' : '\n');
  fprintf(f, "%s\n%s\n", net->act_spec.c_str(), f64 ? "fp64" : "fp32");
  if (f64)
    for (double v : p64) fprintf(f, "%.17g\n", v);
  else
    for (float v : p) fprintf(f, "%.9g\n", v);
  const bool ok = fclose(f) == 0;
  return ok ? NF_OK : fail(NF_EIO, "writing '%s' failed", path);
}

int nf_load_as(const char *path, int math, nf_net **out) {
  if (!out) return fail(NF_EINVAL, "out is NULL");
  *out = nullptr;
  if (!path) return fail(NF_EINVAL, "path is NULL");
  if (math != -1 && math != NF_MATH_FP32 && math != NF_MATH_TF32 && math != NF_MATH_FP64)
    return fail(NF_EINVAL, "unknown math mode %d", math);
  FILE *f = fopen(path, "r");
  if (!f) return fail(NF_EIO, "cannot open '%s'", path);
  char magic[32] = {0}, spec[256] = {0}, prec[16] = {0};
  int ver = 0, nd = 0;
  std::vector<int32_t> dims;
  std::vector<double> p;
  int rc = NF_OK;
  bool f64 = false;
  if (fscanf(f, "%31s", magic) != 1 || strcmp(magic, "nf-b200-net") != 0) {
    rc = fail(NF_EFMT_MAGIC, "'%s' is not an nf-b200 network file (magic)", path);
  } else if (fscanf(f, "%d", &ver) != 1 || (ver != 1 && ver != 2)) {
    rc = fail(NF_EFMT_VERSION, "'%s': unsupported format version", path);
  } else if (fscanf(f, "%d", &nd) != 1 || nd < 2 || nd > 1024) {
    rc = fail(NF_EFMT_DIMS, "'%s': bad number of dims", path);
  } else {
    dims.resize(nd);
    for (int i = 0; i < nd && rc == NF_OK; ++i)
      if (fscanf(f, "%d", &dims[i]) != 1 || dims[i] < 1) rc = fail(NF_EFMT_DIMS, "'%s': bad dims", path);
    if (rc == NF_OK && fscanf(f, "%255s", spec) != 1) rc = fail(NF_EFMT_ACTIVATION, "'%s': no activation", path);
    if (rc == NF_OK) {  // the activation spec: validated before any payload is read
      const std::string sp = spec;
      int names = 0;
      for (size_t b = 0;; ++names) {
        const size_t e = sp.find(',', b);
        if (parse_act(sp.substr(b, e == std::string::npos ? std::string::npos : e - b)) < 0) {
          rc = fail(NF_EFMT_ACTIVATION, "'%s': unknown activation '%s'", path, spec);
          break;
        }
        if (e == std::string::npos) { ++names; break; }
        b = e + 1;
      }
      if (rc == NF_OK && names != 1 && names != 2 && names != nd - 1)
        rc = fail(NF_EFMT_ACTIVATION, "'%s': activation spec '%s' has %d names", path, spec, names);
    }
    if (rc == NF_OK && ver == 2) {
      if (fscanf(f, "%15s", prec) != 1 || (strcmp(prec, "fp32") != 0 && strcmp(prec, "fp64") != 0))
        rc = fail(NF_EFMT_PRECISION, "'%s': unknown precision tag", path);
      f64 = strcmp(prec, "fp64") == 0;
    }
    if (rc == NF_OK && math != -1 && f64 != (math == NF_MATH_FP64))
      rc = fail(NF_EFMT_PRECISION, "'%s' holds %s parameters, %s requested (never narrowed or widened silently)",
                path, f64 ? "fp64" : "fp32", math == NF_MATH_FP64 ? "fp64" : "fp32");
    if (rc == NF_OK) {
      int64_t np = 0;
      for (int l = 1; l < nd; ++l) np += (int64_t)dims[l] * dims[l - 1] + dims[l];
      p.resize(np);
      for (int64_t i = 0; i < np && rc == NF_OK; ++i) {
        float v32 = 0.0f;  // fp32 files: 9 digits parsed to the nearest float = the saved value
        if (f64 ? fscanf(f, "%lf", &p[i]) != 1 : fscanf(f, "%f", &v32) != 1)
          rc = fail(NF_EFMT_TRUNCATED, "'%s': %lld of %lld parameters", path, (long long)i, (long long)np);
        else if (!f64)
          p[i] = v32;
      }
    }
  }
  fclose(f);
  if (rc != NF_OK) return rc;
  nf_net *net = nullptr;
  if ((rc = nf_net_create(dims.data(), nd, spec, 0, &net))) return rc;
  std::vector<float> p32(p.begin(), p.end());
  if ((rc = nf_set_params(net, p32.data(), (int64_t)p32.size()))) {
    nf_net_destroy(net);
    return rc;
  }
  if (f64 || math == NF_MATH_TF32) {
    if ((rc = nf_set_math(net, f64 ? NF_MATH_FP64 : math))) {
      nf_net_destroy(net);
      return rc;
    }
  }
  if (f64) {  // the exact doubles
    cudaError_t e = cudaMemcpy(net->params64, p.data(), p.size() * sizeof(double), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
      nf_net_destroy(net);
      return fail(NF_ECUDA, "nf_load: %s", cudaGetErrorString(e));
    }
  }
  *out = net;
  return NF_OK;
}

int nf_load(const char *path, nf_net **out) { return nf_load_as(path, -1, out); }

void nf_net_destroy(nf_net *net) {
  if (!net) return;
  cudaStreamSynchronize(net->stream);
  if (net->params) cudaFree(net->params);
  if (net->params64) cudaFree(net->params64);
  if (net->params_t) cudaFree(net->params_t);
  if (net->params_lo) cudaFree(net->params_lo);
  net->stash_lo.release();
  net->xlo.release();
  net->stash64.release();
  net->partial64.release();
  net->grad64.release();
  net->stash.release();
  net->partial.release();
  net->red.release();
  net->part_out.release();
  net->stage_x.release();
  net->stage_y.release();
  net->stage_o.release();
  net->stage_g.release();
  net->d_starts.release();
  fused_small_release(net->fused);
  deep_mk_release(net->deep);
  drop_graph(net);
  if (net->cap_stream) cudaStreamDestroy(net->cap_stream);
  for (auto e : net->h2d_ev) if (e) cudaEventDestroy(e);
  if (net->h2d) cudaStreamDestroy(net->h2d);
  if (net->h2d_y) cudaStreamDestroy(net->h2d_y);
  for (auto e : net->ev) if (e) cudaEventDestroy(e);
  if (net->side) cudaStreamDestroy(net->side);
  net->partial2.release();
  delete net;
}

int nf_set_stream(nf_net *net, void *s) {
  if (int rc = check_net(net)) return rc;
  net->stream = static_cast<cudaStream_t>(s);
  return NF_OK;
}

int nf_set_math(nf_net *net, int mode) {
  if (int rc = check_net(net)) return rc;
  if (mode != NF_MATH_FP32 && mode != NF_MATH_TF32 && mode != NF_MATH_FP64)
    return fail(NF_EINVAL, "unknown math mode %d", mode);
  if (mode == NF_MATH_FP64 && net->math != NF_MATH_FP64) {
    // enter: the double parameters start as the exact widening of the fp32 arena
    if (!net->params64) NF_CUDA(cudaMalloc(&net->params64, net->nparams * sizeof(double)));
    NF_CUDA(net->partial64.ensure(kPartial64 * sizeof(double)));
    NF_CUDA(f64_widen(net->stream, net->params, net->params64, net->nparams));
  } else if (mode != NF_MATH_FP64 && net->math == NF_MATH_FP64) {
    // leave: round the double parameters back into the fp32 arena
    NF_CUDA(f64_round(net->stream, net->params64, net->params, net->nparams));
    fused_small_invalidate(net->fused);
  }
  if (mode != net->math) {
    net->shadow_ok = false;
    net->lo_ok = false;
  }
  net->math = mode;
  net->ws.math = mode;
  return NF_OK;
}

int64_t nf_param_count(const nf_net *net) { return net ? net->nparams : -1; }

int nf_get_params(nf_net *net, float *dst, int64_t count) {
  if (int rc = check_net(net)) return rc;
  if (int rc = check_ptr(dst, "dst")) return rc;
  if (count != net->nparams) return fail(NF_EINVAL, "count %lld != %lld", (long long)count, (long long)net->nparams);
  const bool dev = is_device_ptr(dst);
  if (net->math == NF_MATH_FP64) {
    float *d = dst;
    if (!dev) {
      NF_CUDA(net->stage_g.ensure((size_t)count * sizeof(float)));
      d = net->stage_g.as<float>();
    }
    NF_CUDA(f64_round(net->stream, net->params64, d, count));
    if (!dev) {
      NF_CUDA(cudaMemcpyAsync(dst, d, count * sizeof(float), cudaMemcpyDeviceToHost, net->stream));
      NF_CUDA(cudaStreamSynchronize(net->stream));
    }
    return NF_OK;
  }
  NF_CUDA(cudaMemcpyAsync(dst, net->params, count * sizeof(float),
                          dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, net->stream));
  if (!dev) NF_CUDA(cudaStreamSynchronize(net->stream));
  return NF_OK;
}

int nf_set_params(nf_net *net, const float *src, int64_t count) {
  if (int rc = check_net(net)) return rc;
  if (int rc = check_ptr(src, "src")) return rc;
  if (count != net->nparams) return fail(NF_EINVAL, "count %lld != %lld", (long long)count, (long long)net->nparams);
  const bool dev = is_device_ptr(src);
  NF_CUDA(cudaMemcpyAsync(net->params, src, count * sizeof(float),
                          dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, net->stream));
  net->shadow_ok = false;
  net->lo_ok = false;
  if (net->math == NF_MATH_FP64) NF_CUDA(f64_widen(net->stream, net->params, net->params64, count));
  if (!dev) NF_CUDA(cudaStreamSynchronize(net->stream));
  fused_small_invalidate(net->fused);
  return NF_OK;
}

int nf_output(nf_net *net, const float *x, int64_t n, float *out) {
  if (int rc = check_net(net)) return rc;
  if (n < 0) return fail(NF_EINVAL, "n < 0");
  if (n == 0) return NF_OK;
  if (int rc = check_ptr(x, "x")) return rc;
  if (int rc = check_ptr(out, "out")) return rc;
  const int n0 = net->dims[0], nL = net->dims[net->L];
  int rc;
  const float *dx = stage_in(net, x, (size_t)n * n0, net->stage_x, &rc);
  if (rc) return rc;
  const bool host_out = !is_device_ptr(out);
  float *dout = out;
  if (host_out) {
    NF_CUDA(net->stage_o.ensure((size_t)n * nL * sizeof(float)));
    dout = net->stage_o.as<float>();
  }
  if (net->math == NF_MATH_FP64) {
    const int64_t chunk = std::min<int64_t>(n, kEvalChunk);
    if ((rc = ensure_ws64(net, chunk))) return rc;
    for (int64_t r = 0; r < n; r += chunk) {
      const int64_t m = std::min(chunk, n - r);
      if ((rc = forward64(net, dx + r * n0, nullptr, m, 2))) return rc;
      NF_CUDA(f64_round(net->stream, net->A64[net->L], dout + r * nL, m * nL));
    }
  } else if (infer_tc_applicable(net->dims, dx) && getenv("NF_DISABLE_FUSED") == nullptr) {
    if ((rc = ensure_wsplit(net))) return rc;
    NF_CUDA(infer_tc(net->stream, net->dims, net->act_h, net->act_o, net->params, net->params_t, net->params_lo,
                     dx, n, dout));
  } else if (infer_small_applicable(net->dims, dx) && getenv("NF_DISABLE_FUSED") == nullptr) {
    NF_CUDA(infer_small(net->stream, net->dims, net->act_h, net->act_o, net->params, dx, n, dout));
  } else {
    const int64_t chunk = std::min<int64_t>(n, kEvalChunk);
    if ((rc = ensure_ws(net, chunk))) return rc;
    for (int64_t r = 0; r < n; r += chunk) {
      const int64_t m = std::min(chunk, n - r);
      if ((rc = forward(net, dx + r * n0, nullptr, m, 2))) return rc;
      NF_CUDA(cudaMemcpyAsync(dout + r * nL, net->A[net->L], (size_t)m * nL * sizeof(float),
                              cudaMemcpyDeviceToDevice, net->stream));
    }
  }
  if (host_out) {
    NF_CUDA(cudaMemcpyAsync(out, dout, (size_t)n * nL * sizeof(float), cudaMemcpyDeviceToHost, net->stream));
    NF_CUDA(cudaStreamSynchronize(net->stream));
  }
  return NF_OK;
}

int nf_train_batch(nf_net *net, const float *x, const float *y, int64_t n, float eta) {
  if (net && !net->presplit()) net->lo_ok = false;  // (outside the fp32 mode nothing keeps params_lo current)
  if (int rc = check_net(net)) return rc;
  if (n <= 0) return fail(NF_EINVAL, "train needs n >= 1 (S:181)");
  if (!std::isfinite(eta)) return fail(NF_EINVAL, "eta is not finite");
  if (int rc = check_ptr(x, "x")) return rc;
  if (int rc = check_ptr(y, "y")) return rc;
  int rc;
  const float *dx = stage_in(net, x, (size_t)n * net->dims[0], net->stage_x, &rc);
  if (rc) return rc;
  const float *dy = stage_in(net, y, (size_t)n * net->dims[net->L], net->stage_y, &rc);
  if (rc) return rc;
  fused_small_invalidate(net->fused);
  rc = train_batch_dev(net, dx, dy, n, eta, nullptr);
  if (rc == NF_OK && (dx != x || dy != y)) NF_CUDA(cudaStreamSynchronize(net->stream));
  return rc;
}

// The training steps on device-resident data: the single-CTA latency kernel, K6, or the
// generic per-layer kernels (CUDA graph).  st: the steps' first rows in dX / dY (host array).
static int train_steps_device(nf_net *net, const float *dX, const float *dY, int64_t N, int64_t batch,
                              std::vector<int64_t> &st, int64_t n_steps, float eta, float *step_loss,
                              bool allow_graph) {
  const int n0 = net->dims[0], nL = net->dims[net->L];
  const int64_t dN = N;
  // Latency regime (a few rows per step, parameters fit one SM): the single-CTA kernel
  if (net->math != NF_MATH_FP64 && single_cta_applicable(net->dims, batch)) {
    NF_CUDA(net->d_starts.ensure((size_t)n_steps * sizeof(int64_t)));
    NF_CUDA(cudaMemcpyAsync(net->d_starts.p, st.data(), (size_t)n_steps * sizeof(int64_t), cudaMemcpyHostToDevice,
                            net->stream));
    const int src = single_cta_train_steps(net->stream, net->dims, net->acts, net->params, dX, dY,
                                           batch, net->d_starts.as<int64_t>(), n_steps, eta, step_loss);
    if (src == 0) {
      fused_small_invalidate(net->fused);
      net->shadow_ok = false;
  net->lo_ok = false;
      return NF_OK;
    }
    if (src != SINGLE_NOT_APPLICABLE)
      return fail(NF_ECUDA, "single-CTA kernel: %s", cudaGetErrorString((cudaError_t)src));
  }
  // Deep nets of narrow hidden layers in TF32 (config 4): all steps in one task-megakernel launch
  static const bool det = getenv("NF_SPLITK_DETERMINISTIC") != nullptr;
  if (getenv("NF_TRACE_HOST"))
    fprintf(stderr, "[route] det=%d math=%d batch=%lld deep=%d\n", (int)det, net->math, (long long)batch,
            (int)deep_mk_applicable(net->dims, net->math, batch));
  if (!det && deep_mk_applicable(net->dims, net->math, batch)) {
    int rc2;
    if ((rc2 = ensure_ws(net, batch))) return rc2;
    if ((rc2 = ensure_shadow(net))) return rc2;
    rc2 = deep_mk_train_steps(net->deep, net->stream, net->dims, net->acts, net->params, net->params_t, net->offW,
                              net->offB, net->A, net->S, dX, dY, dN, batch, st.data(), n_steps, eta, step_loss);
    if (rc2 == 0) {
      fused_small_invalidate(net->fused);
      return NF_OK;  // (the kernel leaves the TF32 shadow current)
    }
    if (rc2 != DEEP_NOT_APPLICABLE) return fail(NF_ECUDA, "deep-net megakernel: %s", deep_mk_error());
  }
  int rc = net->math == NF_MATH_FP64 ? FUSED_NOT_APPLICABLE : fused_small_train_steps(net->fused, net->stream, net->dims, net->act_h, net->act_o,
                                   net->params, dX, dY, dN, batch, st.data(), n_steps, eta, step_loss);
  if (rc == 0) {  // K6 updated params
    net->shadow_ok = false;
    net->lo_ok = false;
  }
  if (rc == FUSED_NOT_APPLICABLE) {
    // Generic nets: the per-step kernel sequence of all n_steps, captured once as a CUDA
    // graph and replayed while the arguments repeat (removes the host launch gaps between the
    // ~10-50 kernels of each step).  Workspaces are sized before capture.
    if ((rc = net->math == NF_MATH_FP64 ? ensure_ws64(net, batch) : ensure_ws(net, batch))) return rc;
    if ((rc = ensure_side(net))) return rc;
    if ((rc = ensure_shadow(net))) return rc;  // before capture: the graph keeps it current
    if (net->math != NF_MATH_FP64 && (rc = ensure_tpose(net, dX + st[0] * n0, batch))) return rc;
    if ((rc = ensure_lo(net, batch))) return rc;  // (sized before the capture)
    NF_CUDA(net->red.ensure(red_bytes()));
    std::vector<int64_t> key = {(int64_t)(uintptr_t)dX, (int64_t)(uintptr_t)dY, N, batch, n_steps,
                                (int64_t)(uintptr_t)step_loss, (int64_t)(uintptr_t)net->stream, net->math,
                                (int64_t)(uintptr_t)net->stash.p, (int64_t)(uintptr_t)net->stash64.p};
    int32_t eb;
    memcpy(&eb, &eta, 4);
    key.push_back(eb);
    key.insert(key.end(), st.begin(), st.end());
    const bool use_graph = allow_graph && getenv("NF_NO_GRAPH") == nullptr;
    if (use_graph && net->graph && key == net->graph_key) {
      NF_CUDA(cudaGraphLaunch(net->graph, net->stream));
      count_launch((int)net->graph_kernels);
      return NF_OK;
    }
    const int64_t launches0 = nf_launch_count();
    cudaStream_t user = net->stream;
    if (use_graph) {
      drop_graph(net);
      if (!net->cap_stream) NF_CUDA(cudaStreamCreateWithFlags(&net->cap_stream, cudaStreamNonBlocking));
      NF_CUDA(cudaStreamBeginCapture(net->cap_stream, cudaStreamCaptureModeRelaxed));
      net->stream = net->cap_stream;  // the step kernels are recorded, not run
    }
    for (int64_t s = 0; s < n_steps; ++s) {
      rc = train_batch_dev(net, dX + st[s] * n0, dY + st[s] * nL, batch, eta,
                           step_loss ? step_loss + s : nullptr);
      if (rc) break;
    }
    net->stream = user;
    if (use_graph) {
      cudaGraph_t g = nullptr;
      cudaError_t e = cudaStreamEndCapture(net->cap_stream, &g);
      if (rc) {
        if (g) cudaGraphDestroy(g);
        return rc;
      }
      if (e == cudaSuccess) e = cudaGraphInstantiate(&net->graph, g, 0);
      if (g) cudaGraphDestroy(g);
      if (e != cudaSuccess) {
        net->graph = nullptr;
        return fail(NF_ECUDA, "CUDA graph of the training steps: %s", cudaGetErrorString(e));
      }
      net->graph_key = key;
      net->graph_kernels = nf_launch_count() - launches0;
      NF_CUDA(cudaGraphLaunch(net->graph, net->stream));
    }
    if (rc) return rc;
  } else if (rc != 0) {
    return fail(NF_ECUDA, "fused small-net kernel: %s", fused_small_error());
  }
  return NF_OK;
}


int nf_train_steps(nf_net *net, const float *X, const float *Y, int64_t N, int64_t batch,
                   const int64_t *starts, int64_t n_steps, float eta, float *step_loss) {
  host_trace("enter");
  if (net && !net->presplit()) net->lo_ok = false;  // (outside the fp32 mode nothing keeps params_lo current)
  if (int rc = check_net(net)) return rc;
  if (batch <= 0 || N < batch) return fail(NF_EINVAL, "need 1 <= batch <= N");
  if (n_steps < 0) return fail(NF_EINVAL, "n_steps < 0");
  if (n_steps == 0) return NF_OK;
  if (!std::isfinite(eta)) return fail(NF_EINVAL, "eta is not finite");
  if (int rc = check_ptr(X, "X")) return rc;
  if (int rc = check_ptr(Y, "Y")) return rc;
  if (!starts) return fail(NF_EINVAL, "starts is NULL");
  if (is_device_ptr(starts)) return fail(NF_EINVAL, "starts must be a host array");
  for (int64_t s = 0; s < n_steps; ++s)
    if (starts[s] < 0 || starts[s] + batch > N)
      return fail(NF_EINVAL, "starts[%lld] = %lld outside [0, N-batch]", (long long)s, (long long)starts[s]);
  if (step_loss && !is_device_ptr(step_loss)) return fail(NF_EINVAL, "step_loss must be a device array");
  const int n0 = net->dims[0], nL = net->dims[net->L];

  // Device dataset: the steps run straight from it.
  const bool host_in = !is_device_ptr(X) || !is_device_ptr(Y);
  host_trace("checks");
  if (!host_in) {
    std::vector<int64_t> st(starts, starts + n_steps);
    const int rc = train_steps_device(net, X, Y, N, batch, st, n_steps, eta, step_loss, true);
    host_trace("launched");
    return rc;
  }
  // Host dataset (the e2e path): each step's batch is copied host -> device (one copy of its
  // x rows and one of its y rows), in chunks of steps through two staging slots on a copy
  // stream, so that the copies of chunk c+1 overlap the training of chunk c.
  const int64_t row_f = n0 + nL;
  static const int64_t chunk_mb = getenv("NF_H2D_CHUNK_MB") ? atoi(getenv("NF_H2D_CHUNK_MB")) : 16;
  static const bool y_stream = getenv("NF_H2D_Y_STREAM") != nullptr;
  const int64_t chunk = std::max<int64_t>(
      1, std::min<int64_t>(std::min<int64_t>(n_steps, 64), (chunk_mb << 20) / (batch * row_f * 4)));
  // the target rows: read by a gather kernel straight from pinned (mapped) host memory on a
  // second stream, overlapping the x DMA (one small DMA per step cost 8 % of the e2e time)
  const float *Ymap = nullptr;
  {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, Y) == cudaSuccess && at.type == cudaMemoryTypeHost && at.devicePointer)
      Ymap = static_cast<const float *>(at.devicePointer);
    else
      cudaGetLastError();
  }
  static const bool no_gather = getenv("NF_H2D_NO_GATHER") != nullptr;
  if (no_gather) Ymap = nullptr;
  cudaStream_t ys = (y_stream || Ymap) ? net->h2d_y : net->h2d;
  const int64_t slot_f = chunk * batch * row_f;
  NF_CUDA(net->stage_x.ensure((size_t)(2 * slot_f) * sizeof(float)));
  if (!net->h2d) {
    NF_CUDA(cudaStreamCreateWithFlags(&net->h2d, cudaStreamNonBlocking));
    NF_CUDA(cudaStreamCreateWithFlags(&net->h2d_y, cudaStreamNonBlocking));
    for (auto &e : net->h2d_ev) NF_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  NF_CUDA(cudaEventRecord(net->h2d_ev[2], net->stream));  // the caller's prior work on the net
  NF_CUDA(cudaEventRecord(net->h2d_ev[3], net->stream));
  for (int64_t c0 = 0, ci = 0; c0 < n_steps; c0 += chunk, ++ci) {
    const int slot = (int)(ci & 1);
    const int64_t m = std::min(chunk, n_steps - c0);
    float *sx = net->stage_x.as<float>() + slot * slot_f, *sy = sx + chunk * batch * n0;
    NF_CUDA(cudaStreamWaitEvent(net->h2d, net->h2d_ev[2 + slot], 0));  // slot free again
    NF_CUDA(cudaStreamWaitEvent(net->h2d_y, net->h2d_ev[2 + slot], 0));
    std::vector<int64_t> st(m), yoff(m);
    for (int64_t s = 0; s < m; ++s) {
      NF_CUDA(cudaMemcpyAsync(sx + s * batch * n0, X + starts[c0 + s] * n0, (size_t)batch * n0 * sizeof(float),
                              cudaMemcpyDefault, net->h2d));
      if (!Ymap)
        NF_CUDA(cudaMemcpyAsync(sy + s * batch * nL, Y + starts[c0 + s] * nL, (size_t)batch * nL * sizeof(float),
                                cudaMemcpyDefault, ys));
      yoff[s] = starts[c0 + s] * nL;
      st[s] = s * batch;
    }
    if (Ymap) NF_CUDA(gather_steps(ys, Ymap, yoff.data(), (int)m, batch * nL, sy));
    NF_CUDA(cudaEventRecord(net->h2d_ev[slot], net->h2d));            // slot filled
    NF_CUDA(cudaEventRecord(net->h2d_ev[4 + slot], ys));
    NF_CUDA(cudaStreamWaitEvent(net->stream, net->h2d_ev[slot], 0));
    NF_CUDA(cudaStreamWaitEvent(net->stream, net->h2d_ev[4 + slot], 0));
    int rc = train_steps_device(net, sx, sy, m * batch, batch, st, m, eta, step_loss ? step_loss + c0 : nullptr,
                                false);
    if (rc) return rc;
    NF_CUDA(cudaEventRecord(net->h2d_ev[2 + slot], net->stream));     // slot consumed
  }
  NF_CUDA(cudaStreamSynchronize(net->stream));
  return NF_OK;
}

int nf_grad_layers(nf_net *net, const float *x, const float *y, int64_t n, float *grad, void *const *events,
                   int32_t n_events) {
  if (int rc = check_net(net)) return rc;
  if (events && n_events != net->L) return fail(NF_EINVAL, "n_events %d != the %d layers", n_events, net->L);
  if (n <= 0) return fail(NF_EINVAL, "n must be >= 1");
  if (int rc = check_ptr(x, "x")) return rc;
  if (int rc = check_ptr(y, "y")) return rc;
  if (int rc = check_ptr(grad, "grad")) return rc;
  int rc;
  const float *dx = stage_in(net, x, (size_t)n * net->dims[0], net->stage_x, &rc);
  if (rc) return rc;
  const float *dy = stage_in(net, y, (size_t)n * net->dims[net->L], net->stage_y, &rc);
  if (rc) return rc;
  const bool host_out = !is_device_ptr(grad);
  float *dg = grad;
  if (host_out) {
    NF_CUDA(net->stage_g.ensure((size_t)net->nparams * sizeof(float)));
    dg = net->stage_g.as<float>();
  }
  if (net->math == NF_MATH_FP64) {
    NF_CUDA(net->grad64.ensure((size_t)net->nparams * sizeof(double)));
    if ((rc = ensure_ws64(net, n))) return rc;
    if ((rc = forward64(net, dx, dy, n, 0))) return rc;
    if ((rc = backward64(net, dx, n, 0.0, net->grad64.as<double>()))) return rc;
    NF_CUDA(f64_round(net->stream, net->grad64.as<double>(), dg, net->nparams));
  } else {
    if ((rc = ensure_ws(net, n))) return rc;
    if ((rc = ensure_tpose(net, dx, n))) return rc;
    if ((rc = forward(net, dx, dy, n, 0))) return rc;
    if ((rc = backward(net, dx, n, 0.0f, dg, nullptr, events && !host_out ? reinterpret_cast<cudaEvent_t const *>(events)
                                                                            : nullptr)))
      return rc;
  }
  if (events && (host_out || net->math == NF_MATH_FP64))  // no per-layer overlap there: all at the end
    for (int l = 0; l < net->L; ++l)
      if (events[l]) NF_CUDA(cudaEventRecord(static_cast<cudaEvent_t>(events[l]), net->stream));
  if (host_out) {
    NF_CUDA(cudaMemcpyAsync(grad, dg, (size_t)net->nparams * sizeof(float), cudaMemcpyDeviceToHost, net->stream));
    NF_CUDA(cudaStreamSynchronize(net->stream));
  }
  return NF_OK;
}

int nf_grad(nf_net *net, const float *x, const float *y, int64_t n, float *grad) {
  return nf_grad_layers(net, x, y, n, grad, nullptr, 0);
}

int nf_update(nf_net *net, const float *grad, int64_t count, float eta, int64_t n) {
  if (net && !net->presplit()) net->lo_ok = false;  // (outside the fp32 mode nothing keeps params_lo current)
  if (int rc = check_net(net)) return rc;
  if (int rc = check_ptr(grad, "grad")) return rc;
  if (count != net->nparams) return fail(NF_EINVAL, "count %lld != %lld", (long long)count, (long long)net->nparams);
  if (n <= 0) return fail(NF_EINVAL, "n must be >= 1");
  if (!std::isfinite(eta)) return fail(NF_EINVAL, "eta is not finite");
  int rc;
  const float *dg = stage_in(net, grad, (size_t)count, net->stage_g, &rc);
  if (rc) return rc;
  const double scale = (double)eta / (double)n;
  if (net->math == NF_MATH_FP64) NF_CUDA(f64_update(net->stream, net->params64, dg, count, scale));
  else NF_CUDA(sgd_update(net->stream, net->params, dg, count, (float)scale));
  net->shadow_ok = false;
  net->lo_ok = false;
  fused_small_invalidate(net->fused);
  if (dg != grad) NF_CUDA(cudaStreamSynchronize(net->stream));
  return NF_OK;
}

static int eval_loss_acc(nf_net *net, const float *x, const float *y, int64_t n, float *res2) {
  res2[0] = res2[1] = 0.0f;
  if (n == 0) return NF_OK;
  if (int rc = check_ptr(x, "x")) return rc;
  if (int rc = check_ptr(y, "y")) return rc;
  const int n0 = net->dims[0], nL = net->dims[net->L];
  int rc;
  const float *dx = stage_in(net, x, (size_t)n * n0, net->stage_x, &rc);
  if (rc) return rc;
  const float *dy = stage_in(net, y, (size_t)n * nL, net->stage_y, &rc);
  if (rc) return rc;
  const int64_t chunk = std::min<int64_t>(n, kEvalChunk);
  const bool f64 = net->math == NF_MATH_FP64;
  if ((rc = f64 ? ensure_ws64(net, chunk) : ensure_ws(net, chunk))) return rc;
  const int64_t nchunks = (n + chunk - 1) / chunk;
  NF_CUDA(net->red.ensure(red_bytes() + nchunks * 2 * sizeof(float)));
  float *res = reinterpret_cast<float *>(net->red.as<char>() + red_bytes());
  const bool fused_tc = !f64 && infer_tc_applicable(net->dims, dx) && getenv("NF_DISABLE_FUSED") == nullptr;
  const bool fused = !f64 && !fused_tc && infer_small_applicable(net->dims, dx) && getenv("NF_DISABLE_FUSED") == nullptr;
  if (fused_tc && (rc = ensure_wsplit(net))) return rc;
  for (int64_t c = 0; c < nchunks; ++c) {
    const int64_t r = c * chunk, m = std::min(chunk, n - r);
    if (f64) {
      if ((rc = forward64(net, dx + r * n0, nullptr, m, 2))) return rc;
      NF_CUDA(loss_acc64(net->stream, net->A64[net->L], dy + r * nL, m, nL, net->red.as<double2>(), res + 2 * c,
                         nullptr));
      continue;
    }
    if (fused_tc)
      NF_CUDA(infer_tc(net->stream, net->dims, net->act_h, net->act_o, net->params, net->params_t, net->params_lo,
                       dx + r * n0, m, net->A[net->L]));
    else if (fused) NF_CUDA(infer_small(net->stream, net->dims, net->act_h, net->act_o, net->params, dx + r * n0, m,
                                   net->A[net->L]));
    else if ((rc = forward(net, dx + r * n0, nullptr, m, 2))) return rc;
    NF_CUDA(loss_acc(net->stream, net->A[net->L], dy + r * nL, m, nL, net->red.as<double2>(), res + 2 * c, nullptr));
  }
  std::vector<float> h(2 * nchunks);
  NF_CUDA(cudaMemcpyAsync(h.data(), res, h.size() * sizeof(float), cudaMemcpyDeviceToHost, net->stream));
  NF_CUDA(cudaStreamSynchronize(net->stream));
  double l = 0, a = 0;
  for (int64_t c = 0; c < nchunks; ++c) {
    const int64_t m = std::min(chunk, n - c * chunk);
    l += (double)h[2 * c] * m;
    a += (double)h[2 * c + 1] * m;
  }
  res2[0] = (float)(l / n);
  res2[1] = (float)(a / n);
  return NF_OK;
}

int nf_loss(nf_net *net, const float *x, const float *y, int64_t n, float *loss) {
  if (int rc = check_net(net)) return rc;
  if (!loss) return fail(NF_EINVAL, "loss is NULL");
  if (n < 0) return fail(NF_EINVAL, "n < 0");
  float r[2];
  if (int rc = eval_loss_acc(net, x, y, n, r)) return rc;
  *loss = r[0];
  return NF_OK;
}

int nf_accuracy(nf_net *net, const float *x, const float *y, int64_t n, float *acc) {
  if (int rc = check_net(net)) return rc;
  if (!acc) return fail(NF_EINVAL, "acc is NULL");
  if (n < 0) return fail(NF_EINVAL, "n < 0");
  float r[2];
  if (int rc = eval_loss_acc(net, x, y, n, r)) return rc;
  *acc = r[1];
  return NF_OK;
}

}  // extern "C"
