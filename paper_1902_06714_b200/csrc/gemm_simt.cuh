// gemm_simt.cuh -- fp32 FFMA tiled contraction with fused epilogues: the
// generic-width path of the three GEMM-shaped steps of the method
// (SURVEY 8(a) rows a1, a3, a4):
//   K1 forward     Z_l = A_{l-1} W_l^T (+b_l, sigma, stash)      A K-major, B K-major
//   K3 backward    D_l = (D_{l+1} W_{l+1}) .* sigma'(Z_l)        A K-major, B N-major
//   K4 gradient    G_l = D_l^T [A_{l-1} | 1]  (+ SGD epilogue)    A M-major, B N-major
// The bias gradient g_l = 1^T D_l rides along as an extra ones column of the
// B operand (n == nb_real), so one kernel yields dW and db (the paper's
// dw/db tendencies, summed over the batch = the co_sum).
//
// Tiles are staged through double-buffered shared memory (register prefetch
// of tile t+1 while tile t is consumed), each thread owns a TMxTN register
// micro-tile.  Optional split-K over gridDim.z writes partials that a second
// kernel sums in a fixed order (deterministic) before the same epilogue.
#pragma once
#include "nf_common.cuh"
#include "sm100_ptx.cuh"

namespace nf {

struct GemmArgs {
  int M, N, K;
  const float *A; int64_t lda;
  const float *B; int64_t ldb;
  int nb_real;        // B(k, n) = 1 for nb_real <= n < N (ones column for db)
  int kchunk;         // K range per blockIdx.z
  float *partial;     // non-null: write raw partials [z][M][N] instead of the epilogue
};

// ---- epilogues ------------------------------------------------------------
// Each epilogue is split into load(m, n) -> aux (the one global value the element update
// reads, 0 if none) and store(m, n, acc, aux), so that the tensor-core epilogue can issue
// all 32 loads of a tile column before any store (no load-after-store serialisation
// through possibly aliasing pointers).  operator() = store(load()).
//
// Forward: mode 0 hidden (A = sigma(z), S = sigma'(z)); mode 1 output layer in
// training (A = sigma(z), S = (sigma(z) - y) sigma'(z) = delta_L, S:150 /
// quadratic cost P:111); mode 2 inference (A = sigma(z) only).
// rnd (NF_MATH_TF32): the values this epilogue stores as the operand of a later tensor-core
// contraction -- a hidden layer's A, the output layer's delta_L in S -- are rounded to the
// nearest TF32 value (tf32_rn; the output layer's A, the net's output, never is).
// T (tensor-core path only, nullable): a transposed copy [n][ldT] of the value stored -- A for a
// hidden layer, delta_L for the output layer -- so that the weight-gradient contraction reads it
// K-major (the batch is that contraction's K).
struct EpiFwd {
  static constexpr bool kRed = false;
  static constexpr bool kHasT = true;
  const float *bias; float *A; float *S; const float *Y; int ld; int act; int mode; int rnd = 0;
  float *T = nullptr; int ldT = 0;
  // lo / hi (fp32 mode, pre-split 3xTF32 consumers, [rows][ld] like A): a hidden layer's A as the
  // RN split (hi = tf32_rn(A), lo = tf32_lo_rn(A)); the output layer's delta_L as the truncation
  // split (lo only: tf32_lo(delta_L))
  float *lo = nullptr;
  float *hi = nullptr;
  __device__ __forceinline__ float load(int m, int n) const {
    return mode == 1 ? Y[(int64_t)m * ld + n] : 0.0f;
  }
  __device__ __forceinline__ void store(int m, int n, float acc, float y) const {
    const float z = acc + bias[n];
    const int64_t i = (int64_t)m * ld + n;
    if (mode == 2) { const float a = act_only(act, z); A[i] = rnd ? tf32_rn(a) : a; return; }
    float a, s;
    act_fwd(act, z, a, s);
    A[i] = (rnd && mode == 0) ? tf32_rn(a) : a;
    const float sv = mode == 0 ? s : (rnd ? tf32_rn((a - y) * s) : (a - y) * s);
    S[i] = sv;
    if (lo) {
      if (mode == 0) { hi[i] = tf32_rn(a); lo[i] = tf32_lo_rn(a); }
      else lo[i] = tf32_lo(sv);
    }
  }
  __device__ __forceinline__ void operator()(int m, int n, float acc) const { store(m, n, acc, load(m, n)); }

  // Tensor-core epilogue strip: rows m0..m0+31 (valid while < mlim) of column n; value of
  // row r at v[33 r].  The activation and the mode are compile-time inside the strip (one
  // switch per strip), and each 8-row group evaluates its 8 activations unconditionally so the
  // eight dependent exp/rcp chains interleave; only the stores are predicated.
  // (v: the strip's accumulators; each is replaced by the value stored -- the input of the
  // transposed copy, see store_t)
  template <int K, int MODE, bool RND>
  __device__ __forceinline__ void strip_km(int m0, int mlim, int n, float *v) const {
    const float bn = bias[n];
    const int rows = min(32, mlim - m0);
#pragma unroll 1
    for (int r0 = 0; r0 < rows; r0 += 8) {
      float z[8], a[8], s[8], y[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) z[u] = v[33 * (r0 + u)] + bn;
      if (MODE == 1) {
#pragma unroll
        for (int u = 0; u < 8; ++u) y[u] = r0 + u < rows ? Y[(int64_t)(m0 + r0 + u) * ld + n] : 0.0f;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (MODE == 2) a[u] = act_only_t<K>(z[u]);
        else act_fwd_t<K>(z[u], a[u], s[u]);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (r0 + u < rows) {
          const int64_t i = (int64_t)(m0 + r0 + u) * ld + n;
          const float av = (RND && MODE != 1) ? tf32_rn(a[u]) : a[u];
          A[i] = av;
          if (MODE == 0) S[i] = s[u];
          if (MODE == 1) {
            const float d = RND ? tf32_rn((a[u] - y[u]) * s[u]) : (a[u] - y[u]) * s[u];
            S[i] = d;
            v[33 * (r0 + u)] = d;
            if (lo) lo[i] = tf32_lo(d);
          } else {
            v[33 * (r0 + u)] = av;
            if (MODE == 0 && lo) { hi[i] = tf32_rn(av); lo[i] = tf32_lo_rn(av); }
          }
        }
      }
    }
  }
  template <int K>
  __device__ __forceinline__ void strip_t(int m0, int mlim, int n, float *v) const {
    if (rnd) {
      if (mode == 0) strip_km<K, 0, true>(m0, mlim, n, v);
      else if (mode == 1) strip_km<K, 1, true>(m0, mlim, n, v);
      else strip_km<K, 2, true>(m0, mlim, n, v);
    } else {
      if (mode == 0) strip_km<K, 0, false>(m0, mlim, n, v);
      else if (mode == 1) strip_km<K, 1, false>(m0, mlim, n, v);
      else strip_km<K, 2, false>(m0, mlim, n, v);
    }
  }
  __device__ __forceinline__ void strip(int m0, int mlim, int n, float *v) const {
    switch (act) {
      case ACT_SIGMOID: strip_t<ACT_SIGMOID>(m0, mlim, n, v); break;
      case ACT_TANH: strip_t<ACT_TANH>(m0, mlim, n, v); break;
      case ACT_RELU: strip_t<ACT_RELU>(m0, mlim, n, v); break;
      case ACT_GAUSSIAN: strip_t<ACT_GAUSSIAN>(m0, mlim, n, v); break;
      default: strip_t<ACT_STEP>(m0, mlim, n, v); break;
    }
  }
};

// Generic strip for element-wise epilogues with one aux load: all loads first, then stores.
template <class E>
__device__ __forceinline__ void strip_generic(const E &e, int m0, int mlim, int n, const float *v) {
  float aux[32];
#pragma unroll
  for (int r = 0; r < 32; ++r) aux[r] = m0 + r < mlim ? e.load(m0 + r, n) : 0.0f;
#pragma unroll
  for (int r = 0; r < 32; ++r)
    if (m0 + r < mlim) e.store(m0 + r, n, v[33 * r], aux[r]);
}

// Backward: SD holds sigma'(Z_l) on entry and delta_l on exit.
// With bias != nullptr the epilogue also applies the SGD update of the layer's bias from the
// deltas it produces: b[n] -= bscale * sum_m delta[m][n] (its rows' share, an L2 reduction,
// reading R12) -- the bias column sum then needs no kernel of its own.
// rnd (NF_MATH_TF32): the stored delta (the next contractions' operand) is rounded to the
// nearest TF32 value; the fused bias sum uses the unrounded deltas.
struct EpiBwd {
  static constexpr bool kRed = false;
  static constexpr bool kHasT = true;
  float *SD; int ld;
  float *bias = nullptr; float bscale = 0.0f;
  int rnd = 0;
  float *T = nullptr; int ldT = 0;  // transposed copy of delta (tensor-core path), see EpiFwd
  float *lo = nullptr;              // tf32_lo of delta (pre-split 3xTF32 consumers), see EpiFwd
  __device__ __forceinline__ float load(int m, int n) const { return SD[(int64_t)m * ld + n]; }
  __device__ __forceinline__ void store(int m, int n, float acc, float s) const {
    const float d = rnd ? tf32_rn(acc * s) : acc * s;
    SD[(int64_t)m * ld + n] = d;
    if (lo) lo[(int64_t)m * ld + n] = tf32_lo(d);
  }
  __device__ __forceinline__ void operator()(int m, int n, float acc) const {
    const float d = acc * load(m, n);
    SD[(int64_t)m * ld + n] = rnd ? tf32_rn(d) : d;
    if (lo) lo[(int64_t)m * ld + n] = tf32_lo(d);
    if (bias) asm volatile("red.global.add.f32 [%0], %1;" ::"l"(bias + n), "f"(-bscale * d) : "memory");
  }
  __device__ __forceinline__ void strip(int m0, int mlim, int n, float *v) const {
    float aux[32];
#pragma unroll
    for (int r = 0; r < 32; ++r) aux[r] = m0 + r < mlim ? load(m0 + r, n) : 0.0f;
    float sum = 0.0f;
#pragma unroll
    for (int r = 0; r < 32; ++r)
      if (m0 + r < mlim) {
        const float d = v[33 * r] * aux[r];
        const float dr = rnd ? tf32_rn(d) : d;
        SD[(int64_t)(m0 + r) * ld + n] = dr;
        if (lo) lo[(int64_t)(m0 + r) * ld + n] = tf32_lo(dr);
        v[33 * r] = dr;
        sum += d;
      }
    if (bias) asm volatile("red.global.add.f32 [%0], %1;" ::"l"(bias + n), "f"(-bscale * sum) : "memory");
  }
};

// Gradient: store = 0 applies W -= scale*G, b -= scale*g (scale =
// eta/B, reading R3); store = 1 writes G, g (nf_grad).  Column n == nreal is the bias.
// Wt (NF_MATH_TF32, SGD only): the TF32 shadow of W (same layout) the next step's tensor-core
// contractions read; the update also stores tf32_rn(W') there.  (Split-K terms reduced into W
// in L2 cannot: the launcher re-rounds the layer's shadow after such a launch.)
struct EpiGrad {
  static constexpr bool kRed = true;   // the update is additive: split-K terms can go straight in
  static constexpr bool kHasT = false;
  float *W; float *b; int ldw; int nreal; float scale; int store_only;
  float *Wt = nullptr;
  float *T = nullptr; int ldT = 0;     // (unused)
  float *Wlo = nullptr;                // fp32 mode: tf32_lo_rn shadow of W (with Wt = its hi), see EpiFwd
  __device__ __forceinline__ float *at(int m, int n) const { return n < nreal ? W + (int64_t)m * ldw + n : b + m; }
  __device__ __forceinline__ float load(int m, int n) const { return store_only ? 0.0f : *at(m, n); }
  __device__ __forceinline__ void store(int m, int n, float acc, float w) const {
    if (store_only) { *at(m, n) = acc; return; }
    const float w2 = w - scale * acc;
    *at(m, n) = w2;
    if (Wt && n < nreal) Wt[(int64_t)m * ldw + n] = tf32_rn(w2);
    if (Wlo && n < nreal) Wlo[(int64_t)m * ldw + n] = tf32_lo_rn(w2);
  }
  // one split-K term of the update: W[m][n] += -scale * acc as an L2 reduction (red, no return)
  // (store_only: the term itself, into a zeroed tendency block)
  __device__ __forceinline__ void strip_red(int m0, int mlim, int n, const float *v) const {
    const int rows = min(32, mlim - m0);
    const float f = store_only ? 1.0f : -scale;
#pragma unroll 8
    for (int r = 0; r < rows; ++r)
      asm volatile("red.global.add.f32 [%0], %1;" ::"l"(at(m0 + r, n)), "f"(f * v[33 * r]) : "memory");
  }
  __device__ __forceinline__ void operator()(int m, int n, float acc) const { store(m, n, acc, load(m, n)); }
  __device__ __forceinline__ void strip(int m0, int mlim, int n, float *v) const {
    strip_generic(*this, m0, mlim, n, v);
  }
};

// ---- the kernel -------------------------------------------------------------
template <int BM, int BN, int BK, int TM, int TN, bool AK, bool BKM, class Epi>
__global__ void __launch_bounds__((BM / TM) * (BN / TN))
gemm_simt(GemmArgs g, Epi epi) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  constexpr int NT = (BM / TM) * (BN / TN);
  constexpr int APT = BM * BK / NT;
  constexpr int BPT = BN * BK / NT;
  static_assert(APT * NT == BM * BK && BPT * NT == BN * BK, "tile/thread mismatch");
  __shared__ __align__(16) float As[2][BK][BM + 4];
  __shared__ __align__(16) float Bs[2][BK][BN + 4];

  const int tid = threadIdx.x;
  const int tx = tid % (BN / TN), ty = tid / (BN / TN);
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int kbeg = blockIdx.z * g.kchunk;
  const int kend = min(g.K, kbeg + g.kchunk);
  const int nkt = (kend - kbeg + BK - 1) / BK;

  float ra[APT], rb[BPT];
  auto load = [&](int k0) {
#pragma unroll
    for (int i = 0; i < APT; ++i) {
      const int idx = tid + i * NT;
      const int mm = AK ? idx / BK : idx % BM;
      const int kk = AK ? idx % BK : idx / BM;
      const int m = m0 + mm, k = k0 + kk;
      ra[i] = (m < g.M && k < kend) ? __ldg(AK ? g.A + (int64_t)m * g.lda + k
                                               : g.A + (int64_t)k * g.lda + m) : 0.0f;
    }
#pragma unroll
    for (int i = 0; i < BPT; ++i) {
      const int idx = tid + i * NT;
      const int nn = BKM ? idx / BK : idx % BN;
      const int kk = BKM ? idx % BK : idx / BN;
      const int n = n0 + nn, k = k0 + kk;
      float v = 0.0f;
      if (k < kend && n < g.N)
        v = n < g.nb_real ? __ldg(BKM ? g.B + (int64_t)n * g.ldb + k : g.B + (int64_t)k * g.ldb + n)
                          : 1.0f;
      rb[i] = v;
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int i = 0; i < APT; ++i) {
      const int idx = tid + i * NT;
      const int mm = AK ? idx / BK : idx % BM;
      const int kk = AK ? idx % BK : idx / BM;
      As[buf][kk][mm] = ra[i];
    }
#pragma unroll
    for (int i = 0; i < BPT; ++i) {
      const int idx = tid + i * NT;
      const int nn = BKM ? idx / BK : idx % BN;
      const int kk = BKM ? idx % BK : idx / BN;
      Bs[buf][kk][nn] = rb[i];
    }
  };

  float acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = 0.0f;

  if (nkt > 0) {
    load(kbeg);
    store(0);
  }
  __syncthreads();
  for (int t = 0; t < nkt; ++t) {
    const int buf = t & 1;
    if (t + 1 < nkt) load(kbeg + (t + 1) * BK);
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float a[TM], b[TN];
#pragma unroll
      for (int i = 0; i < TM; ++i) a[i] = As[buf][kk][ty * TM + i];
#pragma unroll
      for (int j = 0; j < TN; ++j) b[j] = Bs[buf][kk][tx * TN + j];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    if (t + 1 < nkt) store(buf ^ 1);
    __syncthreads();
  }

#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int m = m0 + ty * TM + i;
    if (m >= g.M) continue;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int n = n0 + tx * TN + j;
      if (n >= g.N) continue;
      if (g.partial)
        g.partial[((int64_t)blockIdx.z * g.M + m) * g.N + n] = acc[i][j];
      else
        epi(m, n, acc[i][j]);
    }
  }
}

// Sum split-K partials in z order (deterministic) and apply the epilogue.
template <class Epi>
__global__ void __launch_bounds__(256)
splitk_epilogue(const float *__restrict__ partial, int splits, int M, int N, Epi epi) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  const int64_t MN = (int64_t)M * N;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < MN;
       i += (int64_t)gridDim.x * blockDim.x) {
    float s = 0.0f;
    int z = 0;
    for (; z + 4 <= splits; z += 4) {  // four loads in flight, summed in order z = 0, 1, ...
      const float v0 = partial[z * MN + i], v1 = partial[(z + 1) * MN + i];
      const float v2 = partial[(z + 2) * MN + i], v3 = partial[(z + 3) * MN + i];
      s += v0; s += v1; s += v2; s += v3;
    }
    for (; z < splits; ++z) s += partial[z * MN + i];
    epi((int)(i / N), (int)(i % N), s);
  }
}

}  // namespace nf
