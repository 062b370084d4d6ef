// fused_small.cu -- ONE persistent kernel running many SGD steps of a two-layer
// net with narrow hidden and output layers (H, O <= 32): configs 1 and 2
// ([3,5,2] and the paper's MNIST net [784,30,10]).
//
// Decomposition:
//   * G clusters x C CTAs.  Cluster g owns rows [r_g, r_{g+1}) of every
//     minibatch (the paper's per-image batch shard); CTA rank c of
//     a cluster owns input columns (pixels) [k_c, k_{c+1}) and keeps that
//     slice of W1 resident in shared memory for all steps.
//   * per step:
//       0  cp.async prefetch of the next step's x tile / y rows (overlaps the step)
//       1  partial Z1 over the pixel slice             (SIMT FFMA, smem operands)
//       2  cluster barrier; each CTA owns ~1/C of the cluster's rows and sums
//          the C partials over DSMEM (fixed rank order), adds b1 -> sigma, sigma'
//          (Eq. 2), then layer 2, delta_2 = (a2 - y) sigma'(z2) and
//          delta_1 = (W2^T delta_2) sigma'(z1) (backprop)
//       3  cluster barrier; all-gather delta_1 over DSMEM; cluster-reduce the
//          W2/b1/b2 tendency partials
//       4  dW1 slice = sum_rows delta_1 (x) x  (SIMT FFMA), red.add into an L2
//          accumulator: the paper's co_sum as an in-GPU reduction
//       5  grid barrier; every CTA applies W -= (eta/B) G to its resident
//          parameters (reading R3), zeroes the accumulator two steps ahead.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "fused_small.cuh"
#include "kernels.cuh"
#include "nf_common.cuh"

namespace cg = cooperative_groups;

namespace nf {

static thread_local char g_fs_err[256] = "";

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kMaxQ = 16;  // nS <= kWarps * kMaxQ = 128 rows per cluster
constexpr int kMaxC = 8;   // cluster size
constexpr int kProf = 16;  // profiler slots per step

struct FusedParams {
  int n0, H, O;          // dims
  int act_h, act_o;
  int B;                 // batch rows per step
  int G;                 // clusters
  int w, wpad;           // pixel-slice width per CTA (max over ranks), padded to 4
  int nSmax;             // max rows per cluster
  int nOwnMax;           // max owned rows per CTA
  int64_t n_steps;
  float scale;           // eta / B
  float inv_B;
  const float *X, *Y;
  const int64_t *starts; // device
  float *params;         // flat [W1 b1 W2 b2]
  float *acc;            // 3 x nparams accumulators (zeroed by the host)
  unsigned *bar;         // grid barrier counter (zeroed by the host)
  float *step_loss;      // nullable, zeroed by the host
  unsigned long long *prof;  // nullable: per-CTA per-step phase timestamps (NF_FUSED_PROF=1)
};

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define PROF(i) \
  if (p.prof && threadIdx.x == 0 && s < 64) p.prof[((int64_t)blockIdx.x * 64 + s) * kProf + (i)] = globaltimer()

__device__ __forceinline__ int row_begin(int g, int B, int G) { return (int)(((int64_t)g * B) / G); }

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__device__ __forceinline__ void grid_barrier(unsigned *ctr, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
    } while (v < target);
  }
  __syncthreads();
}

__device__ __forceinline__ void cp_async4(float *dst, const float *src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async8(float *dst, const float *src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait0() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

__device__ __forceinline__ void red_add(float *p, float v) {
  asm volatile("red.relaxed.gpu.global.add.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}

__global__ void __launch_bounds__(kThreads, 1) fused_small_kernel(const FusedParams p) {
  extern __shared__ __align__(16) float sm[];
  cg::cluster_group cl = cg::this_cluster();
  const int C = (int)cl.num_blocks();
  const int rank = (int)cl.block_rank();
  const int g = blockIdx.x / C;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n0 = p.n0, H = p.H, O = p.O;
  const int nCTA = gridDim.x;

  // pixel slice of this rank
  const int k0 = (int)(((int64_t)rank * n0) / C), k1 = (int)(((int64_t)(rank + 1) * n0) / C);
  const int w = k1 - k0, wpad = p.wpad;
  // rows of this cluster and the rows this CTA owns inside them
  const int r0 = row_begin(g, p.B, p.G), nS = row_begin(g + 1, p.B, p.G) - r0;
  const int o0 = (rank * nS) / C, o1 = ((rank + 1) * nS) / C, nOwn = o1 - o0;

  // ---- shared memory carve-up (floats)
  float *W1t = sm;                                  // [wpad][32]  W1[j][k0+k] at W1t[k*32+j]
  float *W2s = W1t + wpad * 32;                     // [32][33]    W2[o][j] (padded rows)
  float *b1s = W2s + 32 * 33;                       // [32]
  float *b2s = b1s + 32;                            // [32]
  float *xs0 = b2s + 32;                            // 2 x [nSmax][wpad]
  float *ys0 = xs0 + 2 * p.nSmax * wpad;            // 2 x [nOwnMax][32]
  float *P = ys0 + 2 * p.nOwnMax * 32;              // [nSmax][32] partial Z1
  float *D1 = P + p.nSmax * 32;                     // [nSmax][32] delta_1 of all cluster rows
  float *gpart = D1 + p.nSmax * 32;                 // [32*32 + 64]: G2[o][j], g1[j], g2[o]
  const int gsld = wpad + 1;                        // odd row stride: conflict-free row and column access
  float *Gs = gpart + 32 * 32 + 64;                 // [32][gsld] dW1 slice staging
  float *wred = Gs + 32 * gsld;                     // [kWarps][32*32+64] warp partials
  float *lsum = wred + kWarps * (32 * 32 + 64);     // [kWarps]
  const int GP = 32 * 32 + 64;

  // offsets in the flat parameter / accumulator vector
  const int64_t oW1 = 0, ob1 = (int64_t)H * n0, oW2 = ob1 + H, ob2 = oW2 + (int64_t)O * H;
  const int64_t np = ob2 + O;

  // ---- load resident parameters
  for (int i = tid; i < wpad * 32; i += kThreads) {
    const int k = i / 32, j = i % 32;
    W1t[i] = (j < H && k < w) ? p.params[oW1 + (int64_t)j * n0 + k0 + k] : 0.0f;
  }
  for (int i = tid; i < 32 * 33; i += kThreads) {
    const int o = i / 33, j = i % 33;
    W2s[i] = (o < O && j < H) ? p.params[oW2 + (int64_t)o * H + j] : 0.0f;
  }
  for (int i = tid; i < 32; i += kThreads) {
    b1s[i] = i < H ? p.params[ob1 + i] : 0.0f;
    b2s[i] = i < O ? p.params[ob2 + i] : 0.0f;
  }

  const bool vec8 = ((n0 & 1) == 0) && ((k0 & 1) == 0) && ((w & 1) == 0);
  auto prefetch = [&](int64_t s) {
    const int buf = (int)(s & 1);
    const int64_t row0 = p.starts[s] + r0;
    float *xs = xs0 + buf * p.nSmax * wpad;
    if (vec8) {
      for (int r = warp; r < nS; r += kWarps) {
        const float *src = p.X + (row0 + r) * n0 + k0;
        for (int c = lane * 2; c < w; c += 64) cp_async8(xs + r * wpad + c, src + c);
      }
    } else {
      for (int r = warp; r < nS; r += kWarps) {
        const float *src = p.X + (row0 + r) * n0 + k0;
        for (int c = lane; c < w; c += 32) cp_async4(xs + r * wpad + c, src + c);
      }
    }
    float *ys = ys0 + buf * p.nOwnMax * 32;
    for (int i = tid; i < nOwn * O; i += kThreads) {
      const int r = i / O, c = i % O;
      cp_async4(ys + r * 32 + c, p.Y + (row0 + o0 + r) * O + c);
    }
    cp_async_commit();
  };

  // zero the padding columns of both x buffers once (never written by the prefetch)
  for (int i = tid; i < 2 * p.nSmax * wpad; i += kThreads) xs0[i] = 0.0f;
  __syncthreads();
  prefetch(0);

  for (int64_t s = 0; s < p.n_steps; ++s) {
    const int buf = (int)(s & 1);
    const float *xs = xs0 + buf * p.nSmax * wpad;
    const float *ys = ys0 + buf * p.nOwnMax * 32;
    float *accS = p.acc + (s % 3) * np;
    PROF(0);
    if (s + 1 < p.n_steps) prefetch(s + 1);
    else cp_async_commit();
    PROF(1);
    cp_async_wait1();
    __syncthreads();
    PROF(2);

    // ---- 1. partial Z1: P[i][j] = sum_{k<w} x[i][k] W1[j][k0+k]
    //      warp: 8-row chunks (rows warp + 8u), lane: j; 8 independent FMA chains per lane
    for (int rb = 0; rb * kWarps * 8 < nS; ++rb) {
      const float *xr[8];
      int rows[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        rows[u] = warp + kWarps * (rb * 8 + u);
        xr[u] = xs + (rows[u] < nS ? rows[u] : 0) * wpad;
      }
      float a[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      for (int k = 0; k < wpad; k += 4) {
        const float w0 = W1t[(k + 0) * 32 + lane], w1 = W1t[(k + 1) * 32 + lane];
        const float w2 = W1t[(k + 2) * 32 + lane], w3 = W1t[(k + 3) * 32 + lane];
        float4 xv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) xv[u] = *reinterpret_cast<const float4 *>(xr[u] + k);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          a[u] = fmaf(xv[u].x, w0, a[u]);
          a[u] = fmaf(xv[u].y, w1, a[u]);
          a[u] = fmaf(xv[u].z, w2, a[u]);
          a[u] = fmaf(xv[u].w, w3, a[u]);
        }
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (rows[u] < nS) P[rows[u] * 32 + lane] = a[u];
    }
    PROF(3);
    cluster_sync_all();
    PROF(4);

    // ---- 2. owned rows: reduce partials over the cluster, layer 1 epilogue, layer 2, deltas
    float g2acc[32];  // per-lane accumulators: lane j holds G2[o][j] for all o
#pragma unroll
    for (int o = 0; o < 32; ++o) g2acc[o] = 0.0f;
    float g1acc = 0.0f, gb2acc = 0.0f, lacc = 0.0f;
    for (int q = warp; q < nOwn; q += kWarps) {
      const int i = o0 + q;
      float pv[kMaxC];
#pragma unroll
      for (int c = 0; c < kMaxC; ++c)   // all DSMEM loads in flight, then a fixed-order sum
        pv[c] = c < C ? cl.map_shared_rank(P, c)[i * 32 + lane] : 0.0f;
      float z = b1s[lane];
#pragma unroll
      for (int c = 0; c < kMaxC; ++c) z += pv[c];
      float a1, s1;
      act_fwd(p.act_h, z, a1, s1);
      if (lane >= H) { a1 = 0.0f; s1 = 0.0f; }
      // z2[o] at lane o
      float z2 = b2s[lane];
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (j < H) z2 = fmaf(W2s[lane * 33 + j], __shfl_sync(0xffffffffu, a1, j), z2);
      float a2, s2;
      act_fwd(p.act_o, z2, a2, s2);
      const float yv = lane < O ? ys[q * 32 + lane] : 0.0f;
      const float diff = lane < O ? a2 - yv : 0.0f;
      const float d2 = diff * s2;
      lacc += diff * diff;
      // delta_1[j] = s1[j] * sum_o W2[o][j] d2[o];  G2[o][j] += d2[o] a1[j]
      float t = 0.0f;
#pragma unroll
      for (int o = 0; o < 32; ++o) {
        if (o < O) {
          const float d2o = __shfl_sync(0xffffffffu, d2, o);
          t = fmaf(W2s[o * 33 + lane], d2o, t);
          g2acc[o] = fmaf(d2o, a1, g2acc[o]);
        }
      }
      const float d1 = lane < H ? t * s1 : 0.0f;
      D1[i * 32 + lane] = d1;
      g1acc += d1;
      gb2acc += lane < O ? d2 : 0.0f;
    }
    PROF(5);
    // warp partials -> smem
    {
      float *wr = wred + warp * GP;
#pragma unroll
      for (int o = 0; o < 32; ++o) wr[o * 32 + lane] = g2acc[o];
      wr[1024 + lane] = g1acc;
      wr[1056 + lane] = gb2acc;
      const float l = warp_sum(lacc);
      if (lane == 0) lsum[warp] = l;
    }
    __syncthreads();
    for (int i = tid; i < GP; i += kThreads) {
      float v = 0.0f;
#pragma unroll
      for (int ww = 0; ww < kWarps; ++ww) v += wred[ww * GP + i];
      gpart[i] = v;
    }
    if (tid == 0 && p.step_loss) {
      float l = 0.0f;
      for (int ww = 0; ww < kWarps; ++ww) l += lsum[ww];
      red_add(p.step_loss + s, 0.5f * l * p.inv_B);
    }
    PROF(6);
    cluster_sync_all();
    PROF(7);

    // ---- 3. all-gather delta_1 rows of the peers; cluster-reduce the layer-2/bias tendencies
    for (int base = 0; base < nS * 32; base += 8 * kThreads) {
      float v[8];
      int own[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int idx = base + u * kThreads + tid;
        own[u] = -1;
        v[u] = 0.0f;
        if (idx < nS * 32) {
          const int row = idx >> 5;
          int c = 0;
          while (c + 1 < C && ((c + 1) * nS) / C <= row) ++c;
          if (c != rank) { own[u] = c; v[u] = cl.map_shared_rank(D1, c)[idx]; }
        }
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (own[u] >= 0) D1[base + u * kThreads + tid] = v[u];
    }
    PROF(8);
    {
      const int e0 = (rank * GP) / C, e1 = ((rank + 1) * GP) / C;
      for (int e = e0 + tid; e < e1; e += kThreads) {
        float pv[kMaxC];
#pragma unroll
        for (int c = 0; c < kMaxC; ++c) pv[c] = c < C ? cl.map_shared_rank(gpart, c)[e] : 0.0f;
        float v = 0.0f;
#pragma unroll
        for (int c = 0; c < kMaxC; ++c) v += pv[c];
        int64_t dst = -1;
        if (e < 1024) {
          const int o = e / 32, j = e % 32;
          if (o < O && j < H) dst = oW2 + (int64_t)o * H + j;
        } else if (e < 1056) {
          if (e - 1024 < H) dst = ob1 + (e - 1024);
        } else if (e - 1056 < O) {
          dst = ob2 + (e - 1056);
        }
        if (dst >= 0) red_add(accS + dst, v);
      }
    }
    PROF(9);
    __syncthreads();

    PROF(10);
    // ---- 4. dW1 slice: Gs[j][k] = sum_{i<nS} D1[i][j] x[i][k]   (lane: j, warp: 16-column groups)
    {
      const int nchunk = wpad / 4;  // 4-column chunks
      for (int cb = warp * 4; cb < nchunk; cb += kWarps * 4) {
        int cc[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) cc[u] = (cb + u < nchunk ? cb + u : cb) * 4;
        float a[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) a[u] = 0.0f;
        for (int i = 0; i < nS; ++i) {
          const float d = D1[i * 32 + lane];
          const float *xr = xs + i * wpad;
          float4 xv[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) xv[u] = *reinterpret_cast<const float4 *>(xr + cc[u]);
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            a[4 * u + 0] = fmaf(d, xv[u].x, a[4 * u + 0]);
            a[4 * u + 1] = fmaf(d, xv[u].y, a[4 * u + 1]);
            a[4 * u + 2] = fmaf(d, xv[u].z, a[4 * u + 2]);
            a[4 * u + 3] = fmaf(d, xv[u].w, a[4 * u + 3]);
          }
        }
        if (lane < H) {
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (cb + u < nchunk)
#pragma unroll
              for (int e = 0; e < 4; ++e) Gs[lane * gsld + cc[u] + e] = a[4 * u + e];
        }
      }
    }
    __syncthreads();
    PROF(11);
    // co_sum: add this CTA's slice partial into the L2 accumulator (rows j, lanes along k)
    for (int j = warp; j < H; j += kWarps) {
      float *dst = accS + oW1 + (int64_t)j * n0 + k0;
      for (int k = lane; k < w; k += 32) red_add(dst + k, Gs[j * gsld + k]);
    }

    // ---- 5. grid barrier (the co_sum is complete), then the SGD update of the resident parameters
    PROF(12);
    grid_barrier(p.bar, (unsigned)((s + 1) * nCTA));
    PROF(13);
    // fetch the reduced slice rows (coalesced along k, all loads in flight) into Gs
    for (int j = warp; j < H; j += kWarps) {
      const float *src = accS + oW1 + (int64_t)j * n0 + k0;
      float v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int k = lane + 32 * u;
        v[u] = k < w ? __ldcg(src + k) : 0.0f;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int k = lane + 32 * u;
        if (k < w) Gs[j * gsld + k] = v[u];
      }
      for (int k = lane + 256; k < w; k += 32) Gs[j * gsld + k] = __ldcg(src + k);
    }
    float gl2 = 0.0f, gl3 = 0.0f;
    {
      const int e = tid;  // O*H + H + O <= 32*32 + 64 entries of W2/b1/b2 (flat layout order b1, W2, b2)
      if (e < H + O * H + O) gl2 = __ldcg(accS + ob1 + e);
      if (e + kThreads < H + O * H + O) gl3 = __ldcg(accS + ob1 + e + kThreads);
    }
    __syncthreads();
    PROF(14);
    for (int i = tid; i < w * 32; i += kThreads) {
      const int k = i >> 5, j = i & 31;
      if (j < H) W1t[i] -= p.scale * Gs[j * gsld + k];
    }
    for (int e = tid; e < H + O * H + O; e += kThreads) {
      const float gsum = e == tid ? gl2 : (e == tid + kThreads ? gl3 : __ldcg(accS + ob1 + e));
      if (e < H) b1s[e] -= p.scale * gsum;
      else if (e < H + O * H) { const int f = e - H; W2s[(f / H) * 33 + f % H] -= p.scale * gsum; }
      else b2s[e - H - O * H] -= p.scale * gsum;
    }
    PROF(15);
    // zero the accumulator used two steps ahead (its readers finished before this barrier)
    {
      float *z = p.acc + ((s + 2) % 3) * np;
      const int64_t bid = blockIdx.x;
      for (int64_t i = bid * kThreads + tid; i < np; i += (int64_t)nCTA * kThreads) z[i] = 0.0f;
    }
    __syncthreads();
  }
  cp_async_wait0();

  // ---- write the resident parameters back (W1 slice by every CTA of cluster 0; the rest by CTA 0)
  if (g == 0) {
    for (int i = tid; i < H * w; i += kThreads) {
      const int j = i / w, k = i % w;
      p.params[oW1 + (int64_t)j * n0 + k0 + k] = W1t[k * 32 + j];
    }
    if (rank == 0) {
      for (int i = tid; i < O * H; i += kThreads) p.params[oW2 + i] = W2s[(i / H) * 33 + i % H];
      for (int i = tid; i < H; i += kThreads) p.params[ob1 + i] = b1s[i];
      for (int i = tid; i < O; i += kThreads) p.params[ob2 + i] = b2s[i];
    }
  }
}

size_t smem_floats(int wpad, int nSmax, int nOwnMax) {
  return (size_t)wpad * 32 + 32 * 33 + 64 + 2 * (size_t)nSmax * wpad + 2 * (size_t)nOwnMax * 32 +
         2 * (size_t)nSmax * 32 + (32 * 32 + 64) + 32 * (size_t)(wpad + 1) + kWarps * (32 * 32 + 64) + kWarps + 8;
}

int env_int(const char *name, int dflt) {
  const char *v = getenv(name);
  return v ? atoi(v) : dflt;
}

}  // namespace

int fused_small_train_steps(FusedSmall &fs, cudaStream_t st, const std::vector<int> &dims, int act_h,
                            int act_o, float *params, const float *X, const float *Y, int64_t N,
                            int64_t batch, const int64_t *starts, int64_t n_steps, float eta,
                            float *step_loss) {
  (void)N;
  if (env_int("NF_DISABLE_FUSED", 0)) return FUSED_NOT_APPLICABLE;
  if (dims.size() != 3) return FUSED_NOT_APPLICABLE;
  const int n0 = dims[0], H = dims[1], O = dims[2];
  if (H > 32 || O > 32 || batch > 4096) return FUSED_NOT_APPLICABLE;

  // cluster size: pixel slices of >= 32 columns, at most 8 CTAs
  int C = env_int("NF_FUSED_C", 0);
  if (C <= 0) {
    C = 8;
    while (C > 1 && n0 / C < 32) C /= 2;
  }
  C = std::max(1, std::min(C, kMaxC));
  const int w = (n0 + C - 1) / C;
  const int wpad = (w + 3) / 4 * 4;
  // clusters: as many as co-reside (1 CTA per SM), rows per cluster <= 128
  auto smem_for = [&](int G) {
    const int nSmax = (int)((batch + G - 1) / G);
    const int nOwnMax = (nSmax + C - 1) / C;
    return smem_floats(wpad, nSmax, nOwnMax) * sizeof(float);
  };
  int maxG = env_int("NF_FUSED_G", 0);
  int G = 1;
  {
    static bool attr_done = false;
    if (!attr_done) {
      cudaFuncSetAttribute(fused_small_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      cudaFuncSetAttribute(fused_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
      attr_done = true;
    }
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim = {(unsigned)C, 1, 1};
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cfg.blockDim = dim3(kThreads);
    int want = maxG > 0 ? maxG : (int)std::max<int64_t>(1, std::min<int64_t>(batch / 16, 148 / C));
    for (G = want; G >= 1; --G) {
      cfg.gridDim = dim3(G * C);
      cfg.dynamicSmemBytes = smem_for(G);
      if (cfg.dynamicSmemBytes > 227 * 1024) continue;
      int ncl = 0;
      if (cudaOccupancyMaxActiveClusters(&ncl, fused_small_kernel, &cfg) != cudaSuccess) {
        cudaGetLastError();
        continue;
      }
      if (ncl >= G) break;
    }
    if (G < 1) return FUSED_NOT_APPLICABLE;
  }
  const int nSmax = (int)((batch + G - 1) / G);
  if (nSmax > kWarps * kMaxQ) return FUSED_NOT_APPLICABLE;
  const int nOwnMax = (nSmax + C - 1) / C;
  const size_t smem = smem_for(G);

  const int64_t np = (int64_t)H * n0 + H + (int64_t)O * H + O;
  const size_t need = 3 * np * sizeof(float) + 256 + n_steps * sizeof(int64_t);
  if (fs.ws_bytes < need) {
    if (fs.ws) cudaFree(fs.ws);
    fs.ws = nullptr;
    fs.ws_bytes = 0;
    if (cudaMalloc(&fs.ws, need) != cudaSuccess) {
      snprintf(g_fs_err, sizeof g_fs_err, "workspace allocation of %zu bytes failed", need);
      return -1;
    }
    fs.ws_bytes = need;
  }
  char *base = static_cast<char *>(fs.ws);
  FusedParams p{};
  p.n0 = n0; p.H = H; p.O = O; p.act_h = act_h; p.act_o = act_o;
  p.B = (int)batch; p.G = G; p.w = w; p.wpad = wpad; p.nSmax = nSmax; p.nOwnMax = nOwnMax;
  p.n_steps = n_steps;
  p.scale = (float)((double)eta / (double)batch);
  p.inv_B = (float)(1.0 / (double)batch);
  p.X = X; p.Y = Y; p.params = params;
  p.acc = reinterpret_cast<float *>(base);
  p.bar = reinterpret_cast<unsigned *>(base + 3 * np * sizeof(float));
  int64_t *dstarts = reinterpret_cast<int64_t *>(base + 3 * np * sizeof(float) + 256);
  p.starts = dstarts;
  p.step_loss = step_loss;
  static unsigned long long *prof_buf = nullptr;
  const bool prof = env_int("NF_FUSED_PROF", 0) != 0;
  if (prof) {
    if (!prof_buf) cudaMalloc(&prof_buf, sizeof(unsigned long long) * 148 * 64 * kProf);
    cudaMemsetAsync(prof_buf, 0, sizeof(unsigned long long) * 148 * 64 * kProf, st);
    p.prof = prof_buf;
  }

  cudaError_t e = cudaMemsetAsync(base, 0, 3 * np * sizeof(float) + 256, st);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(dstarts, starts, n_steps * sizeof(int64_t), cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess && step_loss) e = cudaMemsetAsync(step_loss, 0, n_steps * sizeof(float), st);
  if (e == cudaSuccess) {
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim = {(unsigned)C, 1, 1};
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cfg.gridDim = dim3(G * C);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    e = cudaLaunchKernelEx(&cfg, fused_small_kernel, p);
    count_launch();
  }
  if (e != cudaSuccess) {
    snprintf(g_fs_err, sizeof g_fs_err, "launch (C=%d G=%d smem=%zu): %s", C, G, smem, cudaGetErrorString(e));
    return -1;
  }
  if (prof) {
    std::vector<unsigned long long> h((size_t)G * C * 64 * kProf);
    cudaStreamSynchronize(st);
    cudaMemcpy(h.data(), prof_buf, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    const int ns = (int)std::min<int64_t>(n_steps, 64);
    double ph[kProf] = {0}, phmax[kProf] = {0};
    int cnt = 0;
    for (int s = 2; s + 1 < ns; ++s, ++cnt) {
      for (int i = 0; i < kProf; ++i) {
        double mx = 0, sum = 0;
        for (int b = 0; b < G * C; ++b) {
          const unsigned long long *t = &h[((size_t)b * 64 + s) * kProf];
          const unsigned long long nxt = i < kProf - 1 ? t[i + 1] : h[((size_t)b * 64 + s + 1) * kProf];
          const double d = (double)(nxt - t[i]);
          sum += d; mx = std::max(mx, d);
        }
        ph[i] += sum / (G * C); phmax[i] += mx;
      }
    }
    fprintf(stderr, "[fused prof] C=%d G=%d nS<=%d w=%d smem=%zu  phase ns (mean over CTAs / max):\n", C, G, nSmax, w, smem);
    const char *names[kProf] = {"prefetch_issue", "wait_x", "z1_partial", "csync1", "owned_rows", "owned_sum",
                                "csync2", "gather_d1", "gpart_red", "sync", "dW1", "red_dW1", "grid_bar",
                                "acc_loads", "update", "tail"};
    for (int i = 0; i < kProf; ++i) fprintf(stderr, "  %-14s %8.0f %8.0f\n", names[i], ph[i] / cnt, phmax[i] / cnt);
  }
  return 0;
}

void fused_small_release(FusedSmall &fs) {
  if (fs.ws) cudaFree(fs.ws);
  fs.ws = nullptr;
  fs.ws_bytes = 0;
}

void fused_small_invalidate(FusedSmall &fs) { fs.valid = false; }

const char *fused_small_error() { return g_fs_err; }

}  // namespace nf
