// fused_small.cu -- ONE persistent kernel running many SGD steps of a two-layer
// net with narrow hidden and output layers (H, O <= 32): configs 1 and 2
// ([3,5,2] and the paper's MNIST net [784,30,10]).
//
// Decomposition:
//   * G clusters x C CTAs, all co-resident (1 CTA per SM).  Cluster g owns rows
//     [r_g, r_{g+1}) of every minibatch (the paper's per-image batch shard,
//     P:511-516); CTA rank c owns input columns (pixels) [k_c, k_c + w_c) and
//     keeps that slice of W1 resident in shared memory for all steps.
//   * per step s:
//       0  TMA 2-D tile load of the NEXT step's x slice (one cp.async.bulk.tensor
//          per CTA, mbarrier completion) -- overlaps the whole step
//       1  partial Z1 over the pixel slice (fp32 FFMA, smem operands)
//       2  DSMEM push: each CTA bulk-copies the partial rows of every peer's owned
//          rows into that peer's shared memory (mbarrier complete_tx, no cluster
//          barrier); the owner sums the C partials in rank order, adds b1, applies
//          sigma / sigma' (Eq. 2), then layer 2, delta_2 = (a2-y) sigma'(z2)
//          and delta_1 = (W2^T delta_2) sigma'(z1) (backprop)
//       3  DSMEM push of the owned delta_1 rows to every peer, and of the W2/b1/b2
//          tendency partials to the rank that reduces them
//       4  dW1 slice = sum_rows delta_1 (x) x (fp32 FFMA); cp.reduce.async.bulk adds
//          it into an L2 accumulator: the paper's co_sum in-GPU
//       5  grid barrier; every CTA applies W -= (eta/B) G to its resident
//          parameters (reading R3) and zeroes the accumulator two steps ahead.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "fused_small.cuh"
#include "kernels.cuh"
#include "nf_common.cuh"
#include "sm100_ptx.cuh"

namespace nf {

static thread_local char g_fs_err[256] = "";

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kMaxC = 8;       // cluster size
constexpr int kMaxRows = 128;  // rows per cluster
constexpr int kProf = 16;      // profiler slots per step
constexpr int kRowsZ = 9;      // rows per warp per pass in the Z1 phase (72 rows per pass)
constexpr int GP = 32 * 32 + 64;  // W2 [32][32] + b1 [32] + b2 [32] tendency partial (padded)

struct FusedParams {
  int n0, H, O;          // dims
  int act_h, act_o;
  int B;                 // batch rows per step
  int G;                 // clusters
  int ws, wpad;          // pixel-slice stride and padded smem row length (floats)
  int aligned;           // 1: n0 % 4 == 0 -> 16-B aligned slices, TMA / bulk paths
  int nSmax, nOwnMax;    // max rows per cluster / per CTA
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
__host__ __device__ __forceinline__ int own_begin(int c, int nS, int C) { return (c * nS) / C; }
__host__ __device__ __forceinline__ int e_begin(int c, int C) { return 4 * (((GP / 4) * c) / C); }
__host__ __device__ __forceinline__ int e_slot(int C) { return ((GP / C + 4) + 3) & ~3; }  // 16-B multiple

__device__ __forceinline__ void cp_async4(float *dst, const float *src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(ptx::smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait0() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

struct Smem {
  // offsets in floats from the 128-B aligned base
  int W1t, W2s, b1s, b2s, xs, ys, Pfull, Pown, D1, gpart, grecv, Gs, Gt, wred, lsum, total;
};

__host__ __device__ inline int al32(int v) { return (v + 31) & ~31; }  // 128-B alignment in floats

__host__ __device__ inline Smem smem_layout(int wpad, int nSmax, int nOwnMax, int C) {
  Smem L;
  int o = 32;  // mbarriers live in the first 128 B
  L.W1t = o;   o = al32(o + wpad * 32);
  L.W2s = o;   o = al32(o + 32 * 33);
  L.b1s = o;   o += 32;
  L.b2s = o;   o = al32(o + 32);
  L.xs = o;    o = al32(o + 2 * al32(nSmax * wpad));  // TMA destinations: 128-B aligned
  L.ys = o;    o = al32(o + 2 * nOwnMax * 32);
  L.Pfull = o; o = al32(o + nSmax * 32);
  L.Pown = o;  o = al32(o + C * nOwnMax * 32);
  L.D1 = o;    o = al32(o + nSmax * 32);
  L.gpart = o; o = al32(o + GP);
  L.grecv = o; o = al32(o + C * e_slot(C));
  L.Gs = o;    o = al32(o + 32 * wpad);
  L.Gt = o;    o = al32(o + wpad * 33);
  L.wred = o;  o = al32(o + kWarps * GP);
  L.lsum = o;  o = al32(o + kWarps);
  L.total = o;
  return L;
}

__global__ void __launch_bounds__(kThreads, 1)
fused_small_kernel(const FusedParams p, const __grid_constant__ CUtensorMap tmX) {
  extern __shared__ __align__(128) float sm[];
  const int C = (int)ptx::cluster_size();
  const int rank = (int)ptx::cluster_rank();
  const int g = blockIdx.x / C;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n0 = p.n0, H = p.H, O = p.O;
  const int nCTA = gridDim.x;

  // pixel slice of this rank
  int k0, w;
  if (p.aligned) {
    k0 = rank * p.ws;
    w = min(p.ws, n0 - k0);
  } else {
    k0 = (int)(((int64_t)rank * n0) / C);
    w = (int)(((int64_t)(rank + 1) * n0) / C) - k0;
  }
  const int wpad = p.wpad;
  // rows of this cluster and the rows each rank owns inside them
  const int r0 = row_begin(g, p.B, p.G), nS = row_begin(g + 1, p.B, p.G) - r0;
  const int o0 = own_begin(rank, nS, C), nOwn = own_begin(rank + 1, nS, C) - o0;
  const int e0 = e_begin(rank, C), ne = e_begin(rank + 1, C) - e0;
  const int eslot = e_slot(C);

  const Smem L = smem_layout(wpad, p.nSmax, p.nOwnMax, C);
  const int xstride = al32(p.nSmax * wpad);
  uint64_t *bar_x = reinterpret_cast<uint64_t *>(sm);  // [2]
  uint64_t *bar_P = bar_x + 2;
  uint64_t *bar_D = bar_x + 3;
  float *W1t = sm + L.W1t, *W2s = sm + L.W2s, *b1s = sm + L.b1s, *b2s = sm + L.b2s;
  float *xs0 = sm + L.xs, *ys0 = sm + L.ys, *Pfull = sm + L.Pfull, *Pown = sm + L.Pown;
  float *D1 = sm + L.D1, *gpart = sm + L.gpart, *grecv = sm + L.grecv, *Gs = sm + L.Gs, *Gt = sm + L.Gt;
  float *wred = sm + L.wred, *lsum = sm + L.lsum;

  const int64_t oW1 = 0, ob1 = (int64_t)H * n0, oW2 = ob1 + H, ob2 = oW2 + (int64_t)O * H;
  const int64_t np = ob2 + O;
  const int64_t npad = (np + 3) & ~int64_t(3);  // accumulator stride (16-B aligned)

  // ---- one-time setup: zero smem, barriers, resident parameters
  for (int i = 32 + tid; i < L.total; i += kThreads) sm[i] = 0.0f;
  if (tid == 0) {
    ptx::mbar_init(&bar_x[0], 1);
    ptx::mbar_init(&bar_x[1], 1);
    ptx::mbar_init(bar_P, 1);
    ptx::mbar_init(bar_D, 1);
    ptx::fence_mbar_init();
    if (p.aligned) ptx::prefetch_tensormap(&tmX);
  }
  __syncthreads();
  for (int i = tid; i < w * 32; i += kThreads) {
    const int k = i >> 5, j = i & 31;
    if (j < H) W1t[i] = p.params[oW1 + (int64_t)j * n0 + k0 + k];
  }
  for (int i = tid; i < O * H; i += kThreads) W2s[(i / H) * 33 + i % H] = p.params[oW2 + i];
  for (int i = tid; i < H; i += kThreads) b1s[i] = p.params[ob1 + i];
  for (int i = tid; i < O; i += kThreads) b2s[i] = p.params[ob2 + i];
  ptx::cluster_sync();  // peers' barriers initialised before any push

  // bytes each exchange delivers to this CTA per step
  uint32_t bytesP = 0, bytesD = 0;
  for (int c = 0; c < C; ++c) {
    if (c == rank) continue;
    bytesP += nOwn * 128;
    bytesD += (own_begin(c + 1, nS, C) - own_begin(c, nS, C)) * 128 + ne * 4;
  }

  const uint32_t xbytes = (uint32_t)(p.nSmax * p.ws * 4);
  auto prefetch = [&](int64_t s) {
    const int buf = (int)(s & 1);
    const int64_t row0 = p.starts[s] + r0;
    float *xs = xs0 + buf * xstride;
    if (p.aligned) {
      if (tid == 0) {
        ptx::mbar_arrive_expect_tx(&bar_x[buf], xbytes);
        ptx::tma_load_2d(xs, &tmX, &bar_x[buf], k0, (int)row0);
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

  prefetch(0);

  for (int64_t s = 0; s < p.n_steps; ++s) {
    const int buf = (int)(s & 1);
    const uint32_t par = (uint32_t)(s & 1);
    const float *xs = xs0 + buf * xstride;
    const float *ys = ys0 + buf * p.nOwnMax * 32;
    float *accS = p.acc + (s % 3) * npad;
    PROF(0);
    if (tid == 0) {  // arm this step's DSMEM receive barriers
      ptx::mbar_arrive_expect_tx(bar_P, bytesP);
      ptx::mbar_arrive_expect_tx(bar_D, bytesD);
    }
    cp_async_wait0();
    if (p.aligned) ptx::mbar_wait(&bar_x[buf], (uint32_t)((s >> 1) & 1));
    __syncthreads();
    if (s + 1 < p.n_steps) prefetch(s + 1);
    PROF(1);

    // ---- 1. partial Z1: Pfull[i][j] = sum_{k<w} x[i][k] W1[j][k0+k]
    //      warp: 8-row chunks (rows warp + 8u), lane: j; 8 independent FMA chains per lane
    for (int rb = 0; rb * kWarps * kRowsZ < nS; ++rb) {
      const float *xr[kRowsZ];
      int rows[kRowsZ];
#pragma unroll
      for (int u = 0; u < kRowsZ; ++u) {
        rows[u] = warp + kWarps * (rb * kRowsZ + u);
        xr[u] = xs + (rows[u] < nS ? rows[u] : 0) * wpad;
      }
      float a[kRowsZ];
#pragma unroll
      for (int u = 0; u < kRowsZ; ++u) a[u] = 0.0f;
      for (int k = 0; k < wpad; k += 4) {
        const float w0 = W1t[(k + 0) * 32 + lane], w1 = W1t[(k + 1) * 32 + lane];
        const float w2 = W1t[(k + 2) * 32 + lane], w3 = W1t[(k + 3) * 32 + lane];
        float4 xv[kRowsZ];
#pragma unroll
        for (int u = 0; u < kRowsZ; ++u) xv[u] = *reinterpret_cast<const float4 *>(xr[u] + k);
#pragma unroll
        for (int u = 0; u < kRowsZ; ++u) {
          a[u] = fmaf(xv[u].x, w0, a[u]);
          a[u] = fmaf(xv[u].y, w1, a[u]);
          a[u] = fmaf(xv[u].z, w2, a[u]);
          a[u] = fmaf(xv[u].w, w3, a[u]);
        }
      }
#pragma unroll
      for (int u = 0; u < kRowsZ; ++u)
        if (rows[u] < nS) Pfull[rows[u] * 32 + lane] = a[u];
    }
    ptx::fence_proxy_async_smem();
    __syncthreads();
    PROF(2);
    // push the partial rows each peer owns into its Pown[rank] slot
    if (warp == 0 && lane < C && lane != rank) {
      const int c = lane;
      const int a0 = own_begin(c, nS, C), na = own_begin(c + 1, nS, C) - a0;
      if (na > 0)
        ptx::bulk_s2peer(Pown + rank * p.nOwnMax * 32, Pfull + a0 * 32, (uint32_t)(na * 128), bar_P, c);
    }
    ptx::mbar_wait(bar_P, par);
    PROF(3);

    // ---- 2. owned rows: reduce partials over the cluster, layer 1 epilogue, layer 2, deltas
    float g2acc[32];  // per-lane accumulators: lane j holds G2[o][j] for all o
#pragma unroll
    for (int o = 0; o < 32; ++o) g2acc[o] = 0.0f;
    float g1acc = 0.0f, gb2acc = 0.0f, lacc = 0.0f;
    for (int q = warp; q < nOwn; q += kWarps) {
      const int i = o0 + q;
      float z = b1s[lane];
#pragma unroll
      for (int c = 0; c < kMaxC; ++c)
        if (c < C) z += (c == rank) ? Pfull[i * 32 + lane] : Pown[(c * p.nOwnMax + q) * 32 + lane];
      if (q == 0) PROF(12);
      float a1, s1;
      act_fwd(p.act_h, z, a1, s1);
      if (lane >= H) { a1 = 0.0f; s1 = 0.0f; }
      // z2[o] at lane o: four interleaved partial chains over j
      const int orow = (lane < O ? lane : 0) * 33;
      float zp[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (j < H) zp[j & 3] = fmaf(W2s[orow + j], __shfl_sync(0xffffffffu, a1, j), zp[j & 3]);
      const float z2 = b2s[lane] + ((zp[0] + zp[1]) + (zp[2] + zp[3]));
      if (q == 0) PROF(13);
      float a2, s2;
      act_fwd(p.act_o, z2, a2, s2);
      const float yv = lane < O ? ys[q * 32 + lane] : 0.0f;
      const float diff = lane < O ? a2 - yv : 0.0f;
      const float d2 = diff * s2;
      lacc += diff * diff;
      // delta_1[j] = s1[j] * sum_o W2[o][j] d2[o];  G2[o][j] += d2[o] a1[j]
      float t0 = 0.0f, t1 = 0.0f;
#pragma unroll
      for (int o = 0; o < 32; ++o) {
        if (o < O) {
          const float d2o = __shfl_sync(0xffffffffu, d2, o);
          if (o & 1) t1 = fmaf(W2s[o * 33 + lane], d2o, t1);
          else t0 = fmaf(W2s[o * 33 + lane], d2o, t0);
          g2acc[o] = fmaf(d2o, a1, g2acc[o]);
        }
      }
      const float d1 = lane < H ? (t0 + t1) * s1 : 0.0f;
      D1[i * 32 + lane] = d1;
      if (q == 0) PROF(14);
      g1acc += d1;
      gb2acc += lane < O ? d2 : 0.0f;
    }
    PROF(15);
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
      ptx::red_add_f32(p.step_loss + s, 0.5f * l * p.inv_B);
    }
    ptx::fence_proxy_async_smem();
    __syncthreads();
    PROF(4);

    // ---- 3. push owned delta_1 rows to every peer; push tendency partial slices to their reducers
    if (warp == 0 && lane < C && lane != rank) {
      const int c = lane;
      if (nOwn > 0) ptx::bulk_s2peer(D1 + o0 * 32, D1 + o0 * 32, (uint32_t)(nOwn * 128), bar_D, c);
      const int ce0 = e_begin(c, C), cne = e_begin(c + 1, C) - ce0;
      if (cne > 0) ptx::bulk_s2peer(grecv + rank * eslot, gpart + ce0, (uint32_t)(cne * 4), bar_D, c);
    }
    ptx::mbar_wait(bar_D, par);
    PROF(5);
    // reduce my slice of the W2/b1/b2 tendencies over the cluster (rank order) -> L2
    for (int e = tid; e < ne; e += kThreads) {
      float v = 0.0f;
      for (int c = 0; c < C; ++c) v += (c == rank) ? gpart[e0 + e] : grecv[c * eslot + e];
      const int ee = e0 + e;
      int64_t dst = -1;
      if (ee < 1024) {
        const int o = ee >> 5, j = ee & 31;
        if (o < O && j < H) dst = oW2 + (int64_t)o * H + j;
      } else if (ee < 1056) {
        if (ee - 1024 < H) dst = ob1 + (ee - 1024);
      } else if (ee - 1056 < O) {
        dst = ob2 + (ee - 1056);
      }
      if (dst >= 0) ptx::red_add_f32(accS + dst, v);
    }
    PROF(6);

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
              *reinterpret_cast<float4 *>(Gs + lane * wpad + cc[u]) =
                  make_float4(a[4 * u + 0], a[4 * u + 1], a[4 * u + 2], a[4 * u + 3]);
        }
      }
    }
    ptx::fence_proxy_async_smem();
    __syncthreads();
    PROF(7);
    // co_sum: add this CTA's dW1 slice into the L2 accumulator
    if (p.aligned) {
      if (warp == 0) {
        if (lane < H) {
          ptx::fence_proxy_async_global();
          ptx::bulk_reduce_add_f32(accS + oW1 + (int64_t)lane * n0 + k0, Gs + lane * wpad, (uint32_t)(w * 4));
          ptx::bulk_commit();
          ptx::bulk_wait_all();
          ptx::fence_proxy_async_global();
        }
        __syncwarp();
      }
    } else {
      for (int j = warp; j < H; j += kWarps) {
        float *dst = accS + oW1 + (int64_t)j * n0 + k0;
        for (int k = lane; k < w; k += 32) ptx::red_add_f32(dst + k, Gs[j * wpad + k]);
      }
    }
    PROF(8);

    // ---- 5. grid barrier (the co_sum is complete), then the SGD update of the resident parameters
    ptx::grid_barrier(p.bar, (unsigned)((s + 1) * nCTA));
    PROF(9);
    // reduced dW1 slice rows (coalesced along k; 16 independent loads per lane) -> Gt[k][j]
    for (int tb = 0; tb * 128 < w; ++tb) {
      float v[4][4];
#pragma unroll
      for (int m = 0; m < 4; ++m)
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const int j = warp + kWarps * m, k = tb * 128 + lane + 32 * t;
          v[m][t] = (j < H && k < w) ? accS[oW1 + (int64_t)j * n0 + k0 + k] : 0.0f;  // L1 invalidated by the barrier
        }
#pragma unroll
      for (int m = 0; m < 4; ++m)
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const int j = warp + kWarps * m, k = tb * 128 + lane + 32 * t;
          if (j < H && k < w) Gt[k * 33 + j] = v[m][t];
        }
    }
    float gl[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int e = tid + u * kThreads;
      gl[u] = e < H + O * H + O ? accS[ob1 + e] : 0.0f;
    }
    __syncthreads();
    PROF(10);
    for (int i = tid; i < w * 32; i += kThreads) {
      const int k = i >> 5, j = i & 31;
      if (j < H) W1t[i] -= p.scale * Gt[k * 33 + j];
    }
    for (int e = tid; e < H + O * H + O; e += kThreads) {
      const float gsum = e < kThreads ? gl[0] : (e < 2 * kThreads ? gl[1] : accS[ob1 + e]);
      if (e < H) b1s[e] -= p.scale * gsum;
      else if (e < H + O * H) { const int f = e - H; W2s[(f / H) * 33 + f % H] -= p.scale * gsum; }
      else b2s[e - H - O * H] -= p.scale * gsum;
    }
    // zero the accumulator used two steps ahead (its readers finished before this barrier)
    {
      float *z = p.acc + ((s + 2) % 3) * npad;
      const int64_t bid = blockIdx.x;
      for (int64_t i = bid * kThreads + tid; i < np; i += (int64_t)nCTA * kThreads) z[i] = 0.0f;
    }
    __syncthreads();
    PROF(11);
  }
  cp_async_wait0();

  // ---- write the resident parameters back (W1 slice by every CTA of cluster 0; the rest by CTA 0)
  if (g == 0) {
    for (int i = tid; i < w * 32; i += kThreads) {
      const int k = i >> 5, j = i & 31;
      if (j < H) p.params[oW1 + (int64_t)j * n0 + k0 + k] = W1t[i];
    }
    if (rank == 0) {
      for (int i = tid; i < O * H; i += kThreads) p.params[oW2 + i] = W2s[(i / H) * 33 + i % H];
      for (int i = tid; i < H; i += kThreads) p.params[ob1 + i] = b1s[i];
      for (int i = tid; i < O; i += kThreads) p.params[ob2 + i] = b2s[i];
    }
  }
  ptx::cluster_sync();  // no CTA exits while a peer may still push into it
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
  if (env_int("NF_DISABLE_FUSED", 0)) return FUSED_NOT_APPLICABLE;
  if (dims.size() != 3) return FUSED_NOT_APPLICABLE;
  const int n0 = dims[0], H = dims[1], O = dims[2];
  if (H > 32 || O > 32 || batch > (int64_t)148 * kMaxRows) return FUSED_NOT_APPLICABLE;

  // cluster size: pixel slices of >= 32 columns, at most 8 CTAs
  int C = env_int("NF_FUSED_C", 0);
  if (C <= 0) {
    C = kMaxC;
    while (C > 1 && n0 / C < 32) C /= 2;
  }
  C = std::max(1, std::min(C, kMaxC));
  const bool aligned = (n0 % 4 == 0) && ((uintptr_t)X % 16 == 0) && env_int("NF_FUSED_NOTMA", 0) == 0;
  int ws, wpad;
  if (aligned) {
    ws = ((n0 + C - 1) / C + 3) / 4 * 4;
    while (C > 1 && (C - 1) * ws >= n0) { --C; ws = ((n0 + C - 1) / C + 3) / 4 * 4; }
    wpad = ws;
  } else {
    ws = (n0 + C - 1) / C;
    wpad = (ws + 3) / 4 * 4;
  }
  if (wpad > 256) return FUSED_NOT_APPLICABLE;  // TMA box limit / smem budget

  static bool attr_done = false;
  if (!attr_done) {
    cudaFuncSetAttribute(fused_small_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(fused_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    attr_done = true;
  }
  auto smem_for = [&](int G) {
    const int nSmax = (int)((batch + G - 1) / G);
    const int nOwnMax = (nSmax + C - 1) / C;
    return (size_t)smem_layout(wpad, nSmax, nOwnMax, C).total * sizeof(float);
  };
  // clusters: as many as co-reside at 1 CTA/SM, with <= kMaxRows rows per cluster
  int G = 0;
  {
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim = {(unsigned)C, 1, 1};
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cfg.blockDim = dim3(kThreads);
    const int maxG = env_int("NF_FUSED_G", 0);
    int want = maxG > 0 ? maxG : (int)std::max<int64_t>(1, std::min<int64_t>(batch / 16, 148 / C));
    for (int cand = want; cand >= 1; --cand) {
      if ((batch + cand - 1) / cand > kMaxRows) break;
      cfg.gridDim = dim3(cand * C);
      cfg.dynamicSmemBytes = smem_for(cand);
      if (cfg.dynamicSmemBytes > 227 * 1024) continue;
      int ncl = 0;
      if (cudaOccupancyMaxActiveClusters(&ncl, fused_small_kernel, &cfg) != cudaSuccess) {
        cudaGetLastError();
        continue;
      }
      if (ncl >= cand) { G = cand; break; }
    }
    if (G < 1) return FUSED_NOT_APPLICABLE;
  }
  const int nSmax = (int)((batch + G - 1) / G);
  const int nOwnMax = (nSmax + C - 1) / C;
  const size_t smem = smem_for(G);

  CUtensorMap tmX;
  memset(&tmX, 0, sizeof tmX);
  if (aligned && !encode_tmap_2d_f32(&tmX, X, (uint64_t)n0, (uint64_t)N, (uint64_t)n0 * 4, (uint32_t)ws,
                                     (uint32_t)nSmax, CU_TENSOR_MAP_SWIZZLE_NONE)) {
    snprintf(g_fs_err, sizeof g_fs_err, "cuTensorMapEncodeTiled failed (cols %d rows %lld box %dx%d)", n0,
             (long long)N, ws, nSmax);
    return -1;
  }

  const int64_t np = (int64_t)H * n0 + H + (int64_t)O * H + O;
  const int64_t npad = (np + 3) & ~int64_t(3);
  const size_t need = 3 * npad * sizeof(float) + 256 + n_steps * sizeof(int64_t);
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
  p.B = (int)batch; p.G = G; p.ws = ws; p.wpad = wpad; p.aligned = aligned ? 1 : 0;
  p.nSmax = nSmax; p.nOwnMax = nOwnMax;
  p.n_steps = n_steps;
  p.scale = (float)((double)eta / (double)batch);
  p.inv_B = (float)(1.0 / (double)batch);
  p.X = X; p.Y = Y; p.params = params;
  p.acc = reinterpret_cast<float *>(base);
  p.bar = reinterpret_cast<unsigned *>(base + 3 * npad * sizeof(float));
  int64_t *dstarts = reinterpret_cast<int64_t *>(base + 3 * npad * sizeof(float) + 256);
  p.starts = dstarts;
  p.step_loss = step_loss;
  static unsigned long long *prof_buf = nullptr;
  const bool prof = env_int("NF_FUSED_PROF", 0) != 0;
  if (prof) {
    if (!prof_buf) cudaMalloc(&prof_buf, sizeof(unsigned long long) * 148 * 64 * kProf);
    cudaMemsetAsync(prof_buf, 0, sizeof(unsigned long long) * 148 * 64 * kProf, st);
    p.prof = prof_buf;
  }

  cudaError_t e = cudaMemsetAsync(base, 0, 3 * npad * sizeof(float) + 256, st);
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
    e = cudaLaunchKernelEx(&cfg, fused_small_kernel, p, tmX);
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
    // slot order in time; CTA-local deltas between consecutive recorded slots
    const int order[16] = {0, 1, 2, 3, 12, 13, 14, 15, 4, 5, 6, 7, 8, 9, 10, 11};
    const int nslot = 16;
    double ph[kProf] = {0}, phmax[kProf] = {0};
    int cnt = 0;
    for (int s = 2; s + 1 < ns; ++s, ++cnt) {
      for (int i = 0; i < nslot; ++i) {
        double mx = 0, sum = 0;
        for (int b = 0; b < G * C; ++b) {
          const unsigned long long *t = &h[((size_t)b * 64 + s) * kProf];
          const unsigned long long a = t[order[i]];
          const unsigned long long nxt = i < nslot - 1 ? t[order[i + 1]] : h[((size_t)b * 64 + s + 1) * kProf];
          const double d = (a && nxt) ? (double)(nxt - a) : 0.0;
          sum += d; mx = std::max(mx, d);
        }
        ph[i] += sum / (G * C); phmax[i] += mx;
      }
    }
    fprintf(stderr, "[fused prof] C=%d G=%d nS<=%d ws=%d aligned=%d smem=%zu  phase ns (mean over CTAs / max):\n",
            C, G, nSmax, ws, (int)aligned, smem);
    const char *names[16] = {"wait_x+issue", "z1_partial", "push_P+wait", "row:z_sum", "row:z2", "row:delta",
                             "rows_rest", "owned_sums", "push_D+wait", "gpart_red", "dW1", "co_sum_red",
                             "grid_bar", "acc_loads", "update", "tail"};
    double tot = 0;
    for (int i = 0; i < nslot; ++i) {
      fprintf(stderr, "  %-14s %8.0f %8.0f\n", names[i], ph[i] / cnt, phmax[i] / cnt);
      tot += ph[i] / cnt;
    }
    fprintf(stderr, "  %-14s %8.0f\n", "step", tot);
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
