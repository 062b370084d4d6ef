// infer_small.cu -- the paper's `output` for two-layer nets with narrow hidden
// and output layers (H, O <= 32; config 2's [784,30,10]): one kernel streams x once and
// writes a2 = sigma(W2 sigma(W1 x + b1) + b2) (Eq. 2) without any stash.
//
// Persistent CTAs (one per SM, 256 threads) walk 64-row tiles of x.  W1 is resident in
// shared memory k-major ([n0][32]); x is staged in 64-pixel chunks by cp.async (double
// buffered, 272-B padded rows: conflict-free float4 reads).  Z1 uses 4-row x 4-neuron
// register tiles with packed FFMA2; layer 2 is a thread-per-(row, output) pass.
#include <algorithm>

#include "infer_small.cuh"
#include "kernels.cuh"
#include "nf_common.cuh"

namespace nf {
namespace {

#ifndef NF_INFER_T
#define NF_INFER_T 256
#endif
#ifndef NF_INFER_S
#define NF_INFER_S 2
#endif
constexpr int kT = NF_INFER_T;                 // threads per tile group
#ifndef NF_INFER_G
#define NF_INFER_G 2
#endif
constexpr int kG = NF_INFER_G;  // independent tile groups per CTA (own ring, own named barrier):
                                // one group's barrier / staging bubbles overlap the other's work
constexpr int kKH = kT / 128;  // pixel parts of a chunk (tasks: 8 neuron groups x 16 row groups x kKH)
constexpr int kRows = 64;      // rows per tile
#ifndef NF_INFER_KC
#define NF_INFER_KC 64
#endif
constexpr int kKC = NF_INFER_KC;        // pixels per staged chunk
constexpr int kXs = kKC + 4;   // padded smem row (floats)
constexpr int kS = NF_INFER_S;  // x chunk ring depth (prefetch distance kS - 1 chunks, across tiles)

__device__ __forceinline__ void cp_async16(float *dst, const float *src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_wait_ring() { asm volatile("cp.async.wait_group %0;" ::"n"(kS - 1) : "memory"); }

__global__ void __launch_bounds__(kT * kG, 1)
infer_small_kernel(const float *__restrict__ X, int64_t n, int n0, int H, int O, int act_h, int act_o,
                   const float *__restrict__ params, float *__restrict__ out) {
  extern __shared__ __align__(16) float sm[];
  const int nchunk = (n0 + kKC - 1) / kKC;
  const int n0p = nchunk * kKC;
  float *W1t = sm;                        // [n0p][32]
  float *W2s = W1t + n0p * 32;            // [32][33]
  float *b1s = W2s + 32 * 33;             // [32]
  float *b2s = b1s + 32;                  // [32]
  const int grp = threadIdx.x / kT;      // this thread's tile group
  float *xs0 = b2s + 32;                  // kG x { kS x [kRows][kXs] ring, [kRows][33] a1s, parts }
  const int gstride = kS * kRows * kXs + kKH * kRows * 33;
  float *xs = xs0 + grp * gstride;        // kS x [kRows][kXs]
  float *a1s = xs + kS * kRows * kXs;     // [kRows][33]
  float *a1p = a1s + kRows * 33;          // (kKH - 1) x [kRows][33] partial Z1 of pixel parts 1..
  const int tid = threadIdx.x % kT;
  auto group_sync = [&]() {
    if (kG == 1) __syncthreads();
    else asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "r"(kT) : "memory");
  };
  const float *W1 = params, *b1 = params + (int64_t)H * n0, *W2 = b1 + H, *b2 = W2 + O * H;

  {  // W1 [H][n0] -> W1t [n0p][32]: a warp per 32-pixel block; coalesced row reads (lane =
     // pixel) into a padded 32 x 33 tile (in the not yet used x ring), then coalesced
     // transposed writes (lane = neuron), conflict-free on both sides
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;  // all groups' warps
    float *tile = xs0 + warp * 32 * 33;
    for (int k0 = warp * 32; k0 < n0p; k0 += (kT * kG / 32) * 32) {
      const int k = k0 + lane;
#pragma unroll 8
      for (int j = 0; j < 32; ++j) tile[j * 33 + lane] = (j < H && k < n0) ? W1[(int64_t)j * n0 + k] : 0.0f;
      __syncwarp();
#pragma unroll 8
      for (int kk = 0; kk < 32; ++kk) W1t[(k0 + kk) * 32 + lane] = tile[lane * 33 + kk];
      __syncwarp();
    }
  }
  __syncthreads();  // the x ring is reused below
  for (int i = threadIdx.x; i < 32 * 33; i += kT * kG) {
    const int o = i / 33, j = i % 33;
    W2s[i] = (o < O && j < H) ? W2[o * H + j] : 0.0f;
  }
  if (threadIdx.x < 32) {
    b1s[threadIdx.x] = threadIdx.x < H ? b1[threadIdx.x] : 0.0f;
    b2s[threadIdx.x] = threadIdx.x < O ? b2[threadIdx.x] : 0.0f;
  }

  // Z1 task (kT = 8 neuron groups x 16 row groups x kKH pixel parts): neurons 4 jg .. 4 jg + 3,
  // rows rgrp + 16 u (u < 4; interleaved so a warp's 4 row groups hit distinct banks)
  const int jg = tid & 7, rg = tid >> 3;
  const int rgrp = rg & 15, kh = rg >> 4;
  const int64_t ntiles = (n + kRows - 1) / kRows;

  // this group's stream of (tile, chunk) pairs: tiles first + k * nstream, k = 0, 1, ...
  const int64_t first = (int64_t)blockIdx.x * kG + grp, nstream = (int64_t)gridDim.x * kG;
  const int64_t my_tiles = ntiles > first ? (ntiles - 1 - first) / nstream + 1 : 0;
  const int64_t T = my_tiles * nchunk;
  // staging cursor (chunk, tile row, ring slot) advanced incrementally: no 64-bit divisions
  int s_c = 0, s_slot = 0;
  int64_t s_r0 = first * kRows, s_t = 0;
  auto stage = [&]() {  // stages the next (tile, chunk); always commits a group (uniform counting)
    if (s_t < T) {
      float *dst = xs + s_slot * kRows * kXs;
#pragma unroll
      for (int i = tid; i < kRows * (kKC / 4); i += kT) {
        const int r = i / (kKC / 4), q = i % (kKC / 4);  // (powers of two: shifts)
        const int k = s_c * kKC + q * 4;
        const int64_t row = s_r0 + r;
        float *d = dst + r * kXs + q * 4;
        if (row < n && k < n0) cp_async16(d, X + row * n0 + k);
        else *reinterpret_cast<float4 *>(d) = make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
    cp_commit();
    ++s_t;
    s_slot = s_slot + 1 == kS ? 0 : s_slot + 1;
    if (++s_c == nchunk) { s_c = 0; s_r0 += nstream * kRows; }
  };
  static_assert((kKC & (kKC - 1)) == 0, "kKC: a power of two");

  __syncthreads();  // parameters staged
  for (int t = 0; t < kS - 1; ++t) stage();
  float2 acc[4][2];
  int c = 0, slot = 0;
  int64_t r0 = first * kRows;
  for (int64_t t = 0; t < T; ++t) {
    if (c == 0) {
#pragma unroll
      for (int u = 0; u < 4; ++u) acc[u][0] = acc[u][1] = make_float2(0.f, 0.f);
    }
    stage();
    cp_wait_ring();   // chunk t has landed (this thread's copies)
    group_sync();  // ... and the group's
    {
      const float *xb = xs + slot * kRows * kXs + rgrp * kXs;
      const float *wb = W1t + (c * kKC) * 32 + jg * 4;
      const int q0 = kh * (kKC / 4 / kKH), q1 = q0 + kKC / 4 / kKH;  // this thread's part (float4 units)
#pragma unroll 2
      for (int q = q0; q < q1; ++q) {
        float4 xv[4], wv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) xv[u] = *reinterpret_cast<const float4 *>(xb + 16 * u * kXs + 4 * q);
#pragma unroll
        for (int v = 0; v < 4; ++v) wv[v] = *reinterpret_cast<const float4 *>(wb + (4 * q + v) * 32);
#pragma unroll
        for (int v = 0; v < 4; ++v) {  // pixel outer: 8 independent accumulators between the
#pragma unroll                          // dependent updates of each (FFMA2 latency hidden)
          for (int u = 0; u < 4; ++u) {
            const float xq = v == 0 ? xv[u].x : v == 1 ? xv[u].y : v == 2 ? xv[u].z : xv[u].w;
            ffma2(acc[u][0], xq, make_float2(wv[v].x, wv[v].y));
            ffma2(acc[u][1], xq, make_float2(wv[v].z, wv[v].w));
          }
        }
      }
    }
    if (c == nchunk - 1) {
      // combine the pixel parts through shared memory (in part order), then the activation
      if (kh >= 1) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          float *d = a1p + (kh - 1) * kRows * 33 + (rgrp + 16 * u) * 33 + jg * 4;
          d[0] = acc[u][0].x; d[1] = acc[u][0].y; d[2] = acc[u][1].x; d[3] = acc[u][1].y;
        }
      }
      group_sync();
      if (kh == 0) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          float *d = a1s + (rgrp + 16 * u) * 33 + jg * 4;
          float z[4] = {acc[u][0].x, acc[u][0].y, acc[u][1].x, acc[u][1].y};
#pragma unroll
          for (int part = 0; part < kKH - 1; ++part) {
            const float *e = a1p + part * kRows * 33 + (rgrp + 16 * u) * 33 + jg * 4;
            z[0] += e[0]; z[1] += e[1]; z[2] += e[2]; z[3] += e[3];
          }
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            const int j = jg * 4 + v;
            d[v] = j < H ? act_only(act_h, z[v] + b1s[j]) : 0.0f;
          }
        }
      }
      group_sync();
      // layer 2: thread per (row, output)
      for (int i = tid; i < kRows * O; i += kT) {
        const int r = i / O, o = i - r * O;
        if (r0 + r >= n) continue;
        const float *a = a1s + r * 33, *w = W2s + o * 33;
        float c0 = 0.f, c1 = 0.f;
        int j = 0;
        for (; j + 2 <= H; j += 2) {
          c0 = fmaf(w[j], a[j], c0);
          c1 = fmaf(w[j + 1], a[j + 1], c1);
        }
        if (j < H) c0 = fmaf(w[j], a[j], c0);
        out[(r0 + r) * O + o] = act_only(act_o, b2s[o] + (c0 + c1));
      }
    }
    group_sync();  // chunk t's buffer is refilled by stage(t + kS) next iteration
    slot = slot + 1 == kS ? 0 : slot + 1;
    if (++c == nchunk) { c = 0; r0 += nstream * kRows; }
  }
  cp_wait_ring();
}

}  // namespace

bool infer_small_applicable(const std::vector<int> &dims, const float *X) {
  return dims.size() == 3 && dims[1] <= 32 && dims[2] <= 32 && dims[0] % 4 == 0 &&
         (reinterpret_cast<uintptr_t>(X) & 15) == 0 && infer_small_smem(dims[0]) <= 227 * 1024;
}

size_t infer_small_smem(int n0) {
  const int n0p = (n0 + kKC - 1) / kKC * kKC;
  return sizeof(float) * ((size_t)n0p * 32 + 32 * 33 + 64 + (size_t)kG * (kS * kRows * kXs + kKH * kRows * 33));
}

cudaError_t infer_small(cudaStream_t st, const std::vector<int> &dims, int act_h, int act_o, const float *params,
                        const float *X, int64_t n, float *out) {
  {
    cudaError_t e = set_max_smem(reinterpret_cast<const void *>(infer_small_kernel), 227 * 1024);
    if (e != cudaSuccess) return e;
  }
  const int64_t ntiles = (n + kRows - 1) / kRows;
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((ntiles + kG - 1) / kG, 148));
  infer_small_kernel<<<blocks, kT * kG, infer_small_smem(dims[0]), st>>>(X, n, dims[0], dims[1], dims[2], act_h,
                                                                         act_o, params, out);
  count_launch();
  log_launch(reinterpret_cast<const void *>(infer_small_kernel), dim3(blocks), dim3(kT * kG), infer_small_smem(dims[0]));
  return cudaGetLastError();
}

}  // namespace nf
