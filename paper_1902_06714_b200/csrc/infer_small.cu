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

constexpr int kT = 256;
constexpr int kRows = 64;      // rows per tile
constexpr int kKC = 64;        // pixels per staged chunk
constexpr int kXs = kKC + 4;   // padded smem row (floats)
constexpr int kS = 4;          // x chunk ring depth (prefetch distance 3 chunks, across tiles)

__device__ __forceinline__ void cp_async16(float *dst, const float *src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_wait_ring() { asm volatile("cp.async.wait_group %0;" ::"n"(kS - 1) : "memory"); }

__global__ void __launch_bounds__(kT, 1)
infer_small_kernel(const float *__restrict__ X, int64_t n, int n0, int H, int O, int act_h, int act_o,
                   const float *__restrict__ params, float *__restrict__ out) {
  extern __shared__ __align__(16) float sm[];
  const int nchunk = (n0 + kKC - 1) / kKC;
  const int n0p = nchunk * kKC;
  float *W1t = sm;                        // [n0p][32]
  float *W2s = W1t + n0p * 32;            // [32][33]
  float *b1s = W2s + 32 * 33;             // [32]
  float *b2s = b1s + 32;                  // [32]
  float *xs = b2s + 32;                   // kS x [kRows][kXs]
  float *a1s = xs + kS * kRows * kXs;     // [kRows][33]
  const int tid = threadIdx.x;
  const float *W1 = params, *b1 = params + (int64_t)H * n0, *W2 = b1 + H, *b2 = W2 + O * H;

  for (int i = tid; i < n0p * 32; i += kT) {
    const int k = i >> 5, j = i & 31;
    W1t[i] = (j < H && k < n0) ? W1[(int64_t)j * n0 + k] : 0.0f;
  }
  for (int i = tid; i < 32 * 33; i += kT) {
    const int o = i / 33, j = i % 33;
    W2s[i] = (o < O && j < H) ? W2[o * H + j] : 0.0f;
  }
  if (tid < 32) {
    b1s[tid] = tid < H ? b1[tid] : 0.0f;
    b2s[tid] = tid < O ? b2[tid] : 0.0f;
  }

  // Z1 task (256 = 8 neuron groups x 16 row groups x 2 pixel halves): neurons 4 jg .. 4 jg + 3,
  // rows rgrp + 16 u (u < 4; interleaved so a warp's 4 row groups hit distinct banks)
  const int jg = tid & 7, rg = tid >> 3;
  const int rgrp = rg & 15, kh = rg >> 4;
  const int64_t ntiles = (n + kRows - 1) / kRows;

  // this CTA's stream of (tile, chunk) pairs: t -> tile blockIdx.x + (t / nchunk) * gridDim.x
  const int64_t my_tiles = ntiles > blockIdx.x ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t T = my_tiles * nchunk;
  auto stage = [&](int64_t t) {  // always commits a group (empty past the end) for uniform counting
    if (t < T) {
      const int64_t tile = blockIdx.x + (t / nchunk) * (int64_t)gridDim.x;
      const int c = (int)(t % nchunk);
      const int64_t r0 = tile * kRows;
      float *dst = xs + (int)(t % kS) * kRows * kXs;
      for (int i = tid; i < kRows * (kKC / 4); i += kT) {
        const int r = i / (kKC / 4), q = i % (kKC / 4);
        const int k = c * kKC + q * 4;
        const int64_t row = r0 + r;
        float *d = dst + r * kXs + q * 4;
        if (row < n && k < n0) cp_async16(d, X + row * n0 + k);
        else *reinterpret_cast<float4 *>(d) = make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
    cp_commit();
  };

  __syncthreads();  // parameters staged
  for (int64_t t = 0; t < kS - 1; ++t) stage(t);
  float2 acc[4][2];
  for (int64_t t = 0; t < T; ++t) {
    const int c = (int)(t % nchunk);
    if (c == 0) {
#pragma unroll
      for (int u = 0; u < 4; ++u) acc[u][0] = acc[u][1] = make_float2(0.f, 0.f);
    }
    stage(t + kS - 1);
    cp_wait_ring();   // chunk t has landed (this thread's copies)
    __syncthreads();  // ... and everyone's
    {
      const float *xb = xs + (int)(t % kS) * kRows * kXs + rgrp * kXs;
      const float *wb = W1t + (c * kKC) * 32 + jg * 4;
      const int q0 = kh * (kKC / 8), q1 = q0 + kKC / 8;  // this thread's half of the chunk (float4 units)
#pragma unroll 2
      for (int q = q0; q < q1; ++q) {
        float4 xv[4], wv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) xv[u] = *reinterpret_cast<const float4 *>(xb + 16 * u * kXs + 4 * q);
#pragma unroll
        for (int v = 0; v < 4; ++v) wv[v] = *reinterpret_cast<const float4 *>(wb + (4 * q + v) * 32);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const float xq[4] = {xv[u].x, xv[u].y, xv[u].z, xv[u].w};
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            ffma2(acc[u][0], xq[v], make_float2(wv[v].x, wv[v].y));
            ffma2(acc[u][1], xq[v], make_float2(wv[v].z, wv[v].w));
          }
        }
      }
    }
    if (c == nchunk - 1) {
      const int64_t r0 = (blockIdx.x + (t / nchunk) * (int64_t)gridDim.x) * kRows;
      // combine the two pixel halves through shared memory, then the layer-1 activation
      if (kh == 1) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          float *d = a1s + (rgrp + 16 * u) * 33 + jg * 4;
          d[0] = acc[u][0].x; d[1] = acc[u][0].y; d[2] = acc[u][1].x; d[3] = acc[u][1].y;
        }
      }
      __syncthreads();
      if (kh == 0) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          float *d = a1s + (rgrp + 16 * u) * 33 + jg * 4;
          const float z[4] = {acc[u][0].x + d[0], acc[u][0].y + d[1], acc[u][1].x + d[2], acc[u][1].y + d[3]};
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            const int j = jg * 4 + v;
            d[v] = j < H ? act_only(act_h, z[v] + b1s[j]) : 0.0f;
          }
        }
      }
      __syncthreads();
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
    __syncthreads();  // chunk t's buffer is refilled by stage(t + kS) next iteration
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
  return sizeof(float) * ((size_t)n0p * 32 + 32 * 33 + 64 + kS * kRows * kXs + kRows * 33);
}

cudaError_t infer_small(cudaStream_t st, const std::vector<int> &dims, int act_h, int act_o, const float *params,
                        const float *X, int64_t n, float *out) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(infer_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    attr = true;
  }
  const int64_t ntiles = (n + kRows - 1) / kRows;
  const int blocks = (int)std::min<int64_t>(ntiles, 148);
  infer_small_kernel<<<blocks, kT, infer_small_smem(dims[0]), st>>>(X, n, dims[0], dims[1], dims[2], act_h, act_o,
                                                                    params, out);
  count_launch();
  return cudaGetLastError();
}

}  // namespace nf
