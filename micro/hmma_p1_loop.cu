// hmma_p1_loop.cu -- what limits K6's warp-MMA P1 loop (3xTF32 mma.sync m16n8k8 over 5 m-tiles,
// operands from shared memory, truncation split of x in registers)?  Variants:
//   0: the K6 loop (LDS.128 x per m-tile, split, 3 HMMA per k-step)
//   1: no split (x raw as hi and lo): ALU removed
//   2: no loads (x from registers, split each time)
//   3: only the HMMAs (no loads, no split)
//   4: 2 HMMAs per k-step instead of 3 (2-term scheme), with loads + split
// 16 warps per CTA, one CTA per SM, 148 CTAs.  Prints clk per loop and per HMMA per SMSP.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 hmma_p1_loop.cu -o hmma_p1_loop
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void hmma(float (&d)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}
__device__ __forceinline__ void split_trunc(float x, uint32_t &hi, uint32_t &lo) {
  hi = __float_as_uint(x);
  lo = __float_as_uint(x - __uint_as_float(hi & 0xffffe000u));
}

template <int V, int NMT>
__global__ void __launch_bounds__(512, 1) k(float *out, long long *clk, int iters) {
  __shared__ __align__(16) float xs[80 * 100 + 64];
  __shared__ __align__(16) float4 W[2 * 4 * 32 * 2];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, gg = lane >> 2, tt = lane & 3;
  for (int i = tid; i < 80 * 100 + 64; i += 512) xs[i] = 0.001f * (i % 97);
  for (int i = tid; i < 2 * 4 * 32 * 2; i += 512) W[i] = make_float4(0.01f * (i % 13), 0.02f, -0.01f, 0.03f);
  __syncthreads();
  const int nb = warp & 3;
  const int pr = (gg >> 1) + 4 * (gg & 1);
  float acc[NMT][4] = {};
  const float *xr = xs + pr * 100 + 4 * tt;
  float4 rx[NMT][2];
#pragma unroll
  for (int m = 0; m < NMT; ++m) rx[m][0] = rx[m][1] = make_float4(1.f + lane, 2.f, 3.f, 4.f);
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const int j = it % 7;
    const float4 wh = W[((j & 1) * 4 + nb) * 32 + lane], wl = W[256 + ((j & 1) * 4 + nb) * 32 + lane];
    float4 xa[NMT], xb[NMT];
#pragma unroll
    for (int m = 0; m < NMT; ++m) {
      if (V == 2 || V == 3) {
        xa[m] = rx[m][0]; xb[m] = rx[m][1];
      } else {
        xa[m] = *reinterpret_cast<const float4 *>(xr + 16 * m * 100 + 16 * j);
        xb[m] = *reinterpret_cast<const float4 *>(xr + (16 * m + 8) * 100 + 16 * j);
      }
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint32_t bh[2] = {__float_as_uint(h ? wh.z : wh.x), __float_as_uint(h ? wh.w : wh.y)};
      const uint32_t bl[2] = {__float_as_uint(h ? wl.z : wl.x), __float_as_uint(h ? wl.w : wl.y)};
      uint32_t ah[NMT][4], al[NMT][4];
#pragma unroll
      for (int m = 0; m < NMT; ++m) {
        const float v[4] = {h ? xa[m].z : xa[m].x, h ? xb[m].z : xb[m].x, h ? xa[m].w : xa[m].y, h ? xb[m].w : xb[m].y};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          if (V == 1 || V == 3) { ah[m][q] = __float_as_uint(v[q]); al[m][q] = __float_as_uint(v[q]); }
          else split_trunc(v[q], ah[m][q], al[m][q]);
        }
      }
#pragma unroll
      for (int m = 0; m < NMT; ++m) hmma(acc[m], al[m], bh);
      if (V != 4) {
#pragma unroll
        for (int m = 0; m < NMT; ++m) hmma(acc[m], ah[m], bl);
      }
#pragma unroll
      for (int m = 0; m < NMT; ++m) hmma(acc[m], ah[m], bh);
    }
  }
  long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int m = 0; m < NMT; ++m) s += acc[m][0] + acc[m][1] + acc[m][2] + acc[m][3];
  out[blockIdx.x * 512 + tid] = s;
  if (tid == 0) clk[blockIdx.x] = t1 - t0;
}

template <int V, int NMT>
void run(const char *name) {
  float *out;
  long long *clk;
  cudaMalloc(&out, 148 * 512 * 4);
  cudaMalloc(&clk, 148 * 8);
  const int iters = 700;
  k<V, NMT><<<148, 512>>>(out, clk, iters);
  k<V, NMT><<<148, 512>>>(out, clk, iters);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("%s\n", cudaGetErrorString(e)); return; }
  long long c;
  cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
  const int per = V == 4 ? 2 : 3;
  const double hmma_per_smsp = (double)iters * 2 * per * NMT * 4;  // 4 warps per SMSP
  printf("%-42s NMT=%d: %8lld clk, %.2f clk per HMMA per SMSP (floor 8)\n", name, NMT, c, c / hmma_per_smsp);
  cudaFree(out);
  cudaFree(clk);
}

int main() {
  run<0, 5>("K6 loop (LDS + split + 3 HMMA)");
  run<1, 5>("no split");
  run<2, 5>("no loads");
  run<3, 5>("HMMA only");
  run<4, 5>("2 HMMA per k-step (LDS + split)");
  run<0, 3>("K6 loop (LDS + split + 3 HMMA)");
  run<3, 3>("HMMA only");
  return 0;
}
