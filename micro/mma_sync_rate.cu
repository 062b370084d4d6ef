// mma_sync_rate.cu -- throughput and latency of the warp-level tensor-core MMA
// (mma.sync.aligned.m16n8k8 tf32, SASS HMMA) on sm_100a, for the small per-CTA contractions of
// the persistent small-net kernel (K6), where tcgen05's issue -> commit -> mbarrier round trip
// (~1.3-3 K cycles measured, micro/tc_atmem_test.cu) is longer than the whole contraction.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 mma_sync_rate.cu -o mma_sync_rate
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void mma_tf32(float (&d)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

// NACC independent accumulators per warp, ITER rounds
template <int NACC>
__global__ void k_rate(float *out, long long *clk, int iters) {
  uint32_t a[4], b[2];
  for (int i = 0; i < 4; ++i) a[i] = __float_as_uint(1.0f + threadIdx.x * 1e-3f + i);
  for (int i = 0; i < 2; ++i) b[i] = __float_as_uint(0.5f + i);
  float d[NACC][4] = {};
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < NACC; ++j) mma_tf32(d[j], a, b);
  }
  __syncthreads();
  const long long t1 = clock64();
  float s = 0;
  for (int j = 0; j < NACC; ++j) s += d[j][0] + d[j][1] + d[j][2] + d[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

template <int NACC>
void run(int warps, int blocks) {
  float *out;
  long long *clk;
  cudaMalloc(&out, blocks * warps * 32 * 4);
  cudaMalloc(&clk, blocks * 8);
  const int iters = 1024;
  k_rate<NACC><<<blocks, warps * 32>>>(out, clk, iters);
  k_rate<NACC><<<blocks, warps * 32>>>(out, clk, iters);
  cudaDeviceSynchronize();
  long long c;
  cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
  const double mmas = (double)iters * NACC * warps;
  printf("warps/SM %2d  acc/warp %d : %8lld clk  %.2f clk per mma per SM  -> %.0f MAC/clk/SM  (per-warp %.1f clk/mma)\n",
         warps, NACC, c, c / mmas, mmas * 1024 / c, (double)c / (iters * NACC));
  cudaFree(out);
  cudaFree(clk);
}

int main() {
  run<1>(1, 1);   // latency of a dependent chain
  run<2>(1, 1);
  run<4>(1, 1);
  run<8>(1, 1);
  run<4>(4, 148);
  run<4>(8, 148);
  run<4>(16, 148);
  run<8>(16, 148);
  return 0;
}
