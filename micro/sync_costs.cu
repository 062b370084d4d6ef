// sync_costs.cu -- per-operation latency of the synchronisation primitives K6 uses, measured
// with clock64 inside one CTA of 512 threads (8-CTA cluster launch): __syncthreads,
// fence.proxy.async.shared::cta (+ __syncthreads), a DSMEM bulk push to a peer + mbarrier wait,
// and an empty mbarrier arrive/wait round.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../paper_1902_06714_b200/csrc -o sync_costs sync_costs.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "sm100_ptx.cuh"

using namespace nf;

__global__ void __cluster_dims__(8, 1, 1) __launch_bounds__(512, 1) k(long long *out, int iters) {
  __shared__ __align__(128) float buf[2048];
  __shared__ __align__(8) uint64_t bar[2];
  const int tid = threadIdx.x;
  const uint32_t rank = ptx::cluster_rank();
  if (tid == 0) {
    ptx::mbar_init(&bar[0], 1);
    ptx::mbar_init(&bar[1], 1);
    ptx::fence_mbar_init();
  }
  for (int i = tid; i < 2048; i += 512) buf[i] = i;
  ptx::cluster_sync();
  long long t0, t1, t2, t3, t4;
  // 1. __syncthreads
  __syncthreads();
  t0 = clock64();
  for (int i = 0; i < iters; ++i) __syncthreads();
  t1 = clock64();
  // 2. fence.proxy.async + __syncthreads
  for (int i = 0; i < iters; ++i) {
    buf[tid] += 1.0f;
    ptx::fence_proxy_async_smem();
    __syncthreads();
  }
  t2 = clock64();
  // 3. DSMEM push round: rank r pushes 1 KB to rank r^1, both wait for their receipt
  for (int i = 0; i < iters; ++i) {
    if (tid == 0) ptx::mbar_arrive_expect_tx(&bar[0], 1024);
    __syncthreads();
    if (tid == 0) ptx::bulk_s2peer(buf + 1024, buf, 1024, &bar[0], rank ^ 1);
    ptx::mbar_wait(&bar[0], (uint32_t)(i & 1));
    __syncthreads();
  }
  t3 = clock64();
  // 4. local mbarrier arrive/wait round
  for (int i = 0; i < iters; ++i) {
    if (tid == 0) ptx::mbar_arrive(&bar[1]);
    ptx::mbar_wait(&bar[1], (uint32_t)(i & 1));
  }
  t4 = clock64();
  if (tid == 0 && blockIdx.x == 0) {
    out[0] = (t1 - t0) / iters;
    out[1] = (t2 - t1) / iters;
    out[2] = (t3 - t2) / iters;
    out[3] = (t4 - t3) / iters;
  }
  ptx::cluster_sync();
}

int main() {
  long long *d, h[4];
  cudaMalloc(&d, 4 * sizeof(long long));
  k<<<8, 512>>>(d, 200);
  cudaDeviceSynchronize();
  k<<<8, 512>>>(d, 200);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  printf("err=%s\n__syncthreads (512 thr)            %lld clk\nSTS + fence.proxy.async + syncthr  %lld clk\n"
         "DSMEM 1 KB push + mbar wait + 2 sync %lld clk\nlocal mbar arrive/wait              %lld clk\n",
         cudaGetErrorString(e), h[0], h[1], h[2], h[3]);
}
