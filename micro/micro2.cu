// micro2.cu -- grid-barrier variants and DSMEM push latency (design data for the
// persistent small-net kernel).  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

namespace cg = cooperative_groups;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

// v0: red.release + ld.acquire poll on the same word
__device__ __forceinline__ void bar_v0(unsigned *ctr, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
    unsigned v;
    do { asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory"); } while (v < target);
  }
  __syncthreads();
}
// v1: relaxed red + relaxed poll, fences outside
__device__ __forceinline__ void bar_v1(unsigned *ctr, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
    asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
    unsigned v;
    do { asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory"); } while (v < target);
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
  }
  __syncthreads();
}
// v2: relaxed, no fences at all (latency floor, not a correct barrier for data)
__device__ __forceinline__ void bar_v2(unsigned *ctr, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
    unsigned v;
    do { asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory"); } while (v < target);
  }
  __syncthreads();
}
// v3: arrive on counter, last arriver publishes generation flag on another line; others poll flag
__device__ __forceinline__ void bar_v3(unsigned *ctr, unsigned *flag, unsigned gen, unsigned n) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned old;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(ctr) : "memory");
    if (old == gen * n - 1) {
      asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flag), "r"(gen) : "memory");
    } else {
      unsigned v;
      do { asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory"); } while (v < gen);
    }
  }
  __syncthreads();
}
// v4: cluster barrier + one global arrive per cluster
__device__ __forceinline__ void bar_v4(unsigned *ctr, unsigned target) {
  cg::cluster_group cl = cg::this_cluster();
  cl.sync();
  if (cl.block_rank() == 0 && threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
    unsigned v;
    do { asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory"); } while (v < target);
  }
  cl.sync();
}
// v5: barrier.cluster.arrive.relaxed / wait split, measuring raw cluster barrier
__device__ __forceinline__ void clbar_raw() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__global__ void k_bar(int v, unsigned *ctr, int iters) {
  for (int i = 1; i <= iters; ++i) {
    if (v == 0) bar_v0(ctr, i * gridDim.x);
    else if (v == 1) bar_v1(ctr, i * gridDim.x);
    else if (v == 2) bar_v2(ctr, i * gridDim.x);
    else if (v == 3) bar_v3(ctr, ctr + 32, i, gridDim.x);
  }
}
__global__ void k_bar4(unsigned *ctr, int iters, int nclusters) {
  for (int i = 1; i <= iters; ++i) bar_v4(ctr, i * nclusters);
}
__global__ void k_clbar(int iters) {
  for (int i = 0; i < iters; ++i) clbar_raw();
}

// DSMEM push: every CTA pushes `bytes` to each peer with cp.async.bulk shared::cluster and a
// complete_tx mbarrier on the receiver; receivers wait on their own mbarrier.  Ping-pong by phase.
__global__ void k_push(int bytes, int iters, float *sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) unsigned long long mbar[2];
  cg::cluster_group cl = cg::this_cluster();
  const int C = cl.num_blocks(), r = cl.block_rank();
  unsigned char *src = sm;                 // bytes
  unsigned char *dst = sm + bytes;         // C * bytes (slot per sender)
  for (int i = threadIdx.x; i < bytes; i += blockDim.x) src[i] = (unsigned char)i;
  if (threadIdx.x == 0) {
    for (int b = 0; b < 2; ++b)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((unsigned)__cvta_generic_to_shared(&mbar[b])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cl.sync();
  for (int it = 0; it < iters; ++it) {
    const int b = it & 1;
    const unsigned phase = (it >> 1) & 1;
    if (threadIdx.x == 0) {
      // expect (C-1)*bytes on my barrier b
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(&mbar[b])),
                   "r"((unsigned)((C - 1) * bytes)) : "memory");
    }
    // make sure all peers armed before pushing (only first iteration matters in real code; here keep
    // it honest by pushing into barrier b which peers armed at this iteration start)
    __syncwarp();
    if (threadIdx.x < C && threadIdx.x != r) {
      const int p = threadIdx.x;
      unsigned ldst = (unsigned)__cvta_generic_to_shared(dst + r * bytes);
      unsigned lbar = (unsigned)__cvta_generic_to_shared(&mbar[b]);
      unsigned rdst, rbar;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rdst) : "r"(ldst), "r"(p));
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rbar) : "r"(lbar), "r"(p));
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(rdst), "r"((unsigned)__cvta_generic_to_shared(src)), "r"(bytes), "r"(rbar) : "memory");
    }
    // wait own barrier
    if (threadIdx.x == 0) {
      unsigned ok = 0;
      while (!ok)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(ok) : "r"((unsigned)__cvta_generic_to_shared(&mbar[b])), "r"(phase) : "memory");
    }
    __syncthreads();
  }
  cl.sync();
  if (dst[5] == 255 && sink) sink[0] = 1;
}

template <class F> float timeit(F f, int reps = 3) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  f(); CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(a); f(); cudaEventRecord(b); CK(cudaEventSynchronize(b));
    float ms; cudaEventElapsedTime(&ms, a, b); best = ms < best ? ms : best;
  }
  return best;
}

int main() {
  unsigned *ctr; CK(cudaMalloc(&ctr, 4096));
  float *sink; CK(cudaMalloc(&sink, 64));
  const int iters = 2000;
  for (int v = 0; v < 4; ++v)
    for (int blocks : {16, 74, 148}) {
      float ms = timeit([&] { cudaMemset(ctr, 0, 4096); k_bar<<<blocks, 128>>>(v, ctr, iters); });
      printf("BAR v%d blocks=%d: %.3f us\n", v, blocks, ms * 1e3 / iters);
    }
  CK(cudaFuncSetAttribute(k_bar4, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  CK(cudaFuncSetAttribute(k_clbar, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  for (int C : {2, 4, 8}) {
    int ncl = (C == 2 ? 74 : C == 4 ? 32 : 15);
    float ms = timeit([&] {
      cudaMemset(ctr, 0, 4096);
      cudaLaunchConfig_t cfg = {}; cfg.gridDim = dim3(C * ncl); cfg.blockDim = dim3(128);
      cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim = {(unsigned)C, 1, 1};
      cfg.attrs = at; cfg.numAttrs = 1;
      CK(cudaLaunchKernelEx(&cfg, k_bar4, ctr, iters, ncl)); });
    printf("BAR v4 (cluster %d x %d): %.3f us\n", C, ncl, ms * 1e3 / iters);
    ms = timeit([&] {
      cudaLaunchConfig_t cfg = {}; cfg.gridDim = dim3(C * ncl); cfg.blockDim = dim3(128);
      cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim = {(unsigned)C, 1, 1};
      cfg.attrs = at; cfg.numAttrs = 1;
      CK(cudaLaunchKernelEx(&cfg, k_clbar, iters)); });
    printf("CLUSTERBAR raw C=%d x %d: %.3f us\n", C, ncl, ms * 1e3 / iters);
  }
  CK(cudaFuncSetAttribute(k_push, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  CK(cudaFuncSetAttribute(k_push, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  for (int C : {2, 4, 8})
    for (int bytes : {1024, 4096, 16384}) {
      int ncl = (C == 2 ? 74 : C == 4 ? 32 : 15);
      float ms = timeit([&] {
        cudaLaunchConfig_t cfg = {}; cfg.gridDim = dim3(C * ncl); cfg.blockDim = dim3(128);
        cfg.dynamicSmemBytes = bytes * (C + 1);
        cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim = {(unsigned)C, 1, 1};
        cfg.attrs = at; cfg.numAttrs = 1;
        CK(cudaLaunchKernelEx(&cfg, k_push, bytes, iters, sink)); });
      printf("PUSH C=%d bytes/peer=%d: %.3f us/round\n", C, bytes, ms * 1e3 / iters);
    }
  CK(cudaDeviceSynchronize());
  printf("done\n");
}
