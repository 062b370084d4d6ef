// micro.cu -- microbenchmarks that decide the persistent small-net kernel's
// design: grid-barrier latency, L2 reduction
// throughput (red.global scalar / v4 / cp.reduce.async.bulk), DSMEM exchange
// and cluster-barrier latency, streaming HBM read bandwidth, co-resident
// cluster counts.  Standalone: nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

namespace cg = cooperative_groups;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

__device__ __forceinline__ void grid_bar(unsigned *ctr, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
    unsigned v;
    do { asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory"); } while (v < target);
  }
  __syncthreads();
}

__global__ void k_barrier(unsigned *ctr, int iters) {
  for (int i = 1; i <= iters; ++i) grid_bar(ctr, i * gridDim.x);
}

// mode 0: scalar red.add.f32, 1: red.global.add.v4.f32, 2: cp.reduce.async.bulk add.f32
__global__ void k_reduce(float *buf, unsigned *ctr, int nf, int groups, int iters, int mode) {
  extern __shared__ __align__(128) float sm[];
  for (int i = threadIdx.x; i < nf; i += blockDim.x) sm[i] = 1.0f;
  __syncthreads();
  float *dst = buf + (size_t)(blockIdx.x % groups) * nf;
  for (int it = 1; it <= iters; ++it) {
    if (mode == 0) {
      for (int i = threadIdx.x; i < nf; i += blockDim.x) atomicAdd(dst + i, sm[i]);
    } else if (mode == 1) {
      for (int i = threadIdx.x * 4; i < nf; i += blockDim.x * 4)
        asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(dst + i), "f"(sm[i]), "f"(sm[i + 1]),
                     "f"(sm[i + 2]), "f"(sm[i + 3]) : "memory");
    } else {
      if (threadIdx.x == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(dst),
                     "r"((unsigned)__cvta_generic_to_shared(sm)), "r"((unsigned)(nf * 4)) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
      }
    }
    grid_bar(ctr, it * gridDim.x);
  }
}

// DSMEM: every CTA of the cluster reads `per_peer` floats from each peer, then cluster barrier.
__global__ void k_dsmem(int per_peer, int iters, float *sink) {
  extern __shared__ __align__(128) float sm[];
  cg::cluster_group cl = cg::this_cluster();
  const int C = cl.num_blocks(), r = cl.block_rank();
  for (int i = threadIdx.x; i < per_peer * C; i += blockDim.x) sm[i] = i;
  cl.sync();
  float acc = 0;
  for (int it = 0; it < iters; ++it) {
    for (int p = 1; p < C; ++p) {
      const float *peer = cl.map_shared_rank(sm, (r + p) % C) + r * per_peer;
      for (int i = threadIdx.x; i < per_peer; i += blockDim.x) acc += peer[i];
    }
    cl.sync();
  }
  if (acc == -1.0f) sink[0] = acc;
}

__global__ void k_clbar(int iters) {
  cg::cluster_group cl = cg::this_cluster();
  for (int it = 0; it < iters; ++it) cl.sync();
}

__global__ void k_read(const float4 *__restrict__ p, size_t n4, float *sink) {
  float4 a = make_float4(0, 0, 0, 0);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
    float4 v = __ldcs(p + i);
    a.x += v.x; a.y += v.y; a.z += v.z; a.w += v.w;
  }
  if (a.x + a.y + a.z + a.w == -1.0f) sink[0] = 1;
}

static float time_kernel(void (*launch)(void *), void *arg, int reps = 3) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  launch(arg);
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    CK(cudaEventRecord(a));
    launch(arg);
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms; CK(cudaEventElapsedTime(&ms, a, b));
    best = ms < best ? ms : best;
  }
  return best;
}

struct BarArg { unsigned *ctr; int blocks, iters; };
struct RedArg { float *buf; unsigned *ctr; int blocks, nf, groups, iters, mode; };
struct DsArg { int C, clusters, per_peer, iters; float *sink; };

int main() {
  int dev = 0; CK(cudaSetDevice(dev));
  cudaDeviceProp pr; CK(cudaGetDeviceProperties(&pr, dev));
  printf("device %s SMs %d L2 %d MB smem/block optin %zu\n", pr.name, pr.multiProcessorCount,
         pr.l2CacheSize >> 20, pr.sharedMemPerBlockOptin);
  unsigned *ctr; CK(cudaMalloc(&ctr, 4096));
  float *sink; CK(cudaMalloc(&sink, 64));

  // --- co-resident clusters (1 CTA/SM forced by 120 KB smem)
  CK(cudaFuncSetAttribute(k_clbar, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  CK(cudaFuncSetAttribute(k_clbar, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  for (int C : {1, 2, 4, 6, 8, 10, 12, 14, 16}) {
    for (int smemkb : {200, 100}) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(C * 32); cfg.blockDim = dim3(256); cfg.dynamicSmemBytes = smemkb * 1024;
      cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim = {(unsigned)C, 1, 1};
      cfg.attrs = at; cfg.numAttrs = 1;
      int ncl = -1; cudaError_t e = cudaOccupancyMaxActiveClusters(&ncl, k_clbar, &cfg);
      printf("MAXCLUSTERS C=%d smem=%dKB -> %d clusters (%d CTAs) %s\n", C, smemkb, ncl, ncl * C, e ? cudaGetErrorString(e) : "");
      cudaGetLastError();
    }
  }

  // --- grid barrier latency
  for (int blocks : {37, 74, 144, 148}) {
    BarArg ba{ctr, blocks, 2000};
    float ms = time_kernel([](void *p) { auto a = (BarArg *)p; cudaMemset(a->ctr, 0, 4);
                             k_barrier<<<a->blocks, 128>>>(a->ctr, a->iters); }, &ba);
    printf("GRIDBAR blocks=%d: %.3f us/barrier\n", blocks, ms * 1e3 / ba.iters);
  }

  // --- L2 reductions + barrier
  float *buf; CK(cudaMalloc(&buf, 64 << 20)); CK(cudaMemset(buf, 0, 64 << 20));
  CK(cudaFuncSetAttribute(k_reduce, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  for (int mode : {0, 1, 2})
    for (auto p : std::vector<std::pair<int, int>>{{2940, 8}, {2940, 16}, {6272, 4}, {23860, 144}, {23860, 1}, {1680, 14}}) {
      RedArg ra{buf, ctr, 144, p.first, 144 / p.second, 200, mode};
      float ms = time_kernel([](void *q) { auto a = (RedArg *)q; cudaMemset(a->ctr, 0, 4);
                               k_reduce<<<a->blocks, 256, a->nf * 4>>>(a->buf, a->ctr, a->nf, a->groups, a->iters, a->mode); }, &ra);
      printf("REDUCE mode=%d floats/CTA=%d contention=%d (%.2f MB/step): %.3f us/step (incl. barrier)\n", mode,
             p.first, p.second, 144.0 * p.first * 4 / 1e6, ms * 1e3 / ra.iters);
    }

  // --- DSMEM exchange + cluster barrier
  CK(cudaFuncSetAttribute(k_dsmem, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  CK(cudaFuncSetAttribute(k_dsmem, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  for (int C : {4, 8, 16})
    for (int per : {0, 210, 840, 2048}) {
      DsArg da{C, 128 / C, per, 2000, sink};
      float ms = time_kernel([](void *q) { auto a = (DsArg *)q;
          cudaLaunchConfig_t cfg = {}; cfg.gridDim = dim3(a->C * a->clusters); cfg.blockDim = dim3(256);
          cfg.dynamicSmemBytes = std::max(a->per_peer * a->C * 4, 4096);
          cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim = {(unsigned)a->C, 1, 1};
          cfg.attrs = at; cfg.numAttrs = 1;
          cudaError_t e = cudaLaunchKernelEx(&cfg, k_dsmem, a->per_peer, a->iters, a->sink);
          if (e) printf("launch err %s\n", cudaGetErrorString(e)); }, &da);
      printf("DSMEM C=%d floats/peer=%d (%d B read/CTA): %.3f us/iter\n", C, per, per * (C - 1) * 4, ms * 1e3 / da.iters);
    }

  // --- HBM streaming read
  size_t bytes = size_t(4) << 30;
  float4 *big; CK(cudaMalloc(&big, bytes)); CK(cudaMemset(big, 0, bytes));
  for (int blocks : {148, 296, 592, 1184}) {
    struct RA { float4 *p; size_t n4; int blocks; float *sink; } rr{big, bytes / 16, blocks, sink};
    float ms = time_kernel([](void *q) { auto a = (RA *)q; k_read<<<a->blocks, 512>>>(a->p, a->n4, a->sink); }, &rr);
    printf("HBMREAD blocks=%d: %.1f GB/s\n", blocks, bytes / ms / 1e6);
  }
  CK(cudaDeviceSynchronize());
  printf("done\n");
  return 0;
}
