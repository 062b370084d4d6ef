// tma_stream.cu -- how fast can 148 persistent CTAs stream config 2's x ([50000][784] fp32, 157 MB,
// rows 3136 B apart) into shared memory with TMA, as a function of the box shape and ring depth?
// (the inference kernel's input stage).  Reference: a plain coalesced LDG.128 read of the same bytes.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_1902_06714_b200/csrc \
//   tma_stream.cu ../paper_1902_06714_b200/csrc/tmap.cu -o tma_stream -lcuda
#include <cstdio>
#include <vector>

#include "sm100_ptx.cuh"

using namespace nf;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

constexpr int N = 50000, K = 784;

// every CTA streams rows [r0, r1) as tiles of TR rows; per tile, K-blocks of BC columns, each
// K-block as TR / BR boxes of {BC, BR}; S-deep ring; consumer warp frees a slot once it lands
template <int BC, int BR, int TR, int S>
__global__ void __launch_bounds__(64, 1) k_tma(const __grid_constant__ CUtensorMap tm, float *sink) {
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t *ring = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  constexpr int SB = TR * BC * 4;
  __shared__ uint64_t full[S], empty[S];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nblk = (N + 31) / 32;
  const int64_t r0 = (int64_t)blockIdx.x * nblk / gridDim.x * 32, r1 = min((int64_t)N, (int64_t)(blockIdx.x + 1) * nblk / gridDim.x * 32);
  const int ntiles = (int)((r1 - r0 + TR - 1) / TR), nkb = (K + BC - 1) / BC;
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) { ptx::mbar_init(&full[i], 1); ptx::mbar_init(&empty[i], 1); }
    ptx::fence_mbar_init();
  }
  __syncthreads();
  float acc = 0;
  if (warp == 0 && lane == 0) {
    int g = 0;
    for (int i = 0; i < ntiles; ++i)
      for (int kb = 0; kb < nkb; ++kb, ++g) {
        const int s = g % S;
        ptx::mbar_wait(&empty[s], ((g / S) & 1) ^ 1);
        ptx::mbar_arrive_expect_tx(&full[s], SB);
        for (int b = 0; b < TR / BR; ++b)
          ptx::tma_load_2d(ring + s * SB + b * BR * BC * 4, &tm, &full[s], kb * BC, (int)(r0 + (int64_t)i * TR + b * BR));
      }
  } else if (warp == 1) {
    int g = 0;
    for (int i = 0; i < ntiles; ++i)
      for (int kb = 0; kb < nkb; ++kb, ++g) {
        const int s = g % S;
        ptx::mbar_wait(&full[s], (g / S) & 1);
        acc += reinterpret_cast<const float *>(ring + s * SB)[lane];
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&empty[s]);
      }
  }
  if (acc == 12345.f) sink[threadIdx.x] = acc;
}

__global__ void k_ldg(const float4 *x, int64_t n4, float *sink) {
  float4 a = make_float4(0, 0, 0, 0);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    const float4 v = __ldcs(x + i);
    a.x += v.x; a.y += v.y; a.z += v.z; a.w += v.w;
  }
  if (a.x + a.y + a.z + a.w == 12345.f) sink[0] = a.x;
}

template <int BC, int BR, int TR, int S>
void run(const float *x, float *sink, float *flush, CUtensorMapSwizzle sw, const char *name) {
  CUtensorMap tm;
  if (!encode_tmap_2d_f32(&tm, x, K, N, K * 4, BC, BR, sw)) { printf("encode failed %s\n", name); return; }
  const int smem = TR * BC * 4 * S + 1024;
  CK(cudaFuncSetAttribute(k_tma<BC, BR, TR, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e9;
  for (int it = 0; it < 6; ++it) {
    CK(cudaMemset(flush, it, 256 << 20));  // evict x from L2
    cudaEventRecord(e0);
    k_tma<BC, BR, TR, S><<<148, 64, smem>>>(tm, sink);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (it) best = std::min(best, ms);
  }
  printf("%-44s box {%3d px, %3d rows} tile %3d rows, ring %2d x %6d B: %6.1f us  %5.0f GB/s\n", name, BC, BR, TR, S,
         TR * BC * 4, best * 1e3, (double)N * K * 4 / best / 1e6);
}

int main() {
  float *x, *sink, *flush;
  CK(cudaMalloc(&x, (size_t)N * K * 4));
  CK(cudaMalloc(&sink, 4096));
  CK(cudaMalloc(&flush, 256 << 20));
  CK(cudaMemset(x, 0, (size_t)N * K * 4));
  {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    float best = 1e9;
    for (int it = 0; it < 6; ++it) {
      CK(cudaMemset(flush, it, 256 << 20));
      cudaEventRecord(e0);
      k_ldg<<<148 * 4, 512>>>(reinterpret_cast<const float4 *>(x), (int64_t)N * K / 4, sink);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      if (it) best = std::min(best, ms);
    }
    printf("%-44s %6.1f us  %5.0f GB/s\n", "LDG.128 coalesced (592 x 512 threads)", best * 1e3, (double)N * K * 4 / best / 1e6);
  }
  run<32, 32, 128, 8>(x, sink, flush, CU_TENSOR_MAP_SWIZZLE_128B, "current: 4 boxes/K-block, SW128");
  run<32, 128, 128, 8>(x, sink, flush, CU_TENSOR_MAP_SWIZZLE_128B, "1 box of 128 rows, SW128");
  run<32, 128, 128, 12>(x, sink, flush, CU_TENSOR_MAP_SWIZZLE_128B, "1 box of 128 rows, SW128, deeper");
  run<32, 256, 256, 6>(x, sink, flush, CU_TENSOR_MAP_SWIZZLE_128B, "256-row tiles, SW128");
  run<64, 128, 128, 6>(x, sink, flush, CU_TENSOR_MAP_SWIZZLE_NONE, "64-px boxes, no swizzle");
  run<128, 64, 64, 6>(x, sink, flush, CU_TENSOR_MAP_SWIZZLE_NONE, "128-px boxes, no swizzle");
  run<196, 32, 32, 6>(x, sink, flush, CU_TENSOR_MAP_SWIZZLE_NONE, "196-px boxes (quarter rows), no swizzle");
  run<196, 64, 64, 4>(x, sink, flush, CU_TENSOR_MAP_SWIZZLE_NONE, "196-px boxes, 64 rows, no swizzle");
  run<32, 32, 32, 16>(x, sink, flush, CU_TENSOR_MAP_SWIZZLE_128B, "32-row tiles, SW128, 16 deep");
  return 0;
}
