// hmma_gemm_test.cu -- standalone timing + check of gemm_hmma (the warp-MMA GEMM engine) at
// config 4's shapes: C[2048][256] = A[2048][256] W[256][256]^T (K-major / K-major), with a plain
// store epilogue, 1xTF32 and 3xTF32, against an fp64 reference.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_1902_06714_b200/csrc \
//   hmma_gemm_test.cu -o hmma_gemm_test
#include <cmath>
#include <cstdio>
#include <vector>

#include "gemm_hmma.cuh"

using namespace nf;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

struct EpiSt {
  float *C; int N;
  __device__ float load(int, int) const { return 0.0f; }
  __device__ void store(int m, int n, float v, float) const { C[(int64_t)m * N + n] = v; }
  __device__ void operator()(int m, int n, float v) const { store(m, n, v, 0.0f); }
};

__global__ void fill(float *x, int64_t n, uint32_t seed) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t h = (uint32_t)i * 2654435761u ^ seed;
    h ^= h >> 13; h *= 0x5bd1e995; h ^= h >> 15;
    x[i] = (h & 0xFFFFFF) / 16777216.0f * 2.0f - 1.0f;
  }
}

template <int SPLIT>
void run(int M, int N, int K, int dbg = 1) {
  float *A, *B, *C;
  CK(cudaMalloc(&A, (size_t)M * K * 4)); CK(cudaMalloc(&B, (size_t)N * K * 4)); CK(cudaMalloc(&C, (size_t)M * N * 4));
  fill<<<256, 256>>>(A, (int64_t)M * K, 1);
  fill<<<256, 256>>>(B, (int64_t)N * K, 2);
  GemmArgs g{M, N, K, A, K, B, K, N, K, nullptr};
  EpiSt epi{C, N};
  auto kern = gemm_hmma<true, true, SPLIT, EpiSt>;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, hm::SMEM));
  dim3 grid((N + 63) / 64, (M + 63) / 64, 1);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e9;
  for (int it = 0; it < 20; ++it) {
    cudaEventRecord(e0);
    kern<<<grid, 256, hm::SMEM>>>(g, epi, dbg);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    best = std::min(best, ms);
  }
  std::vector<float> hA((size_t)M * K), hB((size_t)N * K), hC((size_t)M * N);
  CK(cudaMemcpy(hA.data(), A, hA.size() * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(hB.data(), B, hB.size() * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(hC.data(), C, hC.size() * 4, cudaMemcpyDeviceToHost));
  double maxe = 0, maxr = 0;
  for (int m = 0; m < M; m += 37)
    for (int n = 0; n < N; ++n) {
      double s = 0;
      for (int k = 0; k < K; ++k) s += (double)hA[(size_t)m * K + k] * hB[(size_t)n * K + k];
      maxe = std::max(maxe, std::fabs(s - hC[(size_t)m * N + n]));
      maxr = std::max(maxr, std::fabs(s));
    }
  printf("dbg %d %dxTF32 %dx%dx%d: %.2f us (%.1f TF/s), max err %.2e rel %.2e\n", dbg, SPLIT, M, N, K, best * 1e3,
         2.0 * M * N * K / best / 1e9, maxe, maxe / maxr);
  cudaFree(A); cudaFree(B); cudaFree(C);
}

int main() {
  run<1>(2048, 256, 256);
  run<1>(2048, 256, 256, 3);
  run<1>(2048, 256, 256, 5);
  run<1>(2048, 256, 256, 7);
  run<1>(2048, 256, 256, 0);
  run<3>(2048, 256, 256);
  run<1>(2048, 256, 784);
  run<1>(4096, 1024, 1024);
  return 0;
}
