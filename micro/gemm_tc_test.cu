// gemm_tc_test.cu -- standalone check of the tcgen05 TF32 GEMM core (gemm_tc.cuh):
// correctness against an fp64 reference on the GPU, TF32 rounding behaviour, and
// throughput.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//   -I../paper_1902_06714_b200/csrc gemm_tc_test.cu ../paper_1902_06714_b200/csrc/tmap.cu -o gemm_tc_test
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "gemm_tc.cuh"

using namespace nf;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

struct EpiStore {
  float *C; int N;
  __device__ void operator()(int m, int n, const float (&v)[32]) const {
#pragma unroll
    for (int i = 0; i < 32; ++i)
      if (n + i < N) C[(int64_t)m * N + n + i] = v[i];
  }
};

__global__ void ref_gemm(const float *A, const float *B, double *C, int M, int N, int K) {
  int m = blockIdx.y * 16 + threadIdx.y, n = blockIdx.x * 16 + threadIdx.x;
  if (m >= M || n >= N) return;
  double s = 0;
  for (int k = 0; k < K; ++k) s += (double)A[(int64_t)m * K + k] * (double)B[(int64_t)n * K + k];
  C[(int64_t)m * N + n] = s;
}
__global__ void round_kernel(float *x, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] = tc::round_tf32(x[i]);
}
__global__ void fill(float *x, int64_t n, uint32_t seed) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t h = (uint32_t)i * 2654435761u ^ seed;
    h ^= h >> 13; h *= 0x5bd1e995; h ^= h >> 15;
    x[i] = ((h & 0xFFFFFF) / 16777216.0f) * 2.0f - 1.0f;
  }
}

template <int BN>
float run(const float *A, const float *B, float *C, int M, int N, int K, int reps) {
  CUtensorMap ta, tb;
  if (!encode_tmap_2d_f32(&ta, A, K, M, (uint64_t)K * 4, tc::BK, tc::BM, CU_TENSOR_MAP_SWIZZLE_128B) ||
      !encode_tmap_2d_f32(&tb, B, K, N, (uint64_t)K * 4, tc::BK, BN, CU_TENSOR_MAP_SWIZZLE_128B)) {
    printf("tensor map encode failed\n");
    exit(1);
  }
  auto kern = tc::gemm_tc_kernel<BN, EpiStore>;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, tc::Cfg<BN>::SMEM));
  dim3 grid((N + BN - 1) / BN, (M + tc::BM - 1) / tc::BM);
  EpiStore epi{C, N};
  kern<<<grid, tc::kThreads, tc::Cfg<BN>::SMEM>>>(ta, tb, M, N, K, epi);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) kern<<<grid, tc::kThreads, tc::Cfg<BN>::SMEM>>>(ta, tb, M, N, K, epi);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  return ms / reps;
}

template <int BN>
void check(int M, int N, int K, bool rnd) {
  float *A, *B, *C; double *R;
  CK(cudaMalloc(&A, (size_t)M * K * 4)); CK(cudaMalloc(&B, (size_t)N * K * 4));
  CK(cudaMalloc(&C, (size_t)M * N * 4)); CK(cudaMalloc(&R, (size_t)M * N * 8));
  fill<<<256, 256>>>(A, (int64_t)M * K, 1); fill<<<256, 256>>>(B, (int64_t)N * K, 2);
  if (rnd) { round_kernel<<<256, 256>>>(A, (int64_t)M * K); round_kernel<<<256, 256>>>(B, (int64_t)N * K); }
  run<BN>(A, B, C, M, N, K, 0);
  ref_gemm<<<dim3((N + 15) / 16, (M + 15) / 16), dim3(16, 16)>>>(A, B, R, M, N, K);
  CK(cudaDeviceSynchronize());
  std::vector<float> c((size_t)M * N); std::vector<double> r((size_t)M * N);
  CK(cudaMemcpy(c.data(), C, c.size() * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(r.data(), R, r.size() * 8, cudaMemcpyDeviceToHost));
  double mx = 0, me = 0, se = 0;
  for (size_t i = 0; i < c.size(); ++i) mx = std::max(mx, std::fabs(r[i]));
  for (size_t i = 0; i < c.size(); ++i) {
    double e = std::fabs(c[i] - r[i]) / std::max(std::fabs(r[i]), 0.1 * mx);
    me = std::max(me, e); se += std::fabs(c[i] - r[i]);
  }
  printf("CHECK BN=%d M=%d N=%d K=%d pre-rounded=%d: max rel err (tau=0.1) %.3e  mean abs err %.3e  (max|ref| %.2f)\n",
         BN, M, N, K, (int)rnd, me, se / c.size(), mx);
  cudaFree(A); cudaFree(B); cudaFree(C); cudaFree(R);
}

template <int BN>
void perf(int M, int N, int K) {
  float *A, *B, *C;
  CK(cudaMalloc(&A, (size_t)M * K * 4)); CK(cudaMalloc(&B, (size_t)N * K * 4)); CK(cudaMalloc(&C, (size_t)M * N * 4));
  fill<<<256, 256>>>(A, (int64_t)M * K, 1); fill<<<256, 256>>>(B, (int64_t)N * K, 2);
  float ms = run<BN>(A, B, C, M, N, K, 5);
  printf("PERF BN=%d M=%d N=%d K=%d: %.3f ms  %.1f TFLOP/s\n", BN, M, N, K, ms, 2.0 * M * N * K / ms / 1e9);
  cudaFree(A); cudaFree(B); cudaFree(C);
}

int main() {
  check<256>(256, 512, 64, false);
  check<256>(256, 512, 64, true);
  check<256>(300, 700, 200, false);
  check<256>(1000, 1024, 784, false);
  check<256>(1000, 1024, 784, true);
  check<128>(1000, 1000, 1000, false);
  check<256>(512, 4096, 4096, false);
  perf<256>(16384, 4096, 4096);
  perf<128>(16384, 4096, 4096);
  perf<256>(8192, 8192, 8192);
  printf("done\n");
}
