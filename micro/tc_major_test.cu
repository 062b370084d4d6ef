// tc_major_test.cu -- standalone check of gemm_tc_kernel for the four operand-major
// combinations (K/MN x K/MN), 1xTF32 and 3xTF32, against an fp64 GPU reference.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_1902_06714_b200/csrc \
//   tc_major_test.cu ../paper_1902_06714_b200/csrc/tmap.cu -o tc_major_test -lcuda
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "gemm_tc.cuh"

using namespace nf;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

struct EpiStore {
  float *C; int N;
  __device__ void operator()(int m, int n, float v) const { C[(int64_t)m * N + n] = v; }
};

// A(m,k): amn ? A[k*M + m] : A[m*K + k];  B(n,k): bmn ? B[k*N + n] : B[n*K + k]
__global__ void ref_gemm(const float *A, const float *B, double *C, int M, int N, int K, int amn, int bmn) {
  int m = blockIdx.y * 16 + threadIdx.y, n = blockIdx.x * 16 + threadIdx.x;
  if (m >= M || n >= N) return;
  double s = 0;
  for (int k = 0; k < K; ++k) {
    const double a = amn ? A[(int64_t)k * M + m] : A[(int64_t)m * K + k];
    const double b = bmn ? B[(int64_t)k * N + n] : B[(int64_t)n * K + k];
    s += a * b;
  }
  C[(int64_t)m * N + n] = s;
}
__global__ void fill(float *x, int64_t n, uint32_t seed) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t h = (uint32_t)i * 2654435761u ^ seed;
    h ^= h >> 13; h *= 0x5bd1e995; h ^= h >> 15;
    x[i] = ((h & 0xFFFFFF) / 16777216.0f) * 2.0f - 1.0f;
  }
}

bool map(CUtensorMap *m, const float *p, int rows, int K, bool mn, int box_rows) {
  if (mn) return encode_tmap_2d_f32(m, p, rows, K, (uint64_t)rows * 4, 32, tc::BK, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
  return encode_tmap_2d_f32(m, p, K, rows, (uint64_t)K * 4, tc::BK, box_rows, CU_TENSOR_MAP_SWIZZLE_128B);
}

template <int BN, bool AMN, bool BMN, int SPLIT>
void check(int M, int N, int K) {
  float *A, *B, *C; double *R;
  CK(cudaMalloc(&A, (size_t)M * K * 4)); CK(cudaMalloc(&B, (size_t)N * K * 4));
  CK(cudaMalloc(&C, (size_t)M * N * 4)); CK(cudaMalloc(&R, (size_t)M * N * 8));
  fill<<<256, 256>>>(A, (int64_t)M * K, 1); fill<<<256, 256>>>(B, (int64_t)N * K, 2);
  CK(cudaMemset(C, 0, (size_t)M * N * 4));
  CUtensorMap ta, tb;
  if (!map(&ta, A, M, K, AMN, tc::BM) || !map(&tb, B, N, K, BMN, BN)) { printf("map failed\n"); exit(1); }
  using Cf = tc::Cfg<BN, SPLIT>;
  auto kern = tc::gemm_tc_kernel<BN, AMN, BMN, SPLIT, EpiStore>;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cf::SMEM));
  tc::TileArgs g{M, N, K, ((K + 31) / 32) * 32, nullptr};
  kern<<<dim3((N + BN - 1) / BN, (M + tc::BM - 1) / tc::BM, 1), tc::kThreads, Cf::SMEM>>>(ta, tb, g, EpiStore{C, N});
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  ref_gemm<<<dim3((N + 15) / 16, (M + 15) / 16), dim3(16, 16)>>>(A, B, R, M, N, K, AMN, BMN);
  CK(cudaDeviceSynchronize());
  std::vector<float> c((size_t)M * N); std::vector<double> r((size_t)M * N);
  CK(cudaMemcpy(c.data(), C, c.size() * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(r.data(), R, r.size() * 8, cudaMemcpyDeviceToHost));
  double mx = 0, me = 0;
  int bad = 0;
  for (size_t i = 0; i < c.size(); ++i) mx = std::max(mx, std::fabs(r[i]));
  for (size_t i = 0; i < c.size(); ++i) {
    double e = std::fabs(c[i] - r[i]) / std::max(std::fabs(r[i]), 0.1 * mx);
    if (e > 1e-2 && bad < 6) {
      printf("   bad m=%zu n=%zu got %.5f ref %.5f\n", i / N, i % N, c[i], r[i]);
      ++bad;
    }
    me = std::max(me, e);
  }
  size_t zeros = 0;
  for (size_t i = 0; i < c.size(); ++i) zeros += (c[i] == 0.0f);
  printf("   zeros %zu of %zu; c[0..3] %.4f %.4f %.4f %.4f\n", zeros, c.size(), c[0], c[1], c[2], c[3]);
  printf("CHECK BN=%d AMN=%d BMN=%d SPLIT=%d M=%d N=%d K=%d: max rel err (tau=0.1) %.3e\n", BN, (int)AMN, (int)BMN,
         SPLIT, M, N, K, me);
  // find a transposition pattern: compare c[m][n] with r of other index
  cudaFree(A); cudaFree(B); cudaFree(C); cudaFree(R);
}

int main() {
  check<128, false, false, 1>(256, 256, 64);
  check<128, false, true, 1>(256, 256, 64);
  check<128, true, false, 1>(256, 256, 64);
  check<128, true, true, 1>(256, 256, 64);
  check<128, false, false, 3>(256, 256, 64);
  check<128, false, true, 3>(256, 256, 64);
  check<128, true, true, 3>(300, 136, 72);
  check<256, true, true, 1>(300, 520, 200);
  check<128, false, true, 1>(128, 128, 8);
  check<128, true, false, 1>(128, 128, 8);
  printf("done\n");
}
