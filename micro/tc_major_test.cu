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
  static constexpr bool kRed = false;
  float *C; int N;
  __device__ float load(int, int) const { return 0.0f; }
  __device__ void store(int m, int n, float v, float) const { C[(int64_t)m * N + n] = v; }
  __device__ void strip(int m0, int mlim, int n, const float *v) const {
    for (int r = 0; r < 32 && m0 + r < mlim; ++r) C[(int64_t)(m0 + r) * N + n] = v[33 * r];
  }
};

// the forward epilogue of the library (bias + activation, writes A and S)
#include "gemm_simt.cuh"
struct EpiFwdT : nf::EpiFwd {};

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
__global__ void fill(float *x, int64_t n, uint32_t seed, int positive) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t h = (uint32_t)i * 2654435761u ^ seed;
    h ^= h >> 13; h *= 0x5bd1e995; h ^= h >> 15;
    const float u = (h & 0xFFFFFF) / 16777216.0f;
    x[i] = positive ? u : u * 2.0f - 1.0f;
  }
}
// plain fp32 FMA reference of the same product (the SIMT path's arithmetic)
__global__ void fp32_gemm(const float *A, const float *B, float *C, int M, int N, int K, int amn, int bmn) {
  int m = blockIdx.y * 16 + threadIdx.y, n = blockIdx.x * 16 + threadIdx.x;
  if (m >= M || n >= N) return;
  float s = 0;
  for (int k = 0; k < K; ++k) {
    const float a = amn ? A[(int64_t)k * M + m] : A[(int64_t)m * K + k];
    const float b = bmn ? B[(int64_t)k * N + n] : B[(int64_t)n * K + k];
    s = fmaf(a, b, s);
  }
  C[(int64_t)m * N + n] = s;
}

bool map(CUtensorMap *m, const float *p, int rows, int K, bool mn, int box_rows) {
  if (mn) return encode_tmap_2d_f32(m, p, rows, K, (uint64_t)rows * 4, 32, tc::BK, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
  return encode_tmap_2d_f32(m, p, K, rows, (uint64_t)K * 4, tc::BK, box_rows, CU_TENSOR_MAP_SWIZZLE_128B);
}

template <int BN, bool AMN, bool BMN, int SPLIT>
void check(int M, int N, int K, int positive = 0, int reps = 0) {
  float *A, *B, *C; double *R;
  CK(cudaMalloc(&A, (size_t)M * K * 4)); CK(cudaMalloc(&B, (size_t)N * K * 4));
  CK(cudaMalloc(&C, (size_t)M * N * 4)); CK(cudaMalloc(&R, (size_t)M * N * 8));
  fill<<<256, 256>>>(A, (int64_t)M * K, 1, positive); fill<<<256, 256>>>(B, (int64_t)N * K, 2, 0);
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
  float ms = 0;
  if (reps) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r)
      kern<<<dim3((N + BN - 1) / BN, (M + tc::BM - 1) / tc::BM, 1), tc::kThreads, Cf::SMEM>>>(ta, tb, g, EpiStore{C, N});
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= reps;
  }
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
  // the same metric for plain fp32 FMA accumulation (what the SIMT kernels do)
  double mf = 0;
  {
    float *F; CK(cudaMalloc(&F, (size_t)M * N * 4));
    fp32_gemm<<<dim3((N + 15) / 16, (M + 15) / 16), dim3(16, 16)>>>(A, B, F, M, N, K, AMN, BMN);
    CK(cudaDeviceSynchronize());
    std::vector<float> f((size_t)M * N);
    CK(cudaMemcpy(f.data(), F, f.size() * 4, cudaMemcpyDeviceToHost));
    for (size_t i = 0; i < f.size(); ++i) mf = std::max(mf, std::fabs(f[i] - r[i]) / std::max(std::fabs(r[i]), 0.1 * mx));
    cudaFree(F);
  }
  printf("CHECK BN=%d AMN=%d BMN=%d SPLIT=%d M=%d N=%d K=%d pos=%d: max rel err (tau=0.1) %.3e (fp32 FMA %.3e)",
         BN, (int)AMN, (int)BMN, SPLIT, M, N, K, positive, me, mf);
  if (reps) printf("  %.3f ms %.1f TFLOP/s", ms, 2.0 * M * N * K / ms / 1e9);
  printf("\n");
  // find a transposition pattern: compare c[m][n] with r of other index
  cudaFree(A); cudaFree(B); cudaFree(C); cudaFree(R);
}

template <class Epi, int BNP = 256>
void perf_pers(const char *name, int M, int N, int K, Epi epi, float *A, float *B) {
  CUtensorMap ta, tb;
  map(&ta, A, M, K, false, tc::BM); map(&tb, B, N, K, false, BNP);
  using Cf = tc::Cfg<BNP, 1>;
  auto kern = tc::gemm_tc_persistent<BNP, false, false, Epi>;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cf::SMEM));
  kern<<<148, tc::kThreads, Cf::SMEM>>>(ta, tb, M, N, K, epi);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < 3; ++r) kern<<<148, tc::kThreads, Cf::SMEM>>>(ta, tb, M, N, K, epi);
  cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
  float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 3;
  printf("PERSISTENT BN=%d %-10s M=%d N=%d K=%d: %.3f ms %.1f TFLOP/s\n", BNP, name, M, N, K, ms,
         2.0 * M * N * K / ms / 1e9);
}

template <class Epi, int BNT = 256>
void perf_epi(const char *name, int M, int N, int K, Epi epi, float *A, float *B) {
  CUtensorMap ta, tb;
  map(&ta, A, M, K, false, tc::BM); map(&tb, B, N, K, false, BNT);
  using Cf = tc::Cfg<BNT, 1>;
  auto kern = tc::gemm_tc_kernel<BNT, false, false, 1, Epi>;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cf::SMEM));
  tc::TileArgs g{M, N, K, ((K + 31) / 32) * 32, nullptr};
  dim3 grid((N + BNT - 1) / BNT, (M + 127) / 128, 1);
  kern<<<grid, tc::kThreads, Cf::SMEM>>>(ta, tb, g, epi);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < 3; ++r) kern<<<grid, tc::kThreads, Cf::SMEM>>>(ta, tb, g, epi);
  cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
  float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 3;
  printf("EPI %-10s M=%d N=%d K=%d: %.3f ms %.1f TFLOP/s\n", name, M, N, K, ms, 2.0 * M * N * K / ms / 1e9);
}

int main(int argc, char **argv) {
  if (argc > 1 && argv[1][0] == 't') {  // config-3 layer with the tanh epilogue only (ncu)
    const int M = 4096, N = 1024, K = 1024;
    float *A, *B, *C, *S, *bias;
    CK(cudaMalloc(&A, (size_t)M * K * 4)); CK(cudaMalloc(&B, (size_t)N * K * 4));
    CK(cudaMalloc(&C, (size_t)M * N * 4)); CK(cudaMalloc(&S, (size_t)M * N * 4)); CK(cudaMalloc(&bias, N * 4));
    fill<<<256, 256>>>(A, (int64_t)M * K, 1, 0); fill<<<256, 256>>>(B, (int64_t)N * K, 2, 0);
    fill<<<256, 256>>>(bias, N, 3, 0);
    perf_epi("c3-store", M, N, K, EpiStore{C, N}, A, B);
    perf_epi("c3-tanh", M, N, K, nf::EpiFwd{bias, C, S, nullptr, N, nf::ACT_TANH, 0}, A, B);
    perf_epi("c3-relu", M, N, K, nf::EpiFwd{bias, C, S, nullptr, N, nf::ACT_RELU, 0}, A, B);
    perf_epi("c3-tinf", M, N, K, nf::EpiFwd{bias, C, S, nullptr, N, nf::ACT_TANH, 2}, A, B);
    return 0;
  }
  if (argc > 1 && argv[1][0] == 'c') {  // config-3 shape only (profiling)
    const int M = 4096, N = 1024, K = 1024;
    float *A, *B, *C, *S, *bias;
    CK(cudaMalloc(&A, (size_t)M * K * 4)); CK(cudaMalloc(&B, (size_t)N * K * 4));
    CK(cudaMalloc(&C, (size_t)M * N * 4)); CK(cudaMalloc(&S, (size_t)M * N * 4)); CK(cudaMalloc(&bias, N * 4));
    fill<<<256, 256>>>(A, (int64_t)M * K, 1, 0); fill<<<256, 256>>>(B, (int64_t)N * K, 2, 0);
    fill<<<256, 256>>>(bias, N, 3, 0);
    perf_epi("c3-store", M, N, K, EpiStore{C, N}, A, B);
    perf_epi("c3-tanh", M, N, K, nf::EpiFwd{bias, C, S, nullptr, N, nf::ACT_TANH, 0}, A, B);
    perf_pers<EpiStore, 64>("c3-store", M, N, K, EpiStore{C, N}, A, B);
    perf_pers<nf::EpiFwd, 64>("c3-tanh", M, N, K, nf::EpiFwd{bias, C, S, nullptr, N, nf::ACT_TANH, 0}, A, B);
    perf_pers<EpiStore, 128>("c3-store", M, N, K, EpiStore{C, N}, A, B);
    perf_pers<nf::EpiFwd, 128>("c3-tanh", M, N, K, nf::EpiFwd{bias, C, S, nullptr, N, nf::ACT_TANH, 0}, A, B);
    perf_pers<nf::EpiFwd, 256>("c3-tanh", M, N, K, nf::EpiFwd{bias, C, S, nullptr, N, nf::ACT_TANH, 0}, A, B);
    // config-4 layer shape
    const int M4 = 2048, N4 = 256, K4 = 256;
    perf_pers<nf::EpiFwd, 64>("c4-relu", M4, N4, K4, nf::EpiFwd{bias, C, S, nullptr, N4, nf::ACT_RELU, 0}, A, B);
    perf_pers<nf::EpiFwd, 32>("c4-relu", M4, N4, K4, nf::EpiFwd{bias, C, S, nullptr, N4, nf::ACT_RELU, 0}, A, B);
    return 0;
  }
  if (argc > 1) goto perf;
  check<128, false, false, 1>(256, 256, 64);
  check<128, false, true, 1>(256, 256, 64);
  check<128, true, false, 1>(256, 256, 64);
  check<128, true, true, 1>(256, 256, 64);
  check<128, false, false, 3>(256, 256, 64);
  check<128, false, true, 3>(256, 256, 64);
  check<128, true, true, 3>(300, 136, 72);
  check<64, true, true, 3>(300, 136, 72);
  check<256, true, true, 1>(300, 520, 200);
  check<64, false, true, 1>(128, 200, 8);
  // accuracy at config-5 depth (K = 4096), signed and all-positive A (relu activations)
  check<128, false, false, 3>(512, 512, 4096, 0);
  check<128, false, false, 3>(512, 512, 4096, 1);
  check<128, true, true, 3>(512, 512, 16384, 1);
  // throughput of the four major combinations at the config-5 GEMM shape
  check<256, false, false, 1>(16384, 4096, 4096, 0, 3);
  check<256, false, true, 1>(16384, 4096, 4096, 0, 3);
  check<256, true, true, 1>(4096, 4096, 16384, 0, 3);
  check<128, false, true, 1>(16384, 4096, 4096, 0, 3);
  check<128, false, false, 3>(16384, 4096, 4096, 0, 2);
  check<128, false, true, 3>(16384, 4096, 4096, 0, 2);
perf:
  {  // config-3 layer shape: one wave of 128x256 tiles
    const int M = 4096, N = 1024, K = 1024;
    float *A, *B, *C, *S, *bias;
    CK(cudaMalloc(&A, (size_t)M * K * 4)); CK(cudaMalloc(&B, (size_t)N * K * 4));
    CK(cudaMalloc(&C, (size_t)M * N * 4)); CK(cudaMalloc(&S, (size_t)M * N * 4)); CK(cudaMalloc(&bias, N * 4));
    fill<<<256, 256>>>(A, (int64_t)M * K, 1, 0); fill<<<256, 256>>>(B, (int64_t)N * K, 2, 0);
    fill<<<256, 256>>>(bias, N, 3, 0);
    perf_epi("c3-store", M, N, K, EpiStore{C, N}, A, B);
    perf_epi("c3-tanh", M, N, K, nf::EpiFwd{bias, C, S, nullptr, N, nf::ACT_TANH, 0}, A, B);
    perf_pers("c3-store", M, N, K, EpiStore{C, N}, A, B);
    perf_pers("c3-tanh", M, N, K, nf::EpiFwd{bias, C, S, nullptr, N, nf::ACT_TANH, 0}, A, B);
  }
  {
    const int M = 16384, N = 4096, K = 4096;
    float *A, *B, *C, *S, *bias;
    CK(cudaMalloc(&A, (size_t)M * K * 4)); CK(cudaMalloc(&B, (size_t)N * K * 4));
    CK(cudaMalloc(&C, (size_t)M * N * 4)); CK(cudaMalloc(&S, (size_t)M * N * 4)); CK(cudaMalloc(&bias, N * 4));
    fill<<<256, 256>>>(A, (int64_t)M * K, 1, 0); fill<<<256, 256>>>(B, (int64_t)N * K, 2, 0);
    fill<<<256, 256>>>(bias, N, 3, 0);
    perf_epi("store", M, N, K, EpiStore{C, N}, A, B);
    perf_epi("fwd-relu", M, N, K, nf::EpiFwd{bias, C, S, nullptr, N, nf::ACT_RELU, 0}, A, B);
    perf_epi("fwd-sigm", M, N, K, nf::EpiFwd{bias, C, S, nullptr, N, nf::ACT_SIGMOID, 0}, A, B);
    perf_epi("fwd-infer", M, N, K, nf::EpiFwd{bias, C, S, nullptr, N, nf::ACT_RELU, 2}, A, B);
    perf_epi("bwd", M, N, K, nf::EpiBwd{S, N}, A, B);
    perf_pers("store", M, N, K, EpiStore{C, N}, A, B);
    perf_pers("fwd-relu", M, N, K, nf::EpiFwd{bias, C, S, nullptr, N, nf::ACT_RELU, 0}, A, B);
    perf_pers("fwd-sigm", M, N, K, nf::EpiFwd{bias, C, S, nullptr, N, nf::ACT_SIGMOID, 0}, A, B);
    perf_pers("bwd", M, N, K, nf::EpiBwd{S, N}, A, B);
    // correctness of the persistent kernel against fp64 (and the per-tile kernel's error)
    {
      const int Mc = 1024;  // rows checked (fp64 reference cost)
      float *C2; CK(cudaMalloc(&C2, (size_t)M * N * 4));
      double *R; CK(cudaMalloc(&R, (size_t)Mc * N * 8));
      perf_epi("store-ref", M, N, K, EpiStore{C2, N}, A, B);
      perf_pers("store", M, N, K, EpiStore{C, N}, A, B);
      ref_gemm<<<dim3((N + 15) / 16, (Mc + 15) / 16), dim3(16, 16)>>>(A, B, R, Mc, N, K, 0, 0);
      CK(cudaDeviceSynchronize());
      std::vector<float> h1((size_t)Mc * N), h2((size_t)Mc * N);
      std::vector<double> r((size_t)Mc * N);
      CK(cudaMemcpy(h1.data(), C, h1.size() * 4, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(h2.data(), C2, h2.size() * 4, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(r.data(), R, r.size() * 8, cudaMemcpyDeviceToHost));
      double mx = 0, e1 = 0, e2 = 0;
      for (size_t i = 0; i < r.size(); ++i) mx = std::max(mx, std::fabs(r[i]));
      for (size_t i = 0; i < r.size(); ++i) {
        const double sc = std::max(std::fabs(r[i]), 0.1 * mx);
        e1 = std::max(e1, std::fabs(h1[i] - r[i]) / sc);
        e2 = std::max(e2, std::fabs(h2[i] - r[i]) / sc);
      }
      printf("PERSISTENT max rel err (tau=0.1, first %d rows) %.3e; per-tile kernel %.3e\n", Mc, e1, e2);
    }
  }
  printf("done\n");
}
