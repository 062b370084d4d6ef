// tc_atmem_test.cu -- does the tcgen05 TF32 MMA with the A operand in tensor memory (".kind::tf32
// [d], [a], b_desc") give the right product, and how fast is a chain of small M=128 x N=32 MMAs
// with A in TMEM vs A in shared memory (the K6 P1 / P5 shapes)?
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_1902_06714_b200/csrc \
//   tc_atmem_test.cu -o tc_atmem_test
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "gemm_tc.cuh"

using namespace nf;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

constexpr int M = 128, KMAX = 128;

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const float (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};"
      ::"r"(taddr), "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]),
        "f"(v[8]), "f"(v[9]), "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15]),
        "f"(v[16]), "f"(v[17]), "f"(v[18]), "f"(v[19]), "f"(v[20]), "f"(v[21]), "f"(v[22]), "f"(v[23]),
        "f"(v[24]), "f"(v[25]), "f"(v[26]), "f"(v[27]), "f"(v[28]), "f"(v[29]), "f"(v[30]), "f"(v[31])
      : "memory");
}
__device__ __forceinline__ void mma_tf32_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}"
      ::"r"(tmem_d), "r"(tmem_a), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ int sw128(int r, int c) { return r * 128 + ((((c >> 2) ^ (r & 7))) << 4) + ((c & 3) << 2); }

// A [M][K] fp32, B [N][K] fp32; D[M][N] = sum_k (3xTF32) A B.  mode 0: A in TMEM, 1: A in smem.
template <int N>
__global__ void k_test(const float *A, const float *B, float *D, int K, int mode, int nsplit, long long *clk, int nacc) {
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t *sm = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  // smem: A hi | A lo ([K/32 atoms][128 rows][128 B]), B hi | B lo ([K/32 atoms][N rows][128 B])
  uint8_t *Ah = sm, *Al = Ah + (KMAX / 32) * M * 128, *Bh = Al + (KMAX / 32) * M * 128, *Bl = Bh + (KMAX / 32) * N * 128;
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(ptx::smem_u32(&tslot)), "r"(512u) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (tid == 0) { ptx::mbar_init(&bar, 1); ptx::fence_mbar_init(); }
  for (int i = tid; i < M * KMAX; i += blockDim.x) {
    const int r = i / KMAX, k = i % KMAX;
    const float v = k < K ? A[r * K + k] : 0.0f, h = tc::tf32_hi(v);
    const int off = (k >> 5) * M * 128 + sw128(r, k & 31);
    *reinterpret_cast<float *>(Ah + off) = h;
    *reinterpret_cast<float *>(Al + off) = v - h;
  }
  for (int i = tid; i < N * KMAX; i += blockDim.x) {
    const int r = i / KMAX, k = i % KMAX;
    const float v = k < K ? B[r * K + k] : 0.0f, h = tc::tf32_hi(v);
    const int off = (k >> 5) * N * 128 + sw128(r, k & 31);
    *reinterpret_cast<float *>(Bh + off) = h;
    *reinterpret_cast<float *>(Bl + off) = v - h;
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = tslot;
  // TMEM: D at cols 0..N-1, A hi at 128.., A lo at 256..
  long long t_st0 = clock64();
  if (warp < 4) {
    const int r = tid;
    for (int c0 = 0; c0 < KMAX; c0 += 32) {
      float h[32], l[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const float v = (c0 + j) < K ? A[r * K + c0 + j] : 0.0f;
        h[j] = tc::tf32_hi(v);
        l[j] = v - h[j];
      }
      tmem_st32(tmem + ((uint32_t)(32 * warp) << 16) + 128u + c0, h);
      tmem_st32(tmem + ((uint32_t)(32 * warp) << 16) + 256u + c0, l);
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  long long t_st1 = clock64();
  ptx::fence_proxy_async_smem();
  __syncthreads();
  long long t0 = 0, t1 = 0, tfirst = 0;
  if (tid == 0) {
    constexpr uint32_t idesc = tc::idesc_tf32(M, N, false, false);
    const int nks = (K + 7) / 8;
    for (int rep = 0; rep < 9; ++rep) {
      if (rep == 1) t0 = clock64();
      const long long ta = clock64();
      for (int ks = 0; ks < nks; ++ks) {
        const uint32_t bo = (ks >> 2) * N * 128 + (ks & 3) * 32;
        const uint64_t bh = tc::smem_desc(ptx::smem_u32(Bh) + bo, 16, 1024, 2), bl = tc::smem_desc(ptx::smem_u32(Bl) + bo, 16, 1024, 2);
        if (mode == 0) {
          const uint32_t ah = tmem + 128u + 8 * ks, al = tmem + 256u + 8 * ks;
          const uint32_t dd = tmem + 384u + (uint32_t)(ks % nacc) * 32u;  // nacc > 1: round-robin accumulators
          if (nacc > 1) {
            mma_tf32_ts(dd, ah, bh, idesc, ks >= nacc ? 1u : 0u);
            if (nsplit == 3) {
              mma_tf32_ts(dd, ah, bl, idesc, 1u);
              mma_tf32_ts(dd, al, bh, idesc, 1u);
            }
            continue;
          }
          mma_tf32_ts(tmem, ah, bh, idesc, ks > 0 ? 1u : 0u);
          if (nsplit == 3) {
            mma_tf32_ts(tmem, ah, bl, idesc, 1u);
            mma_tf32_ts(tmem, al, bh, idesc, 1u);
          }
        } else {
          const uint32_t ao = (ks >> 2) * M * 128 + (ks & 3) * 32;
          const uint64_t ah = tc::smem_desc(ptx::smem_u32(Ah) + ao, 16, 1024, 2), al = tc::smem_desc(ptx::smem_u32(Al) + ao, 16, 1024, 2);
          tc::mma_tf32(tmem, ah, bh, idesc, ks > 0 ? 1u : 0u);
          if (nsplit == 3) {
            tc::mma_tf32(tmem, ah, bl, idesc, 1u);
            tc::mma_tf32(tmem, al, bh, idesc, 1u);
          }
        }
      }
      tc::mma_commit(&bar);
      ptx::mbar_wait(&bar, rep & 1);
      tc::tc_fence_after();
      if (rep == 0) tfirst = clock64() - ta;
    }
    t1 = clock64();
  }
  // tcgen05.st rate with the data already in registers: 128 lanes x 256 columns, 4 times
  __syncthreads();
  long long ts0 = clock64();
  if (warp < 4) {
    float h[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) h[j] = (float)(tid + j);
    for (int rep = 0; rep < 4; ++rep)
      for (int c0 = 0; c0 < 256; c0 += 32) tmem_st32(tmem + ((uint32_t)(32 * warp) << 16) + 256u + c0, h);
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  __syncthreads();
  long long ts1 = clock64();
  if (tid == 0) clk[2] = tfirst, clk[3] = ts1 - ts0;
  __syncthreads();
  tc::tc_fence_after();
  if (warp < 4) {
    for (int c0 = 0; c0 < N; c0 += 32) {
      float v[32];
      tc::tmem_ld32(tmem + ((uint32_t)(32 * warp) << 16) + c0, v);
      for (int j = 0; j < 32; ++j) D[tid * N + c0 + j] = v[j];
    }
  }
  if (tid == 0) { clk[0] = (t1 - t0) / 8; clk[1] = t_st1 - t_st0; }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512u) : "memory");
}

template <int N>
void run(int K, int mode, int nsplit, int nacc = 1) {
  std::vector<float> hA(M * K), hB(N * K);
  srand(1);
  for (auto &v : hA) v = (float)rand() / RAND_MAX * 2 - 1;
  for (auto &v : hB) v = (float)rand() / RAND_MAX * 2 - 1;
  float *A, *B, *D;
  long long *clk;
  CK(cudaMalloc(&A, hA.size() * 4)); CK(cudaMalloc(&B, hB.size() * 4)); CK(cudaMalloc(&D, M * N * 4));
  CK(cudaMalloc(&clk, 32));
  CK(cudaMemcpy(A, hA.data(), hA.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(B, hB.data(), hB.size() * 4, cudaMemcpyHostToDevice));
  const int smem = 2 * (KMAX / 32) * (M + N) * 128 + 1024;
  CK(cudaFuncSetAttribute(k_test<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  long long best = 1LL << 60, st = 0, first = 0;
  for (int it = 0; it < 5; ++it) {
    k_test<N><<<1, 256, smem>>>(A, B, D, K, mode, nsplit, clk, nacc);
    CK(cudaDeviceSynchronize());
    long long h[4];
    CK(cudaMemcpy(h, clk, 32, cudaMemcpyDeviceToHost));
    best = std::min(best, h[0]);
    st = h[3];
    first = h[2];
  }
  std::vector<float> hD(M * N);
  CK(cudaMemcpy(hD.data(), D, hD.size() * 4, cudaMemcpyDeviceToHost));
  double maxe = 0, maxr = 0;
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      double s = 0;
      for (int k = 0; k < K; ++k) s += (double)hA[m * K + k] * hB[n * K + k];
      maxe = std::max(maxe, std::fabs(s - hD[m * N + n]));
      maxr = std::max(maxr, std::fabs(s));
    }
  const int nmma = (K + 7) / 8 * nsplit;
  if (nacc > 1) maxe = -1;  // (accumulators not summed: timing only)
  printf("nacc=%d N=%3d K=%3d %s %dxTF32: %2d MMAs, chain+commit+wait %6lld clk warm (%5.1f clk/MMA), first %lld clk; 128x1024 tmem-store %lld clk; max err %.2e (rel %.2e)\n", nacc, N, K,
         mode == 0 ? "A in TMEM" : "A in smem", nsplit, nmma, best, (double)best / nmma, first, st, maxe, maxe / maxr);
  cudaFree(A); cudaFree(B); cudaFree(D); cudaFree(clk);
}

int main() {
  for (int nacc : {2, 4})
    for (int nsplit : {1, 3}) run<32>(104, 0, nsplit, nacc);
  for (int nsplit : {1, 3})
    for (int mode : {0, 1}) {
      run<32>(104, mode, nsplit);
      run<32>(72, mode, nsplit);
      run<64>(104, mode, nsplit);
    }
  return 0;
}
