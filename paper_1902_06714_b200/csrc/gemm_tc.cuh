// gemm_tc.cuh -- tcgen05 (5th-gen tensor core) TF32 contraction for sm_100a with
// fused epilogues: the wide-layer path of the three GEMM-shaped steps of the
// method in NF_MATH_TF32 mode.
//
//   C[M][N] = sum_k A[m][k] * B[n][k]      (both operands K-major, fp32 in HBM,
//                                           TF32 multiply, fp32 accumulate in TMEM)
//
// One CTA computes one BM x BN tile.  Warp roles (192 threads):
//   warp 0      TMA producer: 2-D tensor-map loads of A/B K-blocks (SWIZZLE_128B)
//               into a STAGES-deep shared-memory ring (mbarrier full/empty pairs)
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer; tcgen05.commit
//               releases ring slots and finally signals the accumulator
//   warps 2..5  epilogue: tcgen05.ld 32x32b.x32 (one TMEM lane = one tile row per
//               thread, 32 columns per load) -> functor(m, n, v[32])
#pragma once
#include <cstdint>

#include "nf_common.cuh"
#include "sm100_ptx.cuh"

namespace nf {
namespace tc {

constexpr int BM = 128;
constexpr int BK = 32;              // 32 fp32 = 128 B = one SWIZZLE_128B atom along K
constexpr int kThreads = 192;

template <int BN>
struct Cfg {
  static constexpr int A_BYTES = BM * BK * 4;
  static constexpr int B_BYTES = BN * BK * 4;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = (200 * 1024) / STAGE_BYTES;  // 4 for BN=256, 6 for BN=128
  static constexpr int TMEM_COLS = BN;                        // fp32 accumulator: 1 column per n
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
};

// ---- descriptors ------------------------------------------------------------------
// Shared-memory matrix descriptor, K-major, SWIZZLE_128B: rows of 128 B, 8-row groups
// 1024 B apart (SBO); LBO unused for swizzled K-major; version 1 (sm_100).
__device__ __forceinline__ uint64_t smem_desc_k_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;                    // LBO (ignored)
  d |= (uint64_t)(1024 >> 4) << 32;          // SBO
  d |= (uint64_t)1 << 46;                    // version
  d |= (uint64_t)2 << 61;                    // SWIZZLE_128B
  return d;
}
// Instruction descriptor: D fp32, A/B tf32, both K-major, M x N.
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
      ::"r"(tmem_d), "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
               ::"r"(ptx::smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ float round_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// ---- the kernel ------------------------------------------------------------------------
// Epi: __device__ void operator()(int m, int n, const float (&v)[32]) const -- row m,
// columns n..n+31 (caller guarantees m < M; columns >= N must be ignored by the functor).
template <int BN, class Epi>
__global__ void __launch_bounds__(kThreads, 1)
gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int M, int N,
               int K, Epi epi) {
  using C = Cfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t *empty = full + C::STAGES;
  uint64_t *accum = empty + C::STAGES;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(accum + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n0 = blockIdx.x * BN, m0 = blockIdx.y * BM;
  const int nkb = (K + BK - 1) / BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    ptx::mbar_init(accum, 1);
    ptx::fence_mbar_init();
    ptx::prefetch_tensormap(&tmA);
    ptx::prefetch_tensormap(&tmB);
  }
  if (warp == 1) {  // TMEM allocation (whole warp)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 ::"r"(ptx::smem_u32(tmem_slot)), "r"((uint32_t)C::TMEM_COLS) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = kb % C::STAGES;
        if (kb >= C::STAGES) ptx::mbar_wait(&empty[s], (uint32_t)(((kb / C::STAGES) - 1) & 1));
        uint8_t *sa = smem + s * C::STAGE_BYTES;
        uint8_t *sb = sa + C::A_BYTES;
        ptx::mbar_arrive_expect_tx(&full[s], (uint32_t)C::STAGE_BYTES);
        ptx::tma_load_2d(sa, &tmA, &full[s], kb * BK, m0);
        ptx::tma_load_2d(sb, &tmB, &full[s], kb * BK, n0);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer
      const uint32_t idesc = idesc_tf32(BM, BN);
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = kb % C::STAGES;
        ptx::mbar_wait(&full[s], (uint32_t)((kb / C::STAGES) & 1));
        tc_fence_after();
        const uint32_t sa = ptx::smem_u32(smem + s * C::STAGE_BYTES);
        const uint32_t sb = sa + C::A_BYTES;
#pragma unroll
        for (int k = 0; k < BK / 8; ++k)  // K = 8 tf32 (32 B) per MMA: advance inside the 128-B atom
          mma_tf32(tmem, smem_desc_k_sw128(sa + 32 * k), smem_desc_k_sw128(sb + 32 * k), idesc,
                   (kb | k) != 0 ? 1u : 0u);
        mma_commit(&empty[s]);
      }
      mma_commit(accum);
    }
  } else {  // ---- epilogue warps 2..5: TMEM lane quadrant = warp % 4
    const int q = warp & 3;
    ptx::mbar_wait(accum, 0);
    tc_fence_after();
    const int m = m0 + q * 32 + lane;
#pragma unroll 1
    for (int c = 0; c < BN / 32; ++c) {
      const int n = n0 + c * 32;
      if (n >= N) break;  // warp-uniform
      float v[32];
      tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(c * 32), v);
      if (m < M) epi(m, n, v);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"((uint32_t)C::TMEM_COLS)
                 : "memory");
  }
}

}  // namespace tc
}  // namespace nf
