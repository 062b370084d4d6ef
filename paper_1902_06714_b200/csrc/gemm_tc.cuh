// gemm_tc.cuh -- tcgen05 (5th-gen tensor core) contraction for sm_100a with fused
// epilogues: the wide-layer path of the three GEMM-shaped steps of the method
// (fwdprop P:324-361, backprop P:391-427, the batch-summed
// tendencies of train_batch P:460-476):
//
//   C[m][n] = sum_k A(m,k) * B(n,k)        fp32 operands in HBM, TF32 tensor-core
//                                           multiplies, fp32 accumulation in TMEM
//
//   K1 forward   Z_l = A_{l-1} W_l^T       A K-major [M][K], B K-major [N][K]
//   K3 backward  D_l = D_{l+1} W_{l+1}     A K-major,        B N-major [K][N]
//   K4 gradient  G_l = D_l^T A_{l-1}       A M-major [K][M], B N-major [K][N]
//
// Numerics (reading R13 of DESIGN.md): SPLIT = 1 is plain TF32 (NF_MATH_TF32).
// SPLIT = 3 is 3xTF32 for the fp32 mode: every staged tile x is split in shared memory
// into hi = x rounded to TF32 (written back in place) and lo = (x - hi) rounded to TF32
// (x - hi is exact in fp32), and each K-step issues hi*hi + hi*lo + lo*hi: per-product error
// <= 2^-23 (lo rounding) + 2^-22 (dropped lo*lo) relative.  The tensor core reads fp32 bit patterns and
// drops the low 13 mantissa bits (truncation, measured: micro/tc_major_test.cu), which is
// what SPLIT = 1 gets.
//
// One CTA computes one BM x BN tile (optionally one K-chunk of it: split-K writes raw
// partials that splitk_epilogue sums in fixed order).  Warp roles (320 threads):
//   warp 0      TMA producer: 2-D tensor-map loads (SWIZZLE_128B) into a STAGES-deep ring
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer; tcgen05.commit frees
//               ring slots and finally signals the accumulator
//   warps 2..9  (SPLIT = 3) hi/lo splitters during the main loop; then the epilogue:
//               tcgen05.ld 32x32b.x32 (thread = tile row), transpose through shared memory
//               so that a warp touches 32 consecutive columns of one row per access
//               (coalesced), then epi(m, n, value).
//
// Shared-memory operand layouts (UMMA canonical forms, SWIZZLE_128B):
//   K-major : TMA box {32 k, rows}: row r at r*128 B, 8-row groups 1024 B apart (SBO);
//             the MMA's K = 8 step advances the start address by 32 B inside the row.
//   MN-major: rows/32 TMA boxes {32 mn, 32 k} with the 128B_ATOM_32B swizzle, each 4 KB:
//             k-row at k*128 B, its four 32-B chunks permuted by (k mod 4); 32-element MN
//             blocks 4096 B apart (LBO); 4-k-row atoms 512 B apart (SBO); the K = 8 step
//             advances the start address by 1024 B.
#pragma once
#include <cstdint>

#include "nf_common.cuh"
#include "sm100_ptx.cuh"

namespace nf {
namespace tc {

constexpr int BM = 128;
constexpr int BK = 32;              // 32 fp32 = 128 B = one SWIZZLE_128B row
#ifndef NF_EPI_WARPS
#define NF_EPI_WARPS 8
#endif
constexpr int kEpiWarps = NF_EPI_WARPS;      // epilogue warps: kEpiWarps / 4 per TMEM lane quadrant
constexpr int kThreads = 64 + 32 * kEpiWarps;  // + TMA producer warp + MMA warp
constexpr int kSmemBudget = 232448; // max dynamic shared memory per CTA on sm_100
constexpr int kEpiBytes = kEpiWarps * 32 * 33 * 4;

template <int BN, int SPLIT, int MAXST = 6, int EW = kEpiWarps>
struct Cfg {
  static constexpr int EPI_BYTES = EW * 32 * 33 * 4;  // epilogue transpose buffers
  static constexpr int THREADS = 64 + 32 * EW;
  static constexpr int A_BYTES = BM * BK * 4;
  static constexpr int B_BYTES = BN * BK * 4;
  static constexpr int RAW_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGE_BYTES = SPLIT == 3 ? 2 * RAW_BYTES : RAW_BYTES;  // raw(hi) | lo
  // The per-tile kernel's epilogue transpose buffers may overlay the operand ring (the ring is dead
  // once the accumulator barrier fires: every stage has been consumed): used where that buys a
  // stage (the one-wave 128 x 256 tiles with 16 epilogue warps, config 3: 3 -> 4 stages).  The
  // persistent kernel drains tile i while tile i+1 streams and keeps them apart.
  static constexpr int FIT_SEP = (kSmemBudget - EPI_BYTES - 1024 - 512) / STAGE_BYTES;
  static constexpr int FIT_OVL = (kSmemBudget - 1024 - 512) / STAGE_BYTES;
  static constexpr int ST_SEP = FIT_SEP > MAXST ? MAXST : FIT_SEP;
  static constexpr int ST_OVL = FIT_OVL > MAXST ? MAXST : FIT_OVL;
#ifdef NF_TC_NO_OVERLAY
  static constexpr bool OVL = false;
#else
  static constexpr bool OVL = ST_OVL > ST_SEP;
#endif
  static constexpr int STAGES = OVL ? ST_OVL : ST_SEP;
  static constexpr int RING_BYTES = STAGES * STAGE_BYTES;
  static constexpr int EPI_OFF = OVL ? 0 : RING_BYTES;                                  // epilogue buffers
  static constexpr int BAR_OFF = OVL ? (RING_BYTES > EPI_BYTES ? RING_BYTES : EPI_BYTES) : RING_BYTES + EPI_BYTES;
  // NACC accumulators (all 512 TMEM columns): K-step t accumulates into t % NACC, and
  // the epilogue sums them in fp32.  The tensor core's fp32 accumulation truncates
  // (measured error linear in K, micro/tc_major_test.cu); spreading the K-steps over
  // NACC accumulators divides that error by NACC.
  // 1xTF32 (SPLIT = 1): the operands' TF32 rounding dominates, one accumulator suffices, and
  // allocating only BN columns lets the next kernel's CTA (programmatic dependent launch)
  // take its TMEM while this one drains.
  static constexpr int NACC = SPLIT == 3 ? 512 / BN : 1;
  static constexpr int TMEM_COLS = SPLIT == 3 ? 512 : (BN < 32 ? 32 : BN);
  static constexpr int SMEM = BAR_OFF + 1024 /*align*/ + 512 /*barriers*/;
  static_assert(STAGES >= 2, "ring too shallow");
};

// ---- descriptors ---------------------------------------------------------------------
// Shared-memory matrix descriptor (sm_100 version 1).  layout: 2 = SWIZZLE_128B,
// 1 = SWIZZLE_128B_BASE32B (128-B rows, 32-B swizzle atoms: the only smem layout the
// tensor core accepts for MN-major TF32 operands).
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;                    // version
  d |= (uint64_t)layout << 61;
  return d;
}
// Operand descriptor for K-step `ks` (K = 8 tf32 each) of a staged tile.
//   K-major : SWIZZLE_128B, SBO = 1024 (8-row groups); +32 B per K-step inside the row.
//   MN-major: SWIZZLE_128B_BASE32B, LBO = 4096 (32-element MN blocks = one TMA box),
//             SBO = 512 (4-k-row swizzle atoms); +1024 B (8 k-rows) per K-step.
template <bool MN>
__device__ __forceinline__ uint64_t op_desc(uint32_t base, int ks) {
  if (MN) return smem_desc(base + 1024u * ks, BK * 128, 512, 1);
  return smem_desc(base + 32u * ks, 16, 1024, 2);
}
// Instruction descriptor: D fp32, A/B tf32, majors, M x N.
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N, bool a_mn, bool b_mn) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((a_mn ? 1u : 0u) << 15) | ((b_mn ? 1u : 0u) << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
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

// TF32 part of x, rounded to nearest (ties away): an exact TF32 value, so the tensor core's
// own operand truncation leaves it unchanged; lo = x - hi is exact in fp32 with
// abs(lo) <= 2^-11 abs(x).
__device__ __forceinline__ float tf32_hi(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

struct TileArgs {
  int M, N, K;
  int kchunk;          // K range per blockIdx.z (multiple of BK)
  float *partial;      // non-null: write raw partials [z][M][N] (split-K) instead of epi
  int red;             // split-K with an additive epilogue (EpiGrad update): each split adds
                       // its own term straight into the output (red.global.add), no partials
  int pre = 0;         // SPLIT = 3 with pre-split operands: the lo parts come from their own
                       // tensor maps (written by the producers' epilogues), no in-smem splitting
};

// ---- the kernel ------------------------------------------------------------------------
// MAXST < 6: a shallower ring (less shared memory) so that two CTAs co-reside on an SM and
// one's epilogue overlaps the other's main loop; EW: epilogue warps (a multiple of 4)
template <int BN, bool A_MN, bool B_MN, int SPLIT, class Epi, int MAXST = 6, int EW = kEpiWarps>
__global__ void __launch_bounds__(64 + 32 * EW, 1)
gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, TileArgs g,
               Epi epi, const __grid_constant__ CUtensorMap tmAlo, const __grid_constant__ CUtensorMap tmBlo) {
  using C = Cfg<BN, SPLIT, MAXST, EW>;
  ptx::pdl_trigger();
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  float *epibuf = reinterpret_cast<float *>(smem + C::EPI_OFF);
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + C::BAR_OFF);
  uint64_t *empty = full + C::STAGES;
  uint64_t *conv = empty + C::STAGES;
  uint64_t *accum = conv + C::STAGES;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(accum + 1);

  const int warp = ptx::warp_uniform(threadIdx.x >> 5), lane = threadIdx.x & 31;
  const int n0 = blockIdx.x * BN, m0 = blockIdx.y * BM;
  const int kbeg = blockIdx.z * g.kchunk;
  const int kend = min(g.K, kbeg + g.kchunk);
  const int nkb = (kend - kbeg + BK - 1) / BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
      ptx::mbar_init(&conv[s], EW);
    }
    ptx::mbar_init(accum, 1);
    ptx::fence_mbar_init();
    ptx::prefetch_tensormap(&tmA);
    ptx::prefetch_tensormap(&tmB);
    if (SPLIT == 3 && g.pre) {
      ptx::prefetch_tensormap(&tmAlo);
      ptx::prefetch_tensormap(&tmBlo);
    }
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
  ptx::pdl_wait();  // prologue above overlaps the previous kernel

  // The TMA and MMA warps run their loops and barrier waits with all 32 lanes (warp-uniform control
  // flow, operands in uniform registers) and issue through one elected lane (ptx::elect_one).
  if (warp == 0) {  // ---- TMA producer
    int s = 0;
    for (int it = 0; it < nkb; ++it) {
      if (it >= C::STAGES) ptx::mbar_wait(&empty[s], (uint32_t)(((it / C::STAGES) - 1) & 1));
      uint8_t *sa = smem + s * C::STAGE_BYTES;
      uint8_t *sb = sa + C::A_BYTES;
      const int k = kbeg + it * BK;
      const bool pre = SPLIT == 3 && g.pre;
      if (ptx::elect_one()) {
        ptx::mbar_arrive_expect_tx(&full[s], (uint32_t)(pre ? 2 * C::RAW_BYTES : C::RAW_BYTES));
        // (pre: a second pass with the lo maps into the lo half of the stage)
        for (int half = 0; half < (pre ? 2 : 1); ++half) {
          const CUtensorMap *ma = half ? &tmAlo : &tmA, *mb = half ? &tmBlo : &tmB;
          uint8_t *da = sa + half * C::RAW_BYTES, *db = sb + half * C::RAW_BYTES;
          if (A_MN) {
#pragma unroll
            for (int i = 0; i < BM / 32; ++i) ptx::tma_load_2d(da + i * 4096, ma, &full[s], m0 + 32 * i, k);
          } else {
            ptx::tma_load_2d(da, ma, &full[s], k, m0);
          }
          if (B_MN) {
#pragma unroll
            for (int i = 0; i < BN / 32; ++i) ptx::tma_load_2d(db + i * 4096, mb, &full[s], n0 + 32 * i, k);
          } else {
            ptx::tma_load_2d(db, mb, &full[s], k, n0);
          }
        }
      }
      __syncwarp();
      if (++s == C::STAGES) s = 0;
    }
  } else if (warp == 1) {  // ---- MMA issuer
    constexpr uint32_t idesc = idesc_tf32(BM, BN, A_MN, B_MN);
    const uint32_t tmem_u = (uint32_t)ptx::warp_uniform((int)tmem), smem_u = ptx::smem_u32(smem);
    int s = 0;
    uint32_t par = 0;
    for (int it = 0; it < nkb; ++it) {
      ptx::mbar_wait((SPLIT == 3 && !g.pre) ? &conv[s] : &full[s], par);
      tc_fence_after();
      const uint32_t sa = smem_u + (uint32_t)(s * C::STAGE_BYTES);
      const uint32_t sb = sa + C::A_BYTES;
      if (ptx::elect_one()) {
#pragma unroll
        for (int ks = 0; ks < BK / 8; ++ks) {
          const int t = it * (BK / 8) + ks;                  // global K-step
          const uint32_t d = tmem_u + (uint32_t)((t % C::NACC) * BN);
          const uint32_t acc = t >= C::NACC ? 1u : 0u;       // first use of each accumulator
          const uint64_t ah = op_desc<A_MN>(sa, ks), bh = op_desc<B_MN>(sb, ks);
          mma_tf32(d, ah, bh, idesc, acc);
          if (SPLIT == 3) {
            const uint64_t al = op_desc<A_MN>(sa + C::RAW_BYTES, ks), bl = op_desc<B_MN>(sb + C::RAW_BYTES, ks);
            mma_tf32(d, ah, bl, idesc, 1u);
            mma_tf32(d, al, bh, idesc, 1u);
          }
        }
        mma_commit(&empty[s]);
        if (it == nkb - 1) mma_commit(accum);
      }
      __syncwarp();
      if (++s == C::STAGES) { s = 0; par ^= 1; }
    }
  } else {
    const int t = threadIdx.x - 64;  // 0 .. 32 EW - 1
    if (SPLIT == 3 && !g.pre) {  // ---- hi/lo splitters
      for (int it = 0; it < nkb; ++it) {
        const int s = it % C::STAGES;
        ptx::mbar_wait(&full[s], (uint32_t)((it / C::STAGES) & 1));
        float4 *raw = reinterpret_cast<float4 *>(smem + s * C::STAGE_BYTES);
        float4 *lo = reinterpret_cast<float4 *>(smem + s * C::STAGE_BYTES + C::RAW_BYTES);
#pragma unroll 4
        for (int i = t; i < C::RAW_BYTES / 16; i += 32 * EW) {
          const float4 x = raw[i];
          const float4 h = make_float4(tf32_hi(x.x), tf32_hi(x.y), tf32_hi(x.z), tf32_hi(x.w));
          raw[i] = h;
          lo[i] = make_float4(tf32_hi(x.x - h.x), tf32_hi(x.y - h.y), tf32_hi(x.z - h.z), tf32_hi(x.w - h.w));
        }
        ptx::fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&conv[s]);
      }
    }
    // ---- epilogue: TMEM lane quadrant = warp % 4; the two warps of a quadrant split the
    //      32-column chunks (even / odd)
    const int q = warp & 3, half = (warp - 2) >> 2;
    float *buf = epibuf + (warp - 2) * 32 * 33;
    ptx::mbar_wait(accum, 0);
    tc_fence_after();
    const int mrow0 = m0 + q * 32;
    const int64_t MN = (int64_t)g.M * g.N;
#pragma unroll 1
    for (int c = half; c < BN / 32; c += EW / 4) {
      const int nc = n0 + c * 32;
      if (nc >= g.N) break;  // warp-uniform
      float v[32];
      const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(c * 32);
      tmem_ld32(trow, v);
      const int nk = nkb * (BK / 8);                 // K-steps issued: accumulators in use
#pragma unroll 1
      for (int a = 1; a < C::NACC && a < nk; ++a) {   // fixed order: acc 0 + 1 + ... (RN fp32)
        float w[32];
        tmem_ld32(trow + (uint32_t)(a * BN), w);
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] += w[j];
      }
#pragma unroll
      for (int j = 0; j < 32; ++j) buf[lane * 33 + j] = v[j];
      __syncwarp();
      const int n = nc + lane;
      const bool nok = n < g.N;
      if constexpr (Epi::kRed) {
        if (g.red) {
          if (nok) epi.strip_red(mrow0, g.M, n, buf + lane);
          __syncwarp();
          continue;
        }
      }
      if (g.partial) {
#pragma unroll 4
        for (int r = 0; r < 32; ++r) {
          const int m = mrow0 + r;
          if (m < g.M && nok) g.partial[blockIdx.z * MN + (int64_t)m * g.N + n] = buf[r * 33 + lane];
        }
      } else {
        if (nok) epi.strip(mrow0, g.M, n, buf + lane);  // 32 rows of column n, loads before stores
        if constexpr (Epi::kHasT) {
          if (epi.T) {  // transposed copy from the block of stored values
            __syncwarp();
            store_t(epi.T, epi.ldT, mrow0, g.M, nc, g.N, buf, lane);
          }
        }
      }
      __syncwarp();
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

// ---- persistent variant (1xTF32) -------------------------------------------------------
// One CTA per SM walks tiles tile = blockIdx.x + i * gridDim.x (n fastest, so a wave shares
// A rows and all of B stays hot in L2).  Two TMEM accumulator stages of BN columns: the MMA
// warp fills stage s for tile i+1 while the epilogue warps drain stage s^1 of tile i, so the
// epilogue (bias + activation + stash / x sigma' / SGD RMW) overlaps the next main loop.
template <int BN, bool A_MN, bool B_MN, class Epi>
__global__ void __launch_bounds__(kThreads, 1)
gemm_tc_persistent(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int M, int N,
                   int K, Epi epi) {
  using C = Cfg<BN, 1>;
  static_assert(2 * BN <= 512, "two accumulator stages must fit in TMEM");
  static_assert(!C::OVL, "the persistent kernel's epilogue buffers live beside the ring");
  ptx::pdl_trigger();
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  float *epibuf = reinterpret_cast<float *>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + C::STAGES * C::STAGE_BYTES + kEpiBytes);
  uint64_t *empty = full + C::STAGES;
  uint64_t *tfull = empty + C::STAGES;   // [2] accumulator stage ready (tcgen05.commit)
  uint64_t *tempty = tfull + 2;          // [2] accumulator stage drained (kEpiWarps arrivals)
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty + 2);

  const int warp = ptx::warp_uniform(threadIdx.x >> 5), lane = threadIdx.x & 31;
  const int tn = (N + BN - 1) / BN, ntiles = ((M + BM - 1) / BM) * tn;
  const int nkb = (K + BK - 1) / BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      ptx::mbar_init(&tfull[s], 1);
      ptx::mbar_init(&tempty[s], kEpiWarps);
    }
    ptx::fence_mbar_init();
    ptx::prefetch_tensormap(&tmA);
    ptx::prefetch_tensormap(&tmB);
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 ::"r"(ptx::smem_u32(tmem_slot)), "r"((uint32_t)(2 * BN)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  ptx::pdl_wait();  // prologue above overlaps the previous kernel

  if (warp == 0) {  // ---- TMA producer, continuous over tiles (all lanes loop, one elected lane issues)
    int it = 0, s = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      const int m0 = (tile / tn) * BM, n0 = (tile % tn) * BN;
      for (int kb = 0; kb < nkb; ++kb, ++it) {
        if (it >= C::STAGES) ptx::mbar_wait(&empty[s], (uint32_t)(((it / C::STAGES) - 1) & 1));
        uint8_t *sa = smem + s * C::STAGE_BYTES;
        uint8_t *sb = sa + C::A_BYTES;
        const int k = kb * BK;
        if (ptx::elect_one()) {
          ptx::mbar_arrive_expect_tx(&full[s], (uint32_t)C::RAW_BYTES);
          if (A_MN) {
#pragma unroll
            for (int i = 0; i < BM / 32; ++i) ptx::tma_load_2d(sa + i * 4096, &tmA, &full[s], m0 + 32 * i, k);
          } else {
            ptx::tma_load_2d(sa, &tmA, &full[s], k, m0);
          }
          if (B_MN) {
#pragma unroll
            for (int i = 0; i < BN / 32; ++i) ptx::tma_load_2d(sb + i * 4096, &tmB, &full[s], n0 + 32 * i, k);
          } else {
            ptx::tma_load_2d(sb, &tmB, &full[s], k, n0);
          }
        }
        __syncwarp();
        if (++s == C::STAGES) s = 0;
      }
    }
  } else if (warp == 1) {  // ---- MMA issuer (all lanes loop and wait, one elected lane issues)
    constexpr uint32_t idesc = idesc_tf32(BM, BN, A_MN, B_MN);
    const uint32_t tmem_u = (uint32_t)ptx::warp_uniform((int)tmem), smem_u = ptx::smem_u32(smem);
    int s = 0, lt = 0;
    uint32_t par = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++lt) {
      const int as = lt & 1;
      if (lt >= 2) ptx::mbar_wait(&tempty[as], (uint32_t)(((lt >> 1) - 1) & 1));
      tc_fence_after();
      const uint32_t d = tmem_u + (uint32_t)(as * BN);
      for (int kb = 0; kb < nkb; ++kb) {
        ptx::mbar_wait(&full[s], par);
        tc_fence_after();
        const uint32_t sa = smem_u + (uint32_t)(s * C::STAGE_BYTES);
        const uint32_t sb = sa + C::A_BYTES;
        if (ptx::elect_one()) {
#pragma unroll
          for (int ks = 0; ks < BK / 8; ++ks)
            mma_tf32(d, op_desc<A_MN>(sa, ks), op_desc<B_MN>(sb, ks), idesc, (kb | ks) != 0 ? 1u : 0u);
          mma_commit(&empty[s]);
          if (kb == nkb - 1) mma_commit(&tfull[as]);
        }
        __syncwarp();
        if (++s == C::STAGES) { s = 0; par ^= 1; }
      }
    }
  } else {  // ---- epilogue warps: TMEM lane quadrant = warp % 4, even / odd 32-column chunks
    const int q = warp & 3, half = (warp - 2) >> 2;
    float *buf = epibuf + (warp - 2) * 32 * 33;
    int lt = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++lt) {
      const int as = lt & 1;
      const int m0 = (tile / tn) * BM, n0 = (tile % tn) * BN;
      ptx::mbar_wait(&tfull[as], (uint32_t)((lt >> 1) & 1));
      tc_fence_after();
      const int mrow0 = m0 + q * 32;
#pragma unroll 1
      for (int c = half; c < BN / 32; c += kEpiWarps / 4) {
        const int nc = n0 + c * 32;
        if (nc >= N) break;  // warp-uniform
        float v[32];
        tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(as * BN + c * 32), v);
#pragma unroll
        for (int j = 0; j < 32; ++j) buf[lane * 33 + j] = v[j];
        __syncwarp();
        const int n = nc + lane;
        if (n < N) epi.strip(mrow0, M, n, buf + lane);
        if constexpr (Epi::kHasT) {
          if (epi.T) {
            __syncwarp();
            store_t(epi.T, epi.ldT, mrow0, M, nc, N, buf, lane);
          }
        }
        __syncwarp();
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&tempty[as]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"((uint32_t)(2 * BN))
                 : "memory");
  }
}

}  // namespace tc
}  // namespace nf
