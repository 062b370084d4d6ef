// infer_tc.cu -- the paper's `output` (Eq. 2) for two-layer nets with narrow
// hidden and output layers (H, O <= 32; config 2's [784,30,10]) on the tcgen05 tensor cores.
//
// Why tensor cores: streaming x at the HBM rate (6.5 TB/s = 2.06 G rows/s of 784 pixels) needs
// 2 * 784 * 30 flops per row = 97 TF/s of fp32 FMA, above the 72 TF/s FFMA peak; the FFMA2 kernel
// (infer_small.cu) is shared-memory / issue bound at 19 % of HBM.  Z1 = X W1^T is a dense
// contraction (M = rows, N = 32 neurons, K = pixels), run here in 3xTF32 (hi*hi + hi*lo + lo*hi,
// fp32 accumulate; the fp32 parity bar of 1e-4 rules out 1xTF32).
//
// Design (one persistent CTA per SM, 480 threads, rows split into equal runs of 32-row blocks):
//   warp 0      TMA producer of x: per K-block of 32 pixels, the x tile (4 boxes of 32 rows x 128 B,
//               SWIZZLE_128B) into an 8-deep ring freed by the converters (16 KB per stage)
//   warp 14     TMA producer of the W1 hi / lo K-blocks (RN split kept by the library next to the
//               parameters, L2-resident) into a 4-deep ring freed by the MMA commits: the slow
//               commit round trip never holds an x stage
//   warps 2-9   converters (two groups alternating K-blocks), thread = row: read the row's 32 pixels from the swizzled tile, split
//               them (truncation split: hi = x with the low 13 mantissa bits cleared, lo =
//               rn_tf32(x - hi)) and store hi | lo into a 6-deep TMEM ring with tcgen05.st -- so
//               the MMA reads its A operand from tensor memory (A in TMEM: no shared-memory read
//               of the 128-row operand per MMA; micro/tc_atmem_test.cu: ~14 cycles per M=128 x
//               N=32 x K=8 MMA marginal, vs ~61 with A in shared memory)
//   warp 1      MMA issuer: 4 k-steps x 2 MMAs (x_lo, x_hi) per K-block against B = the W stage's 64
//               rows, W1 hi | W1 lo STACKED along N: accumulator columns 0..31 get x W_hi, columns
//               32..63 x W_lo (all four partial products for two instructions per k-step instead of
//               the three of hi*hi + hi*lo + lo*hi; the epilogue adds the two halves), into one of
//               two 64-column TMEM accumulators (double-buffered per 128-row tile); tcgen05.commit
//               frees the ring slots and hands the finished accumulator to the epilogue
//   warps 10-13 epilogue, thread = row: tcgen05.ld both halves of the Z1 row, + b1, sigma_h, layer 2 (W2, b2 in
//               shared memory, broadcast reads), sigma_o, store the O outputs
// The x tile is read from HBM once; W1 (94 KB) is re-read from L2 per tile.
#include <algorithm>
#include <cstring>
#include <cstdio>
#include <mutex>
#include <vector>

#include "gemm_tc.cuh"
#include "infer_tc.cuh"
#include "kernels.cuh"
#include "nf_common.cuh"
#include "sm100_ptx.cuh"

namespace nf {
namespace {

constexpr int kTileRows = 128;                      // M of the MMA, rows per tile
constexpr int kBoxRows = 32;                        // rows per TMA box (tile tails in 32-row steps)
constexpr int kKB = 32;                             // pixels per K-block (one 128-B swizzle row)
constexpr int kStages = 8;                          // x ring depth (freed by the converters)
constexpr int kWStages = 4;                         // W1 hi | lo ring depth (freed by the MMA commits)
constexpr int kTStages = 6;                         // TMEM x-operand ring depth (64 columns: hi | lo)
constexpr int kCG = 2;                              // converter warp groups (alternating K-blocks)
constexpr int kXBytes = kTileRows * kKB * 4;        // 16 KB
constexpr int kWBytes = 32 * kKB * 4;               // 4 KB (hi or lo)
constexpr int kWStageBytes = 2 * kWBytes;           // 8 KB
constexpr int kAccCol = kTStages * 64;              // accumulators after the x ring: 2 x 64 columns (W hi | lo stacked along N)
constexpr int kThreads = 32 * (2 + 4 * kCG + 4 + 1);  // + the W producer warp
constexpr int kSmem = 1024 + kStages * kXBytes + kWStages * kWStageBytes + (32 * 33 + 64) * 4 + 512;

struct InferTcParams {
  int64_t n;      // rows
  int64_t nblk;   // 32-row blocks
  int n0, H, O, act_h, act_o;
  int nkb;        // K-blocks of 32 pixels
  int exp;        // experiment bits (NF_ITC_EXP, timing only): 1 no W reload, 2 no MMAs, 4 no conversion, 16 no x_lo MMA
  const float *b1, *W2, *b2;  // in the parameter arena
  float *out;
  long long *prof;  // NF_ITC_PROF: per-CTA wait-time counters of the stacked kernel (16 per CTA)
};

#define ITC_T0() const long long t0_ = p.prof ? clock64() : 0
#define ITC_ACC(v) do { if (p.prof) v += clock64() - t0_; } while (0)

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
// D (TMEM) += A (TMEM, M = 128 lanes x 8 columns) * B (shared-memory descriptor)
__device__ __forceinline__ void mma_tf32_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t db, uint32_t idesc,
                                            uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}"
      ::"r"(tmem_d), "r"(tmem_a), "l"(db), "r"(idesc), "r"(acc));
}

__global__ void __launch_bounds__(kThreads, 1)
infer_tc_kernel(const InferTcParams p, const __grid_constant__ CUtensorMap tmX,
                const __grid_constant__ CUtensorMap tmWh, const __grid_constant__ CUtensorMap tmWl) {
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t *ring = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  uint8_t *wring = ring + kStages * kXBytes;
  float *W2s = reinterpret_cast<float *>(wring + kWStages * kWStageBytes);  // [32][33]
  float *b1s = W2s + 32 * 33, *b2s = b1s + 32;
  uint64_t *full = reinterpret_cast<uint64_t *>(b2s + 32);
  uint64_t *empty = full + kStages, *tfull = empty + kStages, *tempty = tfull + kTStages;
  uint64_t *afull = tempty + kTStages, *aempty = afull + 2;
  uint64_t *wfull = aempty + 2, *wempty = wfull + kWStages;
  uint32_t *tslot = reinterpret_cast<uint32_t *>(wempty + kWStages);
  const int tid = threadIdx.x, warp = ptx::warp_uniform(tid >> 5), lane = tid & 31;

  // this CTA's rows: an equal share of the rows (+-1; a TMA box may start at any row, and the rows a
  // last box reads past r1 -- the next CTA's, or zero fill past n -- are computed and not stored)
  const int64_t r0 = (int64_t)blockIdx.x * p.n / gridDim.x, r1 = (int64_t)(blockIdx.x + 1) * p.n / gridDim.x;
  const int ntiles = r1 > r0 ? (int)((r1 - r0 + kTileRows - 1) / kTileRows) : 0;

  if (tid == 0) {
    for (int i = 0; i < kStages; ++i) {
      ptx::mbar_init(&full[i], 1);
      ptx::mbar_init(&empty[i], 4);  // one converter group's four warps have read the x tile
    }
    for (int i = 0; i < kWStages; ++i) {
      ptx::mbar_init(&wfull[i], 1);
      ptx::mbar_init(&wempty[i], 1);  // the MMA commit
    }
    for (int i = 0; i < kTStages; ++i) {
      ptx::mbar_init(&tfull[i], 4);
      ptx::mbar_init(&tempty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&afull[i], 1);
      ptx::mbar_init(&aempty[i], 4);
    }
    ptx::fence_mbar_init();
    // the first ring-full of x K-blocks (all of tile 0) goes out before the rest of the prologue
    // (TMEM allocation, W2 / bias staging): its HBM latency overlaps the set-up
    if (ntiles > 0) {
      const int64_t rows_here = r1 - r0 < kTileRows ? r1 - r0 : kTileRows;
      const int nbox = (int)((rows_here + kBoxRows - 1) / kBoxRows);
      for (int g = 0; g < kStages && g < p.nkb; ++g) {
        ptx::mbar_arrive_expect_tx(&full[g], (uint32_t)(nbox * kBoxRows * kKB * 4));
        for (int b = 0; b < nbox; ++b)
          ptx::tma_load_2d(ring + g * kXBytes + b * (kBoxRows * 128), &tmX, &full[g], g * kKB, (int)(r0 + b * kBoxRows));
      }
    }
    ptx::prefetch_tensormap(&tmWh);
    ptx::prefetch_tensormap(&tmWl);
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(ptx::smem_u32(tslot)),
                 "r"(512u) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  for (int i = tid; i < 32 * 32; i += kThreads) {
    const int o = i >> 5, j = i & 31;
    W2s[o * 33 + j] = (o < p.O && j < p.H) ? p.W2[o * p.H + j] : 0.0f;
  }
  if (tid < 32) {
    b1s[tid] = tid < p.H ? p.b1[tid] : 0.0f;
    b2s[tid] = tid < p.O ? p.b2[tid] : 0.0f;
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tslot;
  const long long tstart = p.prof ? clock64() : 0;
  long long w0 = 0, w1 = 0, w2 = 0;
  long long *prof = p.prof ? p.prof + 16 * blockIdx.x : nullptr;

  if (warp == 0) {
    // ---- TMA producer of the x tiles (all lanes run the loop, one elected lane issues; the first
    //      kStages K-blocks went out in the prologue)
    int g = 0, s = 0;
    uint32_t par = 1;  // parity of the 'empty' phase to wait for (first pass: passes at once)
    for (int i = 0; i < ntiles; ++i) {
      const int64_t row = r0 + (int64_t)i * kTileRows;
      const int64_t rows_here = r1 - row < kTileRows ? r1 - row : kTileRows;
      const int nbox = (int)((rows_here + kBoxRows - 1) / kBoxRows);
      for (int kb = 0; kb < p.nkb; ++kb, ++g) {
        if (g >= kStages || g >= p.nkb) {
          { ITC_T0(); ptx::mbar_wait(&empty[s], par); ITC_ACC(w0); }
          if (ptx::elect_one()) {
            uint8_t *st = ring + s * kXBytes;
            ptx::mbar_arrive_expect_tx(&full[s], (uint32_t)(nbox * kBoxRows * kKB * 4));
            for (int b = 0; b < nbox; ++b)
              ptx::tma_load_2d(st + b * (kBoxRows * 128), &tmX, &full[s], kb * kKB, (int)(row + b * kBoxRows));
          }
          __syncwarp();
        }
        if (++s == kStages) { s = 0; par ^= 1; }
      }
    }
    if (prof && lane == 0) prof[0] = w0;
  } else if (warp == kThreads / 32 - 1) {
    // ---- TMA producer of the W1 hi | lo K-blocks (L2-resident)
    if (lane == 0 && !(p.exp & 8)) {
      int g = 0;
      for (int i = 0; i < ntiles; ++i) {
        for (int kb = 0; kb < p.nkb; ++kb, ++g) {
          const int w = g % kWStages;
          { ITC_T0(); ptx::mbar_wait(&wempty[w], ((g / kWStages) & 1) ^ 1); ITC_ACC(w0); }
          uint8_t *st = wring + w * kWStageBytes;
          if ((p.exp & 1) && g >= kWStages) {  // (timing experiment: no reload)
            ptx::mbar_arrive(&wfull[w]);
            continue;
          }
          ptx::mbar_arrive_expect_tx(&wfull[w], (uint32_t)kWStageBytes);
          ptx::tma_load_2d(st, &tmWh, &wfull[w], kb * kKB, 0);
          ptx::tma_load_2d(st + kWBytes, &tmWl, &wfull[w], kb * kKB, 0);
        }
      }
      if (prof) prof[1] = w0;
    }
  } else if (warp == 1) {
    // ---- MMA issuer: the whole warp runs the loop and the barrier waits (warp-uniform control flow
    //      and operands: descriptors / tensor-memory addresses stay in uniform registers), one
    //      elected lane issues the tcgen05 instructions
    if (!(p.exp & 8)) {
      constexpr uint32_t idesc = tc::idesc_tf32(kTileRows, 64, false, false);  // N = 64: W1 hi rows | W1 lo rows
      const uint32_t tmem_u = (uint32_t)ptx::warp_uniform((int)tmem);
      const uint32_t wring_u = ptx::smem_u32(wring);
      int g = 0, w = 0, t = 0;
      uint32_t wpar = 0, tpar = 0;
      for (int i = 0; i < ntiles; ++i) {
        const int a = i & 1;
        { ITC_T0(); ptx::mbar_wait(&aempty[a], ((i >> 1) & 1) ^ 1); ITC_ACC(w2); }
        tc::tc_fence_after();
        const uint32_t d = tmem_u + kAccCol + 64u * a;
        for (int kb = 0; kb < p.nkb; ++kb, ++g) {
          { ITC_T0(); ptx::mbar_wait(&wfull[w], wpar); ITC_ACC(w0); }    // W K-block landed
          { ITC_T0(); ptx::mbar_wait(&tfull[t], tpar); ITC_ACC(w1); }    // x K-block split into TMEM
          tc::tc_fence_after();
          const uint32_t sw = wring_u + (uint32_t)w * kWStageBytes;
          // B = the stage's 64 rows: W1 hi (rows 0..31) | W1 lo (rows 32..63), so one MMA per x part
          // gives x W_hi in accumulator columns 0..31 and x W_lo in 32..63 (all four partial products)
          const uint64_t bw = tc::smem_desc(sw, 16, 1024, 2);
          const uint32_t ah = tmem_u + 64u * (uint32_t)t;
          if (ptx::elect_one()) {
#pragma unroll
            for (int ks = 0; ks < kKB / 8; ++ks) {
              if (p.exp & 2) break;
              if (!(p.exp & 16)) mma_tf32_ts(d, ah + 8u * ks + 32u, bw + 2u * ks, idesc, (kb | ks) ? 1u : 0u);  // small terms first
              mma_tf32_ts(d, ah + 8u * ks, bw + 2u * ks, idesc, (p.exp & 16) ? ((kb | ks) ? 1u : 0u) : 1u);
            }
            tc::mma_commit(&wempty[w]);
            tc::mma_commit(&tempty[t]);
            if (kb == p.nkb - 1) tc::mma_commit(&afull[a]);
          }
          __syncwarp();
          if (++w == kWStages) { w = 0; wpar ^= 1; }
          if (++t == kTStages) { t = 0; tpar ^= 1; }
        }
      }
      if (prof && lane == 0) { prof[2] = w0; prof[3] = w1; prof[4] = w2; }
    }
  } else if (warp < 2 + 4 * kCG) {
    // ---- converters: thread = row 32 q + lane of the tile (TMEM lane quadrant q = warp % 4); group
    //      cg takes the K-blocks g = cg mod kCG
    const int q = warp & 3, cg = (warp - 2) >> 2;
    int g = 0;
    for (int i = 0; i < ntiles; ++i) {
      for (int kb = 0; kb < p.nkb; ++kb, ++g) {
        if (g % kCG != cg) continue;
        const int s = g % kStages, t = g % kTStages;
        { ITC_T0(); ptx::mbar_wait(&full[s], (g / kStages) & 1); ITC_ACC(w0); }
        if (p.exp & 8) {  // (timing experiment: x streaming alone)
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(&empty[s]);
          continue;
        }
        { ITC_T0(); ptx::mbar_wait(&tempty[t], ((g / kTStages) & 1) ^ 1); ITC_ACC(w1); }
        // this row's 128 B in the swizzled box q: 16-B chunk c at physical chunk c ^ (row % 8)
        const uint8_t *xr = ring + s * kXBytes + q * (kBoxRows * 128) + lane * 128;
        float hi[32], lo[32];
        if (!(p.exp & 4)) {
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const float4 v = *reinterpret_cast<const float4 *>(xr + ((c ^ (lane & 7)) << 4));
          const float xv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            hi[4 * c + e] = __uint_as_float(__float_as_uint(xv[e]) & 0xffffe000u);
            lo[4 * c + e] = tf32_lo(xv[e]);
          }
        }
        const uint32_t ta = tmem + ((uint32_t)(32 * q) << 16) + 64u * t;
        tmem_st32(ta, hi);
        tmem_st32(ta + 32u, lo);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        }
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          ptx::mbar_arrive(&empty[s]);
          ptx::mbar_arrive(&tfull[t]);
        }
      }
    }
    if (prof && tid == 64) { prof[5] = w0; prof[6] = w1; }
  } else if (warp < 2 + 4 * kCG + 4 && !(p.exp & 8)) {
    // ---- epilogue: thread = row 32 q + lane of the tile
    const int q = warp & 3;
    const int H = p.H, O = p.O;
    for (int i = 0; i < ntiles; ++i) {
      const int a = i & 1;
      { ITC_T0(); ptx::mbar_wait(&afull[a], (i >> 1) & 1); ITC_ACC(w0); }
      tc::tc_fence_after();
      float z[32], zl[32];
      tc::tmem_ld32(tmem + ((uint32_t)(32 * q) << 16) + kAccCol + 64u * a, z);
      tc::tmem_ld32(tmem + ((uint32_t)(32 * q) << 16) + kAccCol + 64u * a + 32u, zl);
#pragma unroll
      for (int j = 0; j < 32; ++j) z[j] += zl[j];
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&aempty[a]);
      const int64_t row = r0 + (int64_t)i * kTileRows + 32 * q + lane;
      if (row < r1) {
        float a1[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) a1[j] = j < H ? act_only(p.act_h, z[j] + b1s[j]) : 0.0f;
        float *orow = p.out + row * O;
        for (int o = 0; o < O; ++o) {
          const float *w2 = W2s + o * 33;
          float c0 = b2s[o], c1 = 0.0f, c2 = 0.0f, c3 = 0.0f;
#pragma unroll
          for (int j = 0; j < 32; j += 4) {
            c0 = fmaf(w2[j], a1[j], c0);
            c1 = fmaf(w2[j + 1], a1[j + 1], c1);
            c2 = fmaf(w2[j + 2], a1[j + 2], c2);
            c3 = fmaf(w2[j + 3], a1[j + 3], c3);
          }
          orow[o] = act_only(p.act_o, (c0 + c1) + (c2 + c3));
        }
      }
    }
  }
  if (prof && warp == 2 + 4 * kCG && lane == 0) { prof[7] = w0; prof[9] = clock64() - tstart; }
  tc::tc_fence_before();
  __syncthreads();
  if (prof && tid == 0) { prof[8] = clock64() - tstart; prof[10] = ntiles * p.nkb; }
  if (warp == 1) {
    tc::tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512u) : "memory");
  }
}

// ---- transposed formulation (infer_tcT_kernel, the default): Z1^T = W1 X^T, one MMA per
// (M = 128 neuron lanes, N = 128 rows, K = 8 pixels): a quarter of the M=128 x N=32 instructions
// per row (the instruction cost, not the MMA width, bounds the N = 32 form).  W1 (30 rows of the
// A operand) is read through a K-major descriptor whose rows 32..127 fall on neighbouring shared
// memory: those accumulator lanes are garbage and never read.  x is the B operand straight from
// its TMA tile (the tensor core truncates it: the hi part), the converters write x_lo =
// rn_tf32(x - trunc(x)) into a second tile of the same swizzled layout (elementwise, conflict-free).
// One warp reads the accumulator (lanes = neurons 0..31, columns = rows) and transposes it through
// shared memory; the epilogue warps (thread = row) finish layers 1 and 2.
namespace tt {
#ifndef NF_ITT_ROWS
#define NF_ITT_ROWS 128
#endif
constexpr int kRows = NF_ITT_ROWS;                // rows per tile = N of the MMA (128 or 256)
constexpr int kStages = kRows == 256 ? 2 : 4;
constexpr int kXBytes = kRows * kKB * 4;          // 16 KB
constexpr int kWBytes = 32 * kKB * 4;             // 4 KB: the 32 rows TMA writes of a W K-block
constexpr int kStageBytes = 2 * kXBytes + 2 * kWBytes;   // x | x_lo | W hi | W lo = 40 KB
constexpr int kOverread = 128 * 128 - kWBytes;    // A descriptor rows 32..127 past the last W block
constexpr int kThreads = 32 * (1 + 1 + 4 + 4);    // TMA, MMA, 4 converter warps, 4 epilogue warps
constexpr int kSmem = 1024 + kStages * kStageBytes + kOverread + (kRows * 33 + 32 * 33 + 64) * 4 + 256;
}  // namespace tt

__global__ void __launch_bounds__(tt::kThreads, 1)
infer_tcT_kernel(const InferTcParams p, const __grid_constant__ CUtensorMap tmX,
                 const __grid_constant__ CUtensorMap tmWh, const __grid_constant__ CUtensorMap tmWl) {
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t *ring = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  float *zt = reinterpret_cast<float *>(ring + tt::kStages * tt::kStageBytes + tt::kOverread);  // [rows][33]
  float *W2s = zt + tt::kRows * 33;                 // [32][33]
  float *b1s = W2s + 32 * 33, *b2s = b1s + 32;
  uint64_t *full = reinterpret_cast<uint64_t *>(b2s + 32);
  uint64_t *cvt = full + tt::kStages, *empty = cvt + tt::kStages, *afull = empty + tt::kStages, *aempty = afull + 2;
  uint32_t *tslot = reinterpret_cast<uint32_t *>(aempty + 2);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  const int64_t bb = (int64_t)blockIdx.x * p.nblk / gridDim.x, be = (int64_t)(blockIdx.x + 1) * p.nblk / gridDim.x;
  const int64_t r0 = bb * kBoxRows, r1 = min(p.n, be * kBoxRows);
  const int ntiles = r1 > r0 ? (int)((r1 - r0 + tt::kRows - 1) / tt::kRows) : 0;

  if (tid == 0) {
    for (int i = 0; i < tt::kStages; ++i) {
      ptx::mbar_init(&full[i], 1);
      ptx::mbar_init(&cvt[i], 4);
      ptx::mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&afull[i], 1);
      ptx::mbar_init(&aempty[i], 1);
    }
    ptx::fence_mbar_init();
    ptx::prefetch_tensormap(&tmX);
    ptx::prefetch_tensormap(&tmWh);
    ptx::prefetch_tensormap(&tmWl);
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(ptx::smem_u32(tslot)),
                 "r"((uint32_t)(2 * tt::kRows)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  for (int i = tid; i < 32 * 32; i += tt::kThreads) {
    const int o = i >> 5, j = i & 31;
    W2s[o * 33 + j] = (o < p.O && j < p.H) ? p.W2[o * p.H + j] : 0.0f;
  }
  if (tid < 32) {
    b1s[tid] = tid < p.H ? p.b1[tid] : 0.0f;
    b2s[tid] = tid < p.O ? p.b2[tid] : 0.0f;
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tslot;
  auto sx = [&](int s) { return ring + s * tt::kStageBytes; };           // x tile (B hi)
  auto sxl = [&](int s) { return ring + s * tt::kStageBytes + tt::kXBytes; };  // x_lo tile (B lo)
  auto swh = [&](int s) { return ring + s * tt::kStageBytes + 2 * tt::kXBytes; };
  auto swl = [&](int s) { return ring + s * tt::kStageBytes + 2 * tt::kXBytes + tt::kWBytes; };

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA: x tile (4 boxes of 32 rows) + W1 hi / lo K-blocks
      int g = 0;
      for (int i = 0; i < ntiles; ++i) {
        const int64_t row = r0 + (int64_t)i * tt::kRows;
        const int64_t rows_here = r1 - row < tt::kRows ? r1 - row : tt::kRows;
        const int nbox = (int)((rows_here + kBoxRows - 1) / kBoxRows);
        for (int kb = 0; kb < p.nkb; ++kb, ++g) {
          const int s = g % tt::kStages;
          ptx::mbar_wait(&empty[s], ((g / tt::kStages) & 1) ^ 1);
          ptx::mbar_arrive_expect_tx(&full[s], (uint32_t)(nbox * kBoxRows * 128 + 2 * tt::kWBytes));
          for (int b = 0; b < nbox; ++b)
            ptx::tma_load_2d(sx(s) + b * (kBoxRows * 128), &tmX, &full[s], kb * kKB, (int)(row + b * kBoxRows));
          ptx::tma_load_2d(swh(s), &tmWh, &full[s], kb * kKB, 0);
          ptx::tma_load_2d(swl(s), &tmWl, &full[s], kb * kKB, 0);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer
      constexpr uint32_t idesc = tc::idesc_tf32(128, tt::kRows, false, false);
      int g = 0;
      for (int i = 0; i < ntiles; ++i) {
        const int a = i & 1;
        ptx::mbar_wait(&aempty[a], ((i >> 1) & 1) ^ 1);
        tc::tc_fence_after();
        const uint32_t d = tmem + (uint32_t)(tt::kRows * a);
        for (int kb = 0; kb < p.nkb; ++kb, ++g) {
          const int s = g % tt::kStages;
          ptx::mbar_wait(&cvt[s], (g / tt::kStages) & 1);  // (x landed and its lo part written)
          tc::tc_fence_after();
          const uint32_t xh = ptx::smem_u32(sx(s)), xl = ptx::smem_u32(sxl(s));
          const uint32_t wh = ptx::smem_u32(swh(s)), wl = ptx::smem_u32(swl(s));
#pragma unroll
          for (int ks = 0; ks < kKB / 8; ++ks) {
            if (p.exp & 2) break;
            const uint64_t dwh = tc::smem_desc(wh + 32u * ks, 16, 1024, 2), dwl = tc::smem_desc(wl + 32u * ks, 16, 1024, 2);
            const uint64_t dxh = tc::smem_desc(xh + 32u * ks, 16, 1024, 2), dxl = tc::smem_desc(xl + 32u * ks, 16, 1024, 2);
            tc::mma_tf32(d, dwh, dxl, idesc, (kb | ks) ? 1u : 0u);  // small terms first
            tc::mma_tf32(d, dwl, dxh, idesc, 1u);
            tc::mma_tf32(d, dwh, dxh, idesc, 1u);
          }
          tc::mma_commit(&empty[s]);
          if (kb == p.nkb - 1) tc::mma_commit(&afull[a]);
        }
      }
    }
  } else if (warp < 6) {
    // ---- converters: x_lo = rn_tf32(x - trunc(x)), elementwise over the swizzled tile (the
    //      layouts match: same byte offset), 128 B per thread per K-block
    const int ct = tid - 64;
    int g = 0;
    for (int i = 0; i < ntiles; ++i) {
      for (int kb = 0; kb < p.nkb; ++kb, ++g) {
        const int s = g % tt::kStages;
        ptx::mbar_wait(&full[s], (g / tt::kStages) & 1);
        const float4 *src = reinterpret_cast<const float4 *>(sx(s));
        float4 *dst = reinterpret_cast<float4 *>(sxl(s));
#pragma unroll
        for (int c = 0; c < tt::kXBytes / 16 / 128; ++c) {
          if (p.exp & 4) break;
          const float4 v = src[ct + 128 * c];
          dst[ct + 128 * c] = make_float4(tf32_lo(v.x), tf32_lo(v.y), tf32_lo(v.z), tf32_lo(v.w));
        }
        ptx::fence_proxy_async_smem();  // generic-proxy writes -> visible to the tensor core
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&cvt[s]);
      }
    }
  } else {
    // ---- epilogue: warp 6 + (the warp of TMEM lane quadrant 0) reads Z1^T rows 0..31 (neurons)
    //      x 128 columns (rows) and transposes them into zt; then thread = row finishes
    const int q = warp & 3, et = tid - 192;  // q == 0: warp 8
    const int H = p.H, O = p.O;
    for (int i = 0; i < ntiles; ++i) {
      const int a = i & 1;
      if (q == 0) {
        ptx::mbar_wait(&afull[a], (i >> 1) & 1);
        tc::tc_fence_after();
#pragma unroll
        for (int c0 = 0; c0 < tt::kRows; c0 += 32) {
          float z[32];
          tc::tmem_ld32(tmem + (uint32_t)(tt::kRows * a + c0), z);  // lane = neuron, z[c] = row c0 + c
#pragma unroll
          for (int c = 0; c < 32; ++c) zt[(c0 + c) * 33 + lane] = z[c];
        }
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&aempty[a]);
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");  // zt filled
      for (int rr = et; rr < tt::kRows; rr += 128) {
      const int64_t row = r0 + (int64_t)i * tt::kRows + rr;
      if (row < r1) {
        float a1[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) a1[j] = j < H ? act_only(p.act_h, zt[rr * 33 + j] + b1s[j]) : 0.0f;
        float *orow = p.out + row * O;
        for (int o = 0; o < O; ++o) {
          const float *w2 = W2s + o * 33;
          float c0 = b2s[o], c1 = 0.0f, c2 = 0.0f, c3 = 0.0f;
#pragma unroll
          for (int j = 0; j < 32; j += 4) {
            c0 = fmaf(w2[j], a1[j], c0);
            c1 = fmaf(w2[j + 1], a1[j + 1], c1);
            c2 = fmaf(w2[j + 2], a1[j + 2], c2);
            c3 = fmaf(w2[j + 3], a1[j + 3], c3);
          }
          orow[o] = act_only(p.act_o, (c0 + c1) + (c2 + c3));
        }
      }
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");  // zt free for the next tile
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc::tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"((uint32_t)(2 * tt::kRows)) : "memory");
  }
}

// ---- stacked formulation (infer_tcS_kernel, the default): the transposed contraction with the
// W1 hi and lo parts STACKED along M.  The A descriptor's 128 rows read W1_hi (rows 0..31) and,
// right behind it in shared memory, W1_lo (rows 32..63), so ONE MMA against an x operand gives
// W_hi x in accumulator lanes 0..31 and W_lo x in lanes 32..63 -- the M = 128 instruction costs the
// same as before (the tensor core's floor is max(M,128) N / 256 cycles) but the separate W_lo MMA is
// gone: 2 MMAs per k-step (x_hi, x_lo) instead of 3, and the lo*lo term comes for free (all four
// partial products; lanes 64..127 read neighbouring shared memory and are never looked at).  The
// epilogue adds the two lane groups.  Rings by lifetime: the x tiles (HBM latency) in a 6-deep ring,
// the x_lo tiles the converters write and the W1 K-blocks (L2-resident) in 3-deep rings, all freed
// by the MMA commits; the W1 producer is its own warp so its short ring never delays an x load.
// The last tile of a CTA issues MMAs only as wide (N) as its rows.
namespace ts {
constexpr int kRows = 128;
constexpr int kXS = 6, kLS = 3;                      // x ring / (x_lo, W) ring depths
constexpr int kXBytes = kRows * kKB * 4;             // 16 KB
constexpr int kWStage = 2 * 32 * kKB * 4;            // 8 KB: W hi rows 0..31 | W lo rows 32..63
constexpr int kCvtWarps = 8;
constexpr int kThreads = 32 * (2 + kCvtWarps + 4 + 1);   // x TMA, MMA, converters, epilogue, W TMA
constexpr int kZt = kRows * 33;                      // floats per transposed accumulator half
// the A descriptor of the last W stage reads 8 KB past it: into zt (any bit pattern will do)
constexpr int kSmem = 1024 + kXS * kXBytes + kLS * kXBytes + kLS * kWStage + (2 * kZt + 32 * 33 + 64) * 4 + 256;
static_assert(2 * kZt * 4 >= 128 * 128 - kWStage, "A over-read must stay inside the CTA's shared memory");
static_assert(kSmem <= 232448, "shared memory");
}  // namespace ts

__global__ void __launch_bounds__(ts::kThreads, 1)
infer_tcS_kernel(const InferTcParams p, const __grid_constant__ CUtensorMap tmX,
                 const __grid_constant__ CUtensorMap tmWh, const __grid_constant__ CUtensorMap tmWl) {
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t *xring = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  uint8_t *lring = xring + ts::kXS * ts::kXBytes;
  uint8_t *wring = lring + ts::kLS * ts::kXBytes;
  float *zt = reinterpret_cast<float *>(wring + ts::kLS * ts::kWStage);   // [2][rows][33]
  float *W2s = zt + 2 * ts::kZt;                    // [32][33]
  float *b1s = W2s + 32 * 33, *b2s = b1s + 32;
  uint64_t *xfull = reinterpret_cast<uint64_t *>(b2s + 32);
  uint64_t *xempty = xfull + ts::kXS, *lfull = xempty + ts::kXS, *wfull = lfull + ts::kLS, *mdone = wfull + ts::kLS;
  uint64_t *afull = mdone + ts::kLS, *aempty = afull + 2;
  uint32_t *tslot = reinterpret_cast<uint32_t *>(aempty + 2);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  const int64_t bb = (int64_t)blockIdx.x * p.nblk / gridDim.x, be = (int64_t)(blockIdx.x + 1) * p.nblk / gridDim.x;
  const int64_t r0 = bb * kBoxRows, r1 = min(p.n, be * kBoxRows);
  const int ntiles = r1 > r0 ? (int)((r1 - r0 + ts::kRows - 1) / ts::kRows) : 0;

  if (tid == 0) {
    for (int i = 0; i < ts::kXS; ++i) {
      ptx::mbar_init(&xfull[i], 1);
      ptx::mbar_init(&xempty[i], 1);
    }
    for (int i = 0; i < ts::kLS; ++i) {
      ptx::mbar_init(&lfull[i], ts::kCvtWarps);
      ptx::mbar_init(&wfull[i], 1);
      ptx::mbar_init(&mdone[i], 1);   // the MMAs of this x_lo / W slot have completed
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&afull[i], 1);
      ptx::mbar_init(&aempty[i], 2);
    }
    ptx::fence_mbar_init();
    ptx::prefetch_tensormap(&tmX);
    ptx::prefetch_tensormap(&tmWh);
    ptx::prefetch_tensormap(&tmWl);
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(ptx::smem_u32(tslot)),
                 "r"((uint32_t)(2 * ts::kRows)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  for (int i = tid; i < 32 * 32; i += ts::kThreads) {
    const int o = i >> 5, j = i & 31;
    W2s[o * 33 + j] = (o < p.O && j < p.H) ? p.W2[o * p.H + j] : 0.0f;
  }
  for (int i = tid; i < 2 * ts::kZt; i += ts::kThreads) zt[i] = 0.0f;
  if (tid < 32) {
    b1s[tid] = tid < p.H ? p.b1[tid] : 0.0f;
    b2s[tid] = tid < p.O ? p.b2[tid] : 0.0f;
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tslot;
  const long long tstart = p.prof ? clock64() : 0;
  long long w0 = 0, w1 = 0, w2 = 0;
  long long *prof = p.prof ? p.prof + 16 * blockIdx.x : nullptr;

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA: x tiles (boxes of 32 rows)
      int g = 0;
      for (int i = 0; i < ntiles; ++i) {
        const int64_t row = r0 + (int64_t)i * ts::kRows;
        const int64_t rows_here = r1 - row < ts::kRows ? r1 - row : ts::kRows;
        const int nbox = (int)((rows_here + kBoxRows - 1) / kBoxRows);
        for (int kb = 0; kb < p.nkb; ++kb, ++g) {
          const int s = g % ts::kXS;
          { ITC_T0(); ptx::mbar_wait(&xempty[s], ((g / ts::kXS) & 1) ^ 1); ITC_ACC(w0); }
          uint8_t *st = xring + s * ts::kXBytes;
          ptx::mbar_arrive_expect_tx(&xfull[s], (uint32_t)(nbox * kBoxRows * 128));
          for (int b = 0; b < nbox; ++b)
            ptx::tma_load_2d(st + b * (kBoxRows * 128), &tmX, &xfull[s], kb * kKB, (int)(row + b * kBoxRows));
        }
      }
      if (prof) prof[0] = w0;
    }
  } else if (warp == ts::kThreads / 32 - 1) {
    if (lane == 0) {  // ---- TMA: W1 hi | lo K-blocks
      const int total = ntiles * p.nkb;
      for (int g = 0; g < total; ++g) {
        const int w = g % ts::kLS, kb = g % p.nkb;
        { ITC_T0(); ptx::mbar_wait(&mdone[w], ((g / ts::kLS) & 1) ^ 1); ITC_ACC(w0); }
        uint8_t *st = wring + w * ts::kWStage;
        ptx::mbar_arrive_expect_tx(&wfull[w], (uint32_t)ts::kWStage);
        ptx::tma_load_2d(st, &tmWh, &wfull[w], kb * kKB, 0);
        ptx::tma_load_2d(st + ts::kWStage / 2, &tmWl, &wfull[w], kb * kKB, 0);
      }
      if (prof) prof[1] = w0;
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer
      int g = 0;
      for (int i = 0; i < ntiles; ++i) {
        const int a = i & 1;
        const int64_t left = r1 - (r0 + (int64_t)i * ts::kRows);
        const int nn = left >= ts::kRows ? ts::kRows : (int)((left + 15) & ~int64_t(15));   // N: multiple of 16
        const uint32_t idesc = tc::idesc_tf32(128, nn, false, false);
        { ITC_T0(); ptx::mbar_wait(&aempty[a], ((i >> 1) & 1) ^ 1); ITC_ACC(w2); }
        tc::tc_fence_after();
        const uint32_t d = tmem + (uint32_t)(ts::kRows * a);
        for (int kb = 0; kb < p.nkb; ++kb, ++g) {
          const int s = g % ts::kXS, w = g % ts::kLS;
          { ITC_T0(); ptx::mbar_wait(&wfull[w], (g / ts::kLS) & 1); ITC_ACC(w0); }
          { ITC_T0(); ptx::mbar_wait(&lfull[w], (g / ts::kLS) & 1); ITC_ACC(w1); }  // x landed and its lo part written
          tc::tc_fence_after();
          const uint32_t xh = ptx::smem_u32(xring + s * ts::kXBytes), xl = ptx::smem_u32(lring + w * ts::kXBytes);
          const uint32_t ws = ptx::smem_u32(wring + w * ts::kWStage);
#pragma unroll
          for (int ks = 0; ks < kKB / 8; ++ks) {
            if (p.exp & 2) break;
            const uint64_t dw = tc::smem_desc(ws + 32u * ks, 16, 1024, 2);
            const uint64_t dxh = tc::smem_desc(xh + 32u * ks, 16, 1024, 2), dxl = tc::smem_desc(xl + 32u * ks, 16, 1024, 2);
            tc::mma_tf32(d, dw, dxl, idesc, (kb | ks) ? 1u : 0u);  // small terms first
            tc::mma_tf32(d, dw, dxh, idesc, 1u);
          }
          tc::mma_commit(&xempty[s]);
          tc::mma_commit(&mdone[w]);
          if (kb == p.nkb - 1) tc::mma_commit(&afull[a]);
        }
      }
      if (prof) { prof[2] = w0; prof[3] = w1; prof[4] = w2; }
    }
  } else if (warp < 2 + ts::kCvtWarps) {
    // ---- converters: x_lo = rn_tf32(x - trunc(x)), elementwise over the swizzled tile (the
    //      layouts match: same byte offset), 64 B per thread per K-block
    const int ct = tid - 64;
    const int total = ntiles * p.nkb;
    for (int g = 0; g < total; ++g) {
      const int s = g % ts::kXS, w = g % ts::kLS;
      { ITC_T0(); ptx::mbar_wait(&xfull[s], (g / ts::kXS) & 1); ITC_ACC(w0); }
      { ITC_T0(); ptx::mbar_wait(&mdone[w], ((g / ts::kLS) & 1) ^ 1); ITC_ACC(w1); }
      const float4 *src = reinterpret_cast<const float4 *>(xring + s * ts::kXBytes);
      float4 *dst = reinterpret_cast<float4 *>(lring + w * ts::kXBytes);
      float4 v[ts::kXBytes / 16 / (32 * ts::kCvtWarps)];
#pragma unroll
      for (int c = 0; c < ts::kXBytes / 16 / (32 * ts::kCvtWarps); ++c) v[c] = src[ct + 32 * ts::kCvtWarps * c];
#pragma unroll
      for (int c = 0; c < ts::kXBytes / 16 / (32 * ts::kCvtWarps); ++c) {
        if (p.exp & 4) break;
        dst[ct + 32 * ts::kCvtWarps * c] = make_float4(tf32_lo(v[c].x), tf32_lo(v[c].y), tf32_lo(v[c].z), tf32_lo(v[c].w));
      }
      ptx::fence_proxy_async_smem();  // generic-proxy writes -> visible to the tensor core
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&lfull[w]);
    }
    if (prof && tid == 64) { prof[5] = w0; prof[6] = w1; }
  } else {
    // ---- epilogue: the warps of TMEM lane quadrants 0 and 1 read Z1^T lanes 0..31 (W_hi x) and
    //      32..63 (W_lo x) and transpose them into zt[0] / zt[1]; then thread = row finishes
    const int q = warp & 3, et = tid - 32 * (2 + ts::kCvtWarps);
    const int H = p.H, O = p.O;
    for (int i = 0; i < ntiles; ++i) {
      const int a = i & 1;
      const int64_t left = r1 - (r0 + (int64_t)i * ts::kRows);
      const int nn = left >= ts::kRows ? ts::kRows : (int)((left + 15) & ~int64_t(15));
      if (q < 2) {
        { ITC_T0(); ptx::mbar_wait(&afull[a], (i >> 1) & 1); ITC_ACC(w0); }
        tc::tc_fence_after();
        float *zq = zt + q * ts::kZt;
        for (int c0 = 0; c0 < nn; c0 += 32) {
          float z[32];
          tc::tmem_ld32(tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(ts::kRows * a + c0), z);  // lane = neuron, z[c] = row c0 + c
#pragma unroll
          for (int c = 0; c < 32; ++c) zq[(c0 + c) * 33 + lane] = z[c];
        }
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&aempty[a]);
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");  // zt filled
      const int64_t row = r0 + (int64_t)i * ts::kRows + et;
      if (row < r1) {
        float a1[32];
#pragma unroll
        for (int j = 0; j < 32; ++j)
          a1[j] = j < H ? act_only(p.act_h, (zt[et * 33 + j] + zt[ts::kZt + et * 33 + j]) + b1s[j]) : 0.0f;
        float *orow = p.out + row * O;
        for (int o = 0; o < O; ++o) {
          const float *w2 = W2s + o * 33;
          float c0 = b2s[o], c1 = 0.0f, c2 = 0.0f, c3 = 0.0f;
#pragma unroll
          for (int j = 0; j < 32; j += 4) {
            c0 = fmaf(w2[j], a1[j], c0);
            c1 = fmaf(w2[j + 1], a1[j + 1], c1);
            c2 = fmaf(w2[j + 2], a1[j + 2], c2);
            c3 = fmaf(w2[j + 3], a1[j + 3], c3);
          }
          orow[o] = act_only(p.act_o, (c0 + c1) + (c2 + c3));
        }
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");  // zt free for the next tile
    }
    if (prof && q == 0 && lane == 0) { prof[7] = w0; prof[9] = clock64() - tstart; }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (prof && tid == 0) { prof[8] = clock64() - tstart; prof[10] = ntiles * p.nkb; }
  if (warp == 1) {
    tc::tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"((uint32_t)(2 * ts::kRows)) : "memory");
  }
}

// ---- x as the shared-memory A operand (infer_tcX_kernel): Z1 = X [W1_hi ; W1_lo]^T with A = the x
// tile exactly as TMA wrote it (M = 128 rows, K-major SWIZZLE_128B; the tensor core truncates it to
// its TF32 part) and, second MMA of the k-step, A = the x_lo tile the converters write beside it; B =
// the W stage's 64 rows (W1 hi | W1 lo stacked along N), D = 128 lanes (rows) x 64 columns.  No
// tensor-memory staging of x (tcgen05.st) and no transposition in the epilogue (thread = row).
namespace tx {
constexpr int kRows = 128;
constexpr int kXS = 7, kLS = 4;                      // x ring / (x_lo, W) ring depths
constexpr int kXBytes = kRows * kKB * 4;             // 16 KB
constexpr int kWStage = 2 * 32 * kKB * 4;            // 8 KB: W hi rows 0..31 | W lo rows 32..63
constexpr int kCvtWarps = 8;
constexpr int kThreads = 32 * (2 + kCvtWarps + 4 + 1);   // x TMA, MMA, converters, epilogue, W TMA
constexpr int kSmem = 1024 + kXS * kXBytes + kLS * kXBytes + kLS * kWStage + (32 * 33 + 64) * 4 + 256;
static_assert(kSmem <= 232448, "shared memory");
}  // namespace ts

__global__ void __launch_bounds__(tx::kThreads, 1)
infer_tcX_kernel(const InferTcParams p, const __grid_constant__ CUtensorMap tmX,
                 const __grid_constant__ CUtensorMap tmWh, const __grid_constant__ CUtensorMap tmWl) {
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t *xring = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  uint8_t *lring = xring + tx::kXS * tx::kXBytes;
  uint8_t *wring = lring + tx::kLS * tx::kXBytes;
  float *W2s = reinterpret_cast<float *>(wring + tx::kLS * tx::kWStage);   // [32][33]
  float *b1s = W2s + 32 * 33, *b2s = b1s + 32;
  uint64_t *xfull = reinterpret_cast<uint64_t *>(b2s + 32);
  uint64_t *xempty = xfull + tx::kXS, *lfull = xempty + tx::kXS, *wfull = lfull + tx::kLS, *mdone = wfull + tx::kLS;
  uint64_t *afull = mdone + tx::kLS, *aempty = afull + 2;
  uint32_t *tslot = reinterpret_cast<uint32_t *>(aempty + 2);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  const int64_t bb = (int64_t)blockIdx.x * p.nblk / gridDim.x, be = (int64_t)(blockIdx.x + 1) * p.nblk / gridDim.x;
  const int64_t r0 = bb * kBoxRows, r1 = min(p.n, be * kBoxRows);
  const int ntiles = r1 > r0 ? (int)((r1 - r0 + tx::kRows - 1) / tx::kRows) : 0;

  if (tid == 0) {
    for (int i = 0; i < tx::kXS; ++i) {
      ptx::mbar_init(&xfull[i], 1);
      ptx::mbar_init(&xempty[i], 1);
    }
    for (int i = 0; i < tx::kLS; ++i) {
      ptx::mbar_init(&lfull[i], tx::kCvtWarps);
      ptx::mbar_init(&wfull[i], 1);
      ptx::mbar_init(&mdone[i], 1);   // the MMAs of this x_lo / W slot have completed
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&afull[i], 1);
      ptx::mbar_init(&aempty[i], 4);
    }
    ptx::fence_mbar_init();
    ptx::prefetch_tensormap(&tmX);
    ptx::prefetch_tensormap(&tmWh);
    ptx::prefetch_tensormap(&tmWl);
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(ptx::smem_u32(tslot)),
                 "r"(128u) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  for (int i = tid; i < 32 * 32; i += tx::kThreads) {
    const int o = i >> 5, j = i & 31;
    W2s[o * 33 + j] = (o < p.O && j < p.H) ? p.W2[o * p.H + j] : 0.0f;
  }
  if (tid < 32) {
    b1s[tid] = tid < p.H ? p.b1[tid] : 0.0f;
    b2s[tid] = tid < p.O ? p.b2[tid] : 0.0f;
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tslot;
  const long long tstart = p.prof ? clock64() : 0;
  long long w0 = 0, w1 = 0, w2 = 0;
  long long *prof = p.prof ? p.prof + 16 * blockIdx.x : nullptr;

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA: x tiles (boxes of 32 rows)
      int g = 0;
      for (int i = 0; i < ntiles; ++i) {
        const int64_t row = r0 + (int64_t)i * tx::kRows;
        const int64_t rows_here = r1 - row < tx::kRows ? r1 - row : tx::kRows;
        const int nbox = (int)((rows_here + kBoxRows - 1) / kBoxRows);
        for (int kb = 0; kb < p.nkb; ++kb, ++g) {
          const int s = g % tx::kXS;
          { ITC_T0(); ptx::mbar_wait(&xempty[s], ((g / tx::kXS) & 1) ^ 1); ITC_ACC(w0); }
          uint8_t *st = xring + s * tx::kXBytes;
          ptx::mbar_arrive_expect_tx(&xfull[s], (uint32_t)(nbox * kBoxRows * 128));
          for (int b = 0; b < nbox; ++b)
            ptx::tma_load_2d(st + b * (kBoxRows * 128), &tmX, &xfull[s], kb * kKB, (int)(row + b * kBoxRows));
        }
      }
      if (prof) prof[0] = w0;
    }
  } else if (warp == tx::kThreads / 32 - 1) {
    if (lane == 0) {  // ---- TMA: W1 hi | lo K-blocks
      const int total = ntiles * p.nkb;
      for (int g = 0; g < total; ++g) {
        const int w = g % tx::kLS, kb = g % p.nkb;
        { ITC_T0(); ptx::mbar_wait(&mdone[w], ((g / tx::kLS) & 1) ^ 1); ITC_ACC(w0); }
        uint8_t *st = wring + w * tx::kWStage;
        ptx::mbar_arrive_expect_tx(&wfull[w], (uint32_t)tx::kWStage);
        ptx::tma_load_2d(st, &tmWh, &wfull[w], kb * kKB, 0);
        ptx::tma_load_2d(st + tx::kWStage / 2, &tmWl, &wfull[w], kb * kKB, 0);
      }
      if (prof) prof[1] = w0;
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer
      constexpr uint32_t idesc = tc::idesc_tf32(128, 64, false, false);   // N = 64: W1 hi rows | W1 lo rows
      int g = 0;
      for (int i = 0; i < ntiles; ++i) {
        const int a = i & 1;
        { ITC_T0(); ptx::mbar_wait(&aempty[a], ((i >> 1) & 1) ^ 1); ITC_ACC(w2); }
        tc::tc_fence_after();
        const uint32_t d = tmem + 64u * a;
        for (int kb = 0; kb < p.nkb; ++kb, ++g) {
          const int s = g % tx::kXS, w = g % tx::kLS;
          { ITC_T0(); ptx::mbar_wait(&wfull[w], (g / tx::kLS) & 1); ITC_ACC(w0); }
          { ITC_T0(); ptx::mbar_wait(&lfull[w], (g / tx::kLS) & 1); ITC_ACC(w1); }  // x landed and its lo part written
          tc::tc_fence_after();
          const uint32_t xh = ptx::smem_u32(xring + s * tx::kXBytes), xl = ptx::smem_u32(lring + w * tx::kXBytes);
          const uint32_t ws = ptx::smem_u32(wring + w * tx::kWStage);
#pragma unroll
          for (int ks = 0; ks < kKB / 8; ++ks) {
            if (p.exp & 2) break;
            const uint64_t dw = tc::smem_desc(ws + 32u * ks, 16, 1024, 2);
            const uint64_t dxh = tc::smem_desc(xh + 32u * ks, 16, 1024, 2), dxl = tc::smem_desc(xl + 32u * ks, 16, 1024, 2);
            if (!(p.exp & 16)) tc::mma_tf32(d, dxl, dw, idesc, (kb | ks) ? 1u : 0u);  // small terms first
            tc::mma_tf32(d, dxh, dw, idesc, (p.exp & 16) ? ((kb | ks) ? 1u : 0u) : 1u);
          }
          tc::mma_commit(&xempty[s]);
          tc::mma_commit(&mdone[w]);
          if (kb == p.nkb - 1) tc::mma_commit(&afull[a]);
        }
      }
      if (prof) { prof[2] = w0; prof[3] = w1; prof[4] = w2; }
    }
  } else if (warp < 2 + tx::kCvtWarps) {
    // ---- converters: x_lo = rn_tf32(x - trunc(x)), elementwise over the swizzled tile (the
    //      layouts match: same byte offset), 64 B per thread per K-block
    const int ct = tid - 64;
    const int total = ntiles * p.nkb;
    for (int g = 0; g < total; ++g) {
      const int s = g % tx::kXS, w = g % tx::kLS;
      { ITC_T0(); ptx::mbar_wait(&xfull[s], (g / tx::kXS) & 1); ITC_ACC(w0); }
      { ITC_T0(); ptx::mbar_wait(&mdone[w], ((g / tx::kLS) & 1) ^ 1); ITC_ACC(w1); }
      const float4 *src = reinterpret_cast<const float4 *>(xring + s * tx::kXBytes);
      float4 *dst = reinterpret_cast<float4 *>(lring + w * tx::kXBytes);
      float4 v[tx::kXBytes / 16 / (32 * tx::kCvtWarps)];
#pragma unroll
      for (int c = 0; c < tx::kXBytes / 16 / (32 * tx::kCvtWarps); ++c) v[c] = src[ct + 32 * tx::kCvtWarps * c];
#pragma unroll
      for (int c = 0; c < tx::kXBytes / 16 / (32 * tx::kCvtWarps); ++c) {
        if (p.exp & 4) break;
        dst[ct + 32 * tx::kCvtWarps * c] = make_float4(tf32_lo(v[c].x), tf32_lo(v[c].y), tf32_lo(v[c].z), tf32_lo(v[c].w));
      }
      ptx::fence_proxy_async_smem();  // generic-proxy writes -> visible to the tensor core
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&lfull[w]);
    }
    if (prof && tid == 64) { prof[5] = w0; prof[6] = w1; }
  } else {
    // ---- epilogue, thread = row 32 q + lane of the tile: both halves of the Z1 row from TMEM
    const int q = warp & 3;
    const int H = p.H, O = p.O;
    for (int i = 0; i < ntiles; ++i) {
      const int a = i & 1;
      { ITC_T0(); ptx::mbar_wait(&afull[a], (i >> 1) & 1); ITC_ACC(w0); }
      tc::tc_fence_after();
      float z[32], zl[32];
      tc::tmem_ld32(tmem + ((uint32_t)(32 * q) << 16) + 64u * a, z);
      tc::tmem_ld32(tmem + ((uint32_t)(32 * q) << 16) + 64u * a + 32u, zl);
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&aempty[a]);
      const int64_t row = r0 + (int64_t)i * tx::kRows + 32 * q + lane;
      if (row < r1) {
        float a1[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) a1[j] = j < H ? act_only(p.act_h, (z[j] + zl[j]) + b1s[j]) : 0.0f;
        float *orow = p.out + row * O;
        for (int o = 0; o < O; ++o) {
          const float *w2 = W2s + o * 33;
          float c0 = b2s[o], c1 = 0.0f, c2 = 0.0f, c3 = 0.0f;
#pragma unroll
          for (int j = 0; j < 32; j += 4) {
            c0 = fmaf(w2[j], a1[j], c0);
            c1 = fmaf(w2[j + 1], a1[j + 1], c1);
            c2 = fmaf(w2[j + 2], a1[j + 2], c2);
            c3 = fmaf(w2[j + 3], a1[j + 3], c3);
          }
          orow[o] = act_only(p.act_o, (c0 + c1) + (c2 + c3));
        }
      }
    }
    if (prof && q == 0 && lane == 0) { prof[7] = w0; prof[9] = clock64() - tstart; }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (prof && tid == 0) { prof[8] = clock64() - tstart; prof[10] = ntiles * p.nkb; }
  if (warp == 1) {
    tc::tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(128u) : "memory");
  }
}

}  // namespace

bool infer_tc_applicable(const std::vector<int> &dims, const float *X) {
  return dims.size() == 3 && dims[1] <= 32 && dims[2] <= 32 && dims[0] % 4 == 0 && dims[0] >= kKB &&
         (reinterpret_cast<uintptr_t>(X) & 15) == 0 && getenv("NF_INFER_SIMT") == nullptr;
}

cudaError_t infer_tc(cudaStream_t st, const std::vector<int> &dims, int act_h, int act_o, const float *params,
                     const float *W1hi, const float *W1lo, const float *X, int64_t n, float *out) {
  const int n0 = dims[0], H = dims[1], O = dims[2];
  {
    cudaError_t e = set_max_smem(reinterpret_cast<const void *>(infer_tc_kernel), kSmem);
    if (e == cudaSuccess) e = set_max_smem(reinterpret_cast<const void *>(infer_tcT_kernel), tt::kSmem);
    if (e == cudaSuccess) e = set_max_smem(reinterpret_cast<const void *>(infer_tcS_kernel), ts::kSmem);
    if (e == cudaSuccess) e = set_max_smem(reinterpret_cast<const void *>(infer_tcX_kernel), tx::kSmem);
    if (e != cudaSuccess) return e;
  }
  // tensor maps, cached per (pointer, shape): encoding costs host microseconds per call
  static std::mutex mu;
  static struct {
    const void *x = nullptr, *wh = nullptr, *wl = nullptr;
    int64_t n = 0;
    int n0 = 0, H = 0;
    CUtensorMap mX, mWh, mWl;
  } c;
  CUtensorMap mX, mWh, mWl;
  {
    std::lock_guard<std::mutex> lk(mu);
    if (c.x != X || c.n != n || c.n0 != n0) {
      if (!encode_tmap_2d_f32(&c.mX, X, (uint64_t)n0, (uint64_t)n, (uint64_t)n0 * 4, kKB, kBoxRows,
                              CU_TENSOR_MAP_SWIZZLE_128B))
        return cudaErrorInvalidValue;
      c.x = X; c.n = n; c.n0 = n0;
    }
    if (c.wh != W1hi || c.wl != W1lo || c.H != H || c.n0 != n0) {
      if (!encode_tmap_2d_f32(&c.mWh, W1hi, (uint64_t)n0, (uint64_t)H, (uint64_t)n0 * 4, kKB, 32,
                              CU_TENSOR_MAP_SWIZZLE_128B) ||
          !encode_tmap_2d_f32(&c.mWl, W1lo, (uint64_t)n0, (uint64_t)H, (uint64_t)n0 * 4, kKB, 32,
                              CU_TENSOR_MAP_SWIZZLE_128B))
        return cudaErrorInvalidValue;
      c.wh = W1hi; c.wl = W1lo; c.H = H;
    }
    mX = c.mX; mWh = c.mWh; mWl = c.mWl;
  }
  InferTcParams p{};
  p.n = n;
  p.nblk = (n + kBoxRows - 1) / kBoxRows;
  p.n0 = n0; p.H = H; p.O = O; p.act_h = act_h; p.act_o = act_o;
  p.nkb = (n0 + kKB - 1) / kKB;
  p.b1 = params + (int64_t)H * n0;
  p.W2 = p.b1 + H;
  p.b2 = p.W2 + (int64_t)O * H;
  p.out = out;
  p.exp = getenv("NF_ITC_EXP") ? atoi(getenv("NF_ITC_EXP")) : 0;
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(p.nblk, 148));
  static const bool want_prof = getenv("NF_ITC_PROF") != nullptr;
  static long long *dprof = nullptr;
  if (want_prof && !dprof) cudaMalloc(&dprof, 148 * 16 * sizeof(long long));
  if (want_prof) cudaMemsetAsync(dprof, 0, 148 * 16 * sizeof(long long), st);
  p.prof = want_prof ? dprof : nullptr;
  auto report = [&]() {  // wait-time counters (clocks), mean over CTAs, to stderr
    if (!want_prof) return;
    std::vector<long long> h(148 * 16);
    cudaStreamSynchronize(st);
    cudaMemcpy(h.data(), dprof, h.size() * sizeof(long long), cudaMemcpyDeviceToHost);
    static const char *nm[11] = {"xTMA wait xempty", "wTMA wait mdone", "MMA wait wfull", "MMA wait x ready", "MMA wait aempty",
                                 "cvt wait xfull", "cvt wait slot", "epi wait afull", "CTA total", "epi done", "K-blocks"};
    for (int k = 0; k < 11; ++k) {
      double m = 0, mx = 0;
      for (int b = 0; b < blocks; ++b) { m += (double)h[b * 16 + k]; mx = std::max(mx, (double)h[b * 16 + k]); }
      fprintf(stderr, "[itc] %-18s mean %9.0f  max %9.0f\n", nm[k], m / blocks, mx);
    }
  };
  // 0 (default): x from TMEM, W1 hi | lo stacked along N; 1: transposed, 3 MMAs per k-step; 2: transposed, stacked along M
  const int form = getenv("NF_INFER_TC_FORM") ? atoi(getenv("NF_INFER_TC_FORM")) : 0;
  if (form == 3) {  // x as the shared-memory A operand, W1 hi | lo stacked along N
    infer_tcX_kernel<<<blocks, tx::kThreads, tx::kSmem, st>>>(p, mX, mWh, mWl);
    count_launch();
    log_launch(reinterpret_cast<const void *>(infer_tcX_kernel), dim3(blocks), dim3(tx::kThreads), tx::kSmem);
    report();
    return cudaGetLastError();
  }
  if (form == 2) {  // transposed, W1 hi / lo stacked along M: 2 MMAs per k-step
    infer_tcS_kernel<<<blocks, ts::kThreads, ts::kSmem, st>>>(p, mX, mWh, mWl);
    count_launch();
    log_launch(reinterpret_cast<const void *>(infer_tcS_kernel), dim3(blocks), dim3(ts::kThreads), ts::kSmem);
    report();
    return cudaGetLastError();
  }
  if (form == 1) {  // transposed: Z1^T = W1 X^T, N = 128 rows per MMA, 3 MMAs per k-step
    infer_tcT_kernel<<<blocks, tt::kThreads, tt::kSmem, st>>>(p, mX, mWh, mWl);
    count_launch();
    log_launch(reinterpret_cast<const void *>(infer_tcT_kernel), dim3(blocks), dim3(tt::kThreads), tt::kSmem);
    return cudaGetLastError();
  }
  infer_tc_kernel<<<blocks, kThreads, kSmem, st>>>(p, mX, mWh, mWl);
  count_launch();
  log_launch(reinterpret_cast<const void *>(infer_tc_kernel), dim3(blocks), dim3(kThreads), kSmem);
  report();
  return cudaGetLastError();
}

}  // namespace nf
