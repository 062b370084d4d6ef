// gemm_hmma.cuh -- warp-level tensor-core GEMM (mma.sync.m16n8k8 TF32, SASS HMMA) for the small
// contractions of narrow-deep nets (config 4: 2048 x 256 x 256 per layer, 0.27 GFLOP): the
// forward Z = A W^T (K1), the delta D_{l-1} = D_l W_l (K3) and the weight gradient
// G = D^T [A | 1] (K4, the batch co_sum; ones column = bias) of fwdprop / backprop.
//
// Why not tcgen05 here: at N <= 64 a tcgen05 MMA instruction costs ~100-130 cycles whatever its
// size (micro/tc_atmem_test.cu), so a 128 x 64 tile over K = 256 is 32 serial MMAs (~4 K cycles)
// on 64 of the 148 SMs, plus TMA fill and epilogue; HMMA runs 511 MAC/clk/SM at ~21 cycles latency
// with register operands (micro/mma_sync_rate.cu) and spreads the GEMM over every SM.
//
// C[m][n] = sum_k A(m,k) B(n,k), operand layouts and epilogues as gemm_simt (GemmArgs: A(m,k) =
// AK ? A[m*lda+k] : A[k*lda+m]; B(n,k) = BKM ? B[n*ldb+k] : B[k*ldb+n], = 1 for n >= nb_real;
// split-K partials when g.partial).  CTA tile 64 x 64, BK = 32, 256 threads: warp = (32 x 32
// quadrant, K half); the two K halves of a quadrant are summed through shared memory at the end.
// Operand tiles arrive through a 4-stage cp.async ring (a k-tile is only ~256 cycles of MMA per
// SMSP: the loads of the next three tiles must be in flight), stored in their global layout --
// K-major [rows][BK + 4] or MN-major [BK][64 + 8] -- so every fragment read is conflict-free
// (bank = 4g + t, resp. 8t + g).  16-B copies when rows and bases are 16-B aligned, else 4-B.
// Numerics: SPLIT = 1 (NF_MATH_TF32): operands rounded to nearest TF32 in registers, 1 HMMA;
// SPLIT = 3 (fp32 mode): 3xTF32, A truncation-split, B RN-split (the dropped lo*lo term then has
// zero mean, R13), hi*hi into one accumulator and the two cross terms into another
// (summed in the epilogue), fp32 accumulate.
#pragma once
#include "gemm_simt.cuh"
#include "nf_common.cuh"

namespace nf {

__device__ __forceinline__ void hmma_1688(float (&d)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}
// cp.async of `bytes` (4 / 8 / 12 / 16, <= the copy size) from src, the rest of the copy zero-filled
__device__ __forceinline__ void cp_async16z(float *dst, const float *src, int bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
               "l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_async4z(float *dst, const float *src, int bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
               "l"(src), "r"(bytes) : "memory");
}

namespace hm {
constexpr int BM = 64, BN = 64, BK = 32, NT = 256, STAGES = 4;
constexpr int KP = BK + 4;   // K-major tile row (floats)
constexpr int MP = 64 + 8;   // MN-major tile row (floats)
constexpr int TILE = 64 * KP > BK * MP ? 64 * KP : BK * MP;  // floats per operand tile
constexpr int SMEM = STAGES * 2 * TILE * 4;
}  // namespace hm

template <bool AK, bool BKM, int SPLIT, class Epi>
__global__ void __launch_bounds__(256)
gemm_hmma(GemmArgs g, Epi epi, int vec) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  using namespace hm;
  extern __shared__ __align__(16) float hsm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gg = lane >> 2, tt = lane & 3;
  const int wq = warp & 3, kh = warp >> 2;  // quadrant, K half (k8 steps kh, kh + 2 of a BK tile)
  const int wm = (wq & 1) * 32, wn = (wq >> 1) * 32;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int kbeg = blockIdx.z * g.kchunk;
  const int kend = min(g.K, kbeg + g.kchunk);
  const int nkt = (kend - kbeg + BK - 1) / BK;

  // one operand tile (rows r0.. of a [rows][K] (K-major) or [K][rows] (MN-major) matrix) -> smem
  auto issue_op = [&](float *dst, const float *src, int64_t ld, bool kmaj, int r0, int rlim, int k0) {
    if (vec & 1) {
      // 512 chunks of 4 floats: K-major 64 rows x 8 chunks, MN-major 32 k-rows x 16 chunks
#pragma unroll
      for (int c = tid; c < 512; c += NT) {
        int r, k, bytes;
        float *d;
        const float *s;
        if (kmaj) {
          r = c >> 3; k = k0 + 4 * (c & 7);
          bytes = (r0 + r < rlim) ? 4 * max(0, min(4, kend - k)) : 0;
          d = dst + r * KP + 4 * (c & 7);
          s = src + (int64_t)(r0 + r) * ld + k;
        } else {
          k = k0 + (c >> 4); r = 4 * (c & 15);
          bytes = (k < kend) ? 4 * max(0, min(4, rlim - (r0 + r))) : 0;
          d = dst + (c >> 4) * MP + r;
          s = src + (int64_t)k * ld + r0 + r;
        }
        cp_async16z(d, bytes ? s : src, bytes);
      }
    } else {
#pragma unroll 4
      for (int c = tid; c < 2048; c += NT) {
        int r, k;
        float *d;
        if (kmaj) { r = c >> 5; k = c & 31; d = dst + r * KP + k; }
        else { k = c >> 6; r = c & 63; d = dst + k * MP + r; }
        const bool ok = r0 + r < rlim && k0 + k < kend;
        const float *s = kmaj ? src + (int64_t)(r0 + r) * ld + k0 + k : src + (int64_t)(k0 + k) * ld + r0 + r;
        cp_async4z(d, ok ? s : src, ok ? 4 : 0);
      }
    }
  };
  auto stageA = [&](int s) { return hsm + s * 2 * TILE; };
  auto stageB = [&](int s) { return hsm + s * 2 * TILE + TILE; };
  auto issue = [&](int t) {
    if (t < nkt && !(vec & 4)) {  // (vec bits 2 / 4: timing experiments without MMAs / copies, micro/hmma_gemm_test.cu)
      const int k0 = kbeg + t * BK, s = t % STAGES;
      issue_op(stageA(s), g.A, g.lda, AK, m0, g.M, k0);
      issue_op(stageB(s), g.B, g.ldb, BKM, n0, min(g.N, g.nb_real), k0);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };

  float acc[2][4][4], accl[SPLIT == 3 ? 2 : 1][4][4];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        acc[i][j][q] = 0.0f;
        if constexpr (SPLIT == 3) accl[i][j][q] = 0.0f;
      }

#pragma unroll
  for (int t = 0; t < STAGES - 1; ++t) issue(t);
  const bool ones = n0 + BN > g.nb_real && g.nb_real < g.N;  // this tile holds the ones column(s)
  for (int t = 0; t < nkt; ++t) {
    asm volatile("cp.async.wait_group %0;" ::"n"(STAGES - 2) : "memory");
    const float *sA = stageA(t % STAGES);
    float *sB = stageB(t % STAGES);
    if (ones) {  // B(n, k) = 1 for nb_real <= n < N (the bias column of a weight gradient)
      const int k0 = kbeg + t * BK;
      for (int c = tid; c < BK * BN; c += NT) {
        const int k = BKM ? (c & 31) : (c >> 6), nn = BKM ? (c >> 5) : (c & 63);
        const int n = n0 + nn;
        if (n >= g.nb_real && n < g.N && k0 + k < kend) sB[BKM ? nn * KP + k : k * MP + nn] = 1.0f;
      }
    }
    __syncthreads();
    issue(t + STAGES - 1);  // (its stage was last read in iteration t - 1, before this barrier)
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      if (vec & 2) break;
      const int kk = 8 * (kh + 2 * s);
      // fragments: a0 = A[g][t], a1 = A[g+8][t], a2 = A[g][t+4], a3 = A[g+8][t+4]; b0 = B[t][g], b1 = B[t+4][g]
      float af[2][4], bf[4][2];
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int m = wm + 16 * i + gg;
        if (AK) {
          af[i][0] = sA[m * KP + kk + tt];
          af[i][1] = sA[(m + 8) * KP + kk + tt];
          af[i][2] = sA[m * KP + kk + tt + 4];
          af[i][3] = sA[(m + 8) * KP + kk + tt + 4];
        } else {
          af[i][0] = sA[(kk + tt) * MP + m];
          af[i][1] = sA[(kk + tt) * MP + m + 8];
          af[i][2] = sA[(kk + tt + 4) * MP + m];
          af[i][3] = sA[(kk + tt + 4) * MP + m + 8];
        }
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int n = wn + 8 * j + gg;
        bf[j][0] = BKM ? sB[n * KP + kk + tt] : sB[(kk + tt) * MP + n];
        bf[j][1] = BKM ? sB[n * KP + kk + tt + 4] : sB[(kk + tt + 4) * MP + n];
      }
      if constexpr (SPLIT == 1) {
        uint32_t a[2][4], b[4][2];
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int q = 0; q < 4; ++q) a[i][q] = __float_as_uint(tf32_rn(af[i][q]));
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
          for (int q = 0; q < 2; ++q) b[j][q] = __float_as_uint(tf32_rn(bf[j][q]));
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) hmma_1688(acc[i][j], a[i], b[j]);
      } else {
        uint32_t ah[2][4], al[2][4], bh[4][2], bl[4][2];
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int q = 0; q < 4; ++q) {  // truncation split (hi masked: an exact TF32 value)
            const float h = __uint_as_float(__float_as_uint(af[i][q]) & 0xffffe000u);
            ah[i][q] = __float_as_uint(h);
            al[i][q] = __float_as_uint(af[i][q] - h);
          }
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
          for (int q = 0; q < 2; ++q) {  // RN split
            const float h = tf32_rn(bf[j][q]);
            bh[j][q] = __float_as_uint(h);
            bl[j][q] = __float_as_uint(bf[j][q] - h);
          }
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            hmma_1688(accl[i][j], al[i], bh[j]);
            hmma_1688(accl[i][j], ah[i], bl[j]);
            hmma_1688(acc[i][j], ah[i], bh[j]);
          }
      }
    }
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();

  // both K halves park their quadrant sums (fragment order) in shared memory; then every warp
  // finishes 16 of its quadrant's 32 values per lane: all epilogue loads issued before any store
  // (the load / store split of the epilogues: a dependent global load per element serialised the
  // epilogue), stores in a rolled loop (the inlined activation exists a few times, not 32)
  float *red = hsm + (kh * 4 + wq) * 32 * 33;  // (all copies landed and all reads done: the ring is free)
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        float v = acc[i][j][q];
        if constexpr (SPLIT == 3) v += accl[i][j][q];
        red[((i * 4 + j) * 4 + q) * 33 + lane] = v;
      }
  __syncthreads();
  const float *r0p = hsm + wq * 32 * 33, *r1p = hsm + (4 + wq) * 32 * 33;
  auto coord = [&](int e, int &m, int &n) {
    const int i = e >> 4, j = (e >> 2) & 3, q = e & 3;
    // c0 = C[g][2t], c1 = C[g][2t+1], c2 = C[g+8][2t], c3 = C[g+8][2t+1]
    m = m0 + wm + 16 * i + gg + ((q & 2) ? 8 : 0);
    n = n0 + wn + 8 * j + 2 * tt + (q & 1);
  };
  float aux[16];
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    const int e = 16 * kh + u;
    int m, n;
    coord(e, m, n);
    aux[u] = (!g.partial && m < g.M && n < g.N) ? epi.load(m, n) : 0.0f;
  }
#pragma unroll 4
  for (int u = 0; u < 16; ++u) {
    const int e = 16 * kh + u;
    int m, n;
    coord(e, m, n);
    if (m >= g.M || n >= g.N) continue;
    const float v = r0p[e * 33 + lane] + r1p[e * 33 + lane];
    if (g.partial) g.partial[((int64_t)blockIdx.z * g.M + m) * g.N + n] = v;
    else epi.store(m, n, v, aux[u]);
  }
}

}  // namespace nf
