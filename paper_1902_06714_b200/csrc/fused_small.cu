// fused_small.cu -- ONE persistent kernel running many SGD steps of a two-layer net with
// narrow hidden and output layers (H, O <= 32): configs 1 and 2 ([3,5,2] and the paper's
// MNIST net [784,30,10]).  Every step is the paper's train_batch:
// fwdprop, backprop, tendencies summed over the batch (the co_sum
// of P:536-556) and the update W -= eta/B dW (reading R3).
//
// Decomposition:
//   * G clusters x C CTAs, all co-resident (1 CTA per SM).  Cluster g owns rows
//     [g B/G, (g+1) B/G) of every minibatch (the paper's per-image batch shard,
//     P:511-516); CTA rank c owns input columns (pixels) [c ws, c ws + w) and keeps that
//     slice of W1 resident in shared memory for all steps.
//   * per step s:
//       P0  TMA 2-D tile load of the NEXT step's x slice (mbarrier completion) and
//           cp.async of the next step's owned target rows -- overlaps the whole step
//       P1  partial Z1 over the pixel slice: fp32 FFMA, 5-row x 4-neuron register tiles,
//           K split in two halves across warps, halves summed in shared memory
//       P2  DSMEM push of the partial rows each peer owns (bulk copy, mbarrier
//           complete_tx on the receiver; no cluster barrier)
//       P3  owner rows: sum the C partials in rank order, + b1, sigma/sigma' (Eq. 2,
//           P:319-322), layer 2, delta_2 = (a2 - y) sigma'(z2), delta_1 = (W2^T delta_2)
//           sigma'(z1); W2/b1/b2 tendency partials (one warp per row)
//       P4  DSMEM push of the owned delta_1 rows to every peer and of the W2/b tendency
//           partial slices to the rank that reduces them
//       P5  dW1 slice = sum_rows delta_1 (x) x: 4x4 register tiles
//       P6  co_sum: ONE cp.reduce.async.bulk .add.f32 of the [H][ws] slice into this
//           rank's contiguous slice of the step's L2 accumulator (+ the W2/b slice)
//       P7  grid barrier
//       P8  ONE bulk copy of the reduced slice (+ the W2/b block) back into shared memory
//       P9  W -= (eta/B) G on the resident parameters; zero this CTA's share of the
//           accumulator used two steps ahead
//
// Contraction engines of P1 / P5 (templates TC / MM, chosen per launch):
//   * tcgen05 split-TF32 (TC, the default where it applies: TMA-aligned x, pixel slices <= 128, <= 72
//     rows per cluster): x tiles staged by TMA in the K-major and the MN-major operand layouts, the
//     tensor core truncates them to their hi part, lo = rn_tf32(x - trunc(x)) written beside them;
//     W1 hi | lo and delta_1 hi | lo stacked along N, so two N = 64 MMAs per k-step (x_lo, x_hi)
//     give all four partial products; warp-uniform issue (ptx::warp_uniform / ptx::elect_one);
//     delta_1's operand rows written by their owners in P3 and pushed in P4; neuron-major dW1 slice.
//     9.9 us per config-2 step;
//   * packed FFMA2 SIMT (NF_FUSED_TC=0 and every other shape): 11.0 us;
//   * warp-level tensor-core MMA (mma.sync m16n8k8 TF32, 3xTF32, NF_FUSED_MM=1): three HMMAs per
//     product and m16 / k8 padding of 67 rows x 100 pixels: 11.25 us (profiles/r02_k6_mma_experiment.txt).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "fused_small.cuh"
#include "gemm_tc.cuh"
#include "kernels.cuh"
#include "nf_common.cuh"
#include "sm100_ptx.cuh"

namespace nf {

static thread_local char g_fs_err[256] = "";

namespace {

#ifndef NF_FUSED_THREADS
#define NF_FUSED_THREADS 512
#endif
#ifndef NF_FUSED_MINB
#define NF_FUSED_MINB 1
#endif
constexpr int kThreads = NF_FUSED_THREADS;  // 16 warps: latency hiding for the short dependent phases
constexpr int kMinBlocks = NF_FUSED_MINB;  // CTAs per SM the kernel is built for
constexpr int kWarps = kThreads / 32;
constexpr int kMaxC = 8;       // cluster size
constexpr int kMaxRows = 128;  // rows per cluster
#ifndef NF_KRG
#define NF_KRG 5
#endif
#ifndef NF_KKP
#define NF_KKP 4
#endif
constexpr int kRG = NF_KRG;    // rows per P1 register tile
constexpr int kKP = NF_KKP;    // P1: K (pixel) range split in kKP parts across threads
constexpr int kRH = 2;         // P5: rows split in kRH parts across threads
constexpr int kProf = 16;      // profiler slots per step
// Tensor-core variant (TC): x tiles of kTcRows rows x 4 atoms of 32 pixels, staged twice per
// step by TMA in the two smem layouts the tensor core needs (K-major SWIZZLE_128B for Z1,
// MN-major SWIZZLE_128B_BASE32B for dW1), split in place into TF32 hi + fp32 lo.
constexpr int kTcRows = 72;                     // x rows per tile (>= rows per cluster), 9 K-steps
constexpr int kTcAS = kTcRows * 128;            // bytes per 32-pixel atom
constexpr int kTcXLoK = 44032;                  // K-phase lo offset (hi reads 128 rows per atom)
constexpr int kTcXLoM = 4 * kTcAS;              // M-phase lo offset
constexpr int kTcXBytes = kTcXLoK + 3 * kTcAS + 128 * 128;  // 88064
constexpr int kTcWBytes = 2 * 4 * 32 * 128;     // W1 slice hi | lo, K-major [32 j][128 px]
constexpr int kTcDBytes = 2 * kTcAS;            // delta_1 hi | lo, MN-major [72 rows][32 j]
constexpr int kTcBytes = kTcXBytes + kTcWBytes + kTcDBytes;
constexpr int kSmall = 32 * 32 + 64;  // capacity of the W2/b1/b2 tendency block: O*H + H + O <= 1088
constexpr int kSlots = 4;             // accumulator ring: step s uses slot s % 4; slot (s+2) % 4 is
                                      // zeroed between this step's barrier arrive and wait

// Batch starts of calls with few steps travel in the launch's parameter buffer (no staging copy,
// no event: ~8 us of host time per call), longer runs through a device array.
// The parameter buffer's size costs host time per launch (32 B: 3.0 us, 8 KB: 6.0 us;
// profiles/r02_micro_small_mma_launch.txt): calls of <= 32 steps use the small variant.
constexpr int kInlineSmall = 32;
constexpr int kInlineStarts = 1024;
template <int NI>
struct InlineStarts {
  int64_t v[NI];
};
// MM variant geometry: P1 m-tiles of 16 rows (<= kMT1), P5 m-tiles / W fragment blocks of 16 pixels
constexpr int kMT1 = 8;        // rows per cluster <= 128 (m-tiles mg, mg + 4 per warp)
constexpr int kMJ = 8;         // pixel slice <= 128
constexpr int kDS = 36;        // delta_1 row stride (floats) in the MM variant: conflict-free B fragments
__host__ __device__ inline int mm_rows(int nSmax) { return (nSmax + 15) / 16 * 16; }
__host__ __device__ inline int mm_nj(int wpad) { return (wpad + 15) / 16; }

struct FusedParams {
  int n0, H, O;          // dims
  int act_h, act_o;
  int B;                 // batch rows per step
  int G;                 // clusters
  int ws, wpad;          // pixel-slice stride and padded smem row length (floats)
  int aligned;           // 1: TMA x tiles and bulk reductions (n0 % 4 == 0, 16-B aligned X)
  int nSmax, nOwnMax;    // max rows per cluster / per CTA
  int64_t n_steps;
  int64_t slot;          // accumulator slot stride (floats, multiple of 32)
  int64_t small_off;     // offset of the W2/b1/b2 block inside a slot
  int nsmp;              // W2/b1/b2 block length O*H + H + O, rounded up to a multiple of 4
  int gsl;               // floats of one rank's dW1 slice in an accumulator slot
  float scale;           // eta / B
  float inv_B;
  const float *X, *Y;
  const int64_t *starts; // device array, or null: the starts are in the kernel's InlineStarts
  float *params;         // flat [W1 b1 W2 b2]
  float *acc;            // kSlots accumulator slots (zeroed by the host)
  unsigned *bar;         // grid barrier counter (zeroed by the host)
  float *step_loss;      // nullable; step s's entry zeroed in-kernel before barrier s
  unsigned bar_base;     // barrier counter at launch (it runs on across calls)
  int slot0;             // ring slot of step 0 (the ring runs on across calls)
  long long *prof;       // nullable: per-CTA per-step clock64 stamps (NF_FUSED_PROF=1)
};

#define PROF(i) \
  if (p.prof && threadIdx.x == 0 && s < 64) p.prof[((int64_t)blockIdx.x * 64 + s) * kProf + (i)] = clock64()
// latest arrival over the CTA's warps (lane 0 of each)
#define PROF_MAX(i) \
  if (p.prof && (threadIdx.x & 31) == 0 && s < 64) \
    atomicMax(reinterpret_cast<unsigned long long *>(&p.prof[((int64_t)blockIdx.x * 64 + s) * kProf + (i)]), (unsigned long long)clock64())

__device__ __forceinline__ int row_begin(int g, int B, int G) { return (int)(((int64_t)g * B) / G); }
__host__ __device__ __forceinline__ int own_begin(int c, int nS, int C) { return (c * nS) / C; }
// slice of the W2/b tendency block (nsmp floats) reduced by rank c: 16-B aligned chunks
__host__ __device__ __forceinline__ int e_begin(int c, int C, int nsmp) { return 4 * (((nsmp / 4) * c) / C); }
__host__ __device__ __forceinline__ int e_slot(int C) { return ((kSmall / C + 4) + 3) & ~3; }

__device__ __forceinline__ void cp_async4(float *dst, const float *src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(ptx::smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait0() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

struct Smem {  // offsets in floats from the 128-B aligned base
  int tcr, W1t, W2s, b1s, b2s, xs, ys, Ppart, Pown, D1, A1own, D2own, gpart, grecv, Gs, Gs2, Gr, gsm, lsum, total;
};

__host__ __device__ inline int al32(int v) { return (v + 31) & ~31; }  // 128-B alignment in floats

__host__ __device__ inline int xrows(int nSmax) { return (nSmax + kRG - 1) / kRG * kRG; }

__host__ __device__ inline Smem smem_layout(int wpad, int nSmax, int nOwnMax, int C, bool tc, bool mm) {
  Smem L;
  const int nj = mm_nj(wpad);
  const int xr = mm ? mm_rows(nSmax) : xrows(nSmax);  // x rows staged (MM: whole 16-row m-tiles)
  int o = 32;  // mbarriers (and the TMEM address) live in the first 128 B
  L.tcr = o;   o = al32(o + (tc ? (kTcBytes + 1024) / 4 : 0));  // TC operand tiles (1024-B aligned inside)
  // W1 slice: SIMT [wpad][32] k-major; MM fragment order hi | lo ([j][nb][lane][4] each)
  L.W1t = o;   o = al32(o + (tc ? 0 : mm ? 2 * nj * 512 : wpad * 32));
  L.W2s = o;   o = al32(o + 32 * 33);              // [32][33]
  L.b1s = o;   o += 32;
  L.b2s = o;   o = al32(o + 32);
  // 2 TMA destinations (SIMT / MM); MM reads up to 28 floats past a buffer's last row
  L.xs = o;    o = al32(o + (tc ? 0 : 2 * al32(xr * wpad + (mm ? 32 : 0))));
  L.ys = o;    o = al32(o + 2 * nOwnMax * 32);
  // P1 K-part partials (SIMT: part 0 = Pfull; MM: Pfull [rows][32] only)
  L.Ppart = o; o = al32(o + (tc ? xrows(nSmax) * 32 : mm ? xr * 32 : kKP * xrows(nSmax) * 32));
  L.Pown = o;  o = al32(o + C * nOwnMax * 32);
  L.D1 = o;    o = al32(o + (mm ? ((nSmax + 7) / 8 * 8) * kDS : nSmax * 32));
  L.A1own = o; o = al32(o + nOwnMax * 32);         // a1 of the owned rows
  L.D2own = o; o = al32(o + nOwnMax * 32);         // delta_2 of the owned rows
  L.gpart = o; o = al32(o + kSmall);
  L.grecv = o; o = al32(o + C * e_slot(C));
  L.Gs = o;    o = al32(o + (mm ? nj * 512 : wpad * 32));  // dW1 slice partial (SIMT k-major; MM fragment order)
  L.Gs2 = o;   o = al32(o + (tc || mm ? 0 : wpad * 32)); // second row-half partial (SIMT)
  L.Gr = o;    o = al32(o + (mm ? nj * 512 : wpad * 32));  // reduced slice read back
  L.gsm = o;   o = al32(o + kSmall);               // reduced W2/b block read back
  L.lsum = o;  o = al32(o + kWarps);
  L.total = o;
  return L;
}

// byte offset of element (row r, column c < 32) inside a 32-column atom of 128-B rows
__device__ __forceinline__ int sw128_k(int r, int c) { return r * 128 + ((((c >> 2) ^ (r & 7))) << 4) + ((c & 3) << 2); }
// W1 slice of the TC variant: per 32-pixel atom 8 KB = hi rows 0..31 | lo rows 32..63, so one K-major
// B descriptor of N = 64 rows reads W_hi and W_lo stacked along N
__device__ __forceinline__ int tc_w_off(int j, int k) { return (k >> 5) * 8192 + sw128_k(j, k & 31); }
__device__ __forceinline__ int sw128_32b(int r, int c) { return r * 128 + ((((c >> 3) ^ (r & 3))) << 5) + ((c & 7) << 2); }
// TF32 split of `bytes` of staged fp32 data (the x tiles)
__device__ __forceinline__ void tc_split(const uint8_t *hi, uint8_t *lo, int bytes, int tid, int nthreads = kThreads,
                                         int part = 0, int nparts = 1) {
  // truncation split: the tensor core reads the staged fp32 tile itself as the hi part (it drops the
  // low 13 mantissa bits), so only lo = rn_tf32(x - trunc(x)) is written -- no in-place store, and the
  // loads of successive chunks are independent of the stores
  const int n16 = bytes / 16, i0 = (int)((int64_t)n16 * part / nparts), i1 = (int)((int64_t)n16 * (part + 1) / nparts);
  for (int i = i0 + tid; i < i1; i += nthreads) {
    const float4 x = reinterpret_cast<const float4 *>(hi)[i];
    reinterpret_cast<float4 *>(lo)[i] = make_float4(tf32_lo(x.x), tf32_lo(x.y), tf32_lo(x.z), tf32_lo(x.w));
  }
}

// wait until the monotonically running counter reaches `target` (wrap-safe: the counter runs
// on across calls, bar_base + steps * CTAs may wrap around 2^32)
__device__ __forceinline__ void grid_wait_from(unsigned *ctr, unsigned target) {
  unsigned v;
  do {
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
  } while ((int)(v - target) < 0);
}

// ---- warp-level TF32 MMA (MM variant): D[16x8] += A[16x8] B[8x8], fp32 accumulate.  Fragments
// (g = lane / 4, t = lane % 4): a0 = A[g][t], a1 = A[g+8][t], a2 = A[g][t+4], a3 = A[g+8][t+4];
// b0 = B[t][g], b1 = B[t+4][g]; c0 = C[g][2t], c1 = C[g][2t+1], c2 = C[g+8][2t], c3 = C[g+8][2t+1].
// Row and k indices may be permuted freely (the same way in A and B / in A and C): the loads
// below use that to read 16 or 8 contiguous bytes per lane without shared-memory bank conflicts.
__device__ __forceinline__ void hmma_tf32(float (&d)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}
// 3xTF32 operand split: hi = rn_tf32(x) (an exact TF32 value), lo = x - hi (exact in fp32; the
// tensor core reads its TF32 part)
__device__ __forceinline__ void split_tf32(float x, uint32_t &hi, uint32_t &lo) {
  const float h = tc::tf32_hi(x);
  hi = __float_as_uint(h);
  lo = __float_as_uint(x - h);
}
// truncation split: hi = x itself (the tensor core reads its TF32 part, i.e. x with the low 13
// mantissa bits cleared), lo = x - that part (exact); pairs with an RN-split partner operand so
// the dropped lo*lo term has zero mean (R13)
__device__ __forceinline__ void split_trunc(float x, uint32_t &hi, uint32_t &lo) {
  hi = __float_as_uint(x);
  lo = __float_as_uint(x - __uint_as_float(hi & 0xffffe000u));
}
// D += A B in 3xTF32: small terms first
__device__ __forceinline__ void hmma3(float (&d)[4], const uint32_t (&ah)[4], const uint32_t (&al)[4],
                                      const uint32_t (&bh)[2], const uint32_t (&bl)[2]) {
  hmma_tf32(d, al, bh);
  hmma_tf32(d, ah, bl);
  hmma_tf32(d, ah, bh);
}

// P1 of the MM variant for one warp: Z1 partial rows of the NM m-tiles m0, m0 + MSTEP, ... (16 rows
// each) x one n-block (8 neurons) over the 16-pixel blocks [jb, je) of the slice.  Logical row g of
// an m-tile is physical row pr (the caller picks the permutation that makes the LDS.128
// conflict-free for the slice's row stride); k-step 2j / 2j+1 takes pixels 16 j + 4 t + {0, 1} /
// {2, 3}, matching the W fragment order [j][nb][lane][4].  Output: rows of Pz [rows][32], or (pf
// non-null) fragments pf[(m * 4 + nb) * 32 + lane].
template <int NM, int MSTEP>
__device__ __forceinline__ void p1_mma(const float *xs, int wpad, const float4 *Wh4, const float4 *Wl4, int jb,
                                       int je, int m0, int nb, int lane, int pr, float *Pz, float4 *pf) {
  const int tt = lane & 3;
  float acc[NM][4];
#pragma unroll
  for (int m = 0; m < NM; ++m) acc[m][0] = acc[m][1] = acc[m][2] = acc[m][3] = 0.0f;
  const float *xr = xs + (16 * m0 + pr) * wpad + 4 * tt;
  for (int j = jb; j < je; ++j) {
    const float4 wh = Wh4[(j * 4 + nb) * 32 + lane], wl = Wl4[(j * 4 + nb) * 32 + lane];
    float4 xa[NM], xb[NM];
#pragma unroll
    for (int m = 0; m < NM; ++m) {
      xa[m] = *reinterpret_cast<const float4 *>(xr + 16 * MSTEP * m * wpad + 16 * j);
      xb[m] = *reinterpret_cast<const float4 *>(xr + (16 * MSTEP * m + 8) * wpad + 16 * j);
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {  // k-steps 2j, 2j+1
      const uint32_t bh[2] = {__float_as_uint(h ? wh.z : wh.x), __float_as_uint(h ? wh.w : wh.y)};
      const uint32_t bl[2] = {__float_as_uint(h ? wl.z : wl.x), __float_as_uint(h ? wl.w : wl.y)};
      uint32_t ah[NM][4], al[NM][4];
#pragma unroll
      for (int m = 0; m < NM; ++m) {
        split_trunc(h ? xa[m].z : xa[m].x, ah[m][0], al[m][0]);
        split_trunc(h ? xb[m].z : xb[m].x, ah[m][1], al[m][1]);
        split_trunc(h ? xa[m].w : xa[m].y, ah[m][2], al[m][2]);
        split_trunc(h ? xb[m].w : xb[m].y, ah[m][3], al[m][3]);
      }
#pragma unroll
      for (int m = 0; m < NM; ++m) hmma_tf32(acc[m], al[m], bh);
#pragma unroll
      for (int m = 0; m < NM; ++m) hmma_tf32(acc[m], ah[m], bl);
#pragma unroll
      for (int m = 0; m < NM; ++m) hmma_tf32(acc[m], ah[m], bh);
    }
  }
#pragma unroll
  for (int m = 0; m < NM; ++m) {
    if (pf) {
      pf[(MSTEP * m * 4 + nb) * 32 + lane] = make_float4(acc[m][0], acc[m][1], acc[m][2], acc[m][3]);
    } else {  // c0, c1 = row g (physical pr), neurons 8 nb + 2t, +1; c2, c3 = row g + 8
      float *d = Pz + (16 * (m0 + MSTEP * m) + pr) * 32 + 8 * nb + 2 * tt;
      *reinterpret_cast<float2 *>(d) = make_float2(acc[m][0], acc[m][1]);
      *reinterpret_cast<float2 *>(d + 8 * 32) = make_float2(acc[m][2], acc[m][3]);
    }
  }
}

// AH / AO: compile-time hidden / output activations (-1 = read p.act_h / p.act_o at run time).
// The sigmoid/sigmoid instantiation (configs 1 and 2) keeps the dependent owner-row chain
// short: no activation switch.
template <int AH, int AO>
__device__ __forceinline__ void act_sel(int rt, float z, float &a, float &s) {
  act_fwd(AH >= 0 ? AH : rt, z, a, s);
}

template <bool TC, bool MM, int AH, int AO, int NI>
__global__ void __launch_bounds__(kThreads, kMinBlocks)
fused_small_kernel(const FusedParams p, const __grid_constant__ CUtensorMap tmX,
                   const __grid_constant__ CUtensorMap tmXK, const __grid_constant__ CUtensorMap tmXM,
                   const __grid_constant__ InlineStarts<NI> ist) {
  static_assert(!MM || kThreads == 512, "the MM variant maps 16 warps onto 4 n-blocks x 4 parts");
  constexpr int ds = MM ? kDS : 32;  // delta_1 row stride
  extern __shared__ __align__(128) float sm[];
  const int C = (int)ptx::cluster_size();
  const int rank = (int)ptx::cluster_rank();
  const int g = blockIdx.x / C;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n0 = p.n0, H = p.H, O = p.O;
  const int nCTA = gridDim.x;

  // pixel slice of this rank
  int k0, w;
  if (p.aligned) {
    k0 = rank * p.ws;
    w = min(p.ws, n0 - k0);
  } else {
    k0 = (int)(((int64_t)rank * n0) / C);
    w = (int)(((int64_t)(rank + 1) * n0) / C) - k0;
  }
  const int wpad = p.wpad;
  // rows of this cluster and the rows each rank owns inside them
  const int r0 = row_begin(g, p.B, p.G), nS = row_begin(g + 1, p.B, p.G) - r0;
  const int o0 = own_begin(rank, nS, C), nOwn = own_begin(rank + 1, nS, C) - o0;
  const int nsmp = p.nsmp, nsm = O * H + H + O;
  const int e0 = e_begin(rank, C, nsmp), ne = e_begin(rank + 1, C, nsmp) - e0;
  const int eslot = e_slot(C);

  const Smem L = smem_layout(wpad, p.nSmax, p.nOwnMax, C, TC, MM);
  const int xstride = MM ? al32(mm_rows(p.nSmax) * wpad + 32) : al32(xrows(p.nSmax) * wpad);
  const int nj = mm_nj(wpad);  // MM: 16-pixel blocks of the slice
  uint64_t *bar_x = reinterpret_cast<uint64_t *>(sm);  // [2]
  uint64_t *bar_P = bar_x + 2;
  uint64_t *bar_D = bar_x + 3;
  uint64_t *bar_G = bar_x + 4;
  uint64_t *bar_mma = bar_x + 5;             // TC: tcgen05.commit arrivals (2 per step)
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bar_x + 6);
  // TC operand tiles (1024-B aligned): X (x tile, K- or MN-phase), Wt (W1 hi|lo), Dt (delta_1 hi|lo)
  uint8_t *X = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(sm + L.tcr) + 1023) & ~uintptr_t(1023));
  uint8_t *Wt = X + kTcXBytes, *Dt = Wt + kTcWBytes;
  const uint32_t sX = ptx::smem_u32(X), sW = ptx::smem_u32(Wt), sD = ptx::smem_u32(Dt);
  float *W1t = sm + L.W1t, *W2s = sm + L.W2s, *b1s = sm + L.b1s, *b2s = sm + L.b2s;
  float *xs0 = sm + L.xs, *ys0 = sm + L.ys, *Ppart = sm + L.Ppart, *Pown = sm + L.Pown;
  // row-major Z1 partial rows [rows][32] (SIMT / TC: K part 0 itself; MM: after the 4 fragment-order parts)
  float *Pfull = Ppart;
  const int pstride = xrows(p.nSmax) * 32;  // floats between P1 K-part buffers
  float *D1 = sm + L.D1, *A1own = sm + L.A1own, *D2own = sm + L.D2own;
  float *gpart = sm + L.gpart, *grecv = sm + L.grecv, *Gs = sm + L.Gs, *Gs2 = sm + L.Gs2, *Gr = sm + L.Gr;
  float *gsm = sm + L.gsm, *lsum = sm + L.lsum;

  const int64_t oW1 = 0, ob1 = (int64_t)H * n0, oW2 = ob1 + H, ob2 = oW2 + (int64_t)O * H;
  // accumulator slot layout: [C slices of ws x 32 (k-major)] [W2/b block of nsmp floats]
  const int64_t slice_off = (int64_t)rank * p.gsl;

  // ---- one-time setup: zero smem, barriers, resident parameters
  for (int i = 32 + tid; i < L.total; i += kThreads) sm[i] = 0.0f;
  if (TC) {  // rows >= nS of P5's delta_1 operand (hi and lo blocks) are never written: zero for all steps
             // (the 1024-B alignment pad of the operand area may reach past the loop above)
    for (int t = tid; t < (kTcRows - nS) * 64; t += kThreads) {
      const int r = nS + (t >> 6), c = t & 63;
      *reinterpret_cast<float *>(Dt + (c >= 32 ? kTcAS : 0) + r * 128 + (c & 31) * 4) = 0.0f;
    }
  }
  if (tid == 0) {
    ptx::mbar_init(&bar_x[0], 1);
    ptx::mbar_init(&bar_x[1], 1);
    ptx::mbar_init(bar_P, 1);
    ptx::mbar_init(bar_D, 1);
    ptx::mbar_init(bar_G, 1);
    ptx::mbar_init(bar_mma, 1);
    ptx::fence_mbar_init();
    if (p.aligned) ptx::prefetch_tensormap(&tmX);
    if (TC) {
      ptx::prefetch_tensormap(&tmXK);
      ptx::prefetch_tensormap(&tmXM);
    }
  }
  if (TC && warp == 0) {  // 128 TMEM columns: Z1 partial accumulator (x W_hi | x W_lo) | dW1 accumulator (x^T d_hi | x^T d_lo)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 ::"r"(ptx::smem_u32(tmem_slot)), "r"(128u) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = TC ? *tmem_slot : 0u;
  if (TC && tid == 0 && p.n_steps > 0) {  // step 0's K-layout x tile: its HBM latency overlaps the parameter staging below
    const int64_t row00 = (p.starts ? p.starts[0] : ist.v[0]) + r0;
    ptx::mbar_arrive_expect_tx(&bar_x[0], 4u * kTcAS);
#pragma unroll
    for (int a = 0; a < 4; ++a) ptx::tma_load_2d(X + a * kTcAS, &tmXK, &bar_x[0], k0 + 32 * a, (int)row00);
  }
  if (TC) {  // W1 slice as TF32 hi + fp32 lo in the K-major SWIZZLE_128B B-operand layout
    for (int i = tid; i < 32 * 128; i += kThreads) {
      const int j = i >> 7, k = i & 127;
      const float v = (j < H && k < w) ? p.params[oW1 + (int64_t)j * n0 + k0 + k] : 0.0f;
      const float h = tc::tf32_hi(v);
      const int off = tc_w_off(j, k);
      *reinterpret_cast<float *>(Wt + off) = h;
      *reinterpret_cast<float *>(Wt + 4096 + off) = v - h;
    }
  } else if (MM) {  // fragment order: [j][nb][lane][4] = W1[8 nb + lane / 4][k0 + 16 j + 4 (lane % 4) + e]
    for (int i = tid; i < nj * 512; i += kThreads) {
      const int ln = (i >> 2) & 31, nbj = i >> 7;
      const int n = 8 * (nbj & 3) + (ln >> 2), k = 16 * (nbj >> 2) + 4 * (ln & 3) + (i & 3);
      const float v = (n < H && k < w) ? p.params[oW1 + (int64_t)n * n0 + k0 + k] : 0.0f;
      const float h = tc::tf32_hi(v);
      W1t[i] = h;
      W1t[nj * 512 + i] = v - h;
    }
  } else {  // coalesced row reads (consecutive threads: consecutive pixels of one neuron's row), all
             // loads of a thread issued before its transposed shared-memory stores
    constexpr int kPer = 8;
    for (int i0 = tid; i0 < H * w; i0 += kThreads * kPer) {
      float v[kPer];
#pragma unroll
      for (int u = 0; u < kPer; ++u) {
        const int i = i0 + u * kThreads;
        v[u] = i < H * w ? p.params[oW1 + (int64_t)(i / w) * n0 + k0 + i % w] : 0.0f;
      }
#pragma unroll
      for (int u = 0; u < kPer; ++u) {
        const int i = i0 + u * kThreads;
        if (i < H * w) W1t[(i % w) * 32 + i / w] = v[u];
      }
    }
  }
  for (int i = tid; i < O * H; i += kThreads) W2s[(i / H) * 33 + i % H] = p.params[oW2 + i];
  for (int i = tid; i < H; i += kThreads) b1s[i] = p.params[ob1 + i];
  for (int i = tid; i < O; i += kThreads) b2s[i] = p.params[ob2 + i];
  ptx::cluster_sync();  // peers' barriers initialised before any push

  // bytes each exchange delivers to this CTA per step
  uint32_t bytesP = 0, bytesD = 0;
  for (int c = 0; c < C; ++c) {
    if (c == rank) continue;
    bytesP += nOwn * 128;
    bytesD += (own_begin(c + 1, nS, C) - own_begin(c, nS, C)) * (TC ? 256 : ds * 4) + ne * 4;  // (TC: hi + lo rows of the MMA operand)
  }
  const uint32_t bytesG = (uint32_t)(p.gsl * 4 + nsmp * 4);

  const uint32_t xbytes = (uint32_t)(p.nSmax * p.ws * 4);
  // batch starts are read one step ahead of their use so their global-load latency overlaps
  // a whole step (next_start holds starts[s + 1] while step s runs)
  auto start_of = [&](int64_t s) -> int64_t { return p.starts ? p.starts[s] : ist.v[s]; };
  int64_t next_start = p.n_steps > 0 ? start_of(0) : 0;
  auto prefetch = [&](int64_t s) {
    const int buf = (int)(s & 1);
    const int64_t row0 = next_start + r0;
    next_start = s + 1 < p.n_steps ? start_of(s + 1) : 0;
    float *xs = xs0 + buf * xstride;
    if (TC) {
      // x tiles are staged by tc_issue (two layouts per step); the rows are pulled into L2 a step
      // ahead, so both tile loads of the step hit L2
      if (tid == kThreads - 32) {
#pragma unroll
        for (int a = 0; a < 4; ++a) ptx::tma_prefetch_2d(&tmXK, k0 + 32 * a, (int)row0);
      }
    } else if (p.aligned) {
      // issued by the last warp, which has no P1 task: the issue latency stays off the P1 path
      if (tid == kThreads - 32) {
        ptx::mbar_arrive_expect_tx(&bar_x[buf], xbytes);
        ptx::tma_load_2d(xs, &tmX, &bar_x[buf], k0, (int)row0);
      }
    } else {
      for (int r = warp; r < nS; r += kWarps) {
        const float *src = p.X + (row0 + r) * n0 + k0;
        for (int c = lane; c < w; c += 32) cp_async4(xs + r * wpad + c, src + c);
      }
    }
    float *ys = ys0 + buf * p.nOwnMax * 32;
    for (int i = tid - (kThreads - 64); i >= 0 && i < nOwn * O; i += 64) {  // the last two warps
      const int r = i / O, c = i % O;
      cp_async4(ys + r * 32 + c, p.Y + (row0 + o0 + r) * O + c);
    }
    cp_async_commit();
  };

  // TC: stage the x tile of a step in one layout: four {32 px, kTcRows rows} boxes
  auto tc_issue = [&](const CUtensorMap *map, uint64_t *bar, int64_t row0) {
    ptx::mbar_arrive_expect_tx(bar, 4u * kTcAS);
#pragma unroll
    for (int a = 0; a < 4; ++a) ptx::tma_load_2d(X + a * kTcAS, map, bar, k0 + 32 * a, (int)row0);
  };
  int64_t row_s = next_start + r0;  // first row of step s's batch slice for this cluster
  prefetch(0);
  if (TC && p.n_steps > 0) {  // step 0's K-layout tile (issued at the top of the kernel)
    ptx::mbar_wait(&bar_x[0], 0);
    tc_split(X, X + kTcXLoK, 4 * kTcAS, tid);
    ptx::fence_proxy_async_smem();
    __syncthreads();
  }

  // P1 task geometry: kRG-row x 4-neuron tiles, K in kKP parts of 4-pixel chunks
  const int RG = (nS + kRG - 1) / kRG;
  const int nchunk = wpad / 4;
  // P5 task geometry: 4-neuron x 4-pixel tiles, rows in kRH parts
  const int nP5 = kRH * 8 * nchunk;

  for (int64_t s = 0; s < p.n_steps; ++s) {
    const int buf = (int)(s & 1);
    const uint32_t par = (uint32_t)(s & 1);
    const float *xs = xs0 + buf * xstride;
    const float *ys = ys0 + buf * p.nOwnMax * 32;
    float *accS = p.acc + ((p.slot0 + s) % kSlots) * p.slot;
    PROF(0);
    if (tid == 0) {  // arm this step's receive barriers
      ptx::mbar_arrive_expect_tx(bar_P, bytesP);
      ptx::mbar_arrive_expect_tx(bar_D, bytesD);
    }
    cp_async_wait0();
    if (!TC && p.aligned) ptx::mbar_wait(&bar_x[buf], (uint32_t)((s >> 1) & 1));
    __syncthreads();
    const int64_t row_s1 = next_start + r0;  // step s+1's first row (valid if s+1 < n_steps)
    if (s + 1 < p.n_steps) prefetch(s + 1);
    PROF(1);

    // ---- P1. partial Z1: P[i][j] = sum_{k<w} x[i][k] W1[j][k0+k]
    if constexpr (TC) {
      // 3xTF32 on the tensor core: D[row][j] (TMEM cols 0..31), M = 128 rows, N = 32, K = pixels
      if (ptx::warp_uniform(warp) == 0) {  // warp-uniform loop and operands, one elected lane issues
        tc::tc_fence_after();
        // B = 64 rows per atom: W_hi | W_lo stacked along N -> columns 0..31 x W_hi, 32..63 x W_lo; two
        // MMAs per k-step (x_lo, x_hi) give all four partial products
        constexpr uint32_t idK = tc::idesc_tf32(128, 64, false, false);
        const int nks = (p.ws + 7) / 8;
        const uint32_t tm = (uint32_t)ptx::warp_uniform((int)tmem);
        if (ptx::elect_one()) {
          for (int ks = 0; ks < nks; ++ks) {
            const uint32_t ao = (ks >> 2) * kTcAS + (ks & 3) * 32, bo = (ks >> 2) * 8192 + (ks & 3) * 32;
            const uint64_t ah = tc::smem_desc(sX + ao, 16, 1024, 2), al = tc::smem_desc(sX + kTcXLoK + ao, 16, 1024, 2);
            const uint64_t bw = tc::smem_desc(sW + bo, 16, 1024, 2);
            tc::mma_tf32(tm, al, bw, idK, ks > 0 ? 1u : 0u);
            tc::mma_tf32(tm, ah, bw, idK, 1u);
          }
          tc::mma_commit(bar_mma);
        }
        __syncwarp();
      }
      PROF(13);
      ptx::mbar_wait(bar_mma, 0);
      tc::tc_fence_after();
      PROF(14);
      if (tid == 128) tc_issue(&tmXM, &bar_x[1], row_s);  // the MMAs are done with the K-layout tile (warp 4: not an epilogue warp)
      if (warp < 4) {
        float v[32], vl[32];
        tc::tmem_ld32(tmem + ((uint32_t)(32 * warp) << 16), v);
        tc::tmem_ld32(tmem + ((uint32_t)(32 * warp) << 16) + 32u, vl);
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] += vl[j];
        const int r = 32 * warp + lane;
        if (r < nS) {  // 16-B chunk c of row r at chunk c ^ (r % 8): the eight lanes of a store phase
                       // hit eight different bank groups (P3 reads the rows back with the same key)
#pragma unroll
          for (int j = 0; j < 32; j += 4)
            *reinterpret_cast<float4 *>(Pfull + r * 32 + ((((j >> 2) ^ (r & 7))) << 2)) =
                make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
        }
      }
      tc::tc_fence_before();
    } else if constexpr (MM) {
      // warp = (n-block nb of 8 neurons = the SMSP, mg): m-tiles mg and mg + 4 of 16 rows over all
      // pixels of the slice (p1_mma; no K split, no partial sums).  Measured faster than splitting
      // the fifth m-tile by K quarters for balance (shorter dependent HMMA chains per warp, more
      // fragment re-reads).  Row permutation: rows 4 apart (row stride = 1 mod 8 16-B groups, e.g.
      // config 2's 100-pixel slices) or adjacent (stride = 4 mod 8, 112-pixel slices) share an
      // 8-lane LDS.128 phase, which then covers all 32 banks.
      const int nb = warp & 3, mg = warp >> 2, gg = lane >> 2;
      const int nmt = (nS + 15) >> 4;
      const int pr = (wpad & 31) == 16 ? gg : (gg >> 1) + 4 * (gg & 1);
      const float4 *Wh4 = reinterpret_cast<const float4 *>(W1t), *Wl4 = Wh4 + nj * 128;
      if (mg + 4 < nmt) p1_mma<2, 4>(xs, wpad, Wh4, Wl4, 0, nj, mg, nb, lane, pr, Pfull, nullptr);
      else if (mg < nmt) p1_mma<1, 4>(xs, wpad, Wh4, Wl4, 0, nj, mg, nb, lane, pr, Pfull, nullptr);
      PROF_MAX(13);
    } else {
    // ---- P1. partial Z1: P[i][j] = sum_{k<w} x[i][k] W1[j][k0+k]
      for (int t = tid; t < kKP * RG * 8; t += kThreads) {
        const int jg = t & 7, rg = (t >> 3) % RG, kp = (t >> 3) / RG;
        const int cb = kp * nchunk / kKP, ce = (kp + 1) * nchunk / kKP;
        const float *xr = xs + rg * kRG * wpad;
        const float *wr = W1t + jg * 4;
        float2 a[kRG][2];  // neuron pairs (4jg, 4jg+1), (4jg+2, 4jg+3): packed FFMA2
#pragma unroll
        for (int u = 0; u < kRG; ++u) a[u][0] = a[u][1] = make_float2(0.0f, 0.0f);
#pragma unroll 2
        for (int c = cb; c < ce; ++c) {
          float4 xv[kRG], wv[4];
#pragma unroll
          for (int u = 0; u < kRG; ++u) xv[u] = *reinterpret_cast<const float4 *>(xr + u * wpad + 4 * c);
#pragma unroll
          for (int q = 0; q < 4; ++q) wv[q] = *reinterpret_cast<const float4 *>(wr + (4 * c + q) * 32);
#pragma unroll
          for (int u = 0; u < kRG; ++u) {
            const float xq[4] = {xv[u].x, xv[u].y, xv[u].z, xv[u].w};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              ffma2(a[u][0], xq[q], make_float2(wv[q].x, wv[q].y));
              ffma2(a[u][1], xq[q], make_float2(wv[q].z, wv[q].w));
            }
          }
        }
        float *dst = Pfull + kp * pstride;
#pragma unroll
        for (int u = 0; u < kRG; ++u)
          *reinterpret_cast<float4 *>(dst + (rg * kRG + u) * 32 + jg * 4) = make_float4(a[u][0].x, a[u][0].y, a[u][1].x, a[u][1].y);
      }
      __syncthreads();
      for (int i = tid; i < nS * 8; i += kThreads) {  // parts summed in order 0 + 1 + 2 + 3
        float4 *d = reinterpret_cast<float4 *>(Pfull) + i;
        float4 v = *d;
#pragma unroll
        for (int kp = 1; kp < kKP; ++kp) {
          const float4 h = reinterpret_cast<const float4 *>(Pfull + kp * pstride)[i];
          v.x += h.x; v.y += h.y; v.z += h.z; v.w += h.w;
        }
        *d = v;
      }
    }
    ptx::fence_proxy_async_smem();
    __syncthreads();
    PROF(2);

    // ---- P2. push the partial rows each peer owns into its Pown[rank] slot
    // (one push per warp, lane 0 of warps 0..C-1: a single warp would issue its lanes' bulk copies
    // one after the other, each behind an ELECT / R2UR.BROADCAST sequence)
    if (lane == 0 && warp < C && warp != rank) {
      const int c = warp;
      const int a0 = own_begin(c, nS, C), na = own_begin(c + 1, nS, C) - a0;
      if (na > 0)
        ptx::bulk_s2peer(Pown + rank * p.nOwnMax * 32, Pfull + a0 * 32, (uint32_t)(na * 128), bar_P, c);
    }
    // TC: the M-layout x tile of this step (issued after P1's MMAs) is split for P5 by the warps that
    // have no P3 task (warps >= 9 when a CTA owns <= 9 rows), a third per P3 pass; otherwise here,
    // while the peers' partial rows are still in flight
    const bool split_in_p3 = TC && p.nOwnMax <= 9;
    if constexpr (TC) {
      if (!split_in_p3) {
        ptx::mbar_wait(&bar_x[1], par);
        tc_split(X, X + kTcXLoM, 4 * kTcAS, tid);
      }
    }
    ptx::mbar_wait(bar_P, par);
    PROF(3);

    // ---- P3. owned rows, all rows at once in three CTA-wide passes:
    //      (a) thread (q, j): z1 = b1 + sum of the C partials in rank order, a1, sigma'(z1)
    //      (b) thread (q, o): z2 = b2 + W2 a1, a2, delta_2 = (a2 - y) sigma'(z2), cost
    //      (c) thread (q, j): delta_1 = sigma'(z1) * W2^T delta_2
    float lacc = 0.0f;
    if constexpr (TC) {
      if (split_in_p3 && warp >= 9) {
        ptx::mbar_wait(&bar_x[1], par);
        tc_split(X, X + kTcXLoM, 4 * kTcAS, tid - 288, kThreads - 288, 0, 3);
      }
    }
    for (int t = tid; t < nOwn * 32; t += kThreads) {
      const int q = t >> 5, j = t & 31, i = o0 + q;
      // (TC: the partial rows are stored with their 16-B chunks permuted by the row index)
      const int jc = TC ? ((((j >> 2) ^ (i & 7)) << 2) | (j & 3)) : j;
      float z = b1s[j];
#pragma unroll
      for (int c = 0; c < kMaxC; ++c)
        if (c < C) z += (c == rank) ? Pfull[i * 32 + jc] : Pown[(c * p.nOwnMax + q) * 32 + jc];
      float a1, s1;
      act_sel<AH, AO>(p.act_h, z, a1, s1);
      A1own[t] = j < H ? a1 : 0.0f;
      D1[i * ds + j] = j < H ? s1 : 0.0f;   // sigma'(z1) parked in the delta_1 row
    }
    __syncthreads();
    PROF(11);
    if constexpr (TC) {
      if (split_in_p3 && warp >= 9) tc_split(X, X + kTcXLoM, 4 * kTcAS, tid - 288, kThreads - 288, 1, 3);
    }
    for (int t = tid; t < nOwn * O; t += kThreads) {
      const int q = t / O, o = t - q * O;
      const float *va = A1own + q * 32, *w2 = W2s + o * 33;
      // fully unrolled over the 32-wide rows (W2s and A1own are zero past H): every load is
      // issued up front instead of one iteration at a time
      float c0 = 0.0f, c1 = 0.0f, c2 = 0.0f, c3 = 0.0f;
#pragma unroll
      for (int j = 0; j < 32; j += 4) {
        if (j < H) {  // uniform
          c0 = fmaf(w2[j], va[j], c0);
          c1 = fmaf(w2[j + 1], va[j + 1], c1);
          c2 = fmaf(w2[j + 2], va[j + 2], c2);
          c3 = fmaf(w2[j + 3], va[j + 3], c3);
        }
      }
      const float z2 = b2s[o] + ((c0 + c1) + (c2 + c3));
      float a2, s2;
      act_sel<AO, AO>(p.act_o, z2, a2, s2);
      const float diff = a2 - ys[q * 32 + o];
      lacc = fmaf(diff, diff, lacc);
      D2own[q * 32 + o] = diff * s2;
    }
    __syncthreads();
    PROF(12);
    if constexpr (TC) {
      if (split_in_p3 && warp >= 9) tc_split(X, X + kTcXLoM, 4 * kTcAS, tid - 288, kThreads - 288, 2, 3);
    }
    for (int t = tid; t < nOwn * 32; t += kThreads) {
      const int q = t >> 5, j = t & 31, i = o0 + q;
      const float *vd = D2own + q * 32;
      float t0 = 0.0f, t1 = 0.0f;  // unrolled over <= 32 outputs (D2own, W2s zero past O)
#pragma unroll
      for (int o = 0; o < 32; o += 2) {
        if (o < O) {  // uniform
          t0 = fmaf(W2s[o * 33 + j], vd[o], t0);
          t1 = fmaf(W2s[(o + 1) * 33 + j], vd[o + 1], t1);
        }
      }
      const float d1 = j < H ? (t0 + t1) * D1[i * ds + j] : 0.0f;
      D1[i * ds + j] = d1;
      if constexpr (TC) {  // the owner writes its rows of P5's B operand (delta_1 hi | lo, MN-major, a
        // row = 128 contiguous bytes permuted inside) and pushes those rows: no peer rebuilds them
        const float h = tc::tf32_hi(d1);
        const int off = sw128_32b(i, j);
        *reinterpret_cast<float *>(Dt + off) = h;
        *reinterpret_cast<float *>(Dt + kTcAS + off) = d1 - h;
      }
    }
    {
      const float l = warp_sum(lacc);
      if (lane == 0) lsum[warp] = l;
    }
    ptx::fence_proxy_async_smem();
    __syncthreads();
    PROF(4);

    // ---- P4. push the owned delta_1 rows to every peer at once; then this CTA's W2/b1/b2
    //      tendency partial over its owned rows (a 10x30x9 contraction) and its slices to
    //      the ranks that reduce them
    if (lane == 0 && warp < C && warp != rank && nOwn > 0) {
      if constexpr (TC) {
        ptx::bulk_s2peer(Dt + o0 * 128, Dt + o0 * 128, (uint32_t)(nOwn * 128), bar_D, warp);
        ptx::bulk_s2peer(Dt + kTcAS + o0 * 128, Dt + kTcAS + o0 * 128, (uint32_t)(nOwn * 128), bar_D, warp);
      } else {
        ptx::bulk_s2peer(D1 + o0 * ds, D1 + o0 * ds, (uint32_t)(nOwn * ds * 4), bar_D, warp);
      }
    }
    for (int t = tid; t < nsmp; t += kThreads) {
      float v = 0.0f;
      if (t < O * H) {
        const int o = t / H, j = t - o * H;
#pragma unroll 8
        for (int q = 0; q < nOwn; ++q) v = fmaf(D2own[q * 32 + o], A1own[q * 32 + j], v);
      } else if (t < O * H + H) {
        const int j = t - O * H;
#pragma unroll 8
        for (int q = 0; q < nOwn; ++q) v += D1[(o0 + q) * ds + j];
      } else if (t < nsm) {
        const int o = t - O * H - H;
#pragma unroll 8
        for (int q = 0; q < nOwn; ++q) v += D2own[q * 32 + o];
      }
      gpart[t] = v;
    }
    ptx::fence_proxy_async_smem();
    __syncthreads();
    if (lane == 0 && warp < C && warp != rank) {
      const int c = warp;
      const int ce0 = e_begin(c, C, nsmp), cne = e_begin(c + 1, C, nsmp) - ce0;
      if (cne > 0) ptx::bulk_s2peer(grecv + rank * eslot, gpart + ce0, (uint32_t)(cne * 4), bar_D, c);
    }
    if (TC) ptx::mbar_wait(bar_D, par);  // (the SIMT P5 starts on its own rows and waits inside)
    PROF(5);

    if constexpr (TC) {
      // ---- P5 (tensor core). dW1 slice: D[px][j] = sum_rows x[row][px] delta_1[row][j] with
      //      M = 128 pixels (MN-major x tile), N = 32 neurons (MN-major delta_1), K = rows
      // (the M-layout x tile was split in P2; the delta_1 hi | lo rows were written by their owners in
      //  P3 and pushed in P4: rows >= nS of the operand stay zero from the kernel's set-up)
      PROF(15);
      if (ptx::warp_uniform(warp) == 0) {  // warp-uniform loop and operands, one elected lane issues
        tc::tc_fence_after();
        // B = delta_1 hi | lo: the lo block sits one MN block (LBO = kTcAS) behind the hi block, so an
        // N = 64 descriptor reads them stacked along N: two MMAs per k-step (x_lo, x_hi)
        constexpr uint32_t idM = tc::idesc_tf32(128, 64, true, true);
        const int nks = (nS + 7) / 8;
        const uint32_t tm = (uint32_t)ptx::warp_uniform((int)tmem) + 64u;
        if (ptx::elect_one()) {
          for (int ks = 0; ks < nks; ++ks) {
            const uint64_t ah = tc::smem_desc(sX + 1024 * ks, kTcAS, 512, 1);
            const uint64_t al = tc::smem_desc(sX + kTcXLoM + 1024 * ks, kTcAS, 512, 1);
            const uint64_t bd = tc::smem_desc(sD + 1024 * ks, kTcAS, 512, 1);
            tc::mma_tf32(tm, al, bd, idM, ks > 0 ? 1u : 0u);
            tc::mma_tf32(tm, ah, bd, idM, 1u);
          }
          tc::mma_commit(bar_mma);
        }
        __syncwarp();
      }
      ptx::mbar_wait(bar_mma, 1);
      tc::tc_fence_after();
      if (tid == 128 && s + 1 < p.n_steps) tc_issue(&tmXK, &bar_x[0], row_s1);  // next step's K-layout tile (warp 4: not an epilogue warp)
      if (warp < 4) {
        float v[32], vl[32];
        tc::tmem_ld32(tmem + ((uint32_t)(32 * warp) << 16) + 64u, v);
        tc::tmem_ld32(tmem + ((uint32_t)(32 * warp) << 16) + 96u, vl);
        const int px = 32 * warp + lane;
        if (px < p.ws) {  // neuron-major slice Gs[j][ws]: lanes = consecutive pixels (conflict-free)
#pragma unroll
          for (int j = 0; j < 32; ++j) Gs[j * p.ws + px] = v[j] + vl[j];
        }
      }
      tc::tc_fence_before();
    } else if constexpr (MM) {
      // ---- P5 (MM). dW1 slice, transposed: C(j, px) = sum_rows delta_1[row][j] x[row][px] with
      //      M = neurons (m-tile mt: 16 neurons), N = pixels, K = rows.  warp = (mt, 16-pixel
      //      block j = two n-blocks): n index g of n-block 2j / 2j+1 is pixel 16 j + 2g / +1 (one
      //      8-B load per lane and row), k = t / t + 4 of k-step ks are rows 8 ks + 2t / +1.  Then
      //      lane (g, t) holds exactly the elements it holds of W's fragments [j][nb][lane][4]
      //      (neurons 16 mt + g (nb = 2 mt) and 16 mt + 8 + g (nb = 2 mt + 1), pixels 16 j + 4t + e):
      //      Gs is written in that order and P9 is elementwise.  delta_1 RN-split (A), x
      //      truncation-split (B); delta_1 rows >= nS are zero.
      ptx::mbar_wait(bar_D, par);  // the peers' delta_1 rows (and W2/b slices) have landed
      PROF_MAX(15);
      // warp = (m-tile mt of 16 neurons, 16-pixel block j) over all rows (14 of the 16 warps for
      // config 2's 7 blocks; splitting the rows in halves for balance measured slower)
      const int mt = warp & 1, j = warp >> 1, gg = lane >> 2, tt = lane & 3;
      if (j < nj) {
        const int nks = (nS + 7) >> 3;
        float acc[2][4];
#pragma unroll
        for (int h = 0; h < 2; ++h) acc[h][0] = acc[h][1] = acc[h][2] = acc[h][3] = 0.0f;
        const float *dcol = D1 + 16 * mt + gg;
        const float *xc = xs + 16 * j + 2 * gg;
        for (int ks = 0; ks < nks; ++ks) {
          const int r0 = 8 * ks + 2 * tt;
          uint32_t ah[4], al[4];
          split_tf32(dcol[r0 * kDS], ah[0], al[0]);
          split_tf32(dcol[r0 * kDS + 8], ah[1], al[1]);
          split_tf32(dcol[(r0 + 1) * kDS], ah[2], al[2]);
          split_tf32(dcol[(r0 + 1) * kDS + 8], ah[3], al[3]);
          const float2 u = *reinterpret_cast<const float2 *>(xc + r0 * wpad);        // b0 of n-blocks 2j, 2j+1
          const float2 v = *reinterpret_cast<const float2 *>(xc + (r0 + 1) * wpad);  // b1
          uint32_t bh0[2], bl0[2], bh1[2], bl1[2];
          split_trunc(u.x, bh0[0], bl0[0]); split_trunc(v.x, bh0[1], bl0[1]);
          split_trunc(u.y, bh1[0], bl1[0]); split_trunc(v.y, bh1[1], bl1[1]);
          hmma_tf32(acc[0], al, bh0); hmma_tf32(acc[1], al, bh1);
          hmma_tf32(acc[0], ah, bl0); hmma_tf32(acc[1], ah, bl1);
          hmma_tf32(acc[0], ah, bh0); hmma_tf32(acc[1], ah, bh1);
        }
        // acc[h] = C over n-block 2j + h: c0 / c1 = neuron 16 mt + g, pixels 16 j + 4t + h / + 2 + h;
        // c2 / c3 the same for neuron 16 mt + 8 + g
        float4 *gs4 = reinterpret_cast<float4 *>(Gs);
        gs4[(j * 4 + 2 * mt) * 32 + lane] = make_float4(acc[0][0], acc[1][0], acc[0][1], acc[1][1]);
        gs4[(j * 4 + 2 * mt + 1) * 32 + lane] = make_float4(acc[0][2], acc[1][2], acc[0][3], acc[1][3]);
      }
      PROF_MAX(14);
    } else {

    // ---- P5. dW1 slice partial, k-major like W1t: Gs[k][j] = sum_{i<nS} D1[i][j] x[i][k]
    // Rows of this CTA's own delta_1 first, while the peers' rows are still in flight.
    for (int t = tid; t < nP5; t += kThreads) {
      const int jg = t & 7, kc = (t >> 3) % nchunk, rh = (t >> 3) / nchunk;
      const int ib = rh * nS / kRH, ie = (rh + 1) * nS / kRH;
      const float *dcol = D1 + jg * 4;
      const float *xcol = xs + kc * 4;
      float2 a[4][2];  // neuron u, pixel pairs (4kc, 4kc+1), (4kc+2, 4kc+3): packed FFMA2
#pragma unroll
      for (int u = 0; u < 4; ++u) a[u][0] = a[u][1] = make_float2(0.0f, 0.0f);
      auto rows = [&](int r0_, int r1_) {
#pragma unroll 4
        for (int i = r0_; i < r1_; ++i) {
          const float4 d = *reinterpret_cast<const float4 *>(dcol + i * 32);
          const float4 x = *reinterpret_cast<const float4 *>(xcol + i * wpad);
          const float dv[4] = {d.x, d.y, d.z, d.w};
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            ffma2(a[u][0], dv[u], make_float2(x.x, x.y));
            ffma2(a[u][1], dv[u], make_float2(x.z, x.w));
          }
        }
      };
      const int ob = max(ib, o0), oe = min(ie, o0 + nOwn);
      rows(ob, oe);
      ptx::mbar_wait(bar_D, par);  // the peers' delta_1 rows (and W2/b slices) have landed
      rows(ib, min(ie, ob));
      rows(max(ib, oe), ie);
      float *g = rh ? Gs2 : Gs;
#pragma unroll
      for (int v = 0; v < 4; ++v)
        *reinterpret_cast<float4 *>(g + (kc * 4 + v) * 32 + jg * 4) =
            make_float4(v & 1 ? a[0][v >> 1].y : a[0][v >> 1].x, v & 1 ? a[1][v >> 1].y : a[1][v >> 1].x,
                        v & 1 ? a[2][v >> 1].y : a[2][v >> 1].x, v & 1 ? a[3][v >> 1].y : a[3][v >> 1].x);
    }
    __syncthreads();
    for (int i = tid; i < wpad * 8; i += kThreads) {  // row halves summed in order
      float4 *d = reinterpret_cast<float4 *>(Gs) + i;
      const float4 h = reinterpret_cast<const float4 *>(Gs2)[i];
      float4 v = *d;
      v.x += h.x; v.y += h.y; v.z += h.z; v.w += h.w;
      *d = v;
    }
    ptx::mbar_wait(bar_D, par);  // threads without a P5 task
    }  // !TC
    // reduce my slice of the W2/b1/b2 tendencies over the cluster (rank order); the sum goes
    // to L2 with the dW1 slice in P6 as one more bulk reduction (aligned path: the slice is
    // 16-B aligned, e_begin), in place of gpart's own slice (never pushed to a peer)
    for (int e = tid; e < ne; e += kThreads) {
      float v = 0.0f;
      for (int c = 0; c < C; ++c) v += (c == rank) ? gpart[e0 + e] : grecv[c * eslot + e];
      if (p.aligned) gpart[e0 + e] = v;
      else ptx::red_add_f32(accS + p.small_off + e0 + e, v);
    }
    ptx::fence_proxy_async_smem();
    __syncthreads();
    PROF(6);

    // ---- P6. co_sum: add this CTA's dW1 slice into the L2 accumulator (the paper's co_sum)
    if (p.aligned) {
      if (tid == 0) {
        ptx::fence_proxy_async_global();
        ptx::bulk_reduce_add_f32(accS + slice_off, Gs, (uint32_t)(p.gsl * 4));
        if (ne > 0) ptx::bulk_reduce_add_f32(accS + p.small_off + e0, gpart + e0, (uint32_t)(ne * 4));
        ptx::bulk_commit();
        ptx::bulk_wait_all();
        ptx::fence_proxy_async_global();
      }
    } else {
      for (int i = tid; i < w * 32; i += kThreads)
        if ((i & 31) < H) ptx::red_add_f32(accS + slice_off + i, Gs[i]);
    }
    PROF(7);

    // ---- P7. grid barrier: the co_sum of this step is complete.  Between arrive and wait,
    //      zero this CTA's share of the slot used two steps ahead (its last readers finished
    //      before the previous barrier; its next writers start after the next one).
    __syncthreads();
    if (tid == 0) {
      // step s's cost entry is zeroed by CTA 0 before its arrival; every CTA adds its partial
      // after the barrier, i.e. after that zero (release / acquire through the counter)
      if (blockIdx.x == 0 && p.step_loss) p.step_loss[s] = 0.0f;
      ptx::grid_arrive(p.bar);
    }
    {
      float *z = p.acc + ((p.slot0 + s + 2) % kSlots) * p.slot;
      for (int64_t i = (int64_t)blockIdx.x * kThreads + tid; i < p.slot; i += (int64_t)nCTA * kThreads) z[i] = 0.0f;
    }
    if (TC && s + 1 < p.n_steps) {  // next step's K-layout tile: TF32 split while the barrier fills
      ptx::mbar_wait(&bar_x[0], (uint32_t)((s + 1) & 1));
      tc_split(X, X + kTcXLoK, 4 * kTcAS, tid);
      ptx::fence_proxy_async_smem();
    }
    if (tid == 0) grid_wait_from(p.bar, p.bar_base + (unsigned)((s + 1) * nCTA));
    __syncthreads();
    if (warp == 1 && p.step_loss) {  // this CTA's cost partial (lsum is rewritten in P3)
      const float l = warp_sum(lane < kWarps ? lsum[lane] : 0.0f);
      if (lane == 0) ptx::red_add_f32(p.step_loss + s, 0.5f * l * p.inv_B);
    }
    PROF(8);

    // ---- P8. read the reduced slice and the W2/b block back
    if (p.aligned) {
      if (tid == 0) {
        ptx::fence_proxy_async_global();
        ptx::mbar_arrive_expect_tx(bar_G, bytesG);
        ptx::bulk_g2s(Gr, accS + slice_off, (uint32_t)(p.gsl * 4), bar_G);
        ptx::bulk_g2s(gsm, accS + p.small_off, (uint32_t)(nsmp * 4), bar_G);
      }
      ptx::mbar_wait(bar_G, par);
    } else {
      for (int i = tid; i < w * 32; i += kThreads) Gr[i] = accS[slice_off + i];
      for (int i = tid; i < nsmp; i += kThreads) gsm[i] = accS[p.small_off + i];
      __syncthreads();
    }
    PROF(9);

    // ---- P9. SGD update of the resident parameters (all clusters apply the same sums)
    if constexpr (TC) {  // W = hi + lo exactly; re-split after the update
      // thread = (neuron j, 4 pixels): quarter-warps cover one 128-B row of an atom (conflict-free
      // float4 accesses of W hi / lo; Gr is neuron-major [j][ws])
      const int natom = (w + 31) >> 5;           // 32-pixel atoms of the slice
      for (int i = tid; i < natom * 256; i += kThreads) {
        const int q8 = i >> 5, jj = (i >> 3) & 3, c = i & 7;   // a warp: 8 chunks x 4 neuron rows of one atom
        const int a = q8 >> 3, j = 4 * (q8 & 7) + jj, k = 32 * a + 4 * c;
        if (j < H && k < w) {
          const int off = tc_w_off(j, k);
          float4 *hp = reinterpret_cast<float4 *>(Wt + off), *lp = reinterpret_cast<float4 *>(Wt + 4096 + off);
          const float4 hv = *hp, lv = *lp, gv = *reinterpret_cast<const float4 *>(Gr + j * p.ws + k);
          float wv[4] = {hv.x + lv.x, hv.y + lv.y, hv.z + lv.z, hv.w + lv.w};
          const float gq[4] = {gv.x, gv.y, gv.z, gv.w};
          float hh[4], ll[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            if (k + e < w) wv[e] -= p.scale * gq[e];
            hh[e] = tc::tf32_hi(wv[e]);
            ll[e] = wv[e] - hh[e];
          }
          *hp = make_float4(hh[0], hh[1], hh[2], hh[3]);
          *lp = make_float4(ll[0], ll[1], ll[2], ll[3]);
        }
      }
      ptx::fence_proxy_async_smem();
    } else if constexpr (MM) {  // W = hi + lo exactly; re-split after the update.  Gr has W's fragment order.
      float4 *Wh4 = reinterpret_cast<float4 *>(W1t), *Wl4 = Wh4 + nj * 128;
      const float4 *Gr4 = reinterpret_cast<const float4 *>(Gr);
      for (int i = tid; i < nj * 128; i += kThreads) {
        const int k = 16 * (i >> 7) + 4 * (i & 3);  // first pixel of the 4 (neurons >= H: W = G = 0)
        if (k >= w) continue;
        const float4 h = Wh4[i], l = Wl4[i], gv = Gr4[i];
        float wv[4] = {h.x + l.x, h.y + l.y, h.z + l.z, h.w + l.w};
        const float gq[4] = {gv.x, gv.y, gv.z, gv.w};
        float hh[4], ll[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          if (k + e < w) wv[e] -= p.scale * gq[e];
          hh[e] = tc::tf32_hi(wv[e]);
          ll[e] = wv[e] - hh[e];
        }
        Wh4[i] = make_float4(hh[0], hh[1], hh[2], hh[3]);
        Wl4[i] = make_float4(ll[0], ll[1], ll[2], ll[3]);
      }
    } else {
      for (int i = tid; i < w * 8; i += kThreads) {
        float4 wv = reinterpret_cast<float4 *>(W1t)[i];
        const float4 gv = reinterpret_cast<const float4 *>(Gr)[i];
        wv.x -= p.scale * gv.x; wv.y -= p.scale * gv.y; wv.z -= p.scale * gv.z; wv.w -= p.scale * gv.w;
        reinterpret_cast<float4 *>(W1t)[i] = wv;   // pad neurons j >= H: G = 0, W stays 0
      }
    }
    for (int e = tid; e < nsm; e += kThreads) {
      const float gv = p.scale * gsm[e];
      if (e < O * H) { const int o = e / H; W2s[o * 33 + (e - o * H)] -= gv; }
      else if (e < O * H + H) b1s[e - O * H] -= gv;
      else b2s[e - O * H - H] -= gv;
    }
    __syncthreads();
    PROF(10);
    row_s = row_s1;
  }
  cp_async_wait0();

  // ---- write the resident parameters back (W1 slice by every CTA of cluster 0; the rest by CTA 0)
  if (g == 0) {
    if constexpr (MM) {
      for (int i = tid; i < nj * 512; i += kThreads) {
        const int ln = (i >> 2) & 31, nbj = i >> 7;
        const int n = 8 * (nbj & 3) + (ln >> 2), k = 16 * (nbj >> 2) + 4 * (ln & 3) + (i & 3);
        if (n < H && k < w) p.params[oW1 + (int64_t)n * n0 + k0 + k] = W1t[i] + W1t[nj * 512 + i];
      }
    }
    for (int i = tid; i < (MM ? 0 : w * 32); i += kThreads) {
      const int k = i >> 5, j = i & 31;
      if (j >= H) continue;
      float v;
      if constexpr (TC) {
        const int off = tc_w_off(j, k);
        v = *reinterpret_cast<const float *>(Wt + off) + *reinterpret_cast<const float *>(Wt + 4096 + off);
      } else {
        v = W1t[i];
      }
      p.params[oW1 + (int64_t)j * n0 + k0 + k] = v;
    }
    if (rank == 0) {
      for (int i = tid; i < O * H; i += kThreads) p.params[oW2 + i] = W2s[(i / H) * 33 + i % H];
      for (int i = tid; i < H; i += kThreads) p.params[ob1 + i] = b1s[i];
      for (int i = tid; i < O; i += kThreads) p.params[ob2 + i] = b2s[i];
    }
  }
  ptx::cluster_sync();  // no CTA exits while a peer may still push into it
  if (TC && warp == 0) {
    tc::tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(128u) : "memory");
  }
}

int env_int(const char *name, int dflt) {
  const char *v = getenv(name);
  return v ? atoi(v) : dflt;
}

}  // namespace

int fused_small_train_steps(FusedSmall &fs, cudaStream_t st, const std::vector<int> &dims, int act_h,
                            int act_o, float *params, const float *X, const float *Y, int64_t N,
                            int64_t batch, const int64_t *starts, int64_t n_steps, float eta,
                            float *step_loss) {
  if (env_int("NF_DISABLE_FUSED", 0)) return FUSED_NOT_APPLICABLE;
  // the co_sum here is an L2 bulk-add in arrival order: NF_SPLITK_DETERMINISTIC=1 (bitwise
  // repeatable training, reading R12) takes the generic per-layer path, whose sums are fixed-order
  if (getenv("NF_SPLITK_DETERMINISTIC")) return FUSED_NOT_APPLICABLE;
  if (dims.size() != 3) return FUSED_NOT_APPLICABLE;
  const int n0 = dims[0], H = dims[1], O = dims[2];
  if (H > 32 || O > 32 || batch > (int64_t)148 * kMaxRows) return FUSED_NOT_APPLICABLE;

  const bool aligned_now = (n0 % 4 == 0) && ((uintptr_t)X % 16 == 0) && env_int("NF_FUSED_NOTMA", 0) == 0;
  // ---- launch configuration: decided once per (shape, batch, dataset, switches), then cached
  // (the occupancy query and the tensor-map encodes cost host microseconds per call)
  const std::vector<int64_t> key = {n0, H, O, batch, (int64_t)(uintptr_t)X, N, aligned_now,
                                    env_int("NF_FUSED_C", 0), env_int("NF_FUSED_G", 0), env_int("NF_FUSED_TC", 1),
                                    env_int("NF_FUSED_MM", 0)};
  if (key != fs.cfg_key) {
    fs.cfg_key.clear();
  // cluster size: pixel slices of >= 32 columns, at most 8 CTAs
  int C = env_int("NF_FUSED_C", 0);
  if (C <= 0) {
    C = kMaxC;
    while (C > 1 && n0 / C < 32) C /= 2;
  }
  C = std::max(1, std::min(C, kMaxC));
  const bool aligned = aligned_now;
  int ws, wpad;
  if (aligned) {
    ws = ((n0 + C - 1) / C + 3) / 4 * 4;
    while (C > 1 && (C - 1) * ws >= n0) { --C; ws = ((n0 + C - 1) / C + 3) / 4 * 4; }
    wpad = ws;
  } else {
    ws = (n0 + C - 1) / C;
    wpad = (ws + 3) / 4 * 4;
  }
  if (wpad > 256) return FUSED_NOT_APPLICABLE;  // TMA box limit / smem budget

  {  // (per device: the attributes belong to the device context)
    static std::mutex mu;
    static unsigned done = 0;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    if (!(done & (1u << (dev & 31)))) {
      const void *ks[] = {
          (const void *)fused_small_kernel<false, false, -1, -1, kInlineStarts>,
          (const void *)fused_small_kernel<true, false, -1, -1, kInlineStarts>,
          (const void *)fused_small_kernel<false, false, ACT_SIGMOID, ACT_SIGMOID, kInlineStarts>,
          (const void *)fused_small_kernel<false, true, -1, -1, kInlineStarts>,
          (const void *)fused_small_kernel<false, true, ACT_SIGMOID, ACT_SIGMOID, kInlineStarts>,
          (const void *)fused_small_kernel<false, false, -1, -1, kInlineSmall>,
          (const void *)fused_small_kernel<false, false, ACT_SIGMOID, ACT_SIGMOID, kInlineSmall>,
          (const void *)fused_small_kernel<false, true, -1, -1, kInlineSmall>,
          (const void *)fused_small_kernel<false, true, ACT_SIGMOID, ACT_SIGMOID, kInlineSmall>,
          (const void *)fused_small_kernel<true, false, ACT_SIGMOID, ACT_SIGMOID, kInlineStarts>,
          (const void *)fused_small_kernel<true, false, -1, -1, kInlineSmall>,
          (const void *)fused_small_kernel<true, false, ACT_SIGMOID, ACT_SIGMOID, kInlineSmall>};
      for (const void *k : ks) {
        cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
      }
      done |= 1u << (dev & 31);
    }
  }
  // tensor-core variant (the default where it applies; NF_FUSED_TC=0 selects the FFMA2 path):
  // TMA-aligned x, pixel slices of <= 128 columns, <= kTcRows rows per cluster.  Split-TF32 MMAs with
  // the hi | lo parts of W1 / delta_1 stacked along N (two MMAs per k-step, all four partial
  // products), issued warp-uniformly: 9.9 vs 11.0 us per config-2 step (profiles/r02_k6_tc_stacked.txt)
  bool tc = aligned && ws <= 128 && env_int("NF_FUSED_TC", 1) != 0 && env_int("NF_FUSED_MM", 0) == 0;
  // warp-level MMA contractions (opt-in NF_FUSED_MM=1; TMA-aligned x, <= 128 rows per cluster,
  // pixel slices <= 128): parity-green, but 11.25 vs 11.05 us per config-2 step against the FFMA2
  // SIMT default (profiles/r02_k6_mma_experiment.txt)
  const bool mm_ok = aligned && !tc && mm_nj(wpad) <= kMJ && env_int("NF_FUSED_MM", 0) != 0;
  auto mm_for = [&](int nSmax) { return mm_ok && mm_rows(nSmax) <= 16 * kMT1; };
  auto smem_for = [&](int G) {
    const int nSmax = (int)((batch + G - 1) / G);
    const int nOwnMax = (nSmax + C - 1) / C;
    return (size_t)smem_layout(wpad, nSmax, nOwnMax, C, tc && nSmax <= kTcRows, mm_for(nSmax)).total * sizeof(float) +
           (tc ? 1024 : 0);
  };
  // clusters: as many as co-reside at 1 CTA/SM, with <= kMaxRows rows per cluster
  int G = 0;
  {
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim = {(unsigned)C, 1, 1};
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cfg.blockDim = dim3(kThreads);
    const int maxG = env_int("NF_FUSED_G", 0);
    int want = maxG > 0 ? maxG : (int)std::max<int64_t>(1, std::min<int64_t>(batch / 16, kMinBlocks * 148 / C));
    for (int cand = want; cand >= 1; --cand) {
      if ((batch + cand - 1) / cand > kMaxRows) break;
      cfg.gridDim = dim3(cand * C);
      cfg.dynamicSmemBytes = smem_for(cand);
      if (cfg.dynamicSmemBytes > 227 * 1024) continue;
      int ncl = 0;
      const bool tcc = tc && (batch + cand - 1) / cand <= kTcRows;
      const bool mmc = mm_for((int)((batch + cand - 1) / cand));
      if (cudaOccupancyMaxActiveClusters(&ncl, tcc ? fused_small_kernel<true, false, -1, -1, kInlineStarts>
                                               : mmc ? fused_small_kernel<false, true, -1, -1, kInlineStarts>
                                                     : fused_small_kernel<false, false, -1, -1, kInlineStarts>,
                                         &cfg) !=
          cudaSuccess) {
        cudaGetLastError();
        continue;
      }
      if (ncl >= cand) { G = cand; break; }
    }
    if (G < 1) return FUSED_NOT_APPLICABLE;
  }
  const int nSmax = (int)((batch + G - 1) / G);
  const int nOwnMax = (nSmax + C - 1) / C;
  const size_t smem = smem_for(G);
  tc = tc && nSmax <= kTcRows;
  const bool mm = mm_for(nSmax);

  CUtensorMap tmX, tmXK, tmXM;
  memset(&tmX, 0, sizeof tmX);
  memset(&tmXK, 0, sizeof tmXK);
  memset(&tmXM, 0, sizeof tmXM);
  if (tc && (!encode_tmap_2d_f32(&tmXK, X, (uint64_t)n0, (uint64_t)N, (uint64_t)n0 * 4, 32, kTcRows,
                                 CU_TENSOR_MAP_SWIZZLE_128B) ||
             !encode_tmap_2d_f32(&tmXM, X, (uint64_t)n0, (uint64_t)N, (uint64_t)n0 * 4, 32, kTcRows,
                                 CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B))) {
    snprintf(g_fs_err, sizeof g_fs_err, "cuTensorMapEncodeTiled (TC tiles) failed");
    return -1;
  }
  if (aligned && !encode_tmap_2d_f32(&tmX, X, (uint64_t)n0, (uint64_t)N, (uint64_t)n0 * 4, (uint32_t)ws,
                                     (uint32_t)nSmax, CU_TENSOR_MAP_SWIZZLE_NONE)) {
    snprintf(g_fs_err, sizeof g_fs_err, "cuTensorMapEncodeTiled failed (cols %d rows %lld box %dx%d)", n0,
             (long long)N, ws, nSmax);
    return -1;
  }
    fs.C = C; fs.G = G; fs.ws_cols = ws; fs.wpad = wpad; fs.nSmax = nSmax; fs.nOwnMax = nOwnMax;
    fs.smem = smem; fs.tc = tc; fs.mm = mm; fs.aligned = aligned;
    memcpy(fs.tmaps[0], &tmX, sizeof tmX);
    memcpy(fs.tmaps[1], &tmXK, sizeof tmXK);
    memcpy(fs.tmaps[2], &tmXM, sizeof tmXM);
    fs.cfg_key = key;
  }
  host_trace("k6 config");
  const int C = fs.C, G = fs.G, ws = fs.ws_cols, wpad = fs.wpad, nSmax = fs.nSmax, nOwnMax = fs.nOwnMax;
  const size_t smem = fs.smem;
  const bool tc = fs.tc, mm = fs.mm, aligned = fs.aligned;
  CUtensorMap tmX, tmXK, tmXM;
  memcpy(&tmX, fs.tmaps[0], sizeof tmX);
  memcpy(&tmXK, fs.tmaps[1], sizeof tmXK);
  memcpy(&tmXM, fs.tmaps[2], sizeof tmXM);
  const int nCTA = G * C;

  // accumulator slot: [C][ws][32] dW1 slices (k-major), then the W2/b1/b2 block (16-B aligned)
  const int nsmp = (O * H + H + O + 3) & ~3;
  const int gsl = mm ? mm_nj(wpad) * 512 : ws * 32;  // floats of a rank's dW1 slice
  const int64_t small_off = (int64_t)C * gsl;
  const int64_t slot = (small_off + nsmp + 31) & ~int64_t(31);
  const size_t need = kSlots * slot * sizeof(float) + 256;
  if (fs.ws_bytes < need) {
    if (fs.ws) cudaFree(fs.ws);
    fs.ws = nullptr;
    fs.ws_bytes = 0;
    fs.ws_ready = false;
    if (cudaMalloc(&fs.ws, need) != cudaSuccess) {
      snprintf(g_fs_err, sizeof g_fs_err, "workspace allocation of %zu bytes failed", need);
      return -1;
    }
    fs.ws_bytes = need;
  }
  if (fs.ring_key[0] != slot || fs.ring_key[1] != nCTA) fs.ws_ready = false;
  // batch starts: host array -> pinned staging buffer (double-buffered) -> device, asynchronous
  if (n_steps > kInlineStarts && fs.starts_cap < (size_t)n_steps) {
    for (int i = 0; i < 2; ++i) {
      if (fs.h_ev[i]) cudaEventSynchronize(fs.h_ev[i]);
      if (fs.h_starts[i]) cudaFreeHost(fs.h_starts[i]);
      fs.h_starts[i] = nullptr;
    }
    if (fs.d_starts) cudaFree(fs.d_starts);
    fs.d_starts = nullptr;
    fs.starts_cap = 0;
    const size_t cap = std::max<size_t>(1024, (size_t)n_steps);
    if (cudaMalloc(&fs.d_starts, cap * sizeof(int64_t)) != cudaSuccess ||
        cudaMallocHost(&fs.h_starts[0], cap * sizeof(int64_t)) != cudaSuccess ||
        cudaMallocHost(&fs.h_starts[1], cap * sizeof(int64_t)) != cudaSuccess) {
      snprintf(g_fs_err, sizeof g_fs_err, "batch-start buffers: %s", cudaGetErrorString(cudaGetLastError()));
      return -1;
    }
    for (int i = 0; i < 2; ++i)
      if (!fs.h_ev[i]) cudaEventCreateWithFlags(&fs.h_ev[i], cudaEventDisableTiming);
    fs.starts_cap = cap;
  }
  char *base = static_cast<char *>(fs.ws);
  FusedParams p{};
  p.n0 = n0; p.H = H; p.O = O; p.act_h = act_h; p.act_o = act_o;
  p.B = (int)batch; p.G = G; p.ws = ws; p.wpad = wpad; p.aligned = aligned ? 1 : 0;
  p.nSmax = nSmax; p.nOwnMax = nOwnMax;
  p.n_steps = n_steps;
  p.slot = slot;
  p.small_off = small_off;
  p.nsmp = nsmp;
  p.gsl = gsl;
  p.scale = (float)((double)eta / (double)batch);
  p.inv_B = (float)(1.0 / (double)batch);
  p.X = X; p.Y = Y; p.params = params;
  p.acc = reinterpret_cast<float *>(base);
  p.bar = reinterpret_cast<unsigned *>(base + kSlots * slot * sizeof(float));
  p.starts = fs.d_starts;
  p.step_loss = step_loss;
  static long long *prof_buf = nullptr;
  const bool prof = env_int("NF_FUSED_PROF", 0) != 0;
  if (prof) {
    if (!prof_buf) cudaMalloc(&prof_buf, sizeof(long long) * 148 * 64 * kProf);
    cudaMemsetAsync(prof_buf, 0, sizeof(long long) * 148 * 64 * kProf, st);
    p.prof = prof_buf;
  }

  cudaError_t e = cudaSuccess;
  if (!fs.ws_ready) {  // a fresh ring: all slots zero, counter 0
    e = cudaMemsetAsync(base, 0, kSlots * slot * sizeof(float) + 256, st);
    fs.steps_done = 0;
    fs.bar_base = 0;
    fs.ring_key[0] = slot;
    fs.ring_key[1] = nCTA;
  }
  p.slot0 = (int)(fs.steps_done % kSlots);
  p.bar_base = fs.bar_base;
  static thread_local InlineStarts<kInlineStarts> ist;  // host staging of the launch parameter buffer
  static thread_local InlineStarts<kInlineSmall> ist_s;
  const bool small_ist = n_steps <= kInlineSmall;
  if (small_ist) {
    memcpy(ist_s.v, starts, n_steps * sizeof(int64_t));
    p.starts = nullptr;
  } else if (n_steps <= kInlineStarts) {
    memcpy(ist.v, starts, n_steps * sizeof(int64_t));
    p.starts = nullptr;
  } else {
    const int hb = fs.h_i;
    fs.h_i ^= 1;
    if (e == cudaSuccess) e = cudaEventSynchronize(fs.h_ev[hb]);  // its previous copy has completed
    if (e == cudaSuccess) {
      memcpy(fs.h_starts[hb], starts, n_steps * sizeof(int64_t));
      e = cudaMemcpyAsync(fs.d_starts, fs.h_starts[hb], n_steps * sizeof(int64_t), cudaMemcpyHostToDevice, st);
    }
    if (e == cudaSuccess) e = cudaEventRecord(fs.h_ev[hb], st);
  }
  host_trace("k6 starts");
  if (e == cudaSuccess) {
    static const bool coop = env_int("NF_FUSED_NOCOOP", 0) == 0;
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim = {(unsigned)C, 1, 1};
    // cooperative: the runtime guarantees every CTA is co-resident (the grid barriers need it)
    // or fails the launch, instead of a hang when another stream holds SMs
    at[1].id = cudaLaunchAttributeCooperative;
    at[1].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = coop ? 2 : 1;
    cfg.gridDim = dim3(G * C);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    const bool sig = act_h == ACT_SIGMOID && act_o == ACT_SIGMOID;
    static bool coop_ok = true;
    if (!coop_ok) cfg.numAttrs = 1;
    const void *kern = nullptr;
    auto launch = [&]() {
      if (small_ist) {
        auto k = mm ? (sig ? fused_small_kernel<false, true, ACT_SIGMOID, ACT_SIGMOID, kInlineSmall>
                           : fused_small_kernel<false, true, -1, -1, kInlineSmall>)
                    : tc ? (sig ? fused_small_kernel<true, false, ACT_SIGMOID, ACT_SIGMOID, kInlineSmall>
                                : fused_small_kernel<true, false, -1, -1, kInlineSmall>)
                    : sig ? fused_small_kernel<false, false, ACT_SIGMOID, ACT_SIGMOID, kInlineSmall>
                          : fused_small_kernel<false, false, -1, -1, kInlineSmall>;
        kern = reinterpret_cast<const void *>(k);
        return cudaLaunchKernelEx(&cfg, k, p, tmX, tmXK, tmXM, ist_s);
      }
      auto k = tc   ? (sig ? fused_small_kernel<true, false, ACT_SIGMOID, ACT_SIGMOID, kInlineStarts>
                           : fused_small_kernel<true, false, -1, -1, kInlineStarts>)
               : mm ? (sig ? fused_small_kernel<false, true, ACT_SIGMOID, ACT_SIGMOID, kInlineStarts>
                           : fused_small_kernel<false, true, -1, -1, kInlineStarts>)
               : sig ? fused_small_kernel<false, false, ACT_SIGMOID, ACT_SIGMOID, kInlineStarts>
                     : fused_small_kernel<false, false, -1, -1, kInlineStarts>;
      kern = reinterpret_cast<const void *>(k);
      return cudaLaunchKernelEx(&cfg, k, p, tmX, tmXK, tmXM, ist);
    };
    e = launch();
    if (e != cudaSuccess && cfg.numAttrs == 2 && e != cudaErrorCooperativeLaunchTooLarge) {
      // cooperative + cluster launch unsupported by this driver: plain cluster launch (the grid
      // was sized from cudaOccupancyMaxActiveClusters); a too-large grid is still an error
      cudaGetLastError();
      coop_ok = false;
      cfg.numAttrs = 1;
      e = launch();
    }
    count_launch();
    char nt[64];
    snprintf(nt, sizeof nt, "cluster=%d steps=%lld%s%s", C, (long long)n_steps, cfg.numAttrs == 2 ? " cooperative" : "",
             mm ? " mma" : tc ? " tcgen05" : " simt");
    log_launch(kern, cfg.gridDim, cfg.blockDim, smem, nt);
  }
  host_trace("k6 launch");
  if (e == cudaSuccess) {
    fs.ws_ready = true;
    fs.steps_done += (uint64_t)n_steps;
    fs.bar_base += (unsigned)(n_steps * nCTA);
  } else {
    fs.ws_ready = false;
  }
  if (e != cudaSuccess) {
    snprintf(g_fs_err, sizeof g_fs_err, "launch (C=%d G=%d smem=%zu): %s", C, G, smem, cudaGetErrorString(e));
    return -1;
  }
  if (prof) {
    std::vector<long long> h((size_t)G * C * 64 * kProf);
    cudaStreamSynchronize(st);
    cudaMemcpy(h.data(), prof_buf, h.size() * sizeof(long long), cudaMemcpyDeviceToHost);
    int dev = 0, khz = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, dev);
    const double ns_per_clk = khz > 0 ? 1e6 / khz : 0.5;
    const int ns = (int)std::min<int64_t>(n_steps, 64);
    const int nslot = 11;
    double ph[kProf] = {0}, phmax[kProf] = {0};
    int cnt = 0;
    for (int s = 2; s + 1 < ns; ++s, ++cnt) {
      for (int i = 0; i < nslot; ++i) {
        double mx = 0, sum = 0;
        for (int b = 0; b < G * C; ++b) {
          const long long *t = &h[((size_t)b * 64 + s) * kProf];
          const long long a = t[i];
          const long long nxt = i < nslot - 1 ? t[i + 1] : h[((size_t)b * 64 + s + 1) * kProf];
          const double d = (a && nxt) ? (double)(nxt - a) : 0.0;
          sum += d; mx = std::max(mx, d);
        }
        ph[i] += sum / (G * C); phmax[i] += mx;
      }
    }
    fprintf(stderr, "[fused prof] %s C=%d G=%d nS<=%d ws=%d aligned=%d smem=%zu  phase clk (mean over CTAs / max), "
            "ns at %.0f MHz:\n", tc ? "tcgen05" : mm ? "mma" : "simt", C, G, nSmax, ws, (int)aligned, smem, khz / 1e3);
    const char *names[11] = {"P0 wait_x+issue", "P1 z1_partial", "P2 push_P+wait", "P3 owned_rows",
                             "P4 push_D+gpart", "P5 dW1+small_red", "P6 co_sum_bulk", "P7 grid_bar",
                             "P8 readback", "P9 update+zero", "tail"};
    double tot = 0;
    for (int i = 0; i < nslot; ++i) {
      fprintf(stderr, "  %-18s %8.0f clk %8.0f max  %7.0f ns\n", names[i], ph[i] / cnt, phmax[i] / cnt,
              ph[i] / cnt * ns_per_clk);
      tot += ph[i] / cnt;
    }
    fprintf(stderr, "  %-18s %8.0f clk            %7.0f ns\n", "step", tot, tot * ns_per_clk);
    {  // TC sub-phases of P1 (1 -> 13 issue -> 14 mma wait -> 2) and P5 (5 -> 15 split -> 6)
      double a = 0, b = 0, c = 0, d = 0;
      int n = 0;
      for (int s = 2; s + 1 < ns; ++s)
        for (int bl = 0; bl < G * C; ++bl, ++n) {
          const long long *t = &h[((size_t)bl * 64 + s) * kProf];
          a += (double)(t[13] - t[1]); b += (double)(t[14] - t[13]); c += (double)(t[2] - t[14]);
          d += (double)(t[15] - t[5]);
        }
      if (tc)
        fprintf(stderr, "  P1 split: issue %.0f, mma wait %.0f, epilogue %.0f clk;  P5 split+D build %.0f clk\n",
                a / n, b / n, c / n, d / n);
      if (mm) {  // slots 13 / 15 / 14: last warp done with P1's MMAs / through P5's wait / done with P5's MMAs
        double e1 = 0, e2 = 0, e3 = 0, e4 = 0, e5 = 0;
        int m = 0;
        for (int s = 2; s + 1 < ns; ++s)
          for (int bl = 0; bl < G * C; ++bl, ++m) {
            const long long *t = &h[((size_t)bl * 64 + s) * kProf];
            e1 += (double)(t[13] - t[1]); e2 += (double)(t[2] - t[13]); e3 += (double)(t[15] - t[5]);
            e4 += (double)(t[14] - t[15]); e5 += (double)(t[6] - t[14]);
          }
        fprintf(stderr, "  MM split: P1 mma (last warp) %.0f, P1 K-part sum %.0f;  P5 wait %.0f, P5 mma (last warp) %.0f, "
                "P5 rest %.0f clk\n", e1 / m, e2 / m, e3 / m, e4 / m, e5 / m);
      }
    }
    {  // sub-phases of P3: slots 3 -> 11 -> 12 -> 4
      double a = 0, b = 0, c = 0;
      int n = 0;
      for (int s = 2; s + 1 < ns; ++s)
        for (int bl = 0; bl < G * C; ++bl, ++n) {
          const long long *t = &h[((size_t)bl * 64 + s) * kProf];
          a += (double)(t[11] - t[3]); b += (double)(t[12] - t[11]); c += (double)(t[4] - t[12]);
        }
      fprintf(stderr, "  P3 split: (a) z1/act %.0f clk, (b) layer 2 %.0f clk, (c) delta_1+loss %.0f clk\n", a / n, b / n,
              c / n);
    }
  }
  return 0;
}

void fused_small_release(FusedSmall &fs) {
  if (fs.ws) cudaFree(fs.ws);
  fs.ws = nullptr;
  fs.ws_bytes = 0;
  fs.ws_ready = false;
  for (int i = 0; i < 2; ++i) {
    if (fs.h_ev[i]) {
      cudaEventSynchronize(fs.h_ev[i]);
      cudaEventDestroy(fs.h_ev[i]);
    }
    if (fs.h_starts[i]) cudaFreeHost(fs.h_starts[i]);
    fs.h_ev[i] = nullptr;
    fs.h_starts[i] = nullptr;
  }
  if (fs.d_starts) cudaFree(fs.d_starts);
  fs.d_starts = nullptr;
  fs.starts_cap = 0;
  fs.cfg_key.clear();
}

void fused_small_invalidate(FusedSmall &fs) { fs.valid = false; }

const char *fused_small_error() { return g_fs_err; }

}  // namespace nf
