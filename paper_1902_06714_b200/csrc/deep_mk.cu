// deep_mk.cu -- the deep-net task megakernel (see deep_mk.cuh).
//
// Step s of a call is the task list (built once on the host, same for every step):
//   FWD(l, mb, nb)   l = 1..L-1: tile [128 rows x 64 cols] of Z_l = A_{l-1} W_l^T + b_l,
//                    epilogue A_l = sigma(Z_l) (TF32-rounded), S_l = sigma'(Z_l)
//   OUT(mb)          the narrow output layer for 128 rows (SIMT): z_L, a_L, delta_L, the cost,
//                    delta_{L-1} = (delta_L W_L) .* S_{L-1} in place of S_{L-1}, and the row
//                    block's partial tendency of W_L, b_L
//   BWD(l, mb, nb)   l = L-1..2: tile of delta_{l-1} = (delta_l W_l) .* S_{l-1}, in place
//   GRAD(l, c, mt, nt) l = L-1..1: tile of G_l = delta_l^T A_{l-1} over the rows of chunk c,
//                    added into W_l as -(eta/B) G (L2 reductions; the co_sum P:536-556 and the
//                    update P:423-427); tiles with nt = 0 also reduce the chunk's bias sums
//   GFIN             W_L, b_L update from the OUT partials (fixed order) and the step's cost
//   ROUND(l, q)      slice q of the TF32 shadow of W_l (reading R13) for the next step
// Dependencies are counters in global memory (monotonic within the launch, target = (s + 1) x
// per-step count): FWD(l) of row block mb waits for FWD(l-1) of mb, BWD / GRAD for delta_l of
// their rows, ROUND for every GRAD(l) and BWD(l), step s+1's first layer for all of step s.
// Task t of a step runs on CTA t mod grid; a CTA runs its tasks in list order, which is a
// topological order, so the earliest unfinished task can always run (all CTAs co-resident:
// cooperative launch).
//
// TC tiles: BM = 128 (TMEM lanes), BN = 64, BK = 32 fp32 (one SWIZZLE_128B row), 1xTF32 MMAs
// (kind::tf32) with the shadow / stored operands already RN-rounded; warp 0 TMA producer, warp 1
// MMA issuer, warps 2-5 epilogue (thread = tile row).  The ring state carries across tasks.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "deep_mk.cuh"
#include "gemm_tc.cuh"
#include "kernels.cuh"
#include "nf_common.cuh"
#include "sm100_ptx.cuh"

namespace nf {

static thread_local char g_dmk_err[256] = "";

namespace {

constexpr int BM = 128, BN = 64, BK = 32;
constexpr int kStages = 6;
constexpr int kThreads = 192;               // producer, MMA, 4 epilogue warps
constexpr int kMaxL = 16;
constexpr int A_BYTES = BM * BK * 4, B_BYTES = BN * BK * 4, STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int kNOut = 16;                   // max output width (OUT tasks)
constexpr int BMO = 32;                     // rows per OUT task (4 per 128-row block)
constexpr int kOutPer = BM / BMO;
constexpr int kMaxH = 256;                  // max hidden width
constexpr int kMapsPerLayer = 6;            // fwd A, fwd W, bwd D, bwd W (MN), grad D (MN), grad A (MN)
enum : int { T_FWD = 0, T_OUT = 1, T_BWD = 2, T_GRAD = 3, T_GFIN = 4, T_ROUND = 5 };
enum : int { M_FA = 0, M_FW = 1, M_BD = 2, M_BW = 3, M_GD = 4, M_GA = 5 };

struct Params {
  int L, B, nrb, kc, nchunk, nq, T;
  int dims[kMaxL + 1];
  int act[kMaxL + 1];
  int64_t offW[kMaxL + 1], offB[kMaxL + 1];
  float *A[kMaxL + 1], *S[kMaxL + 1];
  float *params, *params_t;
  const float *X, *Y;
  const int4 *tasks;
  const CUtensorMap *maps;
  const int64_t *starts;
  unsigned *ctr;
  float *part;                              // [nrb][nL][n_{L-1}+1] OUT partial tendencies
  float *lpart;                             // [nrb] OUT partial costs
  float *step_loss;
  float scale, inv_B;
  int64_t n_steps;
  unsigned long long *prof;                 // NF_DMK_PROF=1: [grid][prof_cap][4] globaltimer stamps
  int prof_cap;
};

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// counter layout (uints): fwd[l][mb], dlt[l][mb], grad[l], bwdall[l], oall, step
__device__ __forceinline__ unsigned *c_fwd(const Params &p, int l, int mb) { return p.ctr + l * p.nrb + mb; }
__device__ __forceinline__ unsigned *c_dlt(const Params &p, int l, int mb) {
  return p.ctr + (kMaxL + 1) * p.nrb + l * p.nrb + mb;
}
__device__ __forceinline__ unsigned *c_grad(const Params &p, int l) { return p.ctr + 2 * (kMaxL + 1) * p.nrb + l; }
__device__ __forceinline__ unsigned *c_bwdall(const Params &p, int l) {
  return p.ctr + 2 * (kMaxL + 1) * p.nrb + (kMaxL + 1) + l;
}
__device__ __forceinline__ unsigned *c_oall(const Params &p) { return p.ctr + 2 * (kMaxL + 1) * p.nrb + 2 * (kMaxL + 1); }
__device__ __forceinline__ unsigned *c_step(const Params &p) { return c_oall(p) + 32; }

__device__ __forceinline__ void wait_ge(const unsigned *c, unsigned target) {
  unsigned v;
  do {
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(c) : "memory");
  } while ((int)(v - target) < 0);
}
__device__ __forceinline__ void signal(unsigned *c) {
  asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(c) : "memory");
}
__device__ __forceinline__ void red_v4(float *p, float a, float b, float c, float d) {
  asm volatile("red.relaxed.gpu.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d)
               : "memory");
}

__host__ __device__ inline int cdiv(int a, int b) { return (a + b - 1) / b; }
// per-step counts
__host__ __device__ inline int tn_of(int n) { return cdiv(n, BN); }       // 64-col tiles of width n

// forward epilogue of 32 columns of one row: z = acc + b, A = rn(sigma(z)), S = sigma'(z)
template <int K>
__device__ __forceinline__ void fwd_chunk(float (&v)[32], const float *bias, float *Arow, float *Srow) {
  float4 b4[8];  // every bias load in flight before any store
#pragma unroll
  for (int j = 0; j < 8; ++j) b4[j] = __ldcg(reinterpret_cast<const float4 *>(bias) + j);
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const float bb[4] = {b4[j].x, b4[j].y, b4[j].z, b4[j].w};
    float a[4], sg[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      act_fwd_t<K>(v[4 * j + u] + bb[u], a[u], sg[u]);
      a[u] = tf32_rn(a[u]);
    }
    reinterpret_cast<float4 *>(Arow)[j] = make_float4(a[0], a[1], a[2], a[3]);
    reinterpret_cast<float4 *>(Srow)[j] = make_float4(sg[0], sg[1], sg[2], sg[3]);
  }
}

__global__ void __launch_bounds__(kThreads, 1) deep_mk_kernel(const __grid_constant__ Params p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + kStages * STAGE_BYTES);
  uint64_t *empty = full + kStages;
  uint64_t *accum = empty + kStages;          // [0] accumulator ready, [2] OUT staging
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(accum + 4);
  float *sred = reinterpret_cast<float *>(tmem_slot + 4);  // [kThreads + 8] reduction scratch / stamps

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
  const int L = p.L, nL = p.dims[L], H = p.dims[L - 1];

  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    ptx::mbar_init(accum, 1);
    ptx::mbar_init(accum + 2, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 ::"r"(ptx::smem_u32(tmem_slot)), "r"(64u) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  uint32_t it = 0;       // K-blocks issued by this CTA (ring position, across tasks)
  uint32_t ntc = 0;      // TC tasks run by this CTA (accumulator barrier parity)
  uint32_t nout = 0;     // OUT tasks run by this CTA (staging barrier parity)
  const int T = p.T;
  int np = 0;  // profiled tasks of this CTA
  for (int64_t s = 0; s < p.n_steps; ++s) {
    const int64_t start = p.starts[s];
    const unsigned tgt = (unsigned)(s + 1);
    for (int t = blockIdx.x; t < T; t += gridDim.x) {
      const int4 tk = p.tasks[t];
      const int type = tk.x & 0xff, l = tk.x >> 8;
      // ---- dependencies (one thread spins, then the CTA goes)
      unsigned long long t0 = 0, t1 = 0;
      if (tid == 0) {
        if (p.prof) t0 = gtime();
        if (type == T_FWD) {
          if (l == 1) { if (s > 0) wait_ge(c_step(p), (unsigned)(s * T)); }
          else wait_ge(c_fwd(p, l - 1, tk.y), tgt * tn_of(p.dims[l - 1]));
        } else if (type == T_OUT) {  // rows [y*32, y*32+32) of A_{L-1}
          wait_ge(c_fwd(p, L - 1, tk.y / kOutPer), tgt * tn_of(p.dims[L - 1]));
        } else if (type == T_BWD) {  // delta_l of row block y
          wait_ge(c_dlt(p, l, tk.y), tgt * (l == L - 1 ? (unsigned)kOutPer : (unsigned)tn_of(p.dims[l])));
        } else if (type == T_GRAD) {  // delta_l of every row block of chunk y
          const unsigned per = l == L - 1 ? (unsigned)kOutPer : (unsigned)tn_of(p.dims[l]);
          const int rb0 = tk.y * p.kc / BM, rb1 = min(p.nrb, (tk.y + 1) * p.kc / BM);
          for (int mb = rb0; mb < rb1; ++mb) wait_ge(c_dlt(p, l, mb), tgt * per);
        } else if (type == T_GFIN) {
          wait_ge(c_oall(p), tgt * (unsigned)(p.nrb * kOutPer));
        } else {  // ROUND(l): every GRAD(l) and BWD(l) of this step
          const int tm = cdiv(p.dims[l], BM), tnk = tn_of(p.dims[l - 1]);
          wait_ge(c_grad(p, l), tgt * (unsigned)(p.nchunk * tm * tnk));
          if (l >= 2) wait_ge(c_bwdall(p, l), tgt * (unsigned)(p.nrb * tn_of(p.dims[l - 1])));
        }
        ptx::fence_proxy_async_global();  // the producers' generic writes -> this CTA's TMA reads
        if (p.prof) t1 = gtime();
      }
      __syncthreads();

      if (type == T_FWD || type == T_BWD || type == T_GRAD) {
        // ---- geometry of the tile
        int K, kbeg, nkb, rowA = 0, rowB = 0;
        bool amn = false, bmn = false;
        const CUtensorMap *mA, *mB;
        const CUtensorMap *lm = p.maps + l * kMapsPerLayer;
        if (type == T_FWD) {        // A = A_{l-1} rows (x for l = 1), B = W~_l rows nb
          K = p.dims[l - 1]; kbeg = 0;
          rowA = (l == 1 ? (int)start : 0) + tk.y * BM;
          rowB = tk.z * BN;
          mA = lm + M_FA; mB = lm + M_FW;
        } else if (type == T_BWD) { // A = delta_l rows, B = W~_l (MN-major, n = cols of W)
          K = p.dims[l]; kbeg = 0;
          rowA = tk.y * BM; rowB = tk.z * BN;
          mA = lm + M_BD; mB = lm + M_BW; bmn = true;
        } else {                    // A = delta_l^T (MN), B = A_{l-1} (MN); K = the chunk's rows
          K = min(p.kc, p.B - tk.y * p.kc); kbeg = tk.y * p.kc;
          rowA = tk.z * BM; rowB = tk.w * BN;
          mA = lm + M_GD; mB = lm + M_GA; amn = bmn = true;
        }
        nkb = cdiv(K, BK);
        const int krow0 = (type == T_GRAD && l == 1) ? (int)start : 0;  // x rows of the batch
        if (warp == 0) {
          if (lane == 0) {
            ptx::prefetch_tensormap(mA);
            ptx::prefetch_tensormap(mB);
            for (int kb = 0; kb < nkb; ++kb, ++it) {
              const int st = it % kStages;
              if (it >= kStages) ptx::mbar_wait(&empty[st], ((it / kStages) - 1) & 1);
              uint8_t *sa = smem + st * STAGE_BYTES, *sb = sa + A_BYTES;
              const int k = kbeg + kb * BK;
              ptx::mbar_arrive_expect_tx(&full[st], (uint32_t)STAGE_BYTES);
              if (amn) {
#pragma unroll
                for (int i = 0; i < BM / 32; ++i) ptx::tma_load_2d(sa + i * 4096, mA, &full[st], rowA + 32 * i, k);
              } else {
                ptx::tma_load_2d(sa, mA, &full[st], k, rowA);
              }
              if (bmn) {
#pragma unroll
                for (int i = 0; i < BN / 32; ++i)
                  ptx::tma_load_2d(sb + i * 4096, mB, &full[st], rowB + 32 * i, k + (type == T_GRAD ? krow0 : 0));
              } else {
                ptx::tma_load_2d(sb, mB, &full[st], k, rowB);
              }
            }
          } else {
            it += nkb;  // (lanes 1..31 keep the ring position in step)
          }
        } else if (warp == 1) {
          if (lane == 0) {
            const uint32_t idesc = tc::idesc_tf32(BM, BN, amn, bmn);
            for (int kb = 0; kb < nkb; ++kb, ++it) {
              const int st = it % kStages;
              ptx::mbar_wait(&full[st], (it / kStages) & 1);
              tc::tc_fence_after();
              const uint32_t sa = ptx::smem_u32(smem + st * STAGE_BYTES), sb = sa + A_BYTES;
#pragma unroll
              for (int ks = 0; ks < BK / 8; ++ks) {
                const uint64_t da = amn ? tc::op_desc<true>(sa, ks) : tc::op_desc<false>(sa, ks);
                const uint64_t db = bmn ? tc::op_desc<true>(sb, ks) : tc::op_desc<false>(sb, ks);
                tc::mma_tf32(tmem, da, db, idesc, (kb | ks) != 0 ? 1u : 0u);
              }
              tc::mma_commit(&empty[st]);
            }
            tc::mma_commit(accum);
          } else {
            it += nkb;
          }
        } else {
          it += nkb;
          // ---- epilogue: thread = tile row r (TMEM lane quadrant = warp % 4)
          const int q = warp & 3, r = 32 * q + lane;
          ptx::mbar_wait(accum, ntc & 1);
          tc::tc_fence_after();
          if (p.prof && r == 0) sred[0] = __int_as_float((int)(gtime() & 0x7fffffff));
          if (type == T_FWD) {
            const int N = p.dims[l], n0 = tk.z * BN, m = tk.y * BM + r;
            const float *bias = p.params + p.offB[l] + n0;
            float *Arow = p.A[l] + (int64_t)m * N + n0, *Srow = p.S[l] + (int64_t)m * N + n0;
#pragma unroll 1
            for (int c = 0; c < BN / 32; ++c) {  // 32-column chunks (keeps the code small: it runs once per task)
              float v[32];
              tc::tmem_ld32(tmem + ((uint32_t)(32 * q) << 16) + 32u * c, v);
              switch (p.act[l]) {
                case ACT_SIGMOID: fwd_chunk<ACT_SIGMOID>(v, bias + 32 * c, Arow + 32 * c, Srow + 32 * c); break;
                case ACT_TANH: fwd_chunk<ACT_TANH>(v, bias + 32 * c, Arow + 32 * c, Srow + 32 * c); break;
                case ACT_RELU: fwd_chunk<ACT_RELU>(v, bias + 32 * c, Arow + 32 * c, Srow + 32 * c); break;
                case ACT_GAUSSIAN: fwd_chunk<ACT_GAUSSIAN>(v, bias + 32 * c, Arow + 32 * c, Srow + 32 * c); break;
                default: fwd_chunk<ACT_STEP>(v, bias + 32 * c, Arow + 32 * c, Srow + 32 * c); break;
              }
            }
            tc::tc_fence_before();
          } else if (type == T_BWD) {  // delta_{l-1} = acc .* sigma'(Z_{l-1}), in place of S_{l-1}
            const int N = p.dims[l - 1], n0 = tk.z * BN, m = tk.y * BM + r;
            float *Srow = p.S[l - 1] + (int64_t)m * N + n0;
            float *cs = reinterpret_cast<float *>(smem);  // [BM][65] block of deltas (the idle ring)
#pragma unroll 1
            for (int c = 0; c < BN / 32; ++c) {
              float v[32];
              tc::tmem_ld32(tmem + ((uint32_t)(32 * q) << 16) + 32u * c, v);
              float4 s4[8];  // every sigma' load in flight before any store (N is a multiple of 64)
#pragma unroll
              for (int j = 0; j < 8; ++j) s4[j] = __ldcg(reinterpret_cast<const float4 *>(Srow + 32 * c) + j);
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                const float d0 = v[4 * j] * s4[j].x, d1 = v[4 * j + 1] * s4[j].y, d2 = v[4 * j + 2] * s4[j].z,
                            d3 = v[4 * j + 3] * s4[j].w;
                float *cr = cs + r * 65 + 32 * c + 4 * j;
                cr[0] = d0; cr[1] = d1; cr[2] = d2; cr[3] = d3;
                reinterpret_cast<float4 *>(Srow + 32 * c)[j] = make_float4(tf32_rn(d0), tf32_rn(d1), tf32_rn(d2), tf32_rn(d3));
              }
            }
            tc::tc_fence_before();
            // the block's share of the bias update of layer l-1: b -= (eta/B) sum_rows delta
            asm volatile("bar.sync 1, 128;" ::: "memory");
            if (r < 64 && n0 + r < N) {
              float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
#pragma unroll 8
              for (int i = 0; i < BM; i += 4) {
                s0 += cs[i * 65 + r]; s1 += cs[(i + 1) * 65 + r]; s2 += cs[(i + 2) * 65 + r]; s3 += cs[(i + 3) * 65 + r];
              }
              ptx::red_add_f32(p.params + p.offB[l - 1] + n0 + r, -p.scale * ((s0 + s1) + (s2 + s3)));
            }
          } else {  // GRAD: W_l[m][n] -= scale * acc (one term per chunk, L2 reductions)
            const int M = p.dims[l], N = p.dims[l - 1];
            const int m = tk.z * BM + r, n0 = tk.w * BN;
            float *Wrow = p.params + p.offW[l] + (int64_t)m * N + n0;
            const float sc = -p.scale;
#pragma unroll 1
            for (int c = 0; c < BN / 32; ++c) {
              float v[32];
              tc::tmem_ld32(tmem + ((uint32_t)(32 * q) << 16) + 32u * c, v);
              if (m < M) {
                if ((N & 3) == 0) {
#pragma unroll
                  for (int j = 0; j < 32; j += 4)
                    if (n0 + 32 * c + j < N)
                      red_v4(Wrow + 32 * c + j, sc * v[j], sc * v[j + 1], sc * v[j + 2], sc * v[j + 3]);
                } else {
#pragma unroll
                  for (int j = 0; j < 32; ++j)
                    if (n0 + 32 * c + j < N) ptx::red_add_f32(Wrow + 32 * c + j, sc * v[j]);
                }
              }
            }
            tc::tc_fence_before();
          }
        }
        ++ntc;
      } else if (type == T_OUT) {
        // ---- the narrow output layer for rows [y*32, y*32 + 32) (SIMT).  The task's rows of A_{L-1}
        //      and S_{L-1} and all of W_L are staged into shared memory by bulk copies (one
        //      round trip), then warp w works on rows w, w+6, ... from shared memory.
        const int r0 = tk.y * BMO;
        float *sA = reinterpret_cast<float *>(smem);   // [BMO][H]
        float *sS = sA + BMO * kMaxH;                   // [BMO][H]
        float *sWo = sS + BMO * kMaxH;                  // [nL][H]
        float *sDo = sWo + kNOut * kMaxH;               // [BMO][kNOut] delta_L
        float *sb = sDo + BMO * kNOut;                  // [6][H] per-warp bias sums
        uint64_t *bar = accum + 2;                      // (a spare mbarrier slot, see below)
        const float *AL1 = p.A[L - 1];
        float *SL1 = p.S[L - 1];
        if (tid == 0) {
          const uint32_t rb = (uint32_t)(BMO * H * 4), wb = (uint32_t)(nL * H * 4);
          ptx::mbar_arrive_expect_tx(bar, 2 * rb + wb);
          ptx::bulk_g2s(sA, AL1 + (int64_t)r0 * H, rb, bar);
          ptx::bulk_g2s(sS, SL1 + (int64_t)r0 * H, rb, bar);
          ptx::bulk_g2s(sWo, p.params + p.offW[L], wb, bar);
        }
        const float bl = lane < nL ? __ldcg(p.params + p.offB[L] + lane) : 0.0f;
        float lacc = 0.0f;
        constexpr int kC = kMaxH / 32;  // columns per lane
        float bsum[kC];
#pragma unroll
        for (int i = 0; i < kC; ++i) bsum[i] = 0.0f;
        ptx::mbar_wait(bar, nout & 1);
        ++nout;
        if (p.prof && tid == 0) sred[kThreads + 1] = __int_as_float((int)(gtime() & 0x7fffffff));
#pragma unroll 1
        for (int rr = warp; rr < BMO; rr += kThreads / 32) {
          const int64_t m = r0 + rr;
          const float y = lane < nL ? __ldg(p.Y + (start + m) * nL + lane) : 0.0f;
          const float *ar = sA + rr * H;
          float dl = 0.0f;  // lane o < nL: delta_L[m][o]
#pragma unroll 1
          for (int o = 0; o < nL; ++o) {
            float zpart = 0.0f;
#pragma unroll
            for (int i = 0; i < kC; ++i)
              if (lane + 32 * i < H) zpart = fmaf(ar[lane + 32 * i], sWo[o * H + lane + 32 * i], zpart);
            const float z = warp_sum(zpart);
            if (lane == o) {
              float a_, s_;
              act_fwd(p.act[L], z + bl, a_, s_);
              const float diff = a_ - y;
              lacc = fmaf(diff, diff, lacc);
              dl = diff * s_;
              p.A[L][m * nL + o] = a_;
              p.S[L][m * nL + o] = dl;
            }
          }
          if (lane < kNOut) sDo[rr * kNOut + lane] = lane < nL ? dl : 0.0f;
#pragma unroll
          for (int i = 0; i < kC; ++i) {
            const int j = lane + 32 * i;
            if (j < H) {
              float acc = 0.0f;
#pragma unroll 1
              for (int o = 0; o < nL; ++o) acc = fmaf(__shfl_sync(0xffffffffu, dl, o), sWo[o * H + j], acc);
              const float dv = acc * sS[rr * H + j];
              bsum[i] += dv;
              SL1[m * H + j] = tf32_rn(dv);  // delta_{L-1}: operand of BWD(L-1) / GRAD(L-1)
            } else {
#pragma unroll 1
              for (int o = 0; o < nL; ++o) (void)__shfl_sync(0xffffffffu, dl, o);
            }
          }
        }
        sred[tid] = warp_sum(lacc);
#pragma unroll
        for (int i = 0; i < kC; ++i)
          if (lane + 32 * i < H) sb[warp * H + lane + 32 * i] = bsum[i];
        __syncthreads();
        if (p.prof && tid == 0) sred[kThreads + 2] = __int_as_float((int)(gtime() & 0x7fffffff));
        if (tid == 0) {
          float l2 = 0.0f;
          for (int w = 0; w < kThreads / 32; ++w) l2 += sred[w * 32];
          ptx::red_add_f32(p.lpart, l2);  // the step's cost sum (GFIN reads and re-zeroes it)
        }
        for (int j = tid; j < H; j += kThreads) {  // b_{L-1} -= (eta/B) sum over the task's rows
          float bsv = 0.0f;
#pragma unroll
          for (int w = 0; w < kThreads / 32; ++w) bsv += sb[w * H + j];
          ptx::red_add_f32(p.params + p.offB[L - 1] + j, -p.scale * bsv);
        }
        if (p.prof) { __syncthreads(); if (tid == 0) sred[kThreads + 3] = __int_as_float((int)(gtime() & 0x7fffffff)); }
        // tendency of W_L (columns j < H) and b_L (column H) over the task's rows, added into the
        // step's accumulator (applied by GFIN after every OUT task, so that all of them read the
        // pre-step W_L)
        for (int j = tid; j <= H; j += kThreads) {
          float g[kNOut];
#pragma unroll
          for (int o = 0; o < kNOut; ++o) g[o] = 0.0f;
#pragma unroll 4
          for (int q0 = 0; q0 < BMO; ++q0) {
            const float a = j < H ? sA[q0 * H + j] : 1.0f;
#pragma unroll
            for (int o = 0; o < kNOut; ++o) g[o] = fmaf(sDo[q0 * kNOut + o], a, g[o]);
          }
#pragma unroll
          for (int o = 0; o < kNOut; ++o)
            if (o < nL) ptx::red_add_f32(p.part + o * (H + 1) + j, g[o]);
        }
      } else if (type == T_GFIN) {
        // ---- W_L, b_L -= scale * (partials summed in row-block order); the step's mean cost
        // slice y of nq: W_L, b_L -= scale * accumulated tendency, accumulator re-zeroed; slice 0
        // also writes the step's mean cost
        const int ne = nL * (H + 1);
        const int e0 = ne * tk.y / p.nq, e1 = ne * (tk.y + 1) / p.nq;
        for (int e = e0 + tid; e < e1; e += kThreads) {
          const int o = e / (H + 1), j = e % (H + 1);
          float *dst = j < H ? p.params + p.offW[L] + o * H + j : p.params + p.offB[L] + o;
          const float g = __ldcg(p.part + e), w0 = __ldcg(dst);
          *dst = w0 - p.scale * g;
          p.part[e] = 0.0f;
        }
        if (tk.y == 0 && tid == 0) {
          if (p.step_loss) p.step_loss[s] = 0.5f * __ldcg(p.lpart) * p.inv_B;
          p.lpart[0] = 0.0f;
        }
      } else {  // ROUND(l, q): slice q of W~_l = rn(W_l)
        const int64_t n = (int64_t)p.dims[l] * p.dims[l - 1];
        const int64_t i0 = n * tk.y / p.nq, i1 = n * (tk.y + 1) / p.nq;
        const float *src = p.params + p.offW[l];
        float *dst = p.params_t + p.offW[l];
        int64_t i = i0 + tid;
        for (; i + 3 * kThreads < i1; i += 4 * kThreads) {  // 4 loads in flight per thread
          float t[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) t[u] = __ldcg(src + i + u * kThreads);
#pragma unroll
          for (int u = 0; u < 4; ++u) dst[i + u * kThreads] = tf32_rn(t[u]);
        }
        for (; i < i1; i += kThreads) dst[i] = tf32_rn(__ldcg(src + i));
      }

      // ---- completion: publish this task's writes, then count it (the proxy fence orders this
      //      task's generic smem accesses before the next task's TMA writes into the same bytes)
      ptx::fence_proxy_async_smem();
      tc::tc_fence_before();
      __syncthreads();
      tc::tc_fence_after();
      if (tid == 0) {
        if (p.prof && type == T_OUT) sred[kThreads + 4] = __int_as_float((int)(gtime() & 0x7fffffff));
        ptx::fence_proxy_async_global();
        if (type == T_FWD) signal(c_fwd(p, l, tk.y));
        else if (type == T_OUT) { signal(c_dlt(p, L - 1, tk.y / kOutPer)); signal(c_oall(p)); }
        else if (type == T_BWD) { signal(c_dlt(p, l - 1, tk.y)); signal(c_bwdall(p, l)); }
        else if (type == T_GRAD) signal(c_grad(p, l));
        signal(c_step(p));
        if (p.prof && np < p.prof_cap) {
          unsigned long long *q = p.prof + ((int64_t)blockIdx.x * p.prof_cap + np) * 8;
          for (int k = 1; k <= 4; ++k) q[3 + k] = type == T_OUT ? (unsigned)__float_as_int(sred[kThreads + k]) : 0u;
          const unsigned long long te = gtime();
          // word 3: task word | accumulator-ready time (low 31 bits of globaltimer) << 32 (TC tasks)
          const unsigned long long ta = (type == T_FWD || type == T_BWD || type == T_GRAD)
                                            ? (unsigned long long)(unsigned)__float_as_int(sred[0]) : 0ull;
          q[0] = t0; q[1] = t1; q[2] = te; q[3] = (unsigned long long)(tk.x & 0xffff) | (ta << 32);
        }
        ++np;
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc::tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(64u) : "memory");
  }
}

}  // namespace

bool deep_mk_applicable(const std::vector<int> &dims, int math, int64_t batch) {
  // opt-in (NF_DEEP_MK=1, read per call): measured slower than the per-layer kernels on config 4
  // (196 vs 140 us per step, profiles/r02_deep_mk_experiment.txt) -- each task's fixed latencies
  // (TMA fill, epilogue, release / acquire) are not overlapped across tasks yet
  const char *on = getenv("NF_DEEP_MK");
  if (!on || atoi(on) == 0 || math != 1) return false;
  const int L = (int)dims.size() - 1;
  if (L < 2 || L > kMaxL - 1) return false;
  if (dims[0] % 4 != 0 || dims[0] < 32) return false;
  for (int l = 1; l < L; ++l)
    if (dims[l] % 64 != 0 || dims[l] > kMaxH) return false;
  if (dims[L] > kNOut) return false;
  return batch >= BM && batch % BM == 0 && batch <= 16384;
}

int deep_mk_train_steps(DeepMK &st, cudaStream_t stream, const std::vector<int> &dims, const std::vector<int> &acts,
                        float *params, float *params_t, const std::vector<int64_t> &offW,
                        const std::vector<int64_t> &offB, const std::vector<float *> &A, const std::vector<float *> &S,
                        const float *X, const float *Y, int64_t N, int64_t batch, const int64_t *starts,
                        int64_t n_steps, float eta, float *step_loss) {
  const int L = (int)dims.size() - 1;
  const int B = (int)batch, nrb = B / BM;
  // ---- the configuration (task table, tensor maps, counters): built once per net / batch / dataset
  std::vector<int64_t> key = {B, (int64_t)(uintptr_t)X, N, (int64_t)(uintptr_t)params, (int64_t)(uintptr_t)params_t,
                              (int64_t)(uintptr_t)A[1], (int64_t)(uintptr_t)S[1]};
  for (int d : dims) key.push_back(d);
  // weight-gradient K (batch) chunks: up to 8, at least one 128-row block each
  int nchunk = std::max(1, std::min(nrb, 8));
  const int kc = cdiv(nrb, nchunk) * BM;
  nchunk = cdiv(B, kc);
  const int nq = 16;  // ROUND slices per layer
  if (key != st.key) {
    std::vector<int4> tasks;
    for (int l = 1; l < L; ++l)
      for (int mb = 0; mb < nrb; ++mb)
        for (int nb = 0; nb < tn_of(dims[l]); ++nb) tasks.push_back(make_int4(T_FWD | (l << 8), mb, nb, 0));
    for (int mb = 0; mb < nrb * kOutPer; ++mb) tasks.push_back(make_int4(T_OUT | (L << 8), mb, 0, 0));
    for (int l = L - 1; l >= 1; --l) {
      if (l >= 2)
        for (int mb = 0; mb < nrb; ++mb)
          for (int nb = 0; nb < tn_of(dims[l - 1]); ++nb) tasks.push_back(make_int4(T_BWD | (l << 8), mb, nb, 0));
      for (int c = 0; c < nchunk; ++c)
        for (int mt = 0; mt < cdiv(dims[l], BM); ++mt)
          for (int nt = 0; nt < tn_of(dims[l - 1]); ++nt) tasks.push_back(make_int4(T_GRAD | (l << 8), c, mt, nt));
    }
    for (int q = 0; q < nq; ++q) tasks.push_back(make_int4(T_GFIN | (L << 8), q, 0, 0));
    for (int l = 1; l < L; ++l)
      for (int q = 0; q < nq; ++q) tasks.push_back(make_int4(T_ROUND | (l << 8), q, 0, 0));
    const int T = (int)tasks.size();

    // tensor maps, 6 per layer (index l * 6 + kind)
    std::vector<CUtensorMap> maps((size_t)(L + 1) * kMapsPerLayer);
    memset(maps.data(), 0, maps.size() * sizeof(CUtensorMap));
    for (int l = 1; l < L; ++l) {
      const int nk = dims[l - 1], nl = dims[l];
      const float *Ain = l == 1 ? X : A[l - 1];
      const uint64_t rowsIn = l == 1 ? (uint64_t)N : (uint64_t)B;
      CUtensorMap *m = &maps[(size_t)l * kMapsPerLayer];
      bool ok = encode_tmap_2d_f32(&m[M_FA], Ain, nk, rowsIn, (uint64_t)nk * 4, BK, BM, CU_TENSOR_MAP_SWIZZLE_128B);
      ok = ok && encode_tmap_2d_f32(&m[M_FW], params_t + offW[l], nk, nl, (uint64_t)nk * 4, BK, BN,
                                    CU_TENSOR_MAP_SWIZZLE_128B);
      // BWD(l): A = delta_l [B][nl] K-major; B = W~_l [nl][nk] MN-major (boxes {32 n, 32 k})
      ok = ok && encode_tmap_2d_f32(&m[M_BD], S[l], nl, B, (uint64_t)nl * 4, BK, BM, CU_TENSOR_MAP_SWIZZLE_128B);
      ok = ok && encode_tmap_2d_f32(&m[M_BW], params_t + offW[l], nk, nl, (uint64_t)nk * 4, 32, BK,
                                    CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
      // GRAD(l): A = delta_l^T (MN: delta_l [B][nl], boxes {32 m, 32 k}); B = A_{l-1} (MN)
      ok = ok && encode_tmap_2d_f32(&m[M_GD], S[l], nl, B, (uint64_t)nl * 4, 32, BK, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
      ok = ok && encode_tmap_2d_f32(&m[M_GA], Ain, nk, rowsIn, (uint64_t)nk * 4, 32, BK,
                                    CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
      if (!ok) {
        snprintf(g_dmk_err, sizeof g_dmk_err, "tensor-map encoding failed (layer %d)", l);
        return -1;
      }
    }
    const int H = dims[L - 1], nL = dims[L];
    const size_t ctr_uints = 2 * (kMaxL + 1) * (size_t)nrb + 2 * (kMaxL + 1) + 64;
    size_t o = 0;
    auto take = [&](size_t bytes) { size_t r = o; o = (o + bytes + 255) & ~size_t(255); return r; };
    st.off_maps = take(maps.size() * sizeof(CUtensorMap));
    st.off_tasks = take(tasks.size() * sizeof(int4));
    st.off_ctr = take(ctr_uints * 4);
    st.off_part = take((size_t)nL * (H + 1) * 4);
    st.off_lpart = take(64);
    st.off_starts = o;
    st.ctr_bytes = ctr_uints * 4;
    const size_t need = o + std::max<int64_t>(1024, n_steps) * 8;
    if (st.dev_bytes < need) {
      if (st.dev) cudaFree(st.dev);
      st.dev = nullptr;
      st.dev_bytes = 0;
      if (cudaMalloc(&st.dev, need) != cudaSuccess) {
        snprintf(g_dmk_err, sizeof g_dmk_err, "device state of %zu bytes", need);
        return -1;
      }
      st.dev_bytes = need;
      st.starts_cap = (int64_t)((need - st.off_starts) / 8);
    }
    char *d = static_cast<char *>(st.dev);
    cudaError_t e = cudaMemcpy(d + st.off_maps, maps.data(), maps.size() * sizeof(CUtensorMap), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(d + st.off_tasks, tasks.data(), tasks.size() * sizeof(int4), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
      snprintf(g_dmk_err, sizeof g_dmk_err, "state upload: %s", cudaGetErrorString(e));
      return -1;
    }
    st.tasks_per_step = T;
    st.smem = (size_t)kStages * STAGE_BYTES + 1024 + 512 + kThreads * 4 + 64;
    cudaError_t ea = set_max_smem(reinterpret_cast<const void *>(deep_mk_kernel), (int)st.smem);
    if (ea != cudaSuccess) {
      snprintf(g_dmk_err, sizeof g_dmk_err, "smem attribute: %s", cudaGetErrorString(ea));
      return -1;
    }
    int per_sm = 0, nsm = 0, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, deep_mk_kernel, kThreads, st.smem);
    if (per_sm < 1) {
      snprintf(g_dmk_err, sizeof g_dmk_err, "kernel does not fit an SM");
      return -1;
    }
    st.grid = std::min(nsm, T);
    st.key = key;
  }
  // ---- per call: batch starts (device), counters zeroed, launch
  if (n_steps > st.starts_cap) {
    st.key.clear();  // rebuild with room for the starts
    return deep_mk_train_steps(st, stream, dims, acts, params, params_t, offW, offB, A, S, X, Y, N, batch, starts,
                               n_steps, eta, step_loss);
  }
  if (!st.h_starts || !st.h_ev) {
    if (cudaMallocHost(&st.h_starts, (size_t)st.starts_cap * 8) != cudaSuccess ||
        cudaEventCreateWithFlags(&st.h_ev, cudaEventDisableTiming) != cudaSuccess) {
      snprintf(g_dmk_err, sizeof g_dmk_err, "pinned staging");
      return -1;
    }
  }
  char *d = static_cast<char *>(st.dev);
  cudaError_t e = cudaEventSynchronize(st.h_ev);
  if (e == cudaSuccess) {
    memcpy(st.h_starts, starts, (size_t)n_steps * 8);
    e = cudaMemcpyAsync(d + st.off_starts, st.h_starts, (size_t)n_steps * 8, cudaMemcpyHostToDevice, stream);
  }
  if (e == cudaSuccess) e = cudaEventRecord(st.h_ev, stream);
  if (e == cudaSuccess) e = cudaMemsetAsync(d + st.off_ctr, 0, st.off_starts - st.off_ctr, stream);  // counters,
                                                                    // output-layer accumulators
  Params p{};
  p.L = L; p.B = B; p.nrb = nrb; p.kc = kc; p.nchunk = nchunk; p.nq = nq; p.T = st.tasks_per_step;
  for (int l = 0; l <= L; ++l) {
    p.dims[l] = dims[l];
    p.act[l] = l >= 1 ? acts[l] : 0;
    p.offW[l] = l >= 1 ? offW[l] : 0;
    p.offB[l] = l >= 1 ? offB[l] : 0;
    p.A[l] = l >= 1 ? A[l] : nullptr;
    p.S[l] = l >= 1 ? S[l] : nullptr;
  }
  p.params = params; p.params_t = params_t;
  p.X = X; p.Y = Y;
  p.tasks = reinterpret_cast<const int4 *>(d + st.off_tasks);
  p.maps = reinterpret_cast<const CUtensorMap *>(d + st.off_maps);
  p.starts = reinterpret_cast<const int64_t *>(d + st.off_starts);
  p.ctr = reinterpret_cast<unsigned *>(d + st.off_ctr);
  p.part = reinterpret_cast<float *>(d + st.off_part);
  p.lpart = reinterpret_cast<float *>(d + st.off_lpart);
  p.step_loss = step_loss;
  p.scale = (float)((double)eta / (double)batch);
  p.inv_B = (float)(1.0 / (double)batch);
  p.n_steps = n_steps;
  static const bool prof = getenv("NF_DMK_PROF") != nullptr;
  static unsigned long long *prof_buf = nullptr;
  const int prof_cap = 64;
  if (prof) {
    if (!prof_buf) cudaMalloc(&prof_buf, (size_t)148 * prof_cap * 8 * 8);
    cudaMemsetAsync(prof_buf, 0, (size_t)148 * prof_cap * 8 * 8, stream);
    p.prof = prof_buf;
    p.prof_cap = prof_cap;
  }
  if (e == cudaSuccess) {
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;  // every CTA co-resident (the counters need it)
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cfg.gridDim = dim3(st.grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = st.smem;
    cfg.stream = stream;
    e = cudaLaunchKernelEx(&cfg, deep_mk_kernel, p);
    count_launch();
    char nt[64];
    snprintf(nt, sizeof nt, "tasks/step=%d steps=%lld", st.tasks_per_step, (long long)n_steps);
    log_launch(reinterpret_cast<const void *>(deep_mk_kernel), cfg.gridDim, cfg.blockDim, st.smem, nt);
  }
  if (e != cudaSuccess) {
    snprintf(g_dmk_err, sizeof g_dmk_err, "launch: %s", cudaGetErrorString(e));
    return -1;
  }
  if (prof) {  // per task type: mean dependency wait and run time (the first 64 tasks of each CTA)
    std::vector<unsigned long long> h((size_t)st.grid * prof_cap * 8);
    cudaStreamSynchronize(stream);
    cudaMemcpy(h.data(), prof_buf, h.size() * 8, cudaMemcpyDeviceToHost);
    const char *names[6] = {"FWD", "OUT", "BWD", "GRAD", "GFIN", "ROUND"};
    double wait[6] = {0}, run[6] = {0}, mma[6] = {0};
    int cnt[6] = {0};
    unsigned long long tmin = ~0ull, tmax = 0;
    double osub[5] = {0};
    int ocnt = 0;
    for (size_t i = 0; i < h.size(); i += 8) {
      if (!h[i]) continue;
      if ((int)(h[i + 3] & 0xff) == T_OUT) {  // sub-phase ends relative to t1 (low 31 bits)
        unsigned long long prev = h[i + 1] & 0x7fffffffull;
        for (int k = 1; k <= 4; ++k) {
          const unsigned long long tk2 = h[i + 3 + k];
          osub[k] += (double)((tk2 - prev) & 0x7fffffffull);
          prev = tk2;
        }
        ++ocnt;
      }
      const int ty = (int)(h[i + 3] & 0xff);
      wait[ty] += (double)(h[i + 1] - h[i]);
      run[ty] += (double)(h[i + 2] - h[i + 1]);
      const unsigned long long ta = h[i + 3] >> 32;
      if (ta) {  // accumulator ready (reconstruct the high bits from t1)
        const unsigned long long full = (h[i + 1] & ~0x7fffffffull) | ta;
        mma[ty] += (double)((full >= h[i + 1] ? full : full + 0x80000000ull) - h[i + 1]);
      }
      cnt[ty]++;
      tmin = std::min(tmin, h[i]);
      tmax = std::max(tmax, h[i + 2]);
    }
    fprintf(stderr, "[deep_mk prof] %d CTAs, span of the profiled tasks %.1f us\n", st.grid, (tmax - tmin) / 1e3);
    if (ocnt)
      fprintf(stderr, "  OUT phases: staging %.2f, rows %.2f, bias %.2f, W_L tendency %.2f us\n", osub[1] / ocnt / 1e3,
              osub[2] / ocnt / 1e3, osub[3] / ocnt / 1e3, osub[4] / ocnt / 1e3);
    for (int t = 0; t < 6; ++t)
      if (cnt[t])
        fprintf(stderr, "  %-6s %5d tasks  wait %7.2f us  run %7.2f us (of which to accumulator ready %6.2f us) (mean)\n",
                names[t], cnt[t], wait[t] / cnt[t] / 1e3, run[t] / cnt[t] / 1e3, mma[t] / cnt[t] / 1e3);
  }
  return 0;
}

void deep_mk_release(DeepMK &st) {
  if (st.h_ev) {
    cudaEventSynchronize(st.h_ev);
    cudaEventDestroy(st.h_ev);
  }
  if (st.h_starts) cudaFreeHost(st.h_starts);
  if (st.dev) cudaFree(st.dev);
  st = DeepMK{};
}

const char *deep_mk_error() { return g_dmk_err; }

}  // namespace nf
