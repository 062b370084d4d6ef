// single_cta.cu -- the latency path of small-batch SGD: the paper's train_single (P:429-458,
// batch = 1) and train_batch with a few rows on ONE CTA.
//
// With a handful of rows per step the work of a step is tiny (c1: 120 flops per sample; the
// 784-30-10 net: 95 KFLOP per sample) and the steps are strictly sequential (step s+1 reads
// the parameters step s wrote), so the step time is the latency of its dependent phases.  K6
// spreads a step over clusters and pays a GPU-wide co_sum + barrier per step (~7-8 us at any
// batch); here the whole net lives in one SM's shared memory and a step is a chain of
// CTA barriers:
//   forward (Eq. 2), layer by layer: warp per output (lanes split the K sum) for
//     wide inputs, thread per output otherwise; the epilogue stores a = sigma(z) and
//     sigma'(z) (R6), and for the output layer delta_L = (a - y) sigma'(z) and the cost;
//   deltas, l = L..2: delta_{l-1} = sigma' .* (delta_l W_l);
//   tendencies summed over the rows + update (scale eta/B: R3): warp per
//     neuron row j, lanes over the n_{l-1} + 1 columns (the last one is the bias).
// The next step's x / y rows are prefetched with cp.async while the current step runs.
#include <algorithm>
#include <cstdlib>

#include "kernels.cuh"
#include "nf_common.cuh"
#include "single_cta.cuh"

namespace nf {
namespace {

constexpr int kMaxT = 1024;  // threads: a template parameter (kT) of the kernel, <= kMaxT
constexpr int kMaxL = 16;

struct SingleParams {
  const float *X, *Y;
  const int64_t *starts;
  int64_t n_steps;
  int B, L;
  int dims[kMaxL + 1];
  int kp[kMaxL + 1];                     // widths rounded up to 4 (shared-memory row strides)
  int act[kMaxL + 1];
  int goffW[kMaxL + 1], goffB[kMaxL + 1];  // flat parameters in global memory (include/nf.h)
  int sW[kMaxL + 1], sB[kMaxL + 1];      // shared memory: W_l [n_l][kp_{l-1}], b_l (16-B aligned)
  int sA[kMaxL + 1], sS[kMaxL + 1];      // shared memory: A_l, S_l / delta_l  [B][kp_l]
  int D;                                 // x / y ring depth (steps prefetched ahead), 2..4
  int sX[4], sY[4], sRed, sEnd;
  float *params;
  float scale;                           // eta / B
  float *step_loss;
};

__device__ __forceinline__ void cp_async4(float *dst, const float *src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
// wait until at most n of the most recent groups are pending
__device__ __forceinline__ void cp_async_wait_pending(int n) {
  if (n <= 0) asm volatile("cp.async.wait_group 0;" ::: "memory");
  else if (n == 1) asm volatile("cp.async.wait_group 1;" ::: "memory");
  else asm volatile("cp.async.wait_group 2;" ::: "memory");
}
__device__ __forceinline__ float dot4(float4 a, float4 b, float acc) {
  return fmaf(a.x, b.x, fmaf(a.y, b.y, fmaf(a.z, b.z, fmaf(a.w, b.w, acc))));
}

// kL > 0: the depth is a compile-time constant (layer loops fully unrolled, per-layer parameter
// reads constant-indexed); kL = 0: any depth <= kMaxL
template <int kT, int kL>
__global__ void __launch_bounds__(kT, 1) single_cta_kernel(const __grid_constant__ SingleParams p) {
  constexpr int kWarps = kT / 32;
  extern __shared__ float4 sm4[];
  float *sm = reinterpret_cast<float *>(sm4);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int B = p.B, L = kL ? kL : p.L, n0 = p.dims[0], nL = p.dims[L], x4 = p.kp[0];
  // zero everything (the row paddings stay zero), then the parameters into the padded layout
  for (int i = tid; i < p.sEnd; i += kT) sm[i] = 0.0f;
  __syncthreads();
  for (int l = 1; l <= L; ++l) {
    const int n = p.dims[l], K = p.dims[l - 1], Kp = p.kp[l - 1];
    for (int i = tid; i < n * K; i += kT) sm[p.sW[l] + (i / K) * Kp + i % K] = p.params[p.goffW[l] + i];
    for (int i = tid; i < n; i += kT) sm[p.sB[l] + i] = p.params[p.goffB[l] + i];
  }
  // x / y rows of step s go to ring slot s % D, issued D-1 steps ahead; the start of the next
  // step to issue is loaded a whole step before it is needed (a register, not a stall)
  const int D = p.D;
  auto prefetch = [&](int64_t r0, int slot) {
    const float *xs = p.X + r0 * n0, *ys = p.Y + r0 * nL;
    for (int i = tid; i < B * n0; i += kT) cp_async4(sm + p.sX[slot] + (i / n0) * x4 + i % n0, xs + i);
    for (int i = tid; i < B * nL; i += kT) cp_async4(sm + p.sY[slot] + i, ys + i);
  };
  for (int d = 0; d < D - 1; ++d) {
    if (d < p.n_steps) prefetch(p.starts[d], d);
    cp_async_commit();  // one group per step, empty past the end (uniform counting)
  }
  int64_t st_next = D - 1 < p.n_steps ? p.starts[D - 1] : 0;
  float *red = sm + p.sRed;
  int buf = 0, pbuf = D - 1;  // ring slots of step s and of step s + D - 1
  for (int64_t s = 0; s < p.n_steps; ++s, buf = buf + 1 == D ? 0 : buf + 1, pbuf = pbuf + 1 == D ? 0 : pbuf + 1) {
    cp_async_wait_pending(D - 2);  // step s's group is complete (D - 2 newer ones may pend)
    __syncthreads();  // this step's rows landed; the previous step's update is complete
    if (s > 0 && warp == 0 && p.step_loss) {  // cost of step s-1 from the warp partials
      const float l = warp_sum(red[lane]);
      if (lane == 0) p.step_loss[s - 1] = 0.5f * l / (float)B;
    }
    if (s + D - 1 < p.n_steps) prefetch(st_next, pbuf);
    cp_async_commit();
    if (s + D < p.n_steps) st_next = p.starts[s + D];
    const float *y = sm + p.sY[buf];
    float lacc = 0.0f;

    // ---- forward + delta_L
#pragma unroll
    for (int l = 1; l <= L; ++l) {
      const int n = p.dims[l], np = p.kp[l], K4 = p.kp[l - 1] / 4, act = p.act[l];
      const float4 *W = sm4 + p.sW[l] / 4;
      const float *b = sm + p.sB[l];
      const float4 *ain = sm4 + (l == 1 ? p.sX[buf] : p.sA[l - 1]) / 4;
      float *A = sm + p.sA[l], *S = sm + p.sS[l];
      const bool last = l == L;
      auto epi = [&](int r, int j, float acc) {
        float a, sg;
        act_fwd(act, acc + b[j], a, sg);
        A[r * np + j] = a;
        if (last) {
          const float d = a - y[r * nL + j];
          lacc = fmaf(d, d, lacc);
          S[r * np + j] = d * sg;
        } else {
          S[r * np + j] = sg;
        }
      };
      if (K4 >= 16) {  // warp per output, lanes over 4-column groups
        for (int o = warp; o < B * n; o += kWarps) {
          const int r = o / n, j = o - r * n;
          const float4 *w = W + j * K4, *a = ain + r * K4;
          float acc = 0.0f;
          for (int k = lane; k < K4; k += 32) acc = dot4(w[k], a[k], acc);
          acc = warp_sum(acc);
          if (lane == 0) epi(r, j, acc);
        }
      } else {         // thread per output
        for (int o = tid; o < B * n; o += kT) {
          const int r = o / n, j = o - r * n;
          const float4 *w = W + j * K4, *a = ain + r * K4;
          float acc = 0.0f;
          for (int k = 0; k < K4; ++k) acc = dot4(w[k], a[k], acc);
          epi(r, j, acc);
        }
      }
      __syncthreads();
    }
    lacc = warp_sum(lacc);
    if (lane == 0) red[warp] = lacc;

    // ---- deltas, l = L..2 (W_l read before any update): thread per (row, column)
#pragma unroll
    for (int l = L; l >= 2; --l) {
      const int n = p.dims[l], np = p.kp[l], K = p.dims[l - 1], Kp = p.kp[l - 1];
      const float *W = sm + p.sW[l], *D = sm + p.sS[l];
      float *Sp = sm + p.sS[l - 1];
      for (int o = tid; o < B * K; o += kT) {
        const int r = o / K, k = o - r * K;
        const float *d = D + r * np;
        float a0 = 0.0f, a1 = 0.0f;
        int j = 0;
        for (; j + 2 <= n; j += 2) {
          a0 = fmaf(W[j * Kp + k], d[j], a0);
          a1 = fmaf(W[(j + 1) * Kp + k], d[j + 1], a1);
        }
        if (j < n) a0 = fmaf(W[j * Kp + k], d[j], a0);
        Sp[r * Kp + k] *= a0 + a1;
      }
      __syncthreads();
    }

    // ---- tendencies over the B rows and the update: warp per neuron row (rows of all layers
    //      dealt round-robin to the warps), lanes over 4-column groups; lane 0 also the bias
    {
      int row = warp;
#pragma unroll
      for (int l = 1; l <= L; ++l) {
        const int n = p.dims[l], np = p.kp[l], K4 = p.kp[l - 1] / 4;
        float4 *W = sm4 + p.sW[l] / 4;
        float *b = sm + p.sB[l];
        const float *D = sm + p.sS[l];
        const float4 *ain = sm4 + (l == 1 ? p.sX[buf] : p.sA[l - 1]) / 4;
        for (; row < n; row += kWarps) {
          const int j = row;
          for (int k = lane; k < K4; k += 32) {
            float4 g = make_float4(0.f, 0.f, 0.f, 0.f);
            for (int r = 0; r < B; ++r) {
              const float dv = D[r * np + j];
              const float4 a = ain[r * K4 + k];
              g.x = fmaf(dv, a.x, g.x); g.y = fmaf(dv, a.y, g.y);
              g.z = fmaf(dv, a.z, g.z); g.w = fmaf(dv, a.w, g.w);
            }
            float4 w = W[j * K4 + k];
            w.x = fmaf(-p.scale, g.x, w.x); w.y = fmaf(-p.scale, g.y, w.y);
            w.z = fmaf(-p.scale, g.z, w.z); w.w = fmaf(-p.scale, g.w, w.w);
            W[j * K4 + k] = w;
          }
          if (lane == 0) {
            float g = 0.0f;
            for (int r = 0; r < B; ++r) g += D[r * np + j];
            b[j] = fmaf(-p.scale, g, b[j]);
          }
        }
        row -= n;
      }
    }
  }
  __syncthreads();
  if (p.n_steps > 0 && warp == 0 && p.step_loss) {
    const float l = warp_sum(red[lane]);
    if (lane == 0) p.step_loss[p.n_steps - 1] = 0.5f * l / (float)B;
  }
  for (int l = 1; l <= L; ++l) {
    const int n = p.dims[l], K = p.dims[l - 1], Kp = p.kp[l - 1];
    for (int i = tid; i < n * K; i += kT) p.params[p.goffW[l] + i] = sm[p.sW[l] + (i / K) * Kp + i % K];
    for (int i = tid; i < n; i += kT) p.params[p.goffB[l] + i] = sm[p.sB[l] + i];
  }
}

}  // namespace

// Shared-memory layout (floats) into p; returns the bytes, or 0 if the net / batch is outside
// the latency regime or does not fit.
static size_t single_layout(const std::vector<int> &dims, int64_t batch, SingleParams &p) {
  static const int mode = getenv("NF_SINGLE") ? atoi(getenv("NF_SINGLE")) : -1;  // 0 off, 1 force
  if (mode == 0) return 0;
  const int L = (int)dims.size() - 1;
  if (L < 1 || L > kMaxL || batch < 1 || batch > 4096) return 0;
  auto r4 = [](int64_t v) { return (v + 3) / 4 * 4; };
  int64_t o = 0, macs = 0;
  for (int l = 0; l <= L; ++l) p.kp[l] = (int)r4(dims[l]);
  for (int l = 1; l <= L; ++l) {
    p.goffW[l] = (int)o; o += (int64_t)dims[l] * dims[l - 1];
    p.goffB[l] = (int)o; o += dims[l];
    macs += (int64_t)dims[l] * dims[l - 1];
  }
  // latency regime.  Two-layer nets with <= 32-wide layers have K6 (fused_small.cu, ~7.5 us per
  // step at any batch): one CTA beats it up to ~30 K multiply-adds per step (c1: 200; the
  // 784-30-10 net at batch 1: 23.8 K -> 6.0 vs 7.75 us).  Other nets would run the generic
  // per-layer kernels (tens of us per step): one CTA up to ~1 M multiply-adds per step.
  const bool k6 = L == 2 && dims[1] <= 32 && dims[2] <= 32;
  if (mode != 1 && batch * macs > (k6 ? 30000 : 1000000)) return 0;
  int64_t f = 0;  // shared-memory floats (every block 16-B aligned)
  for (int l = 1; l <= L; ++l) {
    p.sW[l] = (int)f; f += (int64_t)dims[l] * p.kp[l - 1];
    p.sB[l] = (int)f; f += p.kp[l];
  }
  for (int l = 1; l <= L; ++l) {
    p.sA[l] = (int)f; f += batch * p.kp[l];
    p.sS[l] = (int)f; f += batch * p.kp[l];
  }
  const int64_t f0 = f, slot = batch * p.kp[0] + r4(batch * dims[L]);
  const int64_t budget = 227 * 1024 / 4 - kMaxT / 32;
  p.D = 4;  // deepest ring that fits (>= 2)
  while (p.D > 2 && f0 + p.D * slot > budget) --p.D;
  for (int i = 0; i < p.D; ++i) { p.sX[i] = (int)f; f += batch * p.kp[0]; }
  for (int i = 0; i < p.D; ++i) { p.sY[i] = (int)f; f += r4(batch * dims[L]); }
  p.sRed = (int)f; f += kMaxT / 32;
  p.sEnd = (int)f;
  const size_t smem = (size_t)f * 4;
  if (smem > 227 * 1024 || o > (1 << 30)) return 0;
  return smem;
}

bool single_cta_applicable(const std::vector<int> &dims, int64_t batch) {
  SingleParams p{};
  return single_layout(dims, batch, p) != 0;
}

int single_cta_train_steps(cudaStream_t st, const std::vector<int> &dims, const std::vector<int> &acts, float *params,
                           const float *X, const float *Y, int64_t batch, const int64_t *d_starts, int64_t n_steps,
                           float eta, float *step_loss) {
  SingleParams p{};
  const size_t smem = single_layout(dims, batch, p);
  if (smem == 0) return SINGLE_NOT_APPLICABLE;
  const int L = (int)dims.size() - 1;
  p.X = X; p.Y = Y; p.starts = d_starts; p.n_steps = n_steps; p.B = (int)batch; p.L = L;
  for (int l = 0; l <= L; ++l) {
    p.dims[l] = dims[l];
    p.act[l] = l >= 1 ? acts[l] : 0;
  }
  p.params = params;
  p.scale = (float)((double)eta / (double)batch);
  p.step_loss = step_loss;
  // threads: every warp walks every phase of a step, so small steps want few warps
  int64_t macs = 0;
  for (int l = 1; l <= L; ++l) macs += (int64_t)dims[l] * dims[l - 1];
  static const int force_t = getenv("NF_SINGLE_T") ? atoi(getenv("NF_SINGLE_T")) : 0;
  const int T = force_t ? force_t : batch * macs <= 8192 ? 256 : 1024;  // (32: slower, 4.9 vs 2.4 us on c1)
  auto launch = [&](void (*kern)(SingleParams), int threads) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    kern<<<1, threads, smem, st>>>(p);
    log_launch(reinterpret_cast<const void *>(kern), dim3(1), dim3(threads), smem);
  };
  switch ((T == 32 ? 20 : T == 256 ? 0 : 10) + (L <= 4 ? L : 0)) {
    case 21: launch(single_cta_kernel<32, 1>, 32); break;
    case 22: launch(single_cta_kernel<32, 2>, 32); break;
    case 23: launch(single_cta_kernel<32, 3>, 32); break;
    case 24: launch(single_cta_kernel<32, 4>, 32); break;
    case 20: launch(single_cta_kernel<32, 0>, 32); break;
    case 1: launch(single_cta_kernel<256, 1>, 256); break;
    case 2: launch(single_cta_kernel<256, 2>, 256); break;
    case 3: launch(single_cta_kernel<256, 3>, 256); break;
    case 4: launch(single_cta_kernel<256, 4>, 256); break;
    case 0: launch(single_cta_kernel<256, 0>, 256); break;
    case 11: launch(single_cta_kernel<1024, 1>, 1024); break;
    case 12: launch(single_cta_kernel<1024, 2>, 1024); break;
    case 13: launch(single_cta_kernel<1024, 3>, 1024); break;
    case 14: launch(single_cta_kernel<1024, 4>, 1024); break;
    default: launch(single_cta_kernel<1024, 0>, 1024); break;
  }
  count_launch();
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : (int)e;
}

}  // namespace nf
