// kernels.cu -- dispatch of the generic SIMT contraction kernels and the
// loss/accuracy reduction (K5).
#include <algorithm>

#include "kernels.cuh"

namespace nf {

int64_t g_launches = 0;

namespace {

constexpr int kSMs = 148;

enum Cfg { CFG_L, CFG_M, CFG_S, CFG_T };

Cfg choose_cfg(int M, int N) {
  if (N <= 64) return CFG_S;
  if (M <= 64) return CFG_T;
  if (M >= 128 && N >= 128) return CFG_L;
  return CFG_M;
}

template <int BM, int BN, int BK, int TM, int TN, bool AK, bool BKM, class Epi>
cudaError_t launch_cfg(cudaStream_t st, GemmArgs g, const Epi &epi, const Workspace &ws) {
  const int tm = (g.M + BM - 1) / BM, tn = (g.N + BN - 1) / BN;
  const int64_t tiles = (int64_t)tm * tn;
  int splits = 1;
  if (tiles < 2 * kSMs && g.K >= 256) {
    splits = (int)std::min<int64_t>((2 * kSMs + tiles - 1) / tiles, 32);
    splits = std::min(splits, g.K / 128);
    while (splits > 1 && (size_t)splits * g.M * g.N > ws.partial_floats) --splits;
    splits = std::max(splits, 1);
  }
  int kchunk = (g.K + splits - 1) / splits;
  kchunk = (kchunk + BK - 1) / BK * BK;
  splits = std::max(1, (g.K + kchunk - 1) / kchunk);
  g.kchunk = splits > 1 ? kchunk : std::max(g.K, 1);
  g.partial = splits > 1 ? ws.partial : nullptr;
  dim3 grid(tn, tm, splits);
  gemm_simt<BM, BN, BK, TM, TN, AK, BKM, Epi><<<grid, (BM / TM) * (BN / TN), 0, st>>>(g, epi);
  count_launch();
  if (splits > 1) {
    const int64_t MN = (int64_t)g.M * g.N;
    const int blocks = (int)std::min<int64_t>((MN + 255) / 256, 4 * kSMs);
    splitk_epilogue<Epi><<<blocks, 256, 0, st>>>(ws.partial, splits, g.M, g.N, epi);
    count_launch();
  }
  return cudaGetLastError();
}

template <bool AK, bool BKM, class Epi>
cudaError_t run_gemm(cudaStream_t st, GemmArgs g, const Epi &epi, const Workspace &ws) {
  if (g.M <= 0 || g.N <= 0) return cudaSuccess;
  switch (choose_cfg(g.M, g.N)) {
    case CFG_L: return launch_cfg<128, 128, 8, 8, 8, AK, BKM>(st, g, epi, ws);
    case CFG_S: return launch_cfg<128, 32, 16, 8, 2, AK, BKM>(st, g, epi, ws);
    case CFG_T: return launch_cfg<32, 128, 16, 2, 8, AK, BKM>(st, g, epi, ws);
    default: return launch_cfg<64, 64, 16, 4, 4, AK, BKM>(st, g, epi, ws);
  }
}

}  // namespace

cudaError_t gemm_fwd(cudaStream_t st, int M, int N, int K, const float *A, const float *W,
                     const EpiFwd &epi, const Workspace &ws) {
  GemmArgs g{M, N, K, A, K, W, K, N, 0, nullptr};
  return run_gemm<true, true>(st, g, epi, ws);
}

cudaError_t gemm_bwd(cudaStream_t st, int M, int N, int K, const float *D, const float *W,
                     const EpiBwd &epi, const Workspace &ws) {
  GemmArgs g{M, N, K, D, K, W, N, N, 0, nullptr};
  return run_gemm<true, false>(st, g, epi, ws);
}

cudaError_t gemm_grad(cudaStream_t st, int M, int N, int K, const float *D, const float *Aprev,
                      const EpiGrad &epi, const Workspace &ws) {
  // C[M][N+1]: column N is the ones column -> bias gradient.
  GemmArgs g{M, N + 1, K, D, M, Aprev, N, N, 0, nullptr};
  return run_gemm<false, false>(st, g, epi, ws);
}

// ---------------------------------------------------------------------------
// K5: loss / accuracy.  One warp per sample row; per-row cost 1/2 sum (a-y)^2
// in fp32, first-index argmax of a and of y (reading R10); block partials in
// fp64, summed by a single thread in block order (deterministic).
namespace {
constexpr int kLossBlocks = 2 * kSMs;

__device__ __forceinline__ void argmax_merge(float &v, int &i, float v2, int i2) {
  if (v2 > v || (v2 == v && i2 < i)) { v = v2; i = i2; }
}

__global__ void __launch_bounds__(256)
loss_acc_partial(const float *__restrict__ A, const float *__restrict__ Y, int64_t n, int w,
                 double2 *__restrict__ part) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t gw = (int64_t)blockIdx.x * 8 + warp, nw = (int64_t)gridDim.x * 8;
  double lsum = 0.0, csum = 0.0;
  for (int64_t r = gw; r < n; r += nw) {
    const float *a = A + r * w, *y = Y + r * w;
    float l = 0.0f, va = -INFINITY, vy = -INFINITY;
    int ia = 0x7fffffff, iy = 0x7fffffff;
    for (int j = lane; j < w; j += 32) {
      const float aj = a[j], yj = y[j];
      const float d = aj - yj;
      l = fmaf(d, d, l);
      if (aj > va) { va = aj; ia = j; }
      if (yj > vy) { vy = yj; iy = j; }
    }
    l = warp_sum(l);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      argmax_merge(va, ia, __shfl_xor_sync(0xffffffffu, va, o), __shfl_xor_sync(0xffffffffu, ia, o));
      argmax_merge(vy, iy, __shfl_xor_sync(0xffffffffu, vy, o), __shfl_xor_sync(0xffffffffu, iy, o));
    }
    lsum += 0.5 * (double)l;
    csum += (ia == iy) ? 1.0 : 0.0;
  }
  __shared__ double2 sm[8];
  if (lane == 0) sm[warp] = make_double2(lsum, csum);
  __syncthreads();
  if (threadIdx.x == 0) {
    double2 t = make_double2(0.0, 0.0);
    for (int i = 0; i < 8; ++i) { t.x += sm[i].x; t.y += sm[i].y; }
    part[blockIdx.x] = t;
  }
}

__global__ void loss_acc_final(const double2 *__restrict__ part, int nparts, int64_t n,
                               float *out, float *step_loss) {
  if (threadIdx.x != 0) return;
  double l = 0.0, c = 0.0;
  for (int i = 0; i < nparts; ++i) { l += part[i].x; c += part[i].y; }
  const float loss = n > 0 ? (float)(l / (double)n) : 0.0f;
  const float acc = n > 0 ? (float)(c / (double)n) : 0.0f;
  if (out) { out[0] = loss; out[1] = acc; }
  if (step_loss) *step_loss = loss;
}
}  // namespace

int loss_acc_parts() { return kLossBlocks; }

cudaError_t loss_acc(cudaStream_t st, const float *A, const float *Y, int64_t n, int w,
                     double2 *part, float *out, float *step_loss) {
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(kLossBlocks, (n + 7) / 8));
  loss_acc_partial<<<blocks, 256, 0, st>>>(A, Y, n, w, part);
  loss_acc_final<<<1, 32, 0, st>>>(part, blocks, n, out, step_loss);
  count_launch(2);
  return cudaGetLastError();
}

}  // namespace nf
