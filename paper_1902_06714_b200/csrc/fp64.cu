// fp64.cu -- the paper's real64 build (`rk` chosen at compile time) as a
// run-time numerics mode (NF_MATH_FP64): parameters, activations, deltas and all sums in double
// on the B200's FP64 units.  Inputs, targets and results cross the C ABI as fp32 (widened
// exactly on the way in, rounded once on the way out).  Same steps as the fp32 path:
//   K1 forward  Z = A W^T (+ b, sigma, stash sigma'(Z))   K3 backward  D = (D' W) .* sigma'
//   K4 gradient G = D^T [A | 1] (+ SGD update)            loss / accuracy
// One tiled SIMT kernel (64x64 tiles, 4x4 register micro-tiles, double-buffered shared memory)
// with the three fused epilogues; A may be the fp32 input x of layer 1.
#include <algorithm>
#include <cmath>

#include "fp64.cuh"
#include "kernels.cuh"
#include "sm100_ptx.cuh"

namespace nf {
namespace {

constexpr int kSMs = 148;

// sigma, sigma' in double, stable forms from z (reading R6)
__device__ __forceinline__ void act64(int kind, double z, double &a, double &s) {
  switch (kind) {
    case ACT_SIGMOID: {
      const double t = exp(-fabs(z)), r = 1.0 / (1.0 + t);
      a = z >= 0.0 ? r : t * r;
      s = t * r * r;
      break;
    }
    case ACT_TANH: {
      const double t = exp(-2.0 * fabs(z)), r = 1.0 / (1.0 + t);
      a = tanh(z);
      s = 4.0 * t * r * r;
      break;
    }
    case ACT_RELU:
      a = z > 0.0 ? z : 0.0;
      s = z > 0.0 ? 1.0 : 0.0;
      break;
    case ACT_GAUSSIAN: {
      const double e = exp(-z * z);
      a = e;
      s = -2.0 * z * e;
      break;
    }
    default:
      a = z > 0.0 ? 1.0 : 0.0;
      s = 0.0;
      break;
  }
}

struct Args64 {
  int M, N, K;
  const float *Af;  const double *Ad; int64_t lda;  // exactly one of Af / Ad
  const double *B; const float *Bf; int64_t ldb;  // at most one of B / Bf
  int nb_real;      // B(k, n) = 1 for nb_real <= n < N (the bias column of K4)
  int kchunk;
  double *partial;  // split-K partials [z][M][N]
};

// 16 x 16 threads, each a TM x TN micro-tile of rows ty + 16 i, columns tx + 16 j (strided, so
// the shared-memory reads of a warp are one broadcast / one 128-B wavefront each): BM = 16 TM.
template <int TM, int TN, bool AK, bool BKM, class Epi>
__global__ void __launch_bounds__(256)
gemm64_kernel(Args64 g, Epi epi) {
  constexpr int BM = 16 * TM, BN = 16 * TN, BK = 8;
  constexpr int LA = BM * BK / 256, LB = BN * BK / 256;  // staged elements per thread
  __shared__ double As[2][BK][BM + 1];
  __shared__ double Bs[2][BK][BN + 1];
  ptx::pdl_trigger();
  ptx::pdl_wait();
  const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int kbeg = blockIdx.z * g.kchunk, kend = min(g.K, kbeg + g.kchunk);
  const int nkt = (kend - kbeg + BK - 1) / BK;
  double ra[LA], rb[LB];
  auto load = [&](int k0) {
#pragma unroll
    for (int i = 0; i < LA; ++i) {
      const int idx = tid + i * 256;
      const int mm = AK ? idx / BK : idx % BM, kk = AK ? idx % BK : idx / BM;
      const int m = m0 + mm, k = k0 + kk;
      double v = 0.0;
      if (m < g.M && k < kend) {
        const int64_t off = AK ? (int64_t)m * g.lda + k : (int64_t)k * g.lda + m;
        v = g.Af ? (double)g.Af[off] : g.Ad[off];
      }
      ra[i] = v;
    }
#pragma unroll
    for (int i = 0; i < LB; ++i) {
      const int idx = tid + i * 256;
      const int nn = BKM ? idx / BK : idx % BN, kb = BKM ? idx % BK : idx / BN;
      const int n = n0 + nn, kq = k0 + kb;
      double w = 0.0;
      if (kq < kend && n < g.N)
        if (n < g.nb_real) {
          const int64_t off = BKM ? (int64_t)n * g.ldb + kq : (int64_t)kq * g.ldb + n;
          w = g.Bf ? (double)g.Bf[off] : g.B[off];
        } else {
          w = 1.0;
        }
      rb[i] = w;
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int i = 0; i < LA; ++i) {
      const int idx = tid + i * 256;
      const int mm = AK ? idx / BK : idx % BM, kk = AK ? idx % BK : idx / BM;
      As[buf][kk][mm] = ra[i];
    }
#pragma unroll
    for (int i = 0; i < LB; ++i) {
      const int idx = tid + i * 256;
      const int nn = BKM ? idx / BK : idx % BN, kb = BKM ? idx % BK : idx / BN;
      Bs[buf][kb][nn] = rb[i];
    }
  };
  double acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = 0.0;
  if (nkt > 0) {
    load(kbeg);
    store(0);
  }
  __syncthreads();
  for (int t = 0; t < nkt; ++t) {
    const int buf = t & 1;
    if (t + 1 < nkt) load(kbeg + (t + 1) * BK);
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      double a[TM], b[TN];
#pragma unroll
      for (int i = 0; i < TM; ++i) a[i] = As[buf][kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < TN; ++j) b[j] = Bs[buf][kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
    }
    if (t + 1 < nkt) store(buf ^ 1);
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int m = m0 + ty + 16 * i;
    if (m >= g.M) continue;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int n = n0 + tx + 16 * j;
      if (n >= g.N) continue;
      if (g.partial) g.partial[((int64_t)blockIdx.z * g.M + m) * g.N + n] = acc[i][j];
      else epi(m, n, acc[i][j]);
    }
  }
}

template <class Epi>
__global__ void __launch_bounds__(256) splitk64(const double *__restrict__ part, int splits, int M, int N, Epi epi) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  const int64_t MN = (int64_t)M * N;
  for (int64_t i = blockIdx.x * 256 + threadIdx.x; i < MN; i += (int64_t)gridDim.x * 256) {
    double s = 0.0;
    for (int z = 0; z < splits; ++z) s += part[z * MN + i];
    epi((int)(i / N), (int)(i % N), s);
  }
}

template <bool AK, bool BKM, class Epi>
cudaError_t run64(cudaStream_t st, Args64 g, const Epi &epi, double *partial, size_t partial_doubles) {
  if (g.M <= 0 || g.N <= 0) return cudaSuccess;
  // 128 x 128 tiles (8 x 8 per thread: 64 DFMA per 16 shared loads) when they fill the GPU
  const int64_t t128 = (int64_t)((g.M + 127) / 128) * ((g.N + 127) / 128);
  if (t128 >= kSMs) {
    g.kchunk = std::max(g.K, 1);
    g.partial = nullptr;
    gemm64_kernel<8, 8, AK, BKM, Epi><<<dim3((g.N + 127) / 128, (g.M + 127) / 128, 1), 256, 0, st>>>(g, epi);
    count_launch();
    log_launch(reinterpret_cast<const void *>(gemm64_kernel<8, 8, AK, BKM, Epi>), dim3((g.N + 127) / 128, (g.M + 127) / 128, 1), dim3(256), 0);
    return cudaGetLastError();
  }
  const int tm = (g.M + 63) / 64, tn = (g.N + 63) / 64;
  const int tiles = tm * tn;
  int splits = 1;
  if (2 * tiles < kSMs && g.K >= 512) {
    splits = std::min(std::min((2 * kSMs + tiles - 1) / tiles, 32), g.K / 128);
    while (splits > 1 && (size_t)splits * g.M * g.N > partial_doubles) --splits;
    splits = std::max(splits, 1);
  }
  const int kchunk = ((g.K + splits - 1) / splits + 7) / 8 * 8;
  splits = std::max(1, (g.K + kchunk - 1) / kchunk);
  g.kchunk = splits > 1 ? kchunk : std::max(g.K, 1);
  g.partial = splits > 1 ? partial : nullptr;
  gemm64_kernel<4, 4, AK, BKM, Epi><<<dim3(tn, tm, splits), 256, 0, st>>>(g, epi);
  count_launch();
  log_launch(reinterpret_cast<const void *>(gemm64_kernel<4, 4, AK, BKM, Epi>), dim3(tn, tm, splits), dim3(256), 0);
  if (splits > 1) {
    const int64_t MN = (int64_t)g.M * g.N;
    splitk64<Epi><<<(int)std::min<int64_t>((MN + 255) / 256, 4 * kSMs), 256, 0, st>>>(partial, splits, g.M, g.N, epi);
    count_launch();
    log_launch(reinterpret_cast<const void *>(splitk64<Epi>), dim3((int)std::min<int64_t>((MN + 255) / 256, 4 * kSMs)), dim3(256), 0);
  }
  return cudaGetLastError();
}

__global__ void convert_kernel_fd(const float *__restrict__ s, double *__restrict__ d, int64_t n) {
  for (int64_t i = blockIdx.x * 256 + threadIdx.x; i < n; i += (int64_t)gridDim.x * 256) d[i] = (double)s[i];
}
__global__ void convert_kernel_df(const double *__restrict__ s, float *__restrict__ d, int64_t n) {
  ptx::pdl_wait();
  for (int64_t i = blockIdx.x * 256 + threadIdx.x; i < n; i += (int64_t)gridDim.x * 256) d[i] = (float)s[i];
}

__global__ void update_kernel64(double *__restrict__ p, const float *__restrict__ g, int64_t n, double scale) {
  for (int64_t i = blockIdx.x * 256 + threadIdx.x; i < n; i += (int64_t)gridDim.x * 256) p[i] -= scale * (double)g[i];
}

__device__ __forceinline__ void argmax_merge64(double &v, int &i, double v2, int i2) {
  if (v2 > v || (v2 == v && i2 < i)) { v = v2; i = i2; }
}

// one warp per row: cost 1/2 sum (a - y)^2 in double, first-index argmax of a and y
__global__ void __launch_bounds__(256)
loss_acc64_kernel(const double *__restrict__ A, const float *__restrict__ Y, int64_t n, int w, double2 *part) {
  ptx::pdl_wait();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t gw = (int64_t)blockIdx.x * 8 + warp, nw = (int64_t)gridDim.x * 8;
  double lsum = 0.0, csum = 0.0;
  for (int64_t r = gw; r < n; r += nw) {
    double l = 0.0, va = -INFINITY, vy = -INFINITY;
    int ia = 0x7fffffff, iy = 0x7fffffff;
    for (int j = lane; j < w; j += 32) {
      const double aj = A[r * w + j], yj = Y[r * w + j];
      l = fma(aj - yj, aj - yj, l);
      if (aj > va) { va = aj; ia = j; }
      if (yj > vy) { vy = yj; iy = j; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      l += __shfl_xor_sync(0xffffffffu, l, o);
      argmax_merge64(va, ia, __shfl_xor_sync(0xffffffffu, va, o), __shfl_xor_sync(0xffffffffu, ia, o));
      argmax_merge64(vy, iy, __shfl_xor_sync(0xffffffffu, vy, o), __shfl_xor_sync(0xffffffffu, iy, o));
    }
    lsum += 0.5 * l;
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

__global__ void loss_acc64_final(const double2 *__restrict__ part, int nparts, int64_t n, float *out,
                                 float *step_loss) {
  const int lane = threadIdx.x;
  double l = 0.0, c = 0.0;
  for (int i = lane; i < nparts; i += 32) { l += part[i].x; c += part[i].y; }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    l += __shfl_xor_sync(0xffffffffu, l, o);
    c += __shfl_xor_sync(0xffffffffu, c, o);
  }
  if (lane != 0) return;
  const float loss = n > 0 ? (float)(l / (double)n) : 0.0f, acc = n > 0 ? (float)(c / (double)n) : 0.0f;
  if (out) { out[0] = loss; out[1] = acc; }
  if (step_loss) *step_loss = loss;
}

}  // namespace

// ---- epilogues -----------------------------------------------------------------------------
__device__ void Epi64Fwd::operator()(int m, int n, double acc) const {
  const double z = acc + bias[n];
  const int64_t i = (int64_t)m * ld + n;
  double a, s;
  act64(act, z, a, s);
  A[i] = a;
  if (mode == 0) S[i] = s;
  else if (mode == 1) S[i] = (a - (double)Y[i]) * s;
}
__device__ void Epi64Bwd::operator()(int m, int n, double acc) const {
  const int64_t i = (int64_t)m * ld + n;
  SD[i] = acc * SD[i];
}
__device__ void Epi64Grad::operator()(int m, int n, double acc) const {
  double *p = n < nreal ? W + (int64_t)m * ldw + n : b + m;
  *p = store_only ? acc : *p - scale * acc;
}

cudaError_t gemm64_fwd(cudaStream_t st, int M, int N, int K, const float *Af, const double *Ad, const double *W,
                       const Epi64Fwd &epi, double *partial, size_t partial_doubles) {
  // Z[m][n] = sum_k A[m][k] W[n][k]   (A: [M][K] row-major, W: [N][K] row-major)
  Args64 g{M, N, K, Af, Ad, K, W, nullptr, K, N, 0, nullptr};
  return run64<true, true>(st, g, epi, partial, partial_doubles);
}
cudaError_t gemm64_bwd(cudaStream_t st, int M, int N, int K, const double *D, const double *W,
                       const Epi64Bwd &epi, double *partial, size_t partial_doubles) {
  // D[m][n] = sum_k D'[m][k] W[k][n]   (D': [M][K], W: [K][N])
  Args64 g{M, N, K, nullptr, D, K, W, nullptr, N, N, 0, nullptr};
  return run64<true, false>(st, g, epi, partial, partial_doubles);
}
cudaError_t gemm64_grad(cudaStream_t st, int M, int N, int K, const double *D, const float *Af, const double *Ad,
                        const Epi64Grad &epi, double *partial, size_t partial_doubles) {
  // G[m][n] = sum_k D[k][m] [A | 1][k][n]  (D: [K][M], A: [K][N]); column N = the bias tendency
  Args64 g{M, N + 1, K, nullptr, D, M, Ad, Af, N, N, 0, nullptr};
  return run64<false, false>(st, g, epi, partial, partial_doubles);
}

cudaError_t f64_widen(cudaStream_t st, const float *s, double *d, int64_t n) {
  convert_kernel_fd<<<(int)std::min<int64_t>((n + 255) / 256, 8 * kSMs), 256, 0, st>>>(s, d, n);
  count_launch();
  log_launch(reinterpret_cast<const void *>(convert_kernel_fd), dim3((int)std::min<int64_t>((n + 255) / 256, 8 * kSMs)), dim3(256), 0);
  return cudaGetLastError();
}
cudaError_t f64_round(cudaStream_t st, const double *s, float *d, int64_t n) {
  convert_kernel_df<<<(int)std::min<int64_t>((n + 255) / 256, 8 * kSMs), 256, 0, st>>>(s, d, n);
  count_launch();
  log_launch(reinterpret_cast<const void *>(convert_kernel_df), dim3((int)std::min<int64_t>((n + 255) / 256, 8 * kSMs)), dim3(256), 0);
  return cudaGetLastError();
}

cudaError_t f64_update(cudaStream_t st, double *p, const float *g, int64_t n, double scale) {
  if (n <= 0) return cudaSuccess;
  update_kernel64<<<(int)std::min<int64_t>((n + 255) / 256, 8 * kSMs), 256, 0, st>>>(p, g, n, scale);
  count_launch();
  log_launch(reinterpret_cast<const void *>(update_kernel64), dim3((int)std::min<int64_t>((n + 255) / 256, 8 * kSMs)), dim3(256), 0);
  return cudaGetLastError();
}

cudaError_t loss_acc64(cudaStream_t st, const double *A, const float *Y, int64_t n, int w, double2 *part,
                       float *out, float *step_loss) {
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(2 * kSMs, (n + 7) / 8));
  loss_acc64_kernel<<<blocks, 256, 0, st>>>(A, Y, n, w, part);
  loss_acc64_final<<<1, 32, 0, st>>>(part, blocks, n, out, step_loss);
  count_launch(2);
  log_launch(reinterpret_cast<const void *>(loss_acc64_kernel), dim3(blocks), dim3(256), 0);
  log_launch(reinterpret_cast<const void *>(loss_acc64_final), dim3(1), dim3(32), 0);
  return cudaGetLastError();
}

}  // namespace nf
