// fp64.cuh -- the double-precision numerics mode (NF_MATH_FP64; the paper's real64 kind,
// P:113-114): SIMT FP64 GEMMs with the fused forward / backward / gradient epilogues of the
// fp32 path, fp32<->fp64 conversion at the ABI boundary, loss / accuracy in double.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace nf {

// forward: Z = acc + b[n]; A = sigma(Z); mode 0: S = sigma'(Z); 1 (output layer):
// S = (A - Y) sigma'(Z) = delta_L; 2: A only
struct Epi64Fwd {
  const double *bias;
  double *A, *S;
  const float *Y;
  int ld, act, mode;
  __device__ void operator()(int m, int n, double acc) const;
};
// backward: SD holds sigma'(Z_{l-1}) and becomes delta_{l-1} = (delta_l W_l) .* sigma'
struct Epi64Bwd {
  double *SD;
  int ld;
  __device__ void operator()(int m, int n, double acc) const;
};
// gradient: column n < nreal -> W[m][n], column nreal -> b[m]; update p -= scale * acc
// (P:471-474), or store acc (nf_grad)
struct Epi64Grad {
  double *W, *b;
  int ldw, nreal;
  double scale;
  int store_only;
  __device__ void operator()(int m, int n, double acc) const;
};

// A x W^T with A fp32 (layer-1 input) or fp64; W [N][K]
cudaError_t gemm64_fwd(cudaStream_t st, int M, int N, int K, const float *Af, const double *Ad, const double *W,
                       const Epi64Fwd &epi, double *partial, size_t partial_doubles);
// D' [M][K] x W [K][N]
cudaError_t gemm64_bwd(cudaStream_t st, int M, int N, int K, const double *D, const double *W,
                       const Epi64Bwd &epi, double *partial, size_t partial_doubles);
// D^T [M][K] x [A | 1] ([K][N] + ones column), A fp32 (layer-1 input) or fp64
cudaError_t gemm64_grad(cudaStream_t st, int M, int N, int K, const double *D, const float *Af, const double *Ad,
                        const Epi64Grad &epi, double *partial, size_t partial_doubles);

cudaError_t f64_widen(cudaStream_t st, const float *src, double *dst, int64_t n);   // exact
// nf_update in double: p[i] -= scale * g[i] (g fp32, widened exactly)
cudaError_t f64_update(cudaStream_t st, double *p, const float *g, int64_t n, double scale);
cudaError_t f64_round(cudaStream_t st, const double *src, float *dst, int64_t n);   // round to nearest
// loss = 1/n sum 1/2 |a - y|^2, accuracy = share of rows with argmax a == argmax y, both in
// double; out[2] = {loss, acc} (fp32) and/or *step_loss = loss.  part: >= loss_acc64_parts()
cudaError_t loss_acc64(cudaStream_t st, const double *A, const float *Y, int64_t n, int w, double2 *part,
                       float *out, float *step_loss);
constexpr int loss_acc64_parts() { return 2 * 148; }

}  // namespace nf
