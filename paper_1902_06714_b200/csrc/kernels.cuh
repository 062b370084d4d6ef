// kernels.cuh -- host-side launchers of the hot-path kernels (internal, C++).
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "gemm_simt.cuh"

namespace nf {

extern int64_t g_launches;  // kernels launched by this library (nf_launch_count)
inline void count_launch(int n = 1) { __atomic_add_fetch(&g_launches, n, __ATOMIC_RELAXED); }
// launch log (launchlog.cu; NF_LOG_LAUNCHES=1 or nf_debug_log_enable): demangled kernel name,
// grid, block, dynamic smem and a note naming the runtime variant (e.g. "red" split-K terms)
bool launch_log_on();
// NF_TRACE_HOST=1: host-time stamps of one call's phases to stderr (us since the call's "enter")
void host_trace(const char *what);
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device, bytes): the
// attribute is per device context, so a process driving several GPUs sets it on each
cudaError_t set_max_smem(const void *kern, int bytes);
void log_launch(const void *func, dim3 grid, dim3 block, size_t smem, const char *note = nullptr);

// Split-K partial workspace owned by the net (fixed capacity in floats) and the numerics
// mode of the contractions (NF_MATH_FP32 = 0: fp32 SIMT or 3xTF32 tensor cores;
// NF_MATH_TF32 = 1: 1xTF32 tensor cores where a GEMM qualifies).
struct Workspace {
  float *partial = nullptr;
  size_t partial_floats = 0;
  int math = 0;
  // non-null: a split-K SGD launch that reduced terms into W in L2 sets *red_flag instead of
  // re-rounding that layer's TF32 shadow itself (the caller rounds once after the step)
  bool *red_flag = nullptr;
};

// Which engine ran the last gemm_* call (for tests / the bench's kernel attribution).
enum Engine { ENGINE_SIMT = 0, ENGINE_TC1 = 1, ENGINE_TC3 = 3, ENGINE_HMMA1 = 11, ENGINE_HMMA3 = 13 };
Engine last_engine();

// K1: Z = A[M][K] * W[N][K]^T, epilogue EpiFwd.
// Wtc (NF_MATH_TF32, may be null): the TF32-rounded shadow of W, read by the tensor-core path
// instead of W (the SIMT paths read W itself)
// Alo / Wlo (fp32 mode, nullable): tf32_lo parts of the operands (pre-split 3xTF32 when both are given)
cudaError_t gemm_fwd(cudaStream_t st, int M, int N, int K, const float *A, const float *W,
                     const EpiFwd &epi, const Workspace &ws, const float *Wtc = nullptr, const float *Alo = nullptr,
                     const float *Wlo = nullptr, const float *Ahi = nullptr);
// K3: C[M][N] = D[M][K] * W[K][N], epilogue EpiBwd.
cudaError_t gemm_bwd(cudaStream_t st, int M, int N, int K, const float *D, const float *W,
                     const EpiBwd &epi, const Workspace &ws, const float *Wtc = nullptr, const float *Dlo = nullptr,
                     const float *Wlo = nullptr);
// K4: C[M][N+1] = D^T (D is [K][M]) * [Aprev | 1] (Aprev is [K][N]), epilogue EpiGrad.
// bias_done: the layer's bias update was already applied by the delta GEMM (EpiBwd::bias); only
// meaningful on the tensor-core path (the SIMT path carries the bias as a ones column)
// DT [M][K] / AprevT [N][K] (nullable): transposed copies of D / Aprev (written by their producers'
// epilogues, EpiBwd::T / EpiFwd::T) -- the tensor-core path then reads K-major operands
cudaError_t gemm_grad(cudaStream_t st, int M, int N, int K, const float *D, const float *Aprev,
                      const EpiGrad &epi, const Workspace &ws, bool bias_done = false, const float *DT = nullptr,
                      const float *AprevT = nullptr, const float *Dlo = nullptr, const float *Aprevlo = nullptr,
                      const float *Aprevhi = nullptr);
// whether gemm_fwd / gemm_bwd with these operands take the tensor-core path (where EpiFwd::T /
// EpiBwd::T are honoured)
bool gemm_fwd_tc(int M, int N, int K, const float *A, const float *W);
bool gemm_bwd_tc(int M, int N, int K, const float *D, const float *W);
// whether gemm_bwd with these operands takes the path whose epilogue can apply the bias update
bool gemm_bwd_fuses_bias(int M, int N, int K, const float *D, const float *W);
// whether gemm_grad with these operands takes the tensor-core path (bias as a separate sum)
bool gemm_grad_tc(int M, int N, int K, const float *D, const float *Aprev);

// The narrow output layer of a training step fused into one pass (kernels.cu, out_layer_train):
// K1+K2 of layer L, K3 of layer L-1 (in place of S_{L-1}) and the partial tendencies of layer L
// into part[R][nL][H+1] (R = out_layer_blocks(n, H)); out_layer_grad_final then sums them in fixed
// order and applies epi (update or store).
bool out_layer_fusable(int n, int H, int nL, const float *A, const float *S, const float *W);
int out_layer_blocks(int n, int H);
cudaError_t out_layer_train_fused(cudaStream_t st, int n, int H, int nL, const float *A, float *S, const float *W,
                                  const float *bias, const float *Y, float *AL, float *DL, int act, float *part,
                                  int rnd = 0,   // rnd: delta_{L-1} stored TF32-rounded (NF_MATH_TF32)
                                  float *Dlo = nullptr);  // fp32 mode: tf32_lo of delta_{L-1}
// step_loss (nullable): also writes the step's mean cost from the kernel's per-block partials
cudaError_t out_layer_grad_final(cudaStream_t st, int n, int H, int nL, const float *part, const EpiGrad &epi,
                                 float *step_loss = nullptr);

// K5: mean quadratic cost and argmax-accuracy of A_L against Y over n rows of
// width w.  part: scratch of >= loss_acc_parts() double2.  Results: out[0] =
// mean loss, out[1] = accuracy (device floats); step_loss (nullable) gets the
// mean loss too.
int loss_acc_parts();

// The paper's `update` on externally summed tendencies (nf_update): p[i] -= scale * g[i].
cudaError_t sgd_update(cudaStream_t st, float *p, const float *g, int64_t n, float scale);
// dst[i] = tf32_rn(src[i]): the TF32 weight shadow of NF_MATH_TF32
cudaError_t round_tf32(cudaStream_t st, const float *src, float *dst, int64_t n);
// dst[i] = tf32_lo(src[i]): the truncation split of the fp32 mode's pre-split 3xTF32
cudaError_t split_lo(cudaStream_t st, const float *src, float *dst, int64_t n);
// hi[i] = tf32_rn(src[i]), lo[i] = tf32_lo_rn(src[i]): the RN split (weights, input rows)
cudaError_t split_rn(cudaStream_t st, const float *src, float *hi, float *lo, int64_t n);
// copies m <= 64 contiguous runs of len floats, src + off[s] -> dst + s * len (src: device
// memory or mapped pinned host memory; the e2e staging of the per-step target rows)
cudaError_t gather_steps(cudaStream_t st, const float *src, const int64_t *off, int m, int64_t len, float *dst);
cudaError_t loss_acc(cudaStream_t st, const float *A, const float *Y, int64_t n, int w,
                     double2 *part, float *out, float *step_loss);

}  // namespace nf
