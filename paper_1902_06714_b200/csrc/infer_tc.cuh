// infer_tc.cuh -- fused inference (the paper's `output`) for two-layer nets with hidden
// and output widths <= 32 (config 2) on the tcgen05 tensor cores (3xTF32): x streamed once by TMA,
// no stash.
#pragma once
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

namespace nf {

// dims = {n0, H, O} with H, O <= 32, n0 % 4 == 0, n0 >= 32, X 16-B aligned (TMA rows);
// NF_INFER_SIMT=1 selects the FFMA2 kernel (infer_small) instead.
bool infer_tc_applicable(const std::vector<int> &dims, const float *X);
// out [n][O] = sigma_o(W2 sigma_h(W1 x + b1) + b2) for the n rows of X [n][n0].  params: the flat
// arena of nf.h (b1, W2, b2 read from it); W1hi / W1lo: the RN split of W1 (hi = rn_tf32(W1),
// lo = rn_tf32(W1 - hi)), [H][n0] each.
cudaError_t infer_tc(cudaStream_t st, const std::vector<int> &dims, int act_h, int act_o, const float *params,
                     const float *W1hi, const float *W1lo, const float *X, int64_t n, float *out);

}  // namespace nf
