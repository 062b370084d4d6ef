// infer_small.cuh -- fused inference (the paper's `output`) for two-layer nets
// with hidden and output widths <= 32 (config 2): x streamed once, no stash.
#pragma once
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

namespace nf {

bool infer_small_applicable(const std::vector<int> &dims, const float *X);
size_t infer_small_smem(int n0);
// out [n][dims[2]] = sigma_o(W2 sigma_h(W1 x + b1) + b2) for the n rows of X [n][dims[0]];
// params in the flat layout of nf.h.
cudaError_t infer_small(cudaStream_t st, const std::vector<int> &dims, int act_h, int act_o, const float *params,
                        const float *X, int64_t n, float *out);

}  // namespace nf
