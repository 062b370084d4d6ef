// fused_small.cuh -- persistent multi-step SGD kernel for two-layer nets with
// narrow hidden/output layers (configs 1 and 2: [3,5,2], [784,30,10]).
#pragma once
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

namespace nf {

constexpr int FUSED_NOT_APPLICABLE = 1;

struct FusedSmall {
  void *ws = nullptr;        // device workspace: gradient accumulators, barrier counter, starts
  size_t ws_bytes = 0;
  bool valid = false;        // reserved for resident-state caching
};

// Runs n_steps SGD steps (the paper's train_batch per minibatch) in one launch.
// Returns 0 on success, FUSED_NOT_APPLICABLE if the net's shape is not handled
// (the caller then runs the generic per-step kernels), or -1 on a CUDA error
// (text in fused_small_error()).
int fused_small_train_steps(FusedSmall &fs, cudaStream_t st, const std::vector<int> &dims, int act_h,
                            int act_o, float *params, const float *X, const float *Y, int64_t N,
                            int64_t batch, const int64_t *starts, int64_t n_steps, float eta,
                            float *step_loss);
void fused_small_release(FusedSmall &fs);
void fused_small_invalidate(FusedSmall &fs);
const char *fused_small_error();

}  // namespace nf
