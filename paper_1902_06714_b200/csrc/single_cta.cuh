// single_cta.cuh -- small-batch SGD (the paper's train_single / train_batch with a few rows,
// P:429-476) for nets whose parameters fit in one SM's shared memory: all steps in ONE CTA.
#pragma once
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

namespace nf {

constexpr int SINGLE_NOT_APPLICABLE = 1;

// Runs n_steps SGD steps of `batch` rows each (rows starts[s] .. starts[s]+batch-1 of X, Y;
// d_starts: the same starts in device memory) on one CTA: forward, delta_L, backward deltas,
// tendencies summed over the rows and the update, with the parameters resident in shared memory
// and the next step's rows prefetched (cp.async).  step_loss (nullable, device): mean cost per
// step.  Returns 0, SINGLE_NOT_APPLICABLE (shape / batch outside the latency regime: the caller
// uses K6 or the generic kernels), or a cudaError_t value.
bool single_cta_applicable(const std::vector<int> &dims, int64_t batch);
// acts[l]: activation kind of layer l (l = 1..L)
int single_cta_train_steps(cudaStream_t st, const std::vector<int> &dims, const std::vector<int> &acts, float *params,
                           const float *X, const float *Y, int64_t batch, const int64_t *d_starts, int64_t n_steps,
                           float eta, float *step_loss);

}  // namespace nf
