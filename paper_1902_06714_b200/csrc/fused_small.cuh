// fused_small.cuh -- persistent multi-step SGD kernel for two-layer nets with
// narrow hidden/output layers (configs 1 and 2: [3,5,2], [784,30,10]).
#pragma once
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

namespace nf {

constexpr int FUSED_NOT_APPLICABLE = 1;

struct FusedSmall {
  void *ws = nullptr;        // device workspace: gradient accumulator ring + grid-barrier counter
  size_t ws_bytes = 0;
  bool valid = false;        // reserved for resident-state caching
  // Across calls the workspace keeps its state instead of being reset per call: the kernel
  // leaves the slots a next call starts on zeroed, the barrier counter runs on monotonically.
  bool ws_ready = false;     // ring zero / counter known (false: memset before the next launch)
  uint64_t steps_done = 0;   // slot ring position (steps run since the last reset)
  unsigned bar_base = 0;     // barrier counter value at the next launch
  int64_t ring_key[4] = {};  // (slot floats, CTAs) the ring state belongs to
  // device copy of the batch starts, staged through two pinned host buffers (async H2D)
  int64_t *d_starts = nullptr, *h_starts[2] = {nullptr, nullptr};
  size_t starts_cap = 0;
  cudaEvent_t h_ev[2] = {nullptr, nullptr};
  int h_i = 0;
  // launch decision cache: same net shape, batch, dataset and switches -> same configuration
  std::vector<int64_t> cfg_key;
  int C = 0, G = 0, ws_cols = 0, wpad = 0, nSmax = 0, nOwnMax = 0;
  size_t smem = 0;
  bool tc = false, mm = false, aligned = false;
  alignas(64) unsigned char tmaps[3][128];
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
