// deep_mk.cuh -- ONE persistent task kernel per nf_train_steps call for deep nets of narrow
// hidden layers (config 4: [784, 256 x 8, 10]) in NF_MATH_TF32.  Every SGD step (the paper's
// train_batch) becomes a static list of tasks -- tcgen05 GEMM tiles of the forward
// (fwdprop P:324-361), backward delta (backprop P:409-411) and batch-summed weight tendency with
// the SGD update (the co_sum P:536-556), plus SIMT tasks for the narrow output layer,
// its tendency and the TF32 weight shadow -- executed by one co-resident CTA per SM, ordered by
// per-row-block dependency counters in global memory instead of ~26 kernel boundaries per step.
#pragma once
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

namespace nf {

constexpr int DEEP_NOT_APPLICABLE = 1;

struct DeepMK {
  void *dev = nullptr;            // tensor maps | task table | counters | partials | starts
  size_t dev_bytes = 0;
  std::vector<int64_t> key;       // configuration the device state was built for
  int tasks_per_step = 0;
  int grid = 0;
  size_t smem = 0;
  size_t off_maps = 0, off_tasks = 0, off_ctr = 0, off_part = 0, off_lpart = 0, off_starts = 0;
  size_t ctr_bytes = 0;
  int64_t starts_cap = 0;
  int64_t *h_starts = nullptr;    // pinned staging of the batch starts
  cudaEvent_t h_ev = nullptr;
};

// Whether the megakernel handles this net / batch (TF32 mode, 2 <= L <= 15, hidden widths
// multiples of 64 up to 256, output width <= 16, n0 % 4 == 0, batch a multiple of 128 up to 16384).
bool deep_mk_applicable(const std::vector<int> &dims, int math, int64_t batch);

// Runs n_steps SGD steps in one launch.  A[l], S[l] (l = 1..L): the net's stash ([batch][n_l]);
// params / params_t: fp32 master weights and their TF32 shadow (current on entry, current on
// exit); X [N][n0], Y [N][nL] the dataset; starts: host array.  Returns 0, DEEP_NOT_APPLICABLE or
// -1 (CUDA error, text in deep_mk_error()).
int deep_mk_train_steps(DeepMK &st, cudaStream_t stream, const std::vector<int> &dims, const std::vector<int> &acts,
                        float *params, float *params_t, const std::vector<int64_t> &offW,
                        const std::vector<int64_t> &offB, const std::vector<float *> &A, const std::vector<float *> &S,
                        const float *X, const float *Y, int64_t N, int64_t batch, const int64_t *starts,
                        int64_t n_steps, float eta, float *step_loss);
void deep_mk_release(DeepMK &st);
const char *deep_mk_error();

}  // namespace nf
