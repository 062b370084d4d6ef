/*
 * nf.h -- C-ABI of the B200-native hot path of neural-fortran (Curcic,
 * arXiv:1902.06714): minibatch SGD training of a dense feed-forward network.
 *
 * Citations: "P:n" = PAPER.md line n (the paper), "S:n" = SPEC.md line n.
 * The entry points follow the paper's network interface: constructor
 * network_type(dims, activation), output, train on a
 * batch, accuracy and the quadratic cost.
 *
 * Conventions for every call
 *   - All tensors are fp32, row-major [n][width] (one sample per row; the
 *     paper's column-major x(:,i) has the same memory order).
 *   - Caller buffers (x, y, out, grad, params) may be HOST pointers (pageable
 *     or pinned) or CUDA DEVICE pointers; the library tells them apart with
 *     cudaPointerGetAttributes.  Host inputs are copied to device staging
 *     buffers on the net's stream; host outputs are copied back and the call
 *     synchronises before returning.  With device pointers the call is
 *     asynchronous on the net's stream (unless stated) and the caller keeps
 *     the buffers alive until the stream reaches the call.
 *   - Pointers must be 4-byte aligned.  No other alignment is required (the
 *     runtime picks vector widths per pointer).
 *   - Parameters, workspaces and staging buffers are owned by the library.
 *   - Return value: NF_OK (0) or a negative NF_E* code; nf_last_error()
 *     returns a thread-local text for the last failing call.
 *   - A net is used by one stream (one host thread) at a time.
 *
 * Parameter layout ("flat"): for l = 1..L, W_l [n_l][n_{l-1}] row-major, then
 * b_l [n_l].  W_l[i][k] connects input k of layer l-1 to neuron i of layer l;
 * this is the paper's w(k,i) stored in layer l-1 in the same
 * column-major memory order.  b_l lives with layer l.
 */
#ifndef NF_H
#define NF_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct nf_net nf_net;

enum {
    NF_OK = 0,
    NF_EINVAL = -1,       /* bad argument: see nf_last_error()            */
    NF_ECUDA = -2,        /* CUDA runtime error (message has its string)  */
    NF_ENOMEM = -3,       /* device allocation failed                     */
    NF_ENODEV = -4,       /* no sm_100 device: there is NO CPU fallback   */
    /* nf_load / nf_load_as format errors, one code per kind     */
    NF_EFMT_MAGIC = -5,       /* not a file of this library                   */
    NF_EFMT_VERSION = -6,     /* unsupported format version                   */
    NF_EFMT_PRECISION = -7,   /* unknown precision tag, or a precision other
                                 than the one requested (never narrowed)      */
    NF_EFMT_TRUNCATED = -8,   /* fewer parameters than the dims imply         */
    NF_EFMT_ACTIVATION = -9,  /* missing / unknown activation name            */
    NF_EFMT_DIMS = -10,       /* bad dims header                              */
    NF_EIO = -11              /* the file cannot be opened / written          */
};

/* Numerics mode of the contractions (nf_set_math).
 *   NF_MATH_FP32 : fp32 storage; fp32 FMA accumulation or 3xTF32 tensor-core
 *                  tiles (hi*hi + hi*lo + lo*hi, fp32 accumulate) (default; the
 *                  paper's real32).  Parity bar 1e-4 at tau = 0.1
 *                  (BASELINE.json; R14).
 *   NF_MATH_TF32 : 1xTF32 tensor-core tiles on round-to-nearest TF32 operands,
 *                  fp32 accumulate, wherever a contraction has all extents >= 64
 *                  (configs 3, 4 and 5; narrower ones stay fp32).  Parity bar
 *                  5e-3 normwise (tau = 1; R14b).
 *   NF_MATH_FP64 : the paper's real64 build: parameters,
 *                  activations, deltas and every sum in double on the FP64
 *                  units.  Inputs, targets and results still cross this ABI
 *                  as fp32 (widened exactly on entry, rounded once on exit);
 *                  the parameters are held in double while the mode is set
 *                  (nf_get_params rounds them, nf_set_params widens them) and
 *                  rounded back to the fp32 arena when the mode is left.
 *                  Parity bar 2.5e-7 at tau = 0.1 against the fp64 oracle
 *                  (4 fp32 ulps: the rounding at the ABI; R19).   */
enum { NF_MATH_FP32 = 0, NF_MATH_TF32 = 1, NF_MATH_FP64 = 2 };

/* Constructor (network_constructor_listing).
 *   dims[0..n_dims-1] : neurons per layer incl. input and output;
 *                       n_dims >= 2, every dim >= 1.
 *   activation        : "sigmoid" | "tanh" | "relu" | "gaussian" | "step"
 *                        for every layer, or "hidden,output" (e.g.
 *                       "relu,sigmoid": the output layer its own activation,
 *                       reading R7), or n_dims-1 comma-separated names, one
 *                       per layer.  NULL means "sigmoid", the
 *                       paper's default.  An unknown name or
 *                       another count of names -> NF_EINVAL.
 *   seed              : initial parameters are drawn on the host from a
 *                       documented splitmix64/Box-Muller stream:
 *                       W ~ N(0,1)/n_{l-1} ("normalized by the number of
 *                       neurons in the layer"), b ~ N(0,1) (R2).
 *                       Benchmarks and tests overwrite them with nf_set_params.
 *   *out              : receives the new net (owned by the caller, release
 *                       with nf_net_destroy).
 * Fails with NF_ENODEV when no sm_100 GPU is present.                       */
int nf_net_create(const int32_t *dims, int32_t n_dims, const char *activation,
                  uint64_t seed, nf_net **out);

/* Synchronises the net's stream and frees everything the net owns. */
void nf_net_destroy(nf_net *net);

/* Sets the CUDA stream (a cudaStream_t; NULL = legacy default stream) on
 * which every later call of this net is ordered. */
int nf_set_stream(nf_net *net, void *cuda_stream);

/* NF_MATH_FP32, NF_MATH_TF32 or NF_MATH_FP64 (see above); anything else ->
 * NF_EINVAL.  Ordered on the net's stream. */
int nf_set_math(nf_net *net, int mode);

/* Number of parameters: sum_l n_l*n_{l-1} + n_l ([3,5,2] -> 32). */
int64_t nf_param_count(const nf_net *net);

/* Copies the flat parameters out (dst: count floats, host or device).
 * count must equal nf_param_count.  Host dst: synchronous. */
int nf_get_params(nf_net *net, float *dst, int64_t count);

/* Replaces the flat parameters (src: count floats, host or device). */
int nf_set_params(nf_net *net, const float *src, int64_t count);

/* The paper's `output`: forward pass without caching.
 *   x   [n][n_0]  inputs;  out [n][n_L] receives a_L.  n >= 0.            */
int nf_output(nf_net *net, const float *x, int64_t n, float *out);

/* One SGD step on a batch: the paper's train_batch with its
 * fwdprop and backprop per sample, tendencies summed
 * over the batch (the co_sum) and the update
 *   W_l -= (eta/n) * sum_s delta_l(s) a_{l-1}(s)^T,  b_l -= (eta/n) sum_s delta_l(s)
 * (reading R3).  Every sample sees the pre-step parameters.
 *   x [n][n_0], y [n][n_L] (targets, e.g. one-hot labels), n >= 1,
 *   eta finite.  eta = 0 leaves the parameters bitwise unchanged.          */
int nf_train_batch(nf_net *net, const float *x, const float *y, int64_t n, float eta);

/* The MNIST driver's minibatch loop moved on-device (extension):
 * for s = 0..n_steps-1, nf_train_batch on rows [starts[s], starts[s]+batch)
 * of the resident dataset X [N][n_0], Y [N][n_L].
 *   starts     : HOST array of n_steps int64, each in [0, N-batch] (R11).
 *   step_loss  : NULL or a DEVICE array of n_steps floats receiving the mean
 *                quadratic cost of step s's batch under the pre-step
 *                parameters (the cost evaluated by step 1 of SGD).
 * Small nets (two layers, widths <= 32) run as ONE persistent kernel for all
 * steps; others as a sequence of fused kernels per step.                    */
int nf_train_steps(nf_net *net, const float *X, const float *Y, int64_t N, int64_t batch,
                   const int64_t *starts, int64_t n_steps, float eta, float *step_loss);

/* The paper's backprop + co_sum without the update: writes the
 * batch-summed tendencies in the flat parameter layout (grad: count floats).
 * Parameters are unchanged.  (Extension, for gradient parity.)             */
int nf_grad(nf_net *net, const float *x, const float *y, int64_t n, float *grad);

/* nf_grad that announces each layer's tendencies as soon as they are final, so that the
 * data-parallel co_sum of layer l can run while the backward pass still works on
 * layers l-1..1 (bucketed all-reduce overlapped with the backward).
 *   events   : n_events == L cudaEvent_t handles created by the caller (any flags);
 *              events[l-1] is recorded on a stream of the library once the W_l and b_l blocks
 *              of grad are written (layer L first, layer 1 last).  A NULL entry is skipped;
 *              events == NULL is nf_grad.  Another count -> NF_EINVAL.
 * With a HOST grad or in NF_MATH_FP64 every event is recorded at the end (no overlap).
 * The caller makes its communication stream wait on events[l-1] before reading layer l's
 * block and orders nf_update after its collectives (e.g. cudaStreamWaitEvent).           */
int nf_grad_layers(nf_net *net, const float *x, const float *y, int64_t n, float *grad,
                   void *const *events, int32_t n_events);

/* The paper's `update`, applied to externally summed tendencies:
 *   params -= (eta / n) * grad
 * grad: count = nf_param_count floats in the flat parameter layout (host or device), e.g. the
 * nf_grad tendencies of each rank's piece of a batch after the paper's co_sum over ranks
 * (paper_1902_06714_b200.dp.DataParallel does that with an NCCL all-reduce);
 * n = the rows of the WHOLE batch (n >= 1; the eta/B scale of reading R3).  In NF_MATH_FP64
 * the update is applied to the double parameters.  Extension of the north-star list (the
 * data-parallel step of SURVEY 8(e)).  Host grad: synchronous. */
int nf_update(nf_net *net, const float *grad, int64_t count, float eta, int64_t n);

/* Mean quadratic cost (1/n) sum_s 1/2 ||a_L(x_s) - y_s||^2 (reading R9)
 * written to *loss (host).  n = 0 -> 0.  Synchronises. */
int nf_loss(nf_net *net, const float *x, const float *y, int64_t n, float *loss);

/* Accuracy: fraction of samples with
 * argmax a_L(x_s) == argmax y_s, first index on ties (R10), to *acc (host).
 * n = 0 -> 0.0.  Synchronises. */
int nf_accuracy(nf_net *net, const float *x, const float *y, int64_t n, float *acc);

/* Saving and loading networks to and from file (the paper gives no format, this
 * library's is text): a header line "nf-b200-net 2", n_dims, the dims, the activation spec,
 * the precision tag "fp32" or "fp64", then the nf_param_count parameters in the flat layout,
 * one per line -- 9 significant digits for fp32, 17 for fp64 (both exact: a round trip is
 * bitwise).  In NF_MATH_FP64 the double parameters are written, never narrowed.
 * nf_save synchronises; NF_EIO if the file cannot be written.  Host file I/O. */
int nf_save(nf_net *net, const char *path);

/* Loads a file written by nf_save (version 1 files, without a precision line, are fp32):
 * parses and validates the header (magic, version, dims, activation, precision) before the
 * payload, then the whole payload, before any device work; each kind of format error returns
 * its own NF_EFMT_* code.  Then nf_net_create + the parameters; an fp64 file gives a net in
 * NF_MATH_FP64 holding the exact doubles, an fp32 file one in NF_MATH_FP32.  *out is owned by
 * the caller (nf_net_destroy). */
int nf_load(const char *path, nf_net **out);

/* nf_load that also states the numerics mode the caller wants: an fp64 file into
 * NF_MATH_FP32 / NF_MATH_TF32, or an fp32 file into NF_MATH_FP64, is rejected with
 * NF_EFMT_PRECISION (never silently narrowed or widened).  math = -1: as nf_load. */
int nf_load_as(const char *path, int math, nf_net **out);

/* Thread-local text of the last error ("" if none). */
const char *nf_last_error(void);

/* Number of this library's kernels launched since load (for the bench's
 * gpu_launches claim), including the kernels of each replay of the CUDA graph
 * nf_train_steps captures for generic nets. */
int64_t nf_launch_count(void);

/* Debug launch log (tests: which kernel instantiations a workload launches).
 * nf_debug_log_enable(1) clears the log and records every later launch of this library as
 * one line "<demangled kernel name> grid=(x,y,z) block=T smem=S [variant]" (variant: the
 * epilogue mode, split-K "splitk-red" / "splitk-partial", the K6 cluster size); 0 stops
 * recording.  NF_LOG_LAUNCHES=1 in the environment enables it at load.  A CUDA graph's
 * kernels are logged once, when it is captured, not on replay.  Host-only, no errors. */
void nf_debug_log_enable(int on);

/* Copies the launch log (NUL-terminated, truncated to cap bytes) into buf (buf may be NULL,
 * cap <= 0: nothing copied) and returns the bytes the whole log needs including the NUL. */
int64_t nf_debug_log_read(char *buf, int64_t cap);

#ifdef __cplusplus
}
#endif
#endif /* NF_H */
