/*
 * nf_oracle.c -- plain, slow, single-threaded CPU oracle of the neural-fortran
 * method (Curcic, arXiv:1902.06714).  TEST INFRASTRUCTURE ONLY: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load this library.  The product path (paper_1902_06714_b200/) never
 * links, imports or executes anything under oracle/.  It shares no code,
 * header, table or constant with the CUDA path.
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n, "S:n" = SPEC.md line n.
 *
 * Compiled twice from this one file:
 *   REAL=double -> liboracle64.so  (parity reference; inputs are fp32 values
 *                                   widened exactly, results rounded to fp32
 *                                   only at the comparison)
 *   REAL=float  -> liboracle32.so  (the paper-default real32 precision,
 *                                   P:253-256; used only for CPU timing)
 * gcc -O2, NO -ffast-math: IEEE round-to-nearest, libm exp/tanh.
 *
 * Parameter layout (flat, shared convention with the C-ABI by *specification*,
 * not by code): for l = 1..L : W_l[n_l][n_{l-1}] row-major, then b_l[n_l].
 * W_l[i][k] is the paper's w(k,i) of layer l-1 (column-major
 * w(this,next) has the same memory order), reading R4 in DESIGN.md.
 *
 * Every loop below is in the paper's order: per sample, forward layer by layer
 * (P:324-361), backward from the output layer, tendencies summed
 * over the batch in sample order, update once with
 * eta/B after the batch (reading R3).
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>

#ifndef REAL
#define REAL double
#endif

/* activation kinds (P:108-109 lists gaussian, RELU, sigmoid, step, tanh). */
enum { ORC_SIGMOID = 0, ORC_TANH = 1, ORC_RELU = 2, ORC_GAUSSIAN = 3, ORC_STEP = 4 };

#define ORC_MAX_LAYERS 64

/* sigma(x) -- S:40; sigmoid definition P:207-209. */
REAL orc_act(int kind, REAL x)
{
    switch (kind) {
    case ORC_SIGMOID: return (REAL)1 / ((REAL)1 + exp(-x));
    case ORC_TANH: return tanh(x);
    case ORC_RELU: return x > 0 ? x : (REAL)0;
    case ORC_GAUSSIAN: return exp(-x * x);
    case ORC_STEP: return x > 0 ? (REAL)1 : (REAL)0;
    }
    return NAN;
}

/* sigma'(x) -- S:51, written out from each definition; relu'(0)=0 and
 * step'=0 by reading R8. */
REAL orc_act_prime(int kind, REAL x)
{
    REAL s;
    switch (kind) {
    case ORC_SIGMOID: s = (REAL)1 / ((REAL)1 + exp(-x)); return s * ((REAL)1 - s);
    case ORC_TANH: s = tanh(x); return (REAL)1 - s * s;
    case ORC_RELU: return x > 0 ? (REAL)1 : (REAL)0;
    case ORC_GAUSSIAN: return -(REAL)2 * x * exp(-x * x);
    case ORC_STEP: return (REAL)0;
    }
    return NAN;
}

/* the activation of layer l (1-based, l = 1..L) is acts[l-1] (reading R7: the paper has one
 * activation per net; configs 4/5 need relu hidden + sigmoid output, and SURVEY
 * 8(f) generalises to one activation per layer).  The Python wrapper expands "name" and
 * "hidden,output" specs into this array. */
static int act_of(const int *acts, int l) { return acts[l - 1]; }

long orc_param_count(const int *dims, int nd)
{
    long c = 0;
    for (int l = 1; l < nd; ++l) c += (long)dims[l] * dims[l - 1] + dims[l];
    return c;
}

/* offsets of W_l and b_l in the flat parameter vector */
static void layer_offsets(const int *dims, int nd, long *offW, long *offB)
{
    long o = 0;
    for (int l = 1; l < nd; ++l) {
        offW[l] = o; o += (long)dims[l] * dims[l - 1];
        offB[l] = o; o += dims[l];
    }
}

typedef struct {
    int nd, L, maxw;
    const int *acts;             /* acts[l-1]: activation kind of layer l */
    const int *dims;
    long offW[ORC_MAX_LAYERS], offB[ORC_MAX_LAYERS];
    REAL *a[ORC_MAX_LAYERS];     /* a_l, l = 0..L (a_0 = x) */
    REAL *z[ORC_MAX_LAYERS];     /* z_l, l = 1..L ("temp. array") */
    REAL *delta[ORC_MAX_LAYERS]; /* delta_l, l = 1..L (backprop db(n)) */
} net_t;

static int net_open(net_t *t, const int *dims, int nd, const int *acts)
{
    if (nd < 2 || nd > ORC_MAX_LAYERS) return -1;
    memset(t, 0, sizeof *t);
    t->nd = nd; t->L = nd - 1; t->dims = dims; t->acts = acts;
    for (int l = 1; l < nd; ++l)
        if (acts[l - 1] < ORC_SIGMOID || acts[l - 1] > ORC_STEP) return -1;
    for (int l = 0; l < nd; ++l) {
        if (dims[l] < 1) return -1;
        t->a[l] = (REAL *)calloc((size_t)dims[l], sizeof(REAL));
        t->z[l] = (REAL *)calloc((size_t)dims[l], sizeof(REAL));
        t->delta[l] = (REAL *)calloc((size_t)dims[l], sizeof(REAL));
        if (!t->a[l] || !t->z[l] || !t->delta[l]) return -1;
    }
    layer_offsets(dims, nd, t->offW, t->offB);
    return 0;
}

static void net_close(net_t *t)
{
    for (int l = 0; l < t->nd; ++l) { free(t->a[l]); free(t->z[l]); free(t->delta[l]); }
}

/* fwdprop (Eq. 2): a_0 = x; for l = 1..L
 *   z_l[i] = sum_k W_l[i][k] a_{l-1}[k]  (k ascending)  + b_l[i]
 *   a_l    = sigma_l(z_l)                                             */
static void fwdprop(net_t *t, const REAL *p, const float *x)
{
    for (int k = 0; k < t->dims[0]; ++k) t->a[0][k] = (REAL)x[k];
    for (int l = 1; l <= t->L; ++l) {
        const int ni = t->dims[l], nk = t->dims[l - 1];
        const REAL *W = p + t->offW[l], *b = p + t->offB[l];
        const int kind = act_of(t->acts, l);
        for (int i = 0; i < ni; ++i) {
            REAL s = 0;
            for (int k = 0; k < nk; ++k) s += W[(long)i * nk + k] * t->a[l - 1][k];
            t->z[l][i] = s + b[i];
            t->a[l][i] = orc_act(kind, t->z[l][i]);
        }
    }
}

/* backprop: needs a prior fwdprop of the same sample.
 *   delta_L = (a_L - y) * sigma_L'(z_L)               (quadratic cost)
 *   delta_l[k] = (sum_i W_{l+1}[i][k] delta_{l+1}[i]) * sigma_l'(z_l[k]),
 *                l = L-1..1 (no delta for the input layer)
 * and adds the tendencies of this sample to G (same flat layout as params):
 *   dW_l[i][k] += delta_l[i] a_{l-1}[k],  db_l[i] += delta_l[i].            */
static void backprop_accumulate(net_t *t, const REAL *p, const float *y, REAL *G)
{
    const int L = t->L;
    for (int i = 0; i < t->dims[L]; ++i)
        t->delta[L][i] = (t->a[L][i] - (REAL)y[i]) *
                         orc_act_prime(act_of(t->acts, L), t->z[L][i]);
    for (int l = L - 1; l >= 1; --l) {
        const int nk = t->dims[l], ni = t->dims[l + 1];
        const REAL *W = p + t->offW[l + 1];
        const int kind = act_of(t->acts, l);
        for (int k = 0; k < nk; ++k) {
            REAL s = 0;
            for (int i = 0; i < ni; ++i) s += W[(long)i * nk + k] * t->delta[l + 1][i];
            t->delta[l][k] = s * orc_act_prime(kind, t->z[l][k]);
        }
    }
    for (int l = 1; l <= L; ++l) {
        const int ni = t->dims[l], nk = t->dims[l - 1];
        REAL *dW = G + t->offW[l], *db = G + t->offB[l];
        for (int i = 0; i < ni; ++i) {
            for (int k = 0; k < nk; ++k) dW[(long)i * nk + k] += t->delta[l][i] * t->a[l - 1][k];
            db[i] += t->delta[l][i];
        }
    }
}

/* output: the fwdprop recursion, returning a_L only. out[n][n_L]. */
int orc_output(const int *dims, int nd, const int *acts, const REAL *p,
               const float *x, long n, REAL *out)
{
    net_t t;
    if (net_open(&t, dims, nd, acts)) { net_close(&t); return -1; }
    for (long s = 0; s < n; ++s) {
        fwdprop(&t, p, x + s * dims[0]);
        for (int i = 0; i < dims[nd - 1]; ++i) out[s * dims[nd - 1] + i] = t.a[t.L][i];
    }
    net_close(&t);
    return 0;
}

/* summed tendencies over a batch (the batch accumulation of train_batch,
 * P:460-476, and the co_sum total).  G is overwritten. */
int orc_grad(const int *dims, int nd, const int *acts, const REAL *p,
             const float *x, const float *y, long n, REAL *G)
{
    net_t t;
    if (net_open(&t, dims, nd, acts)) { net_close(&t); return -1; }
    memset(G, 0, sizeof(REAL) * (size_t)orc_param_count(dims, nd));
    for (long s = 0; s < n; ++s) {
        fwdprop(&t, p, x + s * dims[0]);
        backprop_accumulate(&t, p, y + s * dims[nd - 1], G);
    }
    net_close(&t);
    return 0;
}

/* update (body omitted in the paper; reading R3):
 *   p -= scale * G */
void orc_update(REAL *p, const REAL *G, long count, REAL scale)
{
    for (long i = 0; i < count; ++i) p[i] -= scale * G[i];
}

/* quadratic cost of one sample, 1/2 sum (a_L - y)^2. */
static REAL sample_cost(const net_t *t, const float *y)
{
    REAL c = 0;
    for (int i = 0; i < t->dims[t->L]; ++i) {
        REAL d = t->a[t->L][i] - (REAL)y[i];
        c += d * d;
    }
    return c / 2;
}

/* train_batch: every sample sees the pre-batch parameters; the
 * summed tendencies are applied once, scaled eta/n (reading R3).
 * If batch_loss != NULL it receives the mean cost of the batch under the
 * pre-update parameters (reading R9). */
int orc_train_batch(const int *dims, int nd, const int *acts, REAL *p,
                    const float *x, const float *y, long n, REAL eta, REAL *batch_loss)
{
    if (n <= 0) return -1;
    const long cnt = orc_param_count(dims, nd);
    REAL *G = (REAL *)calloc((size_t)cnt, sizeof(REAL));
    net_t t;
    if (!G || net_open(&t, dims, nd, acts)) { free(G); return -1; }
    REAL loss = 0;
    for (long s = 0; s < n; ++s) {
        fwdprop(&t, p, x + s * dims[0]);
        loss += sample_cost(&t, y + s * dims[nd - 1]);
        backprop_accumulate(&t, p, y + s * dims[nd - 1], G);
    }
    orc_update(p, G, cnt, eta / (REAL)n);
    if (batch_loss) *batch_loss = loss / (REAL)n;
    net_close(&t);
    free(G);
    return 0;
}

/* The MNIST driver's minibatch loop on a resident dataset:
 * step s trains on rows [starts[s], starts[s]+batch) of X/Y (reading R11:
 * 0-based starts uniform in [0, N-batch]).  step_loss may be NULL. */
int orc_train_steps(const int *dims, int nd, const int *acts, REAL *p,
                    const float *X, const float *Y, long N, long batch,
                    const long *starts, long n_steps, REAL eta, REAL *step_loss)
{
    for (long s = 0; s < n_steps; ++s) {
        if (starts[s] < 0 || starts[s] + batch > N) return -2;
        int rc = orc_train_batch(dims, nd, acts, p, X + starts[s] * dims[0],
                                 Y + starts[s] * dims[nd - 1], batch, eta,
                                 step_loss ? step_loss + s : NULL);
        if (rc) return rc;
    }
    return 0;
}

/* mean quadratic cost over n samples (reading R9). */
int orc_loss(const int *dims, int nd, const int *acts, const REAL *p,
             const float *x, const float *y, long n, REAL *loss)
{
    net_t t;
    if (net_open(&t, dims, nd, acts)) { net_close(&t); return -1; }
    REAL c = 0;
    for (long s = 0; s < n; ++s) {
        fwdprop(&t, p, x + s * dims[0]);
        c += sample_cost(&t, y + s * dims[nd - 1]);
    }
    *loss = n > 0 ? c / (REAL)n : 0;
    net_close(&t);
    return 0;
}

/* index of the first maximum (ties -> lowest index, reading R10). */
static int argmax_first(const REAL *v, int n)
{
    int m = 0;
    for (int i = 1; i < n; ++i) if (v[i] > v[m]) m = i;
    return m;
}
static int argmax_first_f(const float *v, int n)
{
    int m = 0;
    for (int i = 1; i < n; ++i) if (v[i] > v[m]) m = i;
    return m;
}

/* accuracy: fraction of samples whose
 * predicted class argmax(a_L) equals argmax(y).  n = 0 -> 0.0. */
int orc_accuracy(const int *dims, int nd, const int *acts, const REAL *p,
                 const float *x, const float *y, long n, REAL *acc)
{
    net_t t;
    if (net_open(&t, dims, nd, acts)) { net_close(&t); return -1; }
    long good = 0;
    const int no = dims[nd - 1];
    for (long s = 0; s < n; ++s) {
        fwdprop(&t, p, x + s * dims[0]);
        good += argmax_first(t.a[t.L], no) == argmax_first_f(y + s * no, no);
    }
    *acc = n > 0 ? (REAL)good / (REAL)n : 0;
    net_close(&t);
    return 0;
}

/* per-layer stash of one forward pass over a batch, for kernel-level
 * parity (a_l, delta_l and z_l per sample).  A: for l=0..L, [n][n_l] blocks
 * concatenated; D and Z (Z may be NULL): for l=1..L, [n][n_l] blocks. */
int orc_forward_backward_stash(const int *dims, int nd, const int *acts,
                               const REAL *p, const float *x, const float *y,
                               long n, REAL *A, REAL *D, REAL *Z)
{
    net_t t;
    if (net_open(&t, dims, nd, acts)) { net_close(&t); return -1; }
    const long cnt = orc_param_count(dims, nd);
    REAL *G = (REAL *)calloc((size_t)cnt, sizeof(REAL));
    if (!G) { net_close(&t); return -1; }
    for (long s = 0; s < n; ++s) {
        fwdprop(&t, p, x + s * dims[0]);
        backprop_accumulate(&t, p, y + s * dims[nd - 1], G);
        long oa = 0, od = 0;
        for (int l = 0; l < nd; ++l) {
            for (int i = 0; i < dims[l]; ++i) A[oa + s * dims[l] + i] = t.a[l][i];
            oa += n * dims[l];
            if (l >= 1) {
                for (int i = 0; i < dims[l]; ++i) D[od + s * dims[l] + i] = t.delta[l][i];
                if (Z)
                    for (int i = 0; i < dims[l]; ++i) Z[od + s * dims[l] + i] = t.z[l][i];
                od += n * dims[l];
            }
        }
    }
    free(G);
    net_close(&t);
    return 0;
}

int orc_real_bytes(void) { return (int)sizeof(REAL); }
