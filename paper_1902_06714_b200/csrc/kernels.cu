// kernels.cu -- dispatch of the generic SIMT contraction kernels and the
// loss/accuracy reduction (K5).
#include <algorithm>

#include <cstdlib>
#include <cstdio>
#include <cstring>

#include "gemm_tc.cuh"
#include "gemm_hmma.cuh"
#include "kernels.cuh"

namespace nf {

int64_t g_launches = 0;
static thread_local Engine g_last_engine = ENGINE_SIMT;
Engine last_engine() { return g_last_engine; }

namespace {

constexpr int kSMs = 148;

// Every kernel of the generic path is launched with programmatic stream serialization (PDL):
// the next kernel's CTAs are scheduled while the current one drains, run their prologue
// (barrier init, TMEM allocation, tensor-map prefetch) and block in griddepcontrol.wait until
// it has completed.  NF_NO_PDL=1 turns it off.
thread_local const char *g_note = nullptr;  // runtime variant of the next launch (launch log)
thread_local char g_note_buf[96];

// runtime variant of an epilogue for the launch log: forward mode, fused bias update, SGD or store
const char *epi_note(const EpiFwd &e) { return e.mode == 0 ? "fwd-hidden" : e.mode == 1 ? "fwd-output" : "fwd-infer"; }
const char *epi_note(const EpiBwd &e) { return e.bias ? "bwd+bias-red" : "bwd"; }
const char *epi_note(const EpiGrad &e) { return e.store_only ? "grad-store" : "grad-sgd"; }
const char *note(const char *epi, const char *split) {
  if (!launch_log_on()) return nullptr;
  snprintf(g_note_buf, sizeof g_note_buf, "%s%s%s", epi, split ? " " : "", split ? split : "");
  return g_note_buf;
}

bool pdl_enabled() {
  static int v = -1;
  if (v < 0) v = getenv("NF_NO_PDL") ? 0 : 1;
  return v == 1;
}

template <class... KArgs, class... Args>
cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  count_launch();
  log_launch(reinterpret_cast<const void *>(kern), grid, block, smem, g_note);
  g_note = nullptr;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

enum Cfg { CFG_L, CFG_M, CFG_S, CFG_T };

Cfg choose_cfg(int M, int N) {
  if (N <= 64) return CFG_S;
  if (M <= 64) return CFG_T;
  if (M >= 128 && N >= 128) return CFG_L;
  return CFG_M;
}

template <int BM, int BN, int BK, int TM, int TN, bool AK, bool BKM, class Epi>
cudaError_t launch_cfg(cudaStream_t st, GemmArgs g, const Epi &epi, const Workspace &ws) {
  const int tm = (g.M + BM - 1) / BM, tn = (g.N + BN - 1) / BN;
  const int64_t tiles = (int64_t)tm * tn;
  int splits = 1;
  if (tiles < 2 * kSMs && g.K >= 256) {
    splits = (int)std::min<int64_t>((2 * kSMs + tiles - 1) / tiles, 32);
    splits = std::min(splits, g.K / 128);
    while (splits > 1 && (size_t)splits * g.M * g.N > ws.partial_floats) --splits;
    splits = std::max(splits, 1);
  }
  int kchunk = (g.K + splits - 1) / splits;
  kchunk = (kchunk + BK - 1) / BK * BK;
  splits = std::max(1, (g.K + kchunk - 1) / kchunk);
  g.kchunk = splits > 1 ? kchunk : std::max(g.K, 1);
  g.partial = splits > 1 ? ws.partial : nullptr;
  dim3 grid(tn, tm, splits);
  g_note = note(epi_note(epi), splits > 1 ? "splitk-partial" : nullptr);
  cudaError_t e = launch_k(gemm_simt<BM, BN, BK, TM, TN, AK, BKM, Epi>, grid, dim3((BM / TM) * (BN / TN)), 0, st, g, epi);
  if (e != cudaSuccess) return e;
  if (splits > 1) {
    const int64_t MN = (int64_t)g.M * g.N;
    const int blocks = (int)std::min<int64_t>((MN + 255) / 256, 4 * kSMs);
    e = launch_k(splitk_epilogue<Epi>, dim3(blocks), dim3(256), 0, st, ws.partial, splits, g.M, g.N, epi);
    if (e != cudaSuccess) return e;
  }
  return cudaGetLastError();
}

// Warp-level tensor-core engine (gemm_hmma.cuh) for small contractions (<= 2 GFLOP: config 4's
// layers), opt-in NF_HMMA=1: parity-green, but config 4 ran 433 vs 149 us per TF32 step against
// the tcgen05 kernels (profiles/r02_hmma_gemm_experiment.txt)
bool tc_enabled();
bool hmma_engine(int M, int N, int K) {
  const char *e = getenv("NF_HMMA");
  if (!tc_enabled() || !e || atoi(e) == 0) return false;
  return M >= 16 && N >= 16 && K >= 64 && 2.0 * M * N * K <= 2.0e9;
}

template <bool AK, bool BKM, class Epi>
cudaError_t launch_hmma(cudaStream_t st, GemmArgs g, const Epi &epi, const Workspace &ws) {
  constexpr int BM = 64, BN = 64, BK = 32;
  const int tm = (g.M + BM - 1) / BM, tn = (g.N + BN - 1) / BN;
  const int64_t tiles = (int64_t)tm * tn;
  // split-K (fixed-order partials + splitk_epilogue) only under half a wave: the forward / delta
  // GEMMs of config 4 (128 tiles) run unsplit, its weight gradients (20 tiles, K = 2048) split
  int splits = 1;
  if (tiles < kSMs / 2 && g.K >= 256) {
    splits = (int)std::min<int64_t>(kSMs / tiles, g.K / 128);
    while (splits > 1 && (size_t)splits * g.M * g.N > ws.partial_floats) --splits;
    splits = std::max(splits, 1);
  }
  int kchunk = (g.K + splits - 1) / splits;
  kchunk = (kchunk + BK - 1) / BK * BK;
  splits = std::max(1, (g.K + kchunk - 1) / kchunk);
  g.kchunk = splits > 1 ? kchunk : std::max(g.K, 1);
  g.partial = splits > 1 ? ws.partial : nullptr;
  dim3 grid(tn, tm, splits);
  g_note = note(epi_note(epi), splits > 1 ? (ws.math == 1 ? "hmma1 splitk-partial" : "hmma3 splitk-partial")
                                          : (ws.math == 1 ? "hmma1" : "hmma3"));
  g_last_engine = ws.math == 1 ? ENGINE_HMMA1 : ENGINE_HMMA3;
  auto k1 = gemm_hmma<AK, BKM, 1, Epi>;
  auto k3 = gemm_hmma<AK, BKM, 3, Epi>;
  {
    cudaError_t e = set_max_smem(reinterpret_cast<const void *>(ws.math == 1 ? k1 : k3), hm::SMEM);
    if (e != cudaSuccess) return e;
  }
  // 16-B cp.async copies when every operand row starts 16-B aligned
  const int vec = (g.lda % 4 == 0 && g.ldb % 4 == 0 && (reinterpret_cast<uintptr_t>(g.A) & 15) == 0 &&
                   (reinterpret_cast<uintptr_t>(g.B) & 15) == 0) ? 1 : 0;
  cudaError_t e = ws.math == 1 ? launch_k(k1, grid, dim3(256), hm::SMEM, st, g, epi, vec)
                               : launch_k(k3, grid, dim3(256), hm::SMEM, st, g, epi, vec);
  if (e != cudaSuccess) return e;
  if (splits > 1) {
    const int64_t MN = (int64_t)g.M * g.N;
    const int blocks = (int)std::min<int64_t>((MN + 255) / 256, 4 * kSMs);
    e = launch_k(splitk_epilogue<Epi>, dim3(blocks), dim3(256), 0, st, ws.partial, splits, g.M, g.N, epi);
    if (e != cudaSuccess) return e;
  }
  return cudaGetLastError();
}

template <bool AK, bool BKM, class Epi>
cudaError_t run_gemm(cudaStream_t st, GemmArgs g, const Epi &epi, const Workspace &ws) {
  if (g.M <= 0 || g.N <= 0) return cudaSuccess;
  if (ws.math != 2 && hmma_engine(g.M, g.N, g.K)) return launch_hmma<AK, BKM>(st, g, epi, ws);
  g_last_engine = ENGINE_SIMT;
  switch (choose_cfg(g.M, g.N)) {
    case CFG_L: return launch_cfg<128, 128, 8, 8, 8, AK, BKM>(st, g, epi, ws);
    case CFG_S: return launch_cfg<128, 32, 16, 8, 2, AK, BKM>(st, g, epi, ws);
    case CFG_T: return launch_cfg<32, 128, 16, 2, 8, AK, BKM>(st, g, epi, ws);
    default: return launch_cfg<64, 64, 16, 4, 4, AK, BKM>(st, g, epi, ws);
  }
}

// ---------------------------------------------------------------------------
// tcgen05 path.  An operand is K-major ([rows][ld], K contiguous) or MN-major
// ([K][ld], M or N contiguous).  TMA needs 16-B aligned bases and row pitches.
struct TcOp {
  const float *p;
  int64_t ld;
  bool mn;
  const float *lo = nullptr;  // fp32 mode: tf32_lo of the operand, same layout (pre-split 3xTF32)
};

bool tc_enabled() {
  static int v = -1;
  if (v < 0) {
    const char *e = getenv("NF_DISABLE_TC");
    v = (e && atoi(e)) ? 0 : 1;
  }
  return v == 1;
}

bool tc_ok(const TcOp &o) { return (reinterpret_cast<uintptr_t>(o.p) & 15) == 0 && (o.ld * 4) % 16 == 0; }

// The tensor-core path is used for contractions whose three extents are all >= 64
// (the output layer's 10-wide GEMMs stay on the SIMT kernels).
bool use_tc(int M, int N, int K, const TcOp &a, const TcOp &b) {
  return tc_enabled() && M >= 64 && N >= 64 && K >= 64 && tc_ok(a) && tc_ok(b) && !hmma_engine(M, N, K);
}

bool make_map(CUtensorMap *m, const TcOp &o, int rows, int K, int box_rows) {
  if (o.mn)  // [K][rows] with rows contiguous: box {32 mn, 32 k}
    return encode_tmap_2d_f32(m, o.p, (uint64_t)rows, (uint64_t)K, (uint64_t)o.ld * 4, 32, tc::BK,
                              CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
  return encode_tmap_2d_f32(m, o.p, (uint64_t)K, (uint64_t)rows, (uint64_t)o.ld * 4, tc::BK, (uint32_t)box_rows,
                            CU_TENSOR_MAP_SWIZZLE_128B);
}

template <int BN, bool AMN, bool BMN, int SPLIT, class Epi, int MAXST = 6, int EW = tc::kEpiWarps>
cudaError_t launch_tc(cudaStream_t st, int M, int N, int K, const TcOp &a, const TcOp &b, const Epi &epi,
                      const Workspace &ws, int force_splits = 0) {
  using C = tc::Cfg<BN, SPLIT, MAXST, EW>;
  auto kern = tc::gemm_tc_kernel<BN, AMN, BMN, SPLIT, Epi, MAXST, EW>;
  {
    cudaError_t e = set_max_smem(reinterpret_cast<const void *>(kern), C::SMEM);
    if (e != cudaSuccess) return e;
  }
  CUtensorMap ta, tb, tal, tbl;
  if (!make_map(&ta, a, M, K, tc::BM) || !make_map(&tb, b, N, K, BN)) return cudaErrorInvalidValue;
  // pre-split 3xTF32: both operands' lo parts written by their producers -> no in-smem splitting
  static const bool presplit = getenv("NF_PRESPLIT") == nullptr || atoi(getenv("NF_PRESPLIT")) != 0;
  const bool pre = SPLIT == 3 && presplit && a.lo && b.lo;
  memset(&tal, 0, sizeof tal);
  memset(&tbl, 0, sizeof tbl);
  if (pre) {
    TcOp al = a, bl = b;
    al.p = a.lo;
    bl.p = b.lo;
    if (!make_map(&tal, al, M, K, tc::BM) || !make_map(&tbl, bl, N, K, BN)) return cudaErrorInvalidValue;
  }
  const int tm = (M + tc::BM - 1) / tc::BM, tn = (N + BN - 1) / BN;
  const int tiles = tm * tn;
  const int nkb = (K + tc::BK - 1) / tc::BK;
  // An additive epilogue (the SGD update W -= scale G) takes its split-K terms straight into W
  // as L2 reductions (no partial buffer, no second kernel; summation order = arrival order,
  // reading R12); NF_SPLITK_DETERMINISTIC=1 keeps the fixed-order partial path.
  bool red = false;
  if constexpr (Epi::kRed) {
    static const bool det = getenv("NF_SPLITK_DETERMINISTIC") != nullptr;
    // (nf_grad's store-only epilogue takes forced split-K terms the same way, into its zeroed
    // output: the forced splits exist for accuracy, see run_tc)
    red = !det && (!epi.store_only || force_splits > 1);
  }
  // Split-K when under half a wave and K >= 512; for an epilogue that is not additive (needs
  // the partials + a second kernel) only under a quarter wave (c4's layer 1, 64 tiles of
  // K = 784: the split + splitk_epilogue cost more than they saved, 158.9 -> 155.2 us/step)
  int splits = 1;
  if ((red ? 2 : 4) * tiles < kSMs && nkb >= 16) {
    splits = std::min(kSMs / tiles, nkb / 4);  // one wave
    while (!red && splits > 1 && (size_t)splits * M * N > ws.partial_floats) --splits;
    splits = std::max(splits, 1);
  }
  if (force_splits > 1 && red) splits = std::max(splits, std::min(force_splits, nkb));
  if constexpr (Epi::kHasT) {
    if (epi.T) splits = 1;  // the transposed copy is written by the tile epilogue (no split-K partials)
  }
  const int kbper = (nkb + splits - 1) / splits;
  splits = (nkb + kbper - 1) / kbper;  // no empty K-chunk
  red = red && splits > 1;
  if constexpr (Epi::kRed) {
    if (red && epi.store_only) {  // the terms are added into the (zeroed) tendency block
      cudaError_t e = cudaMemsetAsync(epi.W, 0, (size_t)M * epi.ldw * sizeof(float), st);
      if (e != cudaSuccess) return e;
    }
  }
  tc::TileArgs g{M, N, K, kbper * tc::BK, (splits > 1 && !red) ? ws.partial : nullptr, red ? 1 : 0, pre ? 1 : 0};
  g_note = note(epi_note(epi), red ? (pre ? "splitk-red presplit" : "splitk-red")
                                    : (splits > 1 ? (pre ? "splitk-partial presplit" : "splitk-partial")
                                                  : (pre ? "presplit" : nullptr)));
  cudaError_t e = launch_k(kern, dim3(tn, tm, splits), dim3(C::THREADS), C::SMEM, st, ta, tb, g, epi, tal, tbl);
  if (e != cudaSuccess) return e;
  if constexpr (Epi::kRed) {  // split-K terms went into W in L2: the TF32 / lo shadow of W from the sum --
    if (red && (epi.Wt || epi.Wlo)) {  // by the caller in one pass after the step when it asked to (ws.red_flag)
      if (ws.red_flag) *ws.red_flag = true;
      else if (epi.Wlo) return split_rn(st, epi.W, epi.Wt, epi.Wlo, (int64_t)M * epi.ldw);
      else return round_tf32(st, epi.W, epi.Wt, (int64_t)M * epi.ldw);
    }
  }
  if (splits > 1 && !red) {
    const int64_t MN = (int64_t)M * N;
    const int blocks = (int)std::min<int64_t>((MN + 255) / 256, 4 * kSMs);
    e = launch_k(splitk_epilogue<Epi>, dim3(blocks), dim3(256), 0, st, ws.partial, splits, M, N, epi);
    if (e != cudaSuccess) return e;
  }
  return cudaGetLastError();
}

// Persistent 1xTF32 kernel (double-buffered TMEM accumulators, epilogue overlapped with the
// next tile's main loop): for GEMMs of more than one wave of 128x256 tiles.
template <bool AMN, bool BMN, class Epi>
cudaError_t launch_tc_persistent(cudaStream_t st, int M, int N, int K, const TcOp &a, const TcOp &b, const Epi &epi) {
  using C = tc::Cfg<256, 1>;
  auto kern = tc::gemm_tc_persistent<256, AMN, BMN, Epi>;
  {
    cudaError_t e = set_max_smem(reinterpret_cast<const void *>(kern), C::SMEM);
    if (e != cudaSuccess) return e;
  }
  CUtensorMap ta, tb;
  if (!make_map(&ta, a, M, K, tc::BM) || !make_map(&tb, b, N, K, 256)) return cudaErrorInvalidValue;
  const int tiles = ((M + tc::BM - 1) / tc::BM) * ((N + 255) / 256);
  g_note = note(epi_note(epi), nullptr);
  return launch_k(kern, dim3(std::min(tiles, kSMs)), dim3(tc::kThreads), C::SMEM, st, ta, tb, M, N, K, epi);
}

template <bool AMN, bool BMN, class Epi>
cudaError_t run_tc(cudaStream_t st, int M, int N, int K, const TcOp &a, const TcOp &b, const Epi &epi,
                   const Workspace &ws) {
  // Tile width: the widest BN whose tile count still fills the GPU (>= ~0.8 of the SMs);
  // otherwise BN = 64 and split-K over the reduction dimension.
  const int tm = (M + tc::BM - 1) / tc::BM;
  auto tiles = [&](int bn) { return tm * ((N + bn - 1) / bn); };
  const int fill = kSMs * 4 / 5;
  if (ws.math == 1) {
    g_last_engine = ENGINE_TC1;
    if (N > 128 && tiles(256) > kSMs && getenv("NF_TC_NO_PERSISTENT") == nullptr)
      return launch_tc_persistent<AMN, BMN>(st, M, N, K, a, b, epi);
    static const bool dual = getenv("NF_TC_DUAL") != nullptr;  // experiment: 2 CTAs per SM
    if (dual && N > 64 && tiles(128) >= fill && tiles(128) <= 2 * kSMs)
      return launch_tc<128, AMN, BMN, 1, Epi, 2>(st, M, N, K, a, b, epi, ws);
    // one wave of wide tiles: the epilogue is exposed (no next tile to overlap), 16 epilogue
    // warps (c3: 179 -> 171 us per step; the persistent and narrow-tile kernels keep 8)
    static const int ew = getenv("NF_TC_EW8") ? 8 : 16;
    if (N > 128 && tiles(256) >= fill)
      return ew == 16 ? launch_tc<256, AMN, BMN, 1, Epi, 6, 16>(st, M, N, K, a, b, epi, ws)
                      : launch_tc<256, AMN, BMN, 1>(st, M, N, K, a, b, epi, ws);
    // under one wave of 128x256 tiles but deep (the c3 weight gradients, 1024 x 1024 x 4096):
    // keep the wide tile and split K so that tiles x splits fills the GPU in one wave
    {
      const int nkb = (K + tc::BK - 1) / tc::BK;
      const int sp = std::min(kSMs / tiles(256), nkb / 8);
      if (N > 128 && sp >= 2 && tiles(256) * sp >= fill) return launch_tc<256, AMN, BMN, 1>(st, M, N, K, a, b, epi, ws);
    }
    if (N > 64 && tiles(128) >= fill) return launch_tc<128, AMN, BMN, 1>(st, M, N, K, a, b, epi, ws);
    static const bool bn32 = getenv("NF_TC_BN32") != nullptr;  // experiment: narrow tiles, more CTAs
    if (bn32 && tiles(64) < fill && tiles(32) <= 2 * kSMs) return launch_tc<32, AMN, BMN, 1>(st, M, N, K, a, b, epi, ws);
    return launch_tc<64, AMN, BMN, 1>(st, M, N, K, a, b, epi, ws);
  }
  g_last_engine = ENGINE_TC3;
  // 128 x 256 tiles where they fill the GPU leave room for only NACC = 2 accumulators; the
  // truncating accumulation then meets the 1e-4 bar for K <= 1024 (c3 forward / backward: fp32
  // step 366 -> 327 us) but not at c5's K = 4096 (1.9e-4), which keeps BN = 128 unless
  // NF_TC3_BN256=1 (experiment: c5 fp32 31.2 -> 27.2 ms); NF_TC3_NO_SHALLOW256=1 reverts
  static const bool bn256 = getenv("NF_TC3_BN256") != nullptr;
  static const bool shallow256 = getenv("NF_TC3_NO_SHALLOW256") == nullptr;
  if ((bn256 || (shallow256 && K <= 1024)) && N > 128 && tiles(256) >= fill)
    return launch_tc<256, AMN, BMN, 3>(st, M, N, K, a, b, epi, ws);
  if constexpr (Epi::kRed) {  // experiment: deep additive GEMMs in wide tiles, K split so each
    // of the 2 accumulators sums no more than the 128-wide tiles' 4 do over the whole K
    // (only with split-K terms reduced into W: without them -- NF_SPLITK_DETERMINISTIC -- the two
    // accumulators would sum all of K = 16384, which misses the 1e-4 bar)
    static const bool deep256 = getenv("NF_TC3_DEEP256") != nullptr && getenv("NF_SPLITK_DETERMINISTIC") == nullptr;
    if (deep256 && !epi.store_only && N > 128 && tiles(256) >= fill && K > 1024)
      return launch_tc<256, AMN, BMN, 3>(st, M, N, K, a, b, epi, ws, 2);
  }
  // Deep reductions (the c5 weight gradients, K = B = 16384): the tensor core's truncating fp32
  // accumulation errs in proportion to the K-steps one accumulator sums (4 accumulators x 512
  // K-steps: 1.1e-4 > the 1e-4 bar at c5, tests/test_fullsize_gpu.py), so an additive epilogue
  // splits K into chunks of <= NF_TC3_KCHUNK (default 4096) whose terms are reduced into W in L2
  int force = 1;
  if constexpr (Epi::kRed) {
    static const int kchunk = getenv("NF_TC3_KCHUNK") ? atoi(getenv("NF_TC3_KCHUNK")) : 4096;
    if (kchunk > 0 && K > kchunk) force = (K + kchunk - 1) / kchunk;
  }
  if (N > 64 && tiles(128) >= fill) return launch_tc<128, AMN, BMN, 3>(st, M, N, K, a, b, epi, ws, force);
  // under a wave but deep with an additive update (the c3 weight gradients, 1024 x 1024 x
  // 4096): 128 x 256 tiles split 4-way over K (L2 reductions into W) instead of 128 x 64 tiles
  // over the whole K -- 2.5x fewer hi/lo conversions and operand bytes per flop (c3 fp32 step
  // 445 -> 366 us; NF_TC3_NARROW=1 restores BN = 64)
  if constexpr (Epi::kRed) {
    static const bool narrow = getenv("NF_TC3_NARROW") != nullptr;
    if (!narrow && !epi.store_only && N > 128 && 4 * tiles(256) >= fill)
      return launch_tc<256, AMN, BMN, 3>(st, M, N, K, a, b, epi, ws);
  }
  return launch_tc<64, AMN, BMN, 3>(st, M, N, K, a, b, epi, ws);
}

// Bias tendency g[i] = sum_r D[r][i] over n rows (the ones-column of the SIMT path),
// row chunks summed in a fixed order, then the same EpiGrad bias element update.
__global__ void __launch_bounds__(256)
colsum_partial(const float *__restrict__ D, int64_t rows, int cols, int chunk, float *__restrict__ part,
               float *__restrict__ bias, float scale) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  const int c = blockIdx.x * 256 + threadIdx.x;
  if (c >= cols) return;
  const int64_t r0 = (int64_t)blockIdx.y * chunk, r1 = min(rows, r0 + chunk);
  float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
  int64_t r = r0;
  for (; r + 16 <= r1; r += 16) {  // 16 independent loads in flight per thread
    float v[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) v[u] = D[(r + u) * cols + c];
#pragma unroll
    for (int u = 0; u < 16; u += 4) { s0 += v[u]; s1 += v[u + 1]; s2 += v[u + 2]; s3 += v[u + 3]; }
  }
  for (; r < r1; ++r) s0 += D[r * cols + c];
  const float s = (s0 + s1) + (s2 + s3);
  if (bias)  // the update is additive: this chunk's term goes straight into b (L2 reduction, R12)
    asm volatile("red.global.add.f32 [%0], %1;" ::"l"(bias + c), "f"(-scale * s) : "memory");
  else
    part[(int64_t)blockIdx.y * cols + c] = s;
}

__global__ void __launch_bounds__(256)
colsum_final(const float *__restrict__ part, int nchunks, int cols, EpiGrad epi) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  // 32 columns per block; warp w sums the chunks z = w (mod 8), then warp 0 adds the eight
  // warp sums in order w = 0..7 (fixed order: deterministic)
  __shared__ float red[8][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + lane;
  float s = 0.f;
  if (c < cols) {
#pragma unroll 4
    for (int z = w; z < nchunks; z += 8) s += part[(int64_t)z * cols + c];
  }
  red[w][lane] = s;
  __syncthreads();
  if (w == 0 && c < cols) {
    float t = red[0][lane];
#pragma unroll
    for (int i = 1; i < 8; ++i) t += red[i][lane];
    epi(c, epi.nreal, t);  // column nreal of the [M][N+1] gradient = the bias
  }
}

cudaError_t bias_grad(cudaStream_t st, const float *D, int64_t rows, int cols, const EpiGrad &epi,
                      float *part, size_t part_floats) {
  static const bool det = getenv("NF_SPLITK_DETERMINISTIC") != nullptr;
  const int cblocks = (cols + 255) / 256;
  if (!epi.store_only && !det) {
    // SGD update: one kernel, chunk sums reduced into b in L2.  Chunks of >= 64 rows: every
    // b[c] receives one reduction per chunk, and more of them contend for the same L2 line
    // (16-row chunks made the c4 step 164 -> 191 us)
    const int nch = (int)std::min<int64_t>((rows + 63) / 64, 256);
    const int ch = (int)((rows + nch - 1) / nch);
    return launch_k(colsum_partial, dim3(cblocks, (int)((rows + ch - 1) / ch)), dim3(256), 0, st, D, rows, cols, ch,
                    (float *)nullptr, epi.b, epi.scale);
  }
  // ~4 column blocks x 64+ row chunks of <= 64 rows: enough CTAs to stream D at HBM rate
  int nchunks = (int)std::min<int64_t>((rows + 63) / 64, 256);
  while (nchunks > 1 && (size_t)nchunks * cols > part_floats) --nchunks;
  const int chunk = (int)((rows + nchunks - 1) / nchunks);
  const dim3 grid(cblocks, nchunks);
  cudaError_t e = launch_k(colsum_partial, grid, dim3(256), 0, st, D, rows, cols, chunk, part, (float *)nullptr,
                           0.0f);
  if (e != cudaSuccess) return e;
  return launch_k(colsum_final, dim3((cols + 31) / 32), dim3(256), 0, st, (const float *)part, nchunks, cols, epi);
}

// ---------------------------------------------------------------------------
// Narrow output-layer contractions (the 10-wide last layer of configs 3 and 4): one
// extent <= 32, memory-bound on the wide operand.  Dedicated kernels instead of tiles.

// K1 with N <= 32: Z[m][o] = sum_k A[m][k] W[o][k] (+ bias/activation in epi).  One warp per
// row; W [N][K] staged in shared memory; lane-strided K slices, butterfly reductions.
template <int NMAX, bool STAGE>
__global__ void __launch_bounds__(256)
fwd_smalln(const float *__restrict__ A, const float *__restrict__ W, int M, int N, int K, EpiFwd epi) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  extern __shared__ float ws_[];
  const float *wsrc = STAGE ? ws_ : W;   // !STAGE: W read through L1 (16-B aligned W only)
  if (!STAGE) {
  } else if ((reinterpret_cast<uintptr_t>(W) & 15) == 0) {  // N*K % 4 == 0 (K % 4 == 0): float4 staging,
    const int nk4 = N * K / 4;                       // several loads in flight per thread
#pragma unroll 4
    for (int i = threadIdx.x; i < nk4; i += blockDim.x)
      reinterpret_cast<float4 *>(ws_)[i] = __ldg(reinterpret_cast<const float4 *>(W) + i);
  } else {
#pragma unroll 8
    for (int i = threadIdx.x; i < N * K; i += blockDim.x) ws_[i] = __ldg(W + i);
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int m = blockIdx.x * 8 + warp; m < M; m += gridDim.x * 8) {
    const float *a = A + (int64_t)m * K;
    float acc[NMAX];
#pragma unroll
    for (int o = 0; o < NMAX; ++o) acc[o] = 0.0f;
#pragma unroll 4
    for (int k = lane * 4; k < K; k += 128) {
      const float4 av = *reinterpret_cast<const float4 *>(a + k);
#pragma unroll
      for (int o = 0; o < NMAX; ++o) {
        if (o < N) {
          const float4 wv = STAGE ? *reinterpret_cast<const float4 *>(wsrc + o * K + k)
                                  : __ldg(reinterpret_cast<const float4 *>(wsrc + o * K + k));
          acc[o] = fmaf(av.x, wv.x, fmaf(av.y, wv.y, fmaf(av.z, wv.z, fmaf(av.w, wv.w, acc[o]))));
        }
      }
    }
#pragma unroll
    for (int o = 0; o < NMAX; ++o)
      if (o < N) acc[o] = warp_sum(acc[o]);
    float z = 0.0f;
#pragma unroll
    for (int o = 0; o < NMAX; ++o)
      if (o == lane) z = acc[o];
    if (lane < N) epi(m, lane, z);
  }
}

// K3 with K <= 32: SD[m][n] = sigma'[m][n] * sum_k D[m][k] W[k][n].  A thread owns 4 columns
// (W column slice in registers) and walks TM rows; S read and written once, float4.
template <int KMAX>
__global__ void __launch_bounds__(128)
bwd_smallk(const float *__restrict__ D, const float *__restrict__ W, int M, int N, int K, int TM, EpiBwd epi) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  const int n = (blockIdx.x * 128 + threadIdx.x) * 4;
  if (n >= N) return;
  float4 w[KMAX];
#pragma unroll
  for (int k = 0; k < KMAX; ++k)
    w[k] = k < K ? *reinterpret_cast<const float4 *>(W + (int64_t)k * N + n) : make_float4(0.f, 0.f, 0.f, 0.f);
  const int m0 = blockIdx.y * TM, m1 = min(M, m0 + TM);
  for (int mb = m0; mb < m1; mb += 4) {  // 4 rows per pass: their sigma' loads issued together
    float4 sv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (mb + u < m1) sv[u] = *reinterpret_cast<const float4 *>(epi.SD + (int64_t)(mb + u) * epi.ld + n);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int m = mb + u;
      if (m >= m1) break;
      const float *d = D + (int64_t)m * K;
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int k = 0; k < KMAX; ++k) {
        if (k < K) {
          const float dk = __ldg(d + k);
          acc.x = fmaf(dk, w[k].x, acc.x);
          acc.y = fmaf(dk, w[k].y, acc.y);
          acc.z = fmaf(dk, w[k].z, acc.z);
          acc.w = fmaf(dk, w[k].w, acc.w);
        }
      }
      float4 dv = make_float4(acc.x * sv[u].x, acc.y * sv[u].y, acc.z * sv[u].z, acc.w * sv[u].w);
      if (epi.rnd) dv = make_float4(tf32_rn(dv.x), tf32_rn(dv.y), tf32_rn(dv.z), tf32_rn(dv.w));
      *reinterpret_cast<float4 *>(epi.SD + (int64_t)m * epi.ld + n) = dv;
      if (epi.lo)
        *reinterpret_cast<float4 *>(epi.lo + (int64_t)m * epi.ld + n) =
            make_float4(tf32_lo(dv.x), tf32_lo(dv.y), tf32_lo(dv.z), tf32_lo(dv.w));
    }
  }
}

// K4 with M <= 32: G[i][n] = sum_b D[b][i] A[b][n] for n < N, and column n = N with A = 1
// (the bias tendency).  Row chunks -> partials [R][M][N+1], summed in chunk order.
template <int MMAX>
__global__ void __launch_bounds__(128)
grad_smallm_partial(const float *__restrict__ D, const float *__restrict__ A, int M, int N, int K, int chunk,
                    float *__restrict__ part) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  __shared__ __align__(16) float dsm[128 * MMAX];
  const int n = blockIdx.x * 128 + threadIdx.x;
  const int b0 = blockIdx.y * chunk, b1 = min(K, b0 + chunk);
  float acc[MMAX];
#pragma unroll
  for (int i = 0; i < MMAX; ++i) acc[i] = 0.0f;
  for (int bb = b0; bb < b1; bb += 128) {
    const int nb = min(128, b1 - bb);
    __syncthreads();
    for (int t = threadIdx.x; t < nb * M; t += 128) dsm[(t / M) * MMAX + t % M] = D[(int64_t)(bb + t / M) * M + t % M];
    __syncthreads();
    if (n <= N) {
      int r = 0;
      for (; r + 8 <= nb; r += 8) {  // 8 independent row loads in flight
        float a[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) a[u] = n < N ? __ldg(A + (int64_t)(bb + r + u) * N + n) : 1.0f;
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
          for (int i4 = 0; i4 < MMAX; i4 += 4) {
            if (i4 < M) {  // one 16-B shared load per 4 outputs (broadcast)
              const float4 d4 = *reinterpret_cast<const float4 *>(dsm + (r + u) * MMAX + i4);
              acc[i4] = fmaf(d4.x, a[u], acc[i4]);
              if (i4 + 1 < M) acc[i4 + 1] = fmaf(d4.y, a[u], acc[i4 + 1]);
              if (i4 + 2 < M) acc[i4 + 2] = fmaf(d4.z, a[u], acc[i4 + 2]);
              if (i4 + 3 < M) acc[i4 + 3] = fmaf(d4.w, a[u], acc[i4 + 3]);
            }
          }
      }
      for (; r < nb; ++r) {
        const float a = n < N ? __ldg(A + (int64_t)(bb + r) * N + n) : 1.0f;
#pragma unroll
        for (int i = 0; i < MMAX; ++i)
          if (i < M) acc[i] = fmaf(dsm[r * MMAX + i], a, acc[i]);
      }
    }
  }
  if (n <= N) {
#pragma unroll
    for (int i = 0; i < MMAX; ++i)
      if (i < M) part[((int64_t)blockIdx.y * M + i) * (N + 1) + n] = acc[i];
  }
}

// thread t sums the R partials of output t in order r = 0..R-1, four independent loads in
// flight (deterministic)
__global__ void __launch_bounds__(256)
grad_smallm_final(const float *__restrict__ part, int R, int M, int N, EpiGrad epi,
                  const float *__restrict__ lpart = nullptr, float lscale = 0.0f, float *__restrict__ step_loss = nullptr) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  if (step_loss && blockIdx.x == 0 && threadIdx.x < 32) {  // the step's mean cost from the fused
    float l = 0.0f;                                        // output layer's per-block partials
    for (int r = threadIdx.x; r < R; r += 32) l += lpart[r];  // (fixed order)
    l = warp_sum(l);
    if (threadIdx.x == 0) *step_loss = l * lscale;
  }
  // 32 outputs per block; warp w sums the partials r = w (mod 8), warp 0 adds the eight warp
  // sums in order (deterministic)
  __shared__ float red[8][33];
  const int64_t MN = (int64_t)M * (N + 1);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t t = (int64_t)blockIdx.x * 32 + lane;
  float s = 0.0f;
  if (t < MN) {
#pragma unroll 4
    for (int r = w; r < R; r += 8) s += part[r * MN + t];
  }
  red[w][lane] = s;
  __syncthreads();
  if (w == 0 && t < MN) {
    float u = red[0][lane];
#pragma unroll
    for (int i = 1; i < 8; ++i) u += red[i][lane];
    epi((int)(t / (N + 1)), (int)(t % (N + 1)), u);
  }
}

// The narrow output layer of a training step (n_L <= 16 after a wide hidden layer: the 10-wide
// last layer of configs 3 and 4) in ONE pass over its wide operands, instead of fwd_smalln +
// bwd_smallk + grad_smallm_partial:
//   K1+K2 (layer L):  z = A_{L-1} W_L^T + b_L, a = sigma(z), delta_L = (a - y) sigma'(z)
//                      (S:150), a and delta_L stashed for the loss and nf_grad;
//   K3 (layer L-1):   delta_{L-1} = (delta_L W_L) .* sigma'(Z_{L-1}), in place of S_{L-1}
//                      (P:409-411), reading W_L before it is updated;
//   K4 partials:       G_L = delta_L^T [A_{L-1} | 1] over the block's rows -> part[blk][o][0..H]
//                      (the layout grad_smallm_final sums in fixed order, then updates W_L, b_L).
// Phase 1: one warp per row, the A row in registers (HMAX4 float4 slots per lane), W_L staged
// in shared memory.  Phase 2: thread per 4 columns over the block's rows (A re-read from L2).
template <int NMAX, int HMAX4>
__global__ void __launch_bounds__(256)
out_layer_train(const float *__restrict__ A, float *__restrict__ S, const float *__restrict__ W,
                const float *__restrict__ bias, const float *__restrict__ Y, float *__restrict__ AL,
                float *__restrict__ DL, int n, int H, int nL, int act, int rows_per_block, float *__restrict__ part,
                float *__restrict__ lpart, int rnd, float *__restrict__ Dlo) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  __shared__ float lred[8];
  float lacc = 0.0f;  // sum of (a - y)^2 over this warp's rows: the block's cost partial
  extern __shared__ float4 sm4_[];
  float *ws_ = reinterpret_cast<float *>(sm4_);          // [nL][H]
  float *dsm = ws_ + nL * H;                             // [rows_per_block][NMAX] delta_L
  {
    const int nk4 = nL * H / 4;
#pragma unroll 4
    for (int i = threadIdx.x; i < nk4; i += blockDim.x) sm4_[i] = __ldg(reinterpret_cast<const float4 *>(W) + i);
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r0 = blockIdx.x * rows_per_block, r1 = min(n, r0 + rows_per_block);
  const int H4 = H / 4;
  for (int m = r0 + warp; m < r1; m += 8) {
    float4 av[HMAX4];
    const float4 *arow = reinterpret_cast<const float4 *>(A + (int64_t)m * H);
#pragma unroll
    for (int i = 0; i < HMAX4; ++i)
      if (lane + 32 * i < H4) av[i] = __ldg(arow + lane + 32 * i);
    float acc[NMAX];
#pragma unroll
    for (int o = 0; o < NMAX; ++o) {
      acc[o] = 0.0f;
      if (o < nL) {
        float2 p0 = make_float2(0.f, 0.f), p1 = make_float2(0.f, 0.f);  // packed FFMA2 over k pairs
#pragma unroll
        for (int i = 0; i < HMAX4; ++i) {
          if (lane + 32 * i < H4) {
            const float4 w = reinterpret_cast<const float4 *>(ws_ + o * H)[lane + 32 * i];
            ffma2v(p0, make_float2(av[i].x, av[i].y), make_float2(w.x, w.y));
            ffma2v(p1, make_float2(av[i].z, av[i].w), make_float2(w.z, w.w));
          }
        }
        acc[o] = warp_sum((p0.x + p0.y) + (p1.x + p1.y));
      }
    }
    float dl = 0.0f;  // lane o < nL: delta_L[m][o]
#pragma unroll
    for (int o = 0; o < NMAX; ++o)
      if (o == lane && o < nL) {
        float a, sg;
        act_fwd(act, acc[o] + bias[o], a, sg);
        const float diff = a - Y[(int64_t)m * nL + o];
        dl = diff * sg;
        lacc = fmaf(diff, diff, lacc);
        AL[(int64_t)m * nL + o] = a;
        DL[(int64_t)m * nL + o] = dl;
      }
    if (lane < NMAX) dsm[(m - r0) * NMAX + lane] = dl;
    float d[NMAX];
#pragma unroll
    for (int o = 0; o < NMAX; ++o) d[o] = __shfl_sync(0xffffffffu, dl, o);
    float4 *srow = reinterpret_cast<float4 *>(S + (int64_t)m * H);
#pragma unroll
    for (int i = 0; i < HMAX4; ++i) {
      const int k4 = lane + 32 * i;
      if (k4 < H4) {
        const float4 sg = srow[k4];
        float2 t0 = make_float2(0.f, 0.f), t1 = make_float2(0.f, 0.f);
#pragma unroll
        for (int o = 0; o < NMAX; ++o) {
          if (o < nL) {
            const float4 w = reinterpret_cast<const float4 *>(ws_ + o * H)[k4];
            ffma2(t0, d[o], make_float2(w.x, w.y));
            ffma2(t1, d[o], make_float2(w.z, w.w));
          }
        }
        float4 d = make_float4(t0.x * sg.x, t0.y * sg.y, t1.x * sg.z, t1.y * sg.w);
        if (rnd) d = make_float4(tf32_rn(d.x), tf32_rn(d.y), tf32_rn(d.z), tf32_rn(d.w));  // a TC operand next
        srow[k4] = d;
        if (Dlo)  // fp32 mode: its lo part for pre-split 3xTF32 consumers
          reinterpret_cast<float4 *>(Dlo + (int64_t)m * H)[k4] = make_float4(tf32_lo(d.x), tf32_lo(d.y), tf32_lo(d.z), tf32_lo(d.w));
      }
    }
  }
  lacc = warp_sum(lacc);
  if (lane == 0) lred[warp] = lacc;
  __syncthreads();
  if (threadIdx.x == 0) {
    float l = 0.0f;
    for (int i = 0; i < 8; ++i) l += lred[i];
    lpart[blockIdx.x] = l;
  }
  // phase 2: partial tendencies of the block's rows, column group c (4 columns; c == H4: bias)
  float *pb = part + (int64_t)blockIdx.x * nL * (H + 1);
  for (int c = threadIdx.x; c <= H4; c += blockDim.x) {
    float2 g[NMAX][2];  // columns (4c, 4c+1), (4c+2, 4c+3) per output: packed FFMA2
#pragma unroll
    for (int o = 0; o < NMAX; ++o) g[o][0] = g[o][1] = make_float2(0.f, 0.f);
#pragma unroll 4
    for (int m = r0; m < r1; ++m) {  // (unrolled: the rows' A loads overlap)
      const float4 a = c < H4 ? __ldg(reinterpret_cast<const float4 *>(A + (int64_t)m * H) + c)
                              : make_float4(1.f, 0.f, 0.f, 0.f);
      const float *dr = dsm + (m - r0) * NMAX;
#pragma unroll
      for (int o = 0; o < NMAX; ++o) {
        if (o < nL) {
          const float dv = dr[o];
          ffma2(g[o][0], dv, make_float2(a.x, a.y));
          ffma2(g[o][1], dv, make_float2(a.z, a.w));
        }
      }
    }
#pragma unroll
    for (int o = 0; o < NMAX; ++o) {
      if (o < nL) {
        float *p = pb + (int64_t)o * (H + 1) + 4 * c;
        if (c < H4) { p[0] = g[o][0].x; p[1] = g[o][0].y; p[2] = g[o][1].x; p[3] = g[o][1].y; }
        else p[0] = g[o][0].x;  // bias column H
      }
    }
  }
}

// Butterfly reduce-scatter of N per-lane values over the lanes OFF, OFF/2, .., 1: after it lane
// l holds, in v[0], the warp sum of value index (l mod N) (N = 2 * OFF).  N - 1 shuffles instead of
// N * 5 for N separate warp_sums.
template <int N>
__device__ __forceinline__ void warp_reduce_scatter(float (&v)[32], int lane) {
  if constexpr (N >= 2) {
    constexpr int H = N / 2;
    const bool up = (lane & H) != 0;
#pragma unroll
    for (int i = 0; i < H; ++i) {
      const float send = up ? v[i] : v[i + H];
      const float keep = up ? v[i + H] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, H);
    }
    warp_reduce_scatter<H>(v, lane);
  }
}

// The narrow output layer of a training step, register-resident form (hidden width H <= 1024,
// H % 128 == 0; the same three results as out_layer_train above, same part / lpart layout):
// thread = one float4 column group of the hidden layer, W_L's columns and the K4 partial sums
// of those columns held in registers for the whole kernel, so the 40 KB of W_L are never
// re-read per row (the shared-memory bandwidth that bound out_layer_train).  Threads form
// RG = 256 / (H/4) row groups; each iteration a group takes RC = 2 rows:
//   z partials over the thread's 4 columns for 2 rows x 16 outputs -> one 32-value butterfly
//   reduce-scatter per warp (31 shuffles) -> per-warp sums in shared memory -> the group's
//   first warp finishes z, sigma, delta_L, the cost (lane = (row, output)) -> delta_L in shared
//   memory -> every thread: delta_{L-1} of its columns (S read once, written once) and the
//   K4 partials (the A values still in registers).  The next rows' A and S are loaded while
//   the current ones are processed.
constexpr int kOutStages = 8;  // ring stages of out_layer_train_rg (16 KB each: 2 x 2048 floats)
template <int NMAX>
__global__ void __launch_bounds__(256, 1)
out_layer_train_rg(const float *__restrict__ A, float *__restrict__ S, const float *__restrict__ W,
                   const float *__restrict__ bias, const float *__restrict__ Y, float *__restrict__ AL,
                   float *__restrict__ DL, int n, int H, int nL, int act, int rows_per_block, float *__restrict__ part,
                   float *__restrict__ lpart, int rnd, float *__restrict__ Dlo) {
  constexpr int RC = 2;  // rows per group per iteration (RC x 16 = 32 butterfly values)
  ptx::pdl_trigger();
  ptx::pdl_wait();
  __shared__ float red[8][32];      // per-warp butterfly results
  __shared__ float dsm[8][RC][16];  // delta_L of the iteration's rows, per group
  __shared__ float bsm[8][32];      // per-group bias / cost partials
  __shared__ __align__(8) uint64_t full[kOutStages];
  extern __shared__ float4 sm4_[];  // ring: kOutStages x (A rows | S rows), then the groups' K4 partials
  const int H4 = H >> 2;
  const int GS = H4, GW = GS >> 5, RG = 256 / GS;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int grp = tid / GS, gt = tid - grp * GS, gw = gt >> 5;
  const bool act_t = grp < RG;
  const int r0 = blockIdx.x * rows_per_block, r1 = min(n, r0 + rows_per_block);
  const int per_it = RG * RC;             // rows per iteration, contiguous in A and S
  const int stage_f = 2 * per_it * H;     // floats per ring stage
  const int niter = r1 > r0 ? (r1 - r0 + per_it - 1) / per_it : 0;
  float *ring = reinterpret_cast<float *>(sm4_);
  // a stage holds the rows [m0, m0 + nr) of A and of S, copied by two bulk copies
  auto issue = [&](int it) {
    if (it >= niter) return;
    const int st = it % kOutStages, m0 = r0 + it * per_it, nr = min(per_it, r1 - m0);
    const uint32_t bytes = (uint32_t)nr * H * 4;
    ptx::mbar_arrive_expect_tx(&full[st], 2 * bytes);
    ptx::bulk_g2s(ring + (int64_t)st * stage_f, A + (int64_t)m0 * H, bytes, &full[st]);
    ptx::bulk_g2s(ring + (int64_t)st * stage_f + per_it * H, S + (int64_t)m0 * H, bytes, &full[st]);
  };
  if (tid == 0) {
    for (int i = 0; i < kOutStages; ++i) ptx::mbar_init(&full[i], 1);
    ptx::fence_mbar_init();
    for (int i = 0; i < kOutStages; ++i) issue(i);
  }
  float4 w[NMAX], g[NMAX];
#pragma unroll
  for (int o = 0; o < NMAX; ++o) {
    w[o] = (act_t && o < nL) ? __ldg(reinterpret_cast<const float4 *>(W + (int64_t)o * H) + gt) : make_float4(0.f, 0.f, 0.f, 0.f);
    g[o] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  // the block's target rows and the output bias, off the per-iteration critical path
  float *ysm = ring + (int64_t)kOutStages * stage_f + (RG > 1 ? nL * H : 0);
  for (int i = tid; i < (r1 - r0) * nL; i += 256) ysm[i] = Y[(int64_t)r0 * nL + i];
  const float bo = (lane & 15) < nL ? bias[lane & 15] : 0.0f;
  __syncthreads();  // barriers initialised, ysm filled
  float gb = 0.0f, lacc = 0.0f;  // first warp of a group: bias tendency / cost of lane (row slot, output)
  auto row_of = [&](int it, int rr) { return r0 + it * per_it + grp * RC + rr; };
  for (int it = 0; it < niter; ++it) {
    const int st = it % kOutStages;
    ptx::mbar_wait(&full[st], (it / kOutStages) & 1);
    const float4 *sa = reinterpret_cast<const float4 *>(ring + (int64_t)st * stage_f);
    const float4 *ss = sa + per_it * H4;
    float4 a[RC];
#pragma unroll
    for (int rr = 0; rr < RC; ++rr)
      a[rr] = (act_t && row_of(it, rr) < r1) ? sa[(grp * RC + rr) * H4 + gt] : make_float4(0.f, 0.f, 0.f, 0.f);
    float v[32];
#pragma unroll
    for (int rr = 0; rr < RC; ++rr)
#pragma unroll
      for (int o = 0; o < 16; ++o) {
        float z = 0.0f;
        if (o < NMAX) {
          z = a[rr].x * w[o].x;
          z = fmaf(a[rr].y, w[o].y, z);
          z = fmaf(a[rr].z, w[o].z, z);
          z = fmaf(a[rr].w, w[o].w, z);
        }
        v[rr * 16 + o] = z;
      }
    warp_reduce_scatter<32>(v, lane);  // lane l: value (row slot l >> 4, output l & 15)
    red[warp][lane] = v[0];
    __syncthreads();
    // every thread is past iteration it - 1: its stage is refilled with iteration it - 1 + stages
    if (tid == 0 && it >= 1) issue(it - 1 + kOutStages);
    if (act_t && gw == 0) {
      const int rr = lane >> 4, o = lane & 15, m = row_of(it, rr);
      float z = 0.0f;
      for (int q = 0; q < GW; ++q) z += red[grp * GW + q][lane];
      float dl = 0.0f;
      if (o < nL && m < r1) {
        float av, sg;
        act_fwd(act, z + bo, av, sg);
        const float diff = av - ysm[(m - r0) * nL + o];
        dl = diff * sg;
        lacc = fmaf(diff, diff, lacc);
        gb += dl;
        AL[(int64_t)m * nL + o] = av;
        DL[(int64_t)m * nL + o] = dl;
      }
      dsm[grp][rr][o] = dl;
    }
    __syncthreads();
    if (act_t) {
#pragma unroll
      for (int rr = 0; rr < RC; ++rr) {
        const int m = row_of(it, rr);
        float d[NMAX];
#pragma unroll
        for (int o = 0; o < NMAX; ++o) d[o] = dsm[grp][rr][o];
        float4 t = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int o = 0; o < NMAX; ++o) {
          t.x = fmaf(d[o], w[o].x, t.x);
          t.y = fmaf(d[o], w[o].y, t.y);
          t.z = fmaf(d[o], w[o].z, t.z);
          t.w = fmaf(d[o], w[o].w, t.w);
          g[o].x = fmaf(d[o], a[rr].x, g[o].x);
          g[o].y = fmaf(d[o], a[rr].y, g[o].y);
          g[o].z = fmaf(d[o], a[rr].z, g[o].z);
          g[o].w = fmaf(d[o], a[rr].w, g[o].w);
        }
        if (m < r1) {
          const float4 sv = ss[(grp * RC + rr) * H4 + gt];
          float4 dd = make_float4(t.x * sv.x, t.y * sv.y, t.z * sv.z, t.w * sv.w);
          if (rnd) dd = make_float4(tf32_rn(dd.x), tf32_rn(dd.y), tf32_rn(dd.z), tf32_rn(dd.w));  // a TC operand next
          reinterpret_cast<float4 *>(S + (int64_t)m * H)[gt] = dd;
          if (Dlo)
            reinterpret_cast<float4 *>(Dlo + (int64_t)m * H)[gt] =
                make_float4(tf32_lo(dd.x), tf32_lo(dd.y), tf32_lo(dd.z), tf32_lo(dd.w));
        }
      }
    }
  }
  // the groups' K4 partials summed in group order (deterministic), written by group 0
  float *gs = ring + (int64_t)kOutStages * stage_f;
  for (int q = 1; q < RG; ++q) {
    __syncthreads();
    if (grp == q)
#pragma unroll
      for (int o = 0; o < NMAX; ++o)
        if (o < nL) reinterpret_cast<float4 *>(gs + (int64_t)o * H)[gt] = g[o];
    __syncthreads();
    if (grp == 0)
#pragma unroll
      for (int o = 0; o < NMAX; ++o)
        if (o < nL) {
          const float4 u = reinterpret_cast<const float4 *>(gs + (int64_t)o * H)[gt];
          g[o].x += u.x; g[o].y += u.y; g[o].z += u.z; g[o].w += u.w;
        }
  }
  float *pb = part + (int64_t)blockIdx.x * nL * (H + 1);
  if (grp == 0)
#pragma unroll
    for (int o = 0; o < NMAX; ++o)
      if (o < nL) {
        float *p = pb + (int64_t)o * (H + 1) + 4 * gt;
        p[0] = g[o].x; p[1] = g[o].y; p[2] = g[o].z; p[3] = g[o].w;
      }
  // bias column H and the block's cost: lanes (row slot, output) of each group's first warp
  if (act_t && gw == 0) {  // (warp-uniform: GS is a multiple of 32)
    gb += __shfl_xor_sync(0xffffffffu, gb, 16);  // both row slots
    const float lw = warp_sum(lacc);
    bsm[grp][lane] = lane < 16 ? gb : lw;
  }
  __syncthreads();
  if (tid < 16 && tid < nL) {
    float u = 0.0f;
    for (int q = 0; q < RG; ++q) u += bsm[q][tid];
    pb[(int64_t)tid * (H + 1) + H] = u;
  }
  if (tid == 0) {
    float l = 0.0f;
    for (int q = 0; q < RG; ++q) l += bsm[q][16];
    lpart[blockIdx.x] = l;
  }
}

// Host-dataset staging of the small per-step target rows (nf_train_steps e2e path): the rows
// of up to kGatherMax steps read straight from mapped (pinned) host memory by the GPU, one
// kernel per chunk instead of one small DMA per step (their per-copy cost was 8 % of the e2e
// time on c2).  off[s]: first float of step s in src; len floats per step, contiguous.
constexpr int kGatherMax = 64;
struct GatherArgs {
  int64_t off[kGatherMax];
};
__global__ void __launch_bounds__(256) gather_steps_kernel(const float *__restrict__ src, GatherArgs a, int64_t len,
                                                           float *__restrict__ dst) {
  const int s = blockIdx.y;
  const float *p = src + a.off[s];
  float *q = dst + (int64_t)s * len;
  for (int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x; i < len; i += (int64_t)gridDim.x * 256) q[i] = p[i];
}

__global__ void __launch_bounds__(256) round_tf32_kernel(const float *__restrict__ src, float *__restrict__ dst,
                                                          int64_t n) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  for (int64_t i = blockIdx.x * 256 + threadIdx.x; i < n; i += (int64_t)gridDim.x * 256) dst[i] = tf32_rn(src[i]);
}

__global__ void __launch_bounds__(256) split_lo_kernel(const float *__restrict__ src, float *__restrict__ dst,
                                                        int64_t n) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  for (int64_t i = blockIdx.x * 256 + threadIdx.x; i < n; i += (int64_t)gridDim.x * 256) dst[i] = tf32_lo(src[i]);
}

__global__ void __launch_bounds__(256) split_rn_kernel(const float *__restrict__ src, float *__restrict__ hi,
                                                        float *__restrict__ lo, int64_t n) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  for (int64_t i = blockIdx.x * 256 + threadIdx.x; i < n; i += (int64_t)gridDim.x * 256) {
    const float x = src[i];
    hi[i] = tf32_rn(x);
    lo[i] = tf32_lo_rn(x);
  }
}

__global__ void __launch_bounds__(256) sgd_update_kernel(float *__restrict__ p, const float *__restrict__ g, int64_t n,
                                                         float scale) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  for (int64_t i = blockIdx.x * 256 + threadIdx.x; i < n; i += (int64_t)gridDim.x * 256) p[i] = p[i] - scale * g[i];
}

}  // namespace

cudaError_t gather_steps(cudaStream_t st, const float *src, const int64_t *off, int m, int64_t len, float *dst) {
  if (m <= 0) return cudaSuccess;
  if (m > kGatherMax) return cudaErrorInvalidValue;
  GatherArgs a;
  for (int s = 0; s < m; ++s) a.off[s] = off[s];
  const int bx = (int)std::min<int64_t>((len + 255) / 256, 16);
  gather_steps_kernel<<<dim3(bx, m), 256, 0, st>>>(src, a, len, dst);
  count_launch();
  log_launch(reinterpret_cast<const void *>(gather_steps_kernel), dim3(bx, m), dim3(256), 0);
  return cudaGetLastError();
}

cudaError_t round_tf32(cudaStream_t st, const float *src, float *dst, int64_t n) {
  if (n <= 0) return cudaSuccess;
  const int blocks = (int)std::min<int64_t>((n + 255) / 256, 8 * kSMs);
  return launch_k(round_tf32_kernel, dim3(blocks), dim3(256), 0, st, src, dst, n);
}

cudaError_t split_lo(cudaStream_t st, const float *src, float *dst, int64_t n) {
  if (n <= 0) return cudaSuccess;
  const int blocks = (int)std::min<int64_t>((n + 255) / 256, 8 * kSMs);
  return launch_k(split_lo_kernel, dim3(blocks), dim3(256), 0, st, src, dst, n);
}

cudaError_t split_rn(cudaStream_t st, const float *src, float *hi, float *lo, int64_t n) {
  if (n <= 0) return cudaSuccess;
  const int blocks = (int)std::min<int64_t>((n + 255) / 256, 8 * kSMs);
  return launch_k(split_rn_kernel, dim3(blocks), dim3(256), 0, st, src, hi, lo, n);
}

cudaError_t sgd_update(cudaStream_t st, float *p, const float *g, int64_t n, float scale) {
  if (n <= 0) return cudaSuccess;
  const int blocks = (int)std::min<int64_t>((n + 255) / 256, 8 * kSMs);
  return launch_k(sgd_update_kernel, dim3(blocks), dim3(256), 0, st, p, g, n, scale);
}

// blocks of the fused output-layer kernel: >= 8 rows each (>= 8192 / H for narrow hidden
// layers, so that the fixed-order final sum has few partials), at most 2 per SM
// the register-resident form (out_layer_train_rg) for hidden widths 128..1024 in steps of 128;
// NF_OUT_V1=1 keeps out_layer_train
bool out_layer_rg(int H) {
  static const bool v1 = getenv("NF_OUT_V1") != nullptr;
  return !v1 && H % 128 == 0 && H >= 128 && H <= 1024;
}

int out_layer_blocks(int n, int H) {
  // (>= 8192 / H rows for narrow H cut the final sum's partials but made c4 slower)
  const int rmin = 8;
  return std::max(1, std::min((out_layer_rg(H) ? 1 : 2) * kSMs, (n + rmin - 1) / rmin));
}

constexpr int kOutSmemMax = 200 * 1024;
static size_t out_layer_smem(int n, int H, int nL) {
  const int R = out_layer_blocks(n, H);
  return (size_t)nL * H * 4 + (size_t)((n + R - 1) / R) * 16 * 4;
}

bool out_layer_fusable(int n, int H, int nL, const float *A, const float *S, const float *W) {
  auto al16 = [](const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  static const bool off = getenv("NF_NO_OUT_FUSE") != nullptr;
  return !off && nL >= 1 && nL <= 16 && H % 4 == 0 && H >= 128 && H <= 2048 && n >= 256 &&
         out_layer_smem(n, H, nL) <= kOutSmemMax && al16(A) && al16(S) && al16(W);
}

cudaError_t out_layer_train_fused(cudaStream_t st, int n, int H, int nL, const float *A, float *S, const float *W,
                                  const float *bias, const float *Y, float *AL, float *DL, int act, float *part,
                                  int rnd, float *Dlo) {
  const int R = out_layer_blocks(n, H);
  const int rpb = (n + R - 1) / R;
  const int blocks = (n + rpb - 1) / rpb;
  const size_t smem = out_layer_smem(n, H, nL);
  for (const void *k : {reinterpret_cast<const void *>(out_layer_train<16, 4>), reinterpret_cast<const void *>(out_layer_train<16, 8>),
                        reinterpret_cast<const void *>(out_layer_train<16, 16>), reinterpret_cast<const void *>(out_layer_train<10, 4>),
                        reinterpret_cast<const void *>(out_layer_train<10, 8>), reinterpret_cast<const void *>(out_layer_train<10, 16>)}) {
    cudaError_t e = set_max_smem(k, kOutSmemMax);
    if (e != cudaSuccess) return e;
  }
  for (const void *k : {reinterpret_cast<const void *>(out_layer_train_rg<10>), reinterpret_cast<const void *>(out_layer_train_rg<16>)}) {
    cudaError_t e = set_max_smem(k, 200 * 1024);
    if (e != cudaSuccess) return e;
  }
  float *lp = part + (int64_t)blocks * nL * (H + 1);
  if (out_layer_rg(H)) {
    const size_t gsm = (size_t)kOutStages * 2 * 2 * (256 / (H / 4)) * H * 4 + (256 / (H / 4) > 1 ? (size_t)nL * H * 4 : 0) +
                       (size_t)rpb * nL * 4;
    if (gsm > 200 * 1024) return cudaErrorInvalidValue;
    if (nL <= 10)
      return launch_k(out_layer_train_rg<10>, dim3(blocks), dim3(256), gsm, st, A, S, W, bias, Y, AL, DL, n, H, nL,
                      act, rpb, part, lp, rnd, Dlo);
    return launch_k(out_layer_train_rg<16>, dim3(blocks), dim3(256), gsm, st, A, S, W, bias, Y, AL, DL, n, H, nL,
                    act, rpb, part, lp, rnd, Dlo);
  }
  if (nL <= 10) {  // (MNIST-like 10-wide outputs: no idle unrolled output slots)
    if (H <= 512)
      return launch_k(out_layer_train<10, 4>, dim3(blocks), dim3(256), smem, st, A, S, W, bias, Y, AL, DL, n, H, nL,
                      act, rpb, part, lp, rnd, Dlo);
    if (H <= 1024)
      return launch_k(out_layer_train<10, 8>, dim3(blocks), dim3(256), smem, st, A, S, W, bias, Y, AL, DL, n, H, nL,
                      act, rpb, part, lp, rnd, Dlo);
    return launch_k(out_layer_train<10, 16>, dim3(blocks), dim3(256), smem, st, A, S, W, bias, Y, AL, DL, n, H, nL,
                    act, rpb, part, lp, rnd, Dlo);
  }
  if (H <= 512)
    return launch_k(out_layer_train<16, 4>, dim3(blocks), dim3(256), smem, st, A, S, W, bias, Y, AL, DL, n, H, nL,
                    act, rpb, part, part + (int64_t)blocks * nL * (H + 1), rnd, Dlo);
  if (H <= 1024)
    return launch_k(out_layer_train<16, 8>, dim3(blocks), dim3(256), smem, st, A, S, W, bias, Y, AL, DL, n, H, nL,
                    act, rpb, part, part + (int64_t)blocks * nL * (H + 1), rnd, Dlo);
  return launch_k(out_layer_train<16, 16>, dim3(blocks), dim3(256), smem, st, A, S, W, bias, Y, AL, DL, n, H, nL,
                  act, rpb, part, part + (int64_t)blocks * nL * (H + 1), rnd, Dlo);
}

cudaError_t out_layer_grad_final(cudaStream_t st, int n, int H, int nL, const float *part, const EpiGrad &epi,
                                 float *step_loss) {
  const int R = out_layer_blocks(n, H);
  const int rpb = (n + R - 1) / R;
  const int blocks = (n + rpb - 1) / rpb;
  const int64_t MN = (int64_t)nL * (H + 1);
  return launch_k(grad_smallm_final, dim3((int)((MN + 31) / 32)), dim3(256), 0, st, part, blocks, nL, H, epi,
                  (const float *)(part + (int64_t)blocks * nL * (H + 1)), 0.5f / (float)n, step_loss);
}

cudaError_t gemm_fwd(cudaStream_t st, int M, int N, int K, const float *A, const float *W,
                     const EpiFwd &epi, const Workspace &ws, const float *Wtc, const float *Alo, const float *Wlo,
                     const float *Ahi) {
  const TcOp a{Ahi ? Ahi : A, K, false, Alo}, b{Wtc ? Wtc : W, K, false, Wlo};
  if (use_tc(M, N, K, a, b)) return run_tc<false, false>(st, M, N, K, a, b, epi, ws);
  g_last_engine = ENGINE_SIMT;
  if (N <= 16 && K % 4 == 0 && (size_t)N * K * 4 <= 96 * 1024 && tc_ok(a) && tc_ok(b) && M >= 256) {
    {
      cudaError_t e = set_max_smem(reinterpret_cast<const void *>(fwd_smalln<16, true>), 96 * 1024);
      if (e != cudaSuccess) return e;
    }
    static const int per_sm = getenv("NF_SMALLN_PER_SM") ? atoi(getenv("NF_SMALLN_PER_SM")) : 2;
    static const bool nostage = getenv("NF_SMALLN_NOSTAGE") != nullptr;
    const int blocks = std::min((M + 7) / 8, per_sm * kSMs);  // W is staged once per block
    if (nostage && (reinterpret_cast<uintptr_t>(W) & 15) == 0)
      return launch_k(fwd_smalln<16, false>, dim3(blocks), dim3(256), 0, st, A, W, M, N, K, epi);
    return launch_k(fwd_smalln<16, true>, dim3(blocks), dim3(256), (size_t)N * K * 4, st, A, W, M, N, K, epi);
  }
  GemmArgs g{M, N, K, A, K, W, K, N, 0, nullptr};
  return run_gemm<true, true>(st, g, epi, ws);
}

bool gemm_bwd_fuses_bias(int M, int N, int K, const float *D, const float *W) {
  // the tensor-core path only (its strip epilogue sums 32 rows per reduction); up to 16384
  // rows = 512 reductions per bias element (c5: 9.17 -> 9.05 ms per step)
  // NF_SPLITK_DETERMINISTIC=1: off (its L2 reductions arrive in any order; the column-sum
  // kernels then sum the chunks in a fixed order)
  static const bool off = getenv("NF_NO_BIAS_FUSE") != nullptr || getenv("NF_SPLITK_DETERMINISTIC") != nullptr;
  const TcOp a{D, K, false}, b{W, N, true};
  static const int maxm = getenv("NF_BIAS_FUSE_MAXM") ? atoi(getenv("NF_BIAS_FUSE_MAXM")) : 16384;
  return !off && M <= maxm && use_tc(M, N, K, a, b);
}

bool gemm_grad_tc(int M, int N, int K, const float *D, const float *Aprev) {
  const TcOp a{D, M, true}, b{Aprev, N, true};
  return use_tc(M, N, K, a, b);
}

bool gemm_fwd_tc(int M, int N, int K, const float *A, const float *W) {
  const TcOp a{A, K, false}, b{W, K, false};
  return use_tc(M, N, K, a, b);
}

bool gemm_bwd_tc(int M, int N, int K, const float *D, const float *W) {
  const TcOp a{D, K, false}, b{W, N, true};
  return use_tc(M, N, K, a, b);
}

cudaError_t gemm_bwd(cudaStream_t st, int M, int N, int K, const float *D, const float *W,
                     const EpiBwd &epi, const Workspace &ws, const float *Wtc, const float *Dlo, const float *Wlo) {
  const TcOp a{D, K, false, Dlo}, b{Wtc ? Wtc : W, N, true, Wlo};
  if (use_tc(M, N, K, a, b)) return run_tc<false, true>(st, M, N, K, a, b, epi, ws);
  g_last_engine = ENGINE_SIMT;
  if (K <= 16 && N % 4 == 0 && epi.ld % 4 == 0 && (reinterpret_cast<uintptr_t>(W) & 15) == 0 &&
      (reinterpret_cast<uintptr_t>(epi.SD) & 15) == 0 && M >= 256) {
    const int cb = (N / 4 + 127) / 128;
    const int TM = std::max(4, (int)((int64_t)M * cb / (8 * kSMs)));
    return launch_k(bwd_smallk<16>, dim3(cb, (M + TM - 1) / TM), dim3(128), 0, st, D, W, M, N, K, TM, epi);
  }
  GemmArgs g{M, N, K, D, K, W, N, N, 0, nullptr};
  return run_gemm<true, false>(st, g, epi, ws);
}

cudaError_t gemm_grad(cudaStream_t st, int M, int N, int K, const float *D, const float *Aprev,
                      const EpiGrad &epi, const Workspace &ws, bool bias_done, const float *DT,
                      const float *AprevT, const float *Dlo, const float *Aprevlo, const float *Aprevhi) {
  const TcOp a{D, M, true, Dlo}, b{Aprevhi ? Aprevhi : Aprev, N, true, Aprevlo};
  if (use_tc(M, N, K, a, b)) {
    // bias tendencies first (unless the delta GEMM's epilogue applied them): they read D only,
    // and the partial buffer is free again before the split-K GEMM uses it (same stream)
    if (!bias_done) {
      cudaError_t e = bias_grad(st, D, K, M, epi, ws.partial, ws.partial_floats);
      if (e != cudaSuccess) return e;
    }
    // transposed copies written by the producing epilogues make the operands K-major (the MN-major
    // smem layouts run the tensor core at 552 vs 659 TF/s for K/K, profiles/r01_tc_majors_accuracy_perf.txt)
    if (DT) {
      const TcOp at{DT, K, false};
      if (AprevT) return run_tc<false, false>(st, M, N, K, at, TcOp{AprevT, K, false}, epi, ws);
      return run_tc<false, true>(st, M, N, K, at, b, epi, ws);
    }
    return run_tc<true, true>(st, M, N, K, a, b, epi, ws);
  }
  g_last_engine = ENGINE_SIMT;
  if (M <= 16 && K >= 512) {
    const int cb = (N + 1 + 127) / 128;
    int R = std::max(1, std::min(K / 32, (8 * kSMs) / cb));
    while (R > 1 && (size_t)R * M * (N + 1) > ws.partial_floats) --R;
    const int chunk = (K + R - 1) / R;
    R = (K + chunk - 1) / chunk;
    cudaError_t e = launch_k(grad_smallm_partial<16>, dim3(cb, R), dim3(128), 0, st, D, Aprev, M, N, K, chunk,
                             ws.partial);
    if (e != cudaSuccess) return e;
    const int64_t MN = (int64_t)M * (N + 1);
    return launch_k(grad_smallm_final, dim3((int)((MN + 31) / 32)), dim3(256), 0, st,
                    (const float *)ws.partial, R, M, N, epi, (const float *)nullptr, 0.0f, (float *)nullptr);
  }
  // C[M][N+1]: column N is the ones column -> bias gradient.
  GemmArgs g{M, N + 1, K, D, M, Aprev, N, N, 0, nullptr};
  return run_gemm<false, false>(st, g, epi, ws);
}

// ---------------------------------------------------------------------------
// K5: loss / accuracy.  One warp per sample row; per-row cost 1/2 sum (a-y)^2
// in fp32, first-index argmax of a and of y (reading R10); block partials in
// fp64, summed by a single thread in block order (deterministic).
namespace {
constexpr int kLossBlocks = 2 * kSMs;

__device__ __forceinline__ void argmax_merge(float &v, int &i, float v2, int i2) {
  if (v2 > v || (v2 == v && i2 < i)) { v = v2; i = i2; }
}

__global__ void __launch_bounds__(256)
loss_acc_partial(const float *__restrict__ A, const float *__restrict__ Y, int64_t n, int w,
                 double2 *__restrict__ part) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t gw = (int64_t)blockIdx.x * 8 + warp, nw = (int64_t)gridDim.x * 8;
  double lsum = 0.0, csum = 0.0;
  for (int64_t r = gw; r < n; r += nw) {
    const float *a = A + r * w, *y = Y + r * w;
    float l = 0.0f, va = -INFINITY, vy = -INFINITY;
    int ia = 0x7fffffff, iy = 0x7fffffff;
    for (int j = lane; j < w; j += 32) {
      const float aj = a[j], yj = y[j];
      const float d = aj - yj;
      l = fmaf(d, d, l);
      if (aj > va) { va = aj; ia = j; }
      if (yj > vy) { vy = yj; iy = j; }
    }
    l = warp_sum(l);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      argmax_merge(va, ia, __shfl_xor_sync(0xffffffffu, va, o), __shfl_xor_sync(0xffffffffu, ia, o));
      argmax_merge(vy, iy, __shfl_xor_sync(0xffffffffu, vy, o), __shfl_xor_sync(0xffffffffu, iy, o));
    }
    lsum += 0.5 * (double)l;
    csum += (ia == iy) ? 1.0 : 0.0;
  }
  __shared__ double2 sm[8];
  if (lane == 0) sm[warp] = make_double2(lsum, csum);
  __syncthreads();
  if (threadIdx.x == 0) {
    double2 t = make_double2(0.0, 0.0);
    for (int i = 0; i < 8; ++i) { t.x += sm[i].x; t.y += sm[i].y; }
    part[blockIdx.x] = t;
  }
}

// One warp: lane j sums partials j, j+32, ... in order, then a fixed shuffle tree
// (deterministic for a given nparts).
__global__ void loss_acc_final(const double2 *__restrict__ part, int nparts, int64_t n,
                               float *out, float *step_loss) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  const int lane = threadIdx.x;
  double l = 0.0, c = 0.0;
  for (int i = lane; i < nparts; i += 32) { l += part[i].x; c += part[i].y; }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    l += __shfl_xor_sync(0xffffffffu, l, o);
    c += __shfl_xor_sync(0xffffffffu, c, o);
  }
  if (lane != 0) return;
  const float loss = n > 0 ? (float)(l / (double)n) : 0.0f;
  const float acc = n > 0 ? (float)(c / (double)n) : 0.0f;
  if (out) { out[0] = loss; out[1] = acc; }
  if (step_loss) *step_loss = loss;
}
}  // namespace

int loss_acc_parts() { return kLossBlocks; }

cudaError_t loss_acc(cudaStream_t st, const float *A, const float *Y, int64_t n, int w,
                     double2 *part, float *out, float *step_loss) {
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(kLossBlocks, (n + 7) / 8));
  cudaError_t e = launch_k(loss_acc_partial, dim3(blocks), dim3(256), 0, st, A, Y, n, w, part);
  if (e != cudaSuccess) return e;
  return launch_k(loss_acc_final, dim3(1), dim3(32), 0, st, (const double2 *)part, blocks, n, out, step_loss);
}

}  // namespace nf
