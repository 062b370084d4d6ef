"""Parity metric shared by the GPU tests (reading R14 of DESIGN.md).

err = max_i |g_i - o_i| / max(|o_i|, tau * max_j |o_j|), tau = 0.1

The floor tau*max|o| keeps the relative error defined where an entry is tiny
compared with its tensor (saturated sigmoids, relu zeros, cancelling sums).
Bars (BASELINE.json north_star): 1e-4 for the fp32 path, 5e-3 for TF32 tiles.
"""
import numpy as np

TAU = 0.1
FP32_BAR = 1e-4
TF32_BAR = 5e-3        # TF32 tiles, normwise (tau = 1): reading R14b -- at tau = 0.1 even exact
                       # round-to-nearest TF32 operands with an exact sum reach 5.6-8.4e-3 on the
                       # configs (tools/tf32_rounding_emulation.py, profiles/r02_tf32_emulation.txt)
FP64_BAR = 2.5e-7      # NF_MATH_FP64: double arithmetic, one fp32 rounding at the ABI (2^-24 = 6e-8
                       # relative) plus margin; the fp32 path cannot meet it (R19)


def rel_err(got, ref, tau: float = TAU) -> float:
    got = np.asarray(got, dtype=np.float64).ravel()
    ref = np.asarray(ref, dtype=np.float64).ravel()
    assert got.shape == ref.shape, (got.shape, ref.shape)
    if ref.size == 0:
        return 0.0
    if not np.all(np.isfinite(got)):
        return float("inf")
    scale = np.maximum(np.abs(ref), tau * np.max(np.abs(ref)))
    scale = np.where(scale == 0, 1.0, scale)
    return float(np.max(np.abs(got - ref) / scale))


def argmax_agree(got, ref, gap_rel: float = 1e-5):
    """R15: predictions must agree on every row whose oracle top-2 gap exceeds
    gap_rel * max|a|; near-ties are reported, not failed.  Returns (#mismatch, #near_ties)."""
    got = np.asarray(got); ref = np.asarray(ref, dtype=np.float64)
    srt = np.sort(ref, axis=1)
    gap = srt[:, -1] - srt[:, -2] if ref.shape[1] > 1 else np.full(ref.shape[0], np.inf)
    tie = gap <= gap_rel * np.maximum(np.abs(ref).max(axis=1), 1e-30)
    mism = (np.argmax(got, axis=1) != np.argmax(ref, axis=1)) & ~tie
    return int(mism.sum()), int(tie.sum())
