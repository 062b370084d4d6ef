"""What the TF32 format alone costs (reading R14b): numpy emulation of one SGD step's chain of
contractions with TF32 operands -- truncated (what the tensor core does to raw fp32 bit
patterns) or rounded to nearest (cvt.rna, what NF_MATH_TF32 now feeds it) -- products summed
EXACTLY in fp64, stored values rounded to fp32; relu derivative decisions taken on the exact
pre-activations (so kinks do not contribute).  Reports max relative error of the output and of
every layer's batch-summed W / b tendency at tau = 0.1 and normwise (tau = 1) against the exact
fp64 step, on the configs' seeded inputs.  Any TF32 kernel can only add to these numbers.

    python tools/tf32_rounding_emulation.py > profiles/r02_tf32_emulation.txt
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402


def trunc(x):
    x = np.asarray(x, np.float32).copy()
    x.view(np.uint32)[...] &= np.uint32(0xFFFFE000)
    return x.astype(np.float64)


def rn(x):
    v = np.asarray(x, np.float32).copy().view(np.uint32).astype(np.uint64)
    v = (v + 0x1000) & 0xFFFFE000          # ties away from zero, as cvt.rna
    return v.astype(np.uint32).view(np.float32).astype(np.float64)


def ident(x):
    return np.asarray(x, np.float64)


def f32(x):
    return np.asarray(x, np.float32).astype(np.float64)


def sig(z):
    return 1 / (1 + np.exp(-z))


ACT = {"tanh": (np.tanh, lambda z: 1 - np.tanh(z) ** 2),
       "relu": (lambda z: np.maximum(z, 0), lambda z: (z > 0) * 1.0),
       "sigmoid": (sig, lambda z: sig(z) * (1 - sig(z)))}


def step(dims, spec, p, X, Y, rop, store, xop=None, zref=None):
    parts = spec.split(",")
    L = len(dims) - 1
    names = [parts[0]] * (L - 1) + [parts[-1]] if len(parts) == 2 else parts * L
    Ws, o = [], 0
    for l in range(1, len(dims)):
        W = p[o:o + dims[l] * dims[l - 1]].reshape(dims[l], dims[l - 1]).astype(np.float64); o += W.size
        b = p[o:o + dims[l]].astype(np.float64); o += dims[l]
        Ws.append((W, b))
    xop = xop or rop
    A, S, Z = [X.astype(np.float64)], [], []
    for l, (W, b) in enumerate(Ws):
        f, fp = ACT[names[l]]
        z = (xop if l == 0 else rop)(A[-1]) @ rop(W).T + b
        Z.append(z)
        A.append(store(f(z)))
        S.append(store(fp(zref[l] if zref is not None else z)))
    D = [None] * L
    D[L - 1] = store((A[L] - Y) * S[L - 1])
    for l in range(L - 2, -1, -1):
        D[l] = store((rop(D[l + 1]) @ rop(Ws[l + 1][0])) * S[l])
    G = [(rop(D[l]).T @ (xop if l == 0 else rop)(A[l]), D[l].sum(0)) for l in range(L)]
    return A[-1], G, Z


def err(g, r, tau):
    s = np.maximum(np.abs(r), tau * np.abs(r).max())
    return float(np.max(np.abs(g - r) / s))


def main():
    print("max relative error vs the exact fp64 step; 'a/b' = tau 0.1 / normwise (tau 1)")
    for cid, B in [(3, 4096), (4, 2048), (5, 1024)]:
        cfg = synth.CONFIGS[cid]
        p = synth.init_params(cid)
        X, Y = synth.dataset(cid, N=B)
        ref = step(cfg["dims"], cfg["act"], p, X, Y, ident, ident)
        for name, rop, xop in [("truncated operands", trunc, None), ("RN operands", rn, None),
                               ("RN operands, x truncated", rn, trunc)]:
            got = step(cfg["dims"], cfg["act"], p, X, Y, rop, f32, xop=xop, zref=ref[2])
            gs = "  ".join(f"L{l + 1} W {err(a[0], b[0], .1):.2e}/{err(a[0], b[0], 1):.2e} "
                           f"b {err(a[1], b[1], .1):.2e}/{err(a[1], b[1], 1):.2e}"
                           for l, (a, b) in enumerate(zip(got[1], ref[1])))
            print(f"c{cid} B={B} {name:26s} out {err(got[0], ref[0], .1):.2e}/{err(got[0], ref[0], 1):.2e}  {gs}",
                  flush=True)


if __name__ == "__main__":
    main()
