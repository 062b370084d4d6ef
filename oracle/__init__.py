"""CPU oracle of the neural-fortran method (arXiv:1902.06714) -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` leg may import this package.  The product package
``paper_1902_06714_b200`` never imports it and shares no code with it.

The arithmetic lives in ``nf_oracle.c`` (plain C, strict left-to-right sums, no
fast-math), compiled twice: ``REAL=double`` (the parity reference) and
``REAL=float`` (the paper's default real32, used for CPU timing).
This module only marshals numpy arrays into it.

Parity status: every exported function is pinned by ``tests/test_oracle.py``
(closed forms, finite differences, split-batch identity, SPEC examples); the
one unpinned item is the MNIST accuracy trajectory (dataset absent),
which this oracle does not attempt.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "nf_oracle.c")

# Activation names of P:108-109 / S:30 -> the oracle's own enum (nf_oracle.c).
ACT = {"sigmoid": 0, "tanh": 1, "relu": 2, "gaussian": 3, "step": 4}


def parse_activation(spec: str, L: int = 2) -> list[int]:
    """Activation kind of each of the L layers: 'sigmoid' -> every layer; 'relu,sigmoid' ->
    hidden layers / output layer (reading R7); L comma-separated names -> one per layer
    (SURVEY 8(f)).  Unknown names or other counts raise (never a silent default)."""
    parts = [s.strip().lower() for s in spec.split(",")]
    if any(p not in ACT for p in parts):
        raise ValueError(f"unknown activation spec {spec!r}")
    if len(parts) == 1:
        parts = parts * L
    elif len(parts) == 2:
        parts = [parts[0]] * (L - 1) + [parts[1]]
    elif len(parts) != L:
        raise ValueError(f"activation spec {spec!r}: need 1, 2 or {L} names")
    return [ACT[p] for p in parts]


def build(force: bool = False) -> None:
    """Compile liboracle64.so and liboracle32.so next to the source (gcc -O2, no fast-math)."""
    for real, name in (("double", "liboracle64.so"), ("float", "liboracle32.so")):
        out = os.path.join(_HERE, name)
        if not force and os.path.exists(out) and os.path.getmtime(out) >= os.path.getmtime(_SRC):
            continue
        subprocess.check_call(
            ["gcc", "-O2", "-std=c99", "-fPIC", "-shared", "-fno-fast-math",
             "-ffp-contract=off", f"-DREAL={real}", _SRC, "-o", out, "-lm"])


_LIBS: dict[int, ctypes.CDLL] = {}


def _lib(bits: int = 64) -> ctypes.CDLL:
    if bits not in _LIBS:
        build()
        lib = ctypes.CDLL(os.path.join(_HERE, f"liboracle{bits}.so"))
        lib.orc_act.restype = ctypes.c_double if bits == 64 else ctypes.c_float
        lib.orc_act_prime.restype = lib.orc_act.restype
        lib.orc_act.argtypes = [ctypes.c_int, lib.orc_act.restype]
        lib.orc_act_prime.argtypes = lib.orc_act.argtypes
        lib.orc_param_count.restype = ctypes.c_long
        assert lib.orc_real_bytes() == bits // 8
        _LIBS[bits] = lib
    return _LIBS[bits]


def _real(bits):
    return np.float64 if bits == 64 else np.float32


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _dims(dims):
    d = np.ascontiguousarray(np.asarray(dims, dtype=np.int32))
    return d, ctypes.c_int(len(d))


def _f32(a) -> np.ndarray:
    a = np.asarray(a)
    if a.dtype != np.float32:
        raise TypeError("oracle inputs x/y are fp32 values (the GPU path's storage type)")
    return np.ascontiguousarray(a)


class Oracle:
    """A network description (dims, activation) evaluated by the C oracle.

    ``bits=64`` is the parity reference; ``bits=32`` is the real32 build used
    only as the timed CPU baseline.
    """

    def __init__(self, dims, activation: str = "sigmoid", bits: int = 64):
        self.dims = [int(d) for d in dims]
        if len(self.dims) < 2 or min(self.dims) < 1:
            raise ValueError("dims needs >= 2 entries, each >= 1 (S:118-124)")
        self.acts = parse_activation(activation, len(self.dims) - 1)
        self.act_h, self.act_o = self.acts[0], self.acts[-1]
        self._acts = np.ascontiguousarray(np.asarray(self.acts, dtype=np.int32))
        self.bits = bits
        self.lib = _lib(bits)
        self.real = _real(bits)

    # -- helpers -----------------------------------------------------------
    @property
    def n_params(self) -> int:
        d, nd = _dims(self.dims)
        return int(self.lib.orc_param_count(_ptr(d), nd))

    def _p(self, params) -> np.ndarray:
        p = np.ascontiguousarray(np.asarray(params, dtype=self.real))
        if p.size != self.n_params:
            raise ValueError(f"expected {self.n_params} params, got {p.size}")
        return p

    def _head(self):
        d, nd = _dims(self.dims)
        self._keep = d
        return _ptr(d), nd, _ptr(self._acts)

    def layers(self, params):
        """Split a flat vector into [(W_l [n_l][n_{l-1}], b_l [n_l])] views."""
        out, o = [], 0
        for l in range(1, len(self.dims)):
            ni, nk = self.dims[l], self.dims[l - 1]
            W = params[o:o + ni * nk].reshape(ni, nk); o += ni * nk
            b = params[o:o + ni]; o += ni
            out.append((W, b))
        return out

    # -- the method --------------------------------------------------------
    def act(self, kind: str, x: float) -> float:
        return float(self.lib.orc_act(ACT[kind], x))

    def act_prime(self, kind: str, x: float) -> float:
        return float(self.lib.orc_act_prime(ACT[kind], x))

    def output(self, params, x) -> np.ndarray:
        p, x = self._p(params), _f32(x)
        n = x.shape[0]
        out = np.zeros((n, self.dims[-1]), dtype=self.real)
        rc = self.lib.orc_output(*self._head(), _ptr(p), _ptr(x), ctypes.c_long(n), _ptr(out))
        assert rc == 0
        return out

    def grad(self, params, x, y) -> np.ndarray:
        """Summed tendencies over the batch (flat, params layout)."""
        p, x, y = self._p(params), _f32(x), _f32(y)
        G = np.zeros(self.n_params, dtype=self.real)
        rc = self.lib.orc_grad(*self._head(), _ptr(p), _ptr(x), _ptr(y),
                               ctypes.c_long(x.shape[0]), _ptr(G))
        assert rc == 0
        return G

    def train_batch(self, params, x, y, eta: float):
        """Returns (updated params, mean batch loss before the update)."""
        p, x, y = self._p(params).copy(), _f32(x), _f32(y)
        loss = np.zeros(1, dtype=self.real)
        rc = self.lib.orc_train_batch(*self._head(), _ptr(p), _ptr(x), _ptr(y),
                                      ctypes.c_long(x.shape[0]), _scalar(self.bits, eta), _ptr(loss))
        if rc != 0:
            raise ValueError("train_batch: empty batch")
        return p, float(loss[0])

    def train_steps(self, params, X, Y, batch: int, starts, eta: float):
        """Returns (params after len(starts) steps, per-step pre-update batch loss)."""
        p, X, Y = self._p(params).copy(), _f32(X), _f32(Y)
        st = np.ascontiguousarray(np.asarray(starts, dtype=np.int64))
        losses = np.zeros(len(st), dtype=self.real)
        rc = self.lib.orc_train_steps(*self._head(), _ptr(p), _ptr(X), _ptr(Y),
                                      ctypes.c_long(X.shape[0]), ctypes.c_long(batch),
                                      _ptr(st), ctypes.c_long(len(st)),
                                      _scalar(self.bits, eta), _ptr(losses))
        if rc != 0:
            raise ValueError(f"train_steps failed rc={rc}")
        return p, losses

    def loss(self, params, x, y) -> float:
        p, x, y = self._p(params), _f32(x), _f32(y)
        out = np.zeros(1, dtype=self.real)
        rc = self.lib.orc_loss(*self._head(), _ptr(p), _ptr(x), _ptr(y),
                               ctypes.c_long(x.shape[0]), _ptr(out))
        assert rc == 0
        return float(out[0])

    def accuracy(self, params, x, y) -> float:
        p, x, y = self._p(params), _f32(x), _f32(y)
        out = np.zeros(1, dtype=self.real)
        rc = self.lib.orc_accuracy(*self._head(), _ptr(p), _ptr(x), _ptr(y),
                                   ctypes.c_long(x.shape[0]), _ptr(out))
        assert rc == 0
        return float(out[0])

    def stash(self, params, x, y, with_z: bool = False):
        """Per-layer activations a_0..a_L and deltas delta_1..delta_L of one batch
        (and pre-activations z_1..z_L with with_z=True)."""
        p, x, y = self._p(params), _f32(x), _f32(y)
        n = x.shape[0]
        A = np.zeros(n * sum(self.dims), dtype=self.real)
        D = np.zeros(n * sum(self.dims[1:]), dtype=self.real)
        Z = np.zeros(n * sum(self.dims[1:]), dtype=self.real) if with_z else None
        rc = self.lib.orc_forward_backward_stash(*self._head(), _ptr(p), _ptr(x), _ptr(y),
                                                 ctypes.c_long(n), _ptr(A), _ptr(D),
                                                 _ptr(Z) if with_z else None)
        assert rc == 0
        As, Ds, Zs, oa, od = [], [], [], 0, 0
        for l, w in enumerate(self.dims):
            As.append(A[oa:oa + n * w].reshape(n, w)); oa += n * w
            if l >= 1:
                Ds.append(D[od:od + n * w].reshape(n, w))
                if with_z:
                    Zs.append(Z[od:od + n * w].reshape(n, w))
                od += n * w
        return (As, Ds, Zs) if with_z else (As, Ds)

    def kink_free_rows(self, params, x, y, margin: float = 1e-4):
        """Rows whose hidden pre-activations all keep |z| > margin, where a relu/step
        derivative is a discrete decision: the fp32 GPU sum and this fp64 sum may take it
        differently within rounding (reading R8 of DESIGN.md).  Parity compares these rows."""
        _, _, Zs = self.stash(params, x, y, with_z=True)
        ok = np.ones(x.shape[0], dtype=bool)
        for l, z in enumerate(Zs, start=1):
            if self.acts[l - 1] in (ACT["relu"], ACT["step"]):
                ok &= np.all(np.abs(z) > margin, axis=1)
        return ok


def _scalar(bits, v):
    return ctypes.c_double(v) if bits == 64 else ctypes.c_float(v)

