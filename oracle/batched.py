"""Batched fp64 oracle of the neural-fortran method -- TEST INFRASTRUCTURE.

Same import rule as the rest of ``oracle/``: only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s CPU legs may use it; the product package never imports it.

This is the *definition* of one SGD step (SURVEY.md 8(c) "Definition") written out over a
whole batch, with numpy's fp64 matrix product as the one library primitive (the paper's own
``matmul``, fwdprop P:337, and the outer products of backprop P:406-413):

    A_0 = X                                  (rows = samples)
    Z_l = A_{l-1} W_l^T + 1 b_l^T            Eq. 2; fwdprop P:324-361
    A_l = sigma_l(Z_l)
    D_L = (A_L - Y) .* sigma_L'(Z_L)         quadratic cost
    D_l = (D_{l+1} W_{l+1}) .* sigma_l'(Z_l) backprop P:409-411 (no D_0)
    G_l = D_l^T A_{l-1},  g_l = 1^T D_l      tendencies summed over the batch = the co_sum,
                                             P:406-413, P:460-462, P:536-556
    W_l -= (eta/B) G_l,  b_l -= (eta/B) g_l  update, reading R3

It computes the same numbers as ``nf_oracle.c`` (per sample, per neuron, in the paper's
loop order) up to the summation order inside the products; at the sizes of the bench
configurations (c5: 4.8 TFLOP per step) the per-sample C loops would take hours, this takes
seconds on the host's BLAS threads.  Inputs are fp32 values widened exactly; everything is
fp64; results are rounded to fp32 only by the comparing test.

Pins (tests/test_oracle_batched.py, ``-m "not gpu"``): equality with the independently
pinned C oracle on random nets of every activation, the closed-form single sigmoid neuron,
centered finite differences, and the co_sum split identity.

Relu / step derivatives are a 0/1 decision taken from a float (reading R8).  ``zdec``
(optional, per layer) supplies the pre-activations the decision is taken on -- used by the
tests only to select rows whose decisions are unambiguous (``kink_margin``); by default the
decision is on the oracle's own fp64 Z.
"""
from __future__ import annotations

import numpy as np

from . import parse_activation

SIGMOID, TANH, RELU, GAUSSIAN, STEP = range(5)


def act(kind: int, z: np.ndarray) -> np.ndarray:
    """sigma(z), S:40 (sigmoid P:207-209)."""
    if kind == SIGMOID:
        return 1.0 / (1.0 + np.exp(-z))
    if kind == TANH:
        return np.tanh(z)
    if kind == RELU:
        return np.where(z > 0, z, 0.0)
    if kind == GAUSSIAN:
        return np.exp(-z * z)
    if kind == STEP:
        return np.where(z > 0, 1.0, 0.0)
    raise ValueError(kind)


def act_prime(kind: int, z: np.ndarray) -> np.ndarray:
    """sigma'(z); relu'(0) = 0, step' = 0 (reading R8)."""
    if kind == SIGMOID:
        s = 1.0 / (1.0 + np.exp(-z))
        return s * (1.0 - s)
    if kind == TANH:
        t = np.tanh(z)
        return 1.0 - t * t
    if kind == RELU:
        return np.where(z > 0, 1.0, 0.0)
    if kind == GAUSSIAN:
        return -2.0 * z * np.exp(-z * z)
    if kind == STEP:
        return np.zeros_like(z)
    raise ValueError(kind)


class BatchedOracle:
    """A network (dims, activation spec) evaluated batch-wise in fp64."""

    def __init__(self, dims, activation: str = "sigmoid"):
        self.dims = [int(d) for d in dims]
        if len(self.dims) < 2 or min(self.dims) < 1:
            raise ValueError("dims needs >= 2 entries, each >= 1 (S:118-124)")
        self.L = len(self.dims) - 1
        self.acts = parse_activation(activation, self.L)

    @property
    def n_params(self) -> int:
        return sum(self.dims[l] * self.dims[l - 1] + self.dims[l] for l in range(1, self.L + 1))

    def layers(self, params):
        """[(W_l [n_l][n_{l-1}], b_l [n_l])] views of a flat vector (include/nf.h layout)."""
        out, o = [], 0
        for l in range(1, self.L + 1):
            ni, nk = self.dims[l], self.dims[l - 1]
            W = params[o:o + ni * nk].reshape(ni, nk); o += ni * nk
            b = params[o:o + ni]; o += ni
            out.append((W, b))
        return out

    def _p64(self, params) -> np.ndarray:
        p = np.asarray(params)
        if p.size != self.n_params:
            raise ValueError(f"expected {self.n_params} params, got {p.size}")
        return p.astype(np.float64).ravel()

    # -- fwdprop over the batch ------------------------------------------------------
    def forward(self, params, X):
        """Returns (A, Z): A[0..L] activations (A[0] = X), Z[1..L] pre-activations (Z[0] = None)."""
        Wb = self.layers(self._p64(params))
        A = [np.asarray(X, dtype=np.float64)]
        Z = [None]
        for l in range(1, self.L + 1):
            W, b = Wb[l - 1]
            z = A[l - 1] @ W.T + b
            Z.append(z)
            A.append(act(self.acts[l - 1], z))
        return A, Z

    def output(self, params, X) -> np.ndarray:
        """output: a_L of every row."""
        return self.forward(params, X)[0][-1]

    # -- backprop + batch sum ----------------------------------------------------------
    def backward(self, params, A, Z, Y, zdec=None):
        """Deltas D[1..L] (D[0] = None) from a forward pass.  zdec[l]: the pre-activations the
        relu/step derivative decision of layer l is taken on (default Z[l])."""
        Wb = self.layers(self._p64(params))
        Y = np.asarray(Y, dtype=np.float64)
        zd = zdec if zdec is not None else Z

        def sp(l):
            k = self.acts[l - 1]
            if k in (RELU, STEP):
                return act_prime(k, zd[l])
            return act_prime(k, Z[l])

        D = [None] * (self.L + 1)
        D[self.L] = (A[self.L] - Y) * sp(self.L)
        for l in range(self.L - 1, 0, -1):
            D[l] = (D[l + 1] @ Wb[l][0]) * sp(l)
        return D

    def tendencies(self, A, D) -> np.ndarray:
        """Flat [G_1 | g_1 | ... ]: G_l = D_l^T A_{l-1}, g_l = 1^T D_l (summed over the batch)."""
        out = []
        for l in range(1, self.L + 1):
            out.append((D[l].T @ A[l - 1]).ravel())
            out.append(D[l].sum(axis=0))
        return np.concatenate(out)

    def grad(self, params, X, Y, zdec=None) -> np.ndarray:
        A, Z = self.forward(params, X)
        return self.tendencies(A, self.backward(params, A, Z, Y, zdec))

    def train_batch(self, params, X, Y, eta: float, zdec=None):
        """One SGD step (train_batch P:460-476): returns (updated params fp64, mean pre-update
        cost 1/2 |a_L - y|^2 (reading R9), summed tendencies)."""
        p = self._p64(params)
        A, Z = self.forward(p, X)
        D = self.backward(p, A, Z, Y, zdec)
        G = self.tendencies(A, D)
        B = np.asarray(X).shape[0]
        loss = 0.5 * float(np.sum((A[-1] - np.asarray(Y, dtype=np.float64)) ** 2)) / B
        return p - (float(eta) / B) * G, loss, G

    def loss(self, params, X, Y) -> float:
        a = self.output(params, X)
        return 0.5 * float(np.sum((a - np.asarray(Y, dtype=np.float64)) ** 2)) / max(1, a.shape[0])

    def accuracy(self, params, X, Y) -> float:
        """Fraction with argmax a_L == argmax y, first index on ties (R10)."""
        a = self.output(params, X)
        if a.shape[0] == 0:
            return 0.0
        return float(np.mean(np.argmax(a, axis=1) == np.argmax(np.asarray(Y), axis=1)))

    # -- test helper: rows whose relu/step decisions are unambiguous --------------------
    def kink_free_rows(self, Z, margin_rel: float) -> np.ndarray:
        """Rows whose relu/step pre-activations all keep |z| > margin_rel * rms(Z_l) in every
        such layer (reading R8: inside that band an fp32 / TF32 sum and this fp64 sum may take
        the 0/1 decision differently; parity compares rows outside it)."""
        ok = np.ones(Z[1].shape[0], dtype=bool)
        for l in range(1, self.L + 1):
            if self.acts[l - 1] in (RELU, STEP):
                z = Z[l]
                m = margin_rel * float(np.sqrt(np.mean(z * z)))
                ok &= np.all(np.abs(z) > m, axis=1)
        return ok
