"""B200-native hot path of neural-fortran (Curcic, arXiv:1902.06714): minibatch SGD
training of a dense feed-forward network, behind the C-ABI of ``include/nf.h``.

This module is a thin ctypes binding: argument marshalling only.  Every step of
the method runs in the CUDA kernels of ``libnf_b200.so`` (built in-tree by
``paper_1902_06714_b200.build``).  There is no CPU fallback: if the library is
missing, the first call raises ImportError; if no sm_100 GPU is present, ``nf_net_create``
fails with ``NF_ENODEV``.

The functions carry the C names (``nf_net_create``, ``nf_output``,
``nf_train_batch``, ``nf_train_steps``, ``nf_grad``, ``nf_loss``,
``nf_accuracy``, ...).  Array arguments may be torch tensors (CUDA or CPU) or
numpy arrays; they must be contiguous fp32 (int64 for ``starts``).
``Net`` is a small object wrapper over the same calls.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libnf_b200.so")

NF_OK, NF_EINVAL, NF_ECUDA, NF_ENOMEM, NF_ENODEV = 0, -1, -2, -3, -4
# nf_load format errors (one code per kind) and file I/O
NF_EFMT_MAGIC, NF_EFMT_VERSION, NF_EFMT_PRECISION, NF_EFMT_TRUNCATED = -5, -6, -7, -8
NF_EFMT_ACTIVATION, NF_EFMT_DIMS, NF_EIO = -9, -10, -11
NF_MATH_FP32, NF_MATH_TF32, NF_MATH_FP64 = 0, 1, 2


class NFError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"nf error {code}: {msg}")
        self.code = code


def _load() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_1902_06714_b200.build` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    P, I64, I32, F, U64 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_float, ctypes.c_uint64
    sig = {
        "nf_net_create": (ctypes.c_int, [P, I32, ctypes.c_char_p, U64, ctypes.POINTER(P)]),
        "nf_net_destroy": (None, [P]),
        "nf_set_stream": (ctypes.c_int, [P, P]),
        "nf_set_math": (ctypes.c_int, [P, ctypes.c_int]),
        "nf_param_count": (I64, [P]),
        "nf_get_params": (ctypes.c_int, [P, P, I64]),
        "nf_set_params": (ctypes.c_int, [P, P, I64]),
        "nf_output": (ctypes.c_int, [P, P, I64, P]),
        "nf_train_batch": (ctypes.c_int, [P, P, P, I64, F]),
        "nf_train_steps": (ctypes.c_int, [P, P, P, I64, I64, P, I64, F, P]),
        "nf_grad": (ctypes.c_int, [P, P, P, I64, P]),
        "nf_grad_layers": (ctypes.c_int, [P, P, P, I64, P, P, I32]),
        "nf_update": (ctypes.c_int, [P, P, I64, F, I64]),
        "nf_save": (ctypes.c_int, [P, ctypes.c_char_p]),
        "nf_load": (ctypes.c_int, [ctypes.c_char_p, ctypes.POINTER(P)]),
        "nf_load_as": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_int, ctypes.POINTER(P)]),
        "nf_debug_log_enable": (None, [ctypes.c_int]),
        "nf_debug_log_read": (I64, [ctypes.c_char_p, I64]),
        "nf_loss": (ctypes.c_int, [P, P, P, I64, ctypes.POINTER(F)]),
        "nf_accuracy": (ctypes.c_int, [P, P, P, I64, ctypes.POINTER(F)]),
        "nf_last_error": (ctypes.c_char_p, []),
        "nf_launch_count": (I64, []),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype, fn.argtypes = res, args
    return lib


_lib = None


def lib() -> ctypes.CDLL:
    """The loaded libnf_b200.so.  Loaded on first use so that the build step can import
    ``paper_1902_06714_b200.build`` before the library exists; every C call goes through
    here and raises ImportError when the library is missing (no CPU fallback)."""
    global _lib
    if _lib is None:
        _lib = _load()
    return _lib

# Every symbol include/nf.h declares (checked by tests/test_abi.py).
EXPORTS = ("nf_net_create", "nf_net_destroy", "nf_set_stream", "nf_set_math", "nf_param_count",
           "nf_get_params", "nf_set_params", "nf_output", "nf_train_batch", "nf_train_steps",
           "nf_grad", "nf_grad_layers", "nf_update", "nf_save", "nf_load", "nf_load_as", "nf_loss", "nf_accuracy", "nf_last_error",
           "nf_launch_count", "nf_debug_log_enable", "nf_debug_log_read")


def _check(rc: int):
    if rc != NF_OK:
        raise NFError(rc, lib().nf_last_error().decode())


_TORCH_DT = {}


def _ptr(a, dtype=np.float32):
    """Data pointer of a contiguous torch tensor or numpy array (no copies)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        if a.dtype != dtype or not a.flags.c_contiguous:
            raise TypeError(f"expected a C-contiguous {np.dtype(dtype).name} array")
        return a.ctypes.data
    if hasattr(a, "data_ptr"):          # torch.Tensor
        want = _TORCH_DT.get(dtype)
        if want is None:
            import torch
            want = _TORCH_DT.setdefault(dtype, {np.float32: torch.float32, np.int64: torch.int64}[dtype])
        if a.dtype != want or not a.is_contiguous():
            raise TypeError(f"expected a contiguous {want} tensor")
        return a.data_ptr()
    raise TypeError(f"expected a C-contiguous {np.dtype(dtype).name} array or tensor")


# ---------------------------------------------------------------- C-named functions
def nf_net_create(dims, activation: str = "sigmoid", seed: int = 0):
    d = np.ascontiguousarray(np.asarray(dims, dtype=np.int32))
    out = ctypes.c_void_p()
    _check(lib().nf_net_create(d.ctypes.data_as(ctypes.c_void_p), len(d),
                              None if activation is None else activation.encode(), seed, ctypes.byref(out)))
    return out


def nf_net_destroy(net):
    lib().nf_net_destroy(net)


def nf_set_stream(net, stream):
    """stream: a torch.cuda.Stream, a raw cudaStream_t int, or None (legacy default)."""
    h = getattr(stream, "cuda_stream", stream)
    _check(lib().nf_set_stream(net, ctypes.c_void_p(h or 0)))


def nf_set_math(net, mode: int):
    _check(lib().nf_set_math(net, mode))


def nf_param_count(net) -> int:
    return int(lib().nf_param_count(net))


def nf_get_params(net, dst):
    _check(lib().nf_get_params(net, _ptr(dst), _numel(dst)))


def nf_set_params(net, src):
    _check(lib().nf_set_params(net, _ptr(src), _numel(src)))


def nf_output(net, x, n: int, out):
    _check(lib().nf_output(net, _ptr(x), n, _ptr(out)))


def nf_train_batch(net, x, y, n: int, eta: float):
    _check(lib().nf_train_batch(net, _ptr(x), _ptr(y), n, eta))


def nf_train_steps(net, X, Y, N: int, batch: int, starts, n_steps: int, eta: float, step_loss=None):
    _check(lib().nf_train_steps(net, _ptr(X), _ptr(Y), N, batch, _ptr(starts, np.int64), n_steps, eta,
                               _ptr(step_loss)))


def nf_grad(net, x, y, n: int, grad):
    _check(lib().nf_grad(net, _ptr(x), _ptr(y), n, _ptr(grad)))


def nf_grad_layers(net, x, y, n: int, grad, events):
    """events: one torch.cuda.Event (or raw cudaEvent_t int) per layer; events[l-1] is recorded
    when layer l's tendency block of grad is final (include/nf.h)."""
    handles = [int(getattr(e, "cuda_event", e) or 0) for e in events]
    arr = (ctypes.c_void_p * len(handles))(*handles)
    _check(lib().nf_grad_layers(net, _ptr(x), _ptr(y), n, _ptr(grad), ctypes.cast(arr, ctypes.c_void_p), len(handles)))


def nf_update(net, grad, count: int, eta: float, n: int):
    _check(lib().nf_update(net, _ptr(grad), count, eta, n))


def nf_save(net, path: str):
    _check(lib().nf_save(net, os.fsencode(path)))


def nf_load(path: str):
    h = ctypes.c_void_p()
    _check(lib().nf_load(os.fsencode(path), ctypes.byref(h)))
    return h


def nf_load_as(path: str, math: int):
    h = ctypes.c_void_p()
    _check(lib().nf_load_as(os.fsencode(path), math, ctypes.byref(h)))
    return h


def nf_debug_log_enable(on: bool = True):
    lib().nf_debug_log_enable(1 if on else 0)


def nf_debug_log_read() -> list[str]:
    """The launch log as a list of lines (see include/nf.h)."""
    need = int(lib().nf_debug_log_read(None, 0))
    buf = ctypes.create_string_buffer(need)
    lib().nf_debug_log_read(buf, need)
    return [l for l in buf.value.decode().split("\n") if l]


def nf_loss(net, x, y, n: int) -> float:
    v = ctypes.c_float()
    _check(lib().nf_loss(net, _ptr(x), _ptr(y), n, ctypes.byref(v)))
    return v.value


def nf_accuracy(net, x, y, n: int) -> float:
    v = ctypes.c_float()
    _check(lib().nf_accuracy(net, _ptr(x), _ptr(y), n, ctypes.byref(v)))
    return v.value


def nf_last_error() -> str:
    return lib().nf_last_error().decode()


def nf_launch_count() -> int:
    return int(lib().nf_launch_count())


def _numel(a) -> int:
    return int(a.numel()) if hasattr(a, "numel") else int(a.size)


# ---------------------------------------------------------------- object wrapper
class Net:
    """network_type(dims, activation) on the GPU."""

    def __init__(self, dims, activation: str = "sigmoid", seed: int = 0, stream=None):
        self.dims = [int(d) for d in dims]
        self.activation = activation
        self.h = nf_net_create(self.dims, activation, seed)
        if stream is not None:
            nf_set_stream(self.h, stream)

    def close(self):
        if getattr(self, "h", None):
            nf_net_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def n_params(self) -> int:
        return nf_param_count(self.h)

    def set_stream(self, stream):
        nf_set_stream(self.h, stream)

    def set_math(self, mode: int):
        nf_set_math(self.h, mode)

    def get_params(self, out=None):
        if out is None:
            out = np.empty(self.n_params, np.float32)
        nf_get_params(self.h, out)
        return out

    def set_params(self, p):
        nf_set_params(self.h, p)

    def output(self, x, out=None):
        n = x.shape[0]
        if out is None:
            out = _empty_like_rows(x, n, self.dims[-1])
        nf_output(self.h, x, n, out)
        return out

    def train_batch(self, x, y, eta: float):
        nf_train_batch(self.h, x, y, x.shape[0], eta)

    def train_steps(self, X, Y, batch: int, starts, eta: float, step_loss=None):
        if not (isinstance(starts, np.ndarray) and starts.dtype == np.int64 and starts.flags.c_contiguous):
            starts = np.ascontiguousarray(np.asarray(starts, dtype=np.int64))
        nf_train_steps(self.h, X, Y, X.shape[0], batch, starts, len(starts), eta, step_loss)

    def grad(self, x, y, out=None):
        if out is None:
            out = _empty_like_rows(x, self.n_params, None)
        nf_grad(self.h, x, y, x.shape[0], out)
        return out

    def grad_layers(self, x, y, out, events):
        """nf_grad into `out`, recording events[l-1] when layer l's block is final."""
        nf_grad_layers(self.h, x, y, x.shape[0], out, events)
        return out

    def layer_slices(self):
        """(offset, count) of each layer's W_l, b_l block in the flat layout, l = 1..L."""
        out, o = [], 0
        for l in range(1, len(self.dims)):
            c = self.dims[l] * self.dims[l - 1] + self.dims[l]
            out.append((o, c))
            o += c
        return out

    def update(self, grad, eta: float, n: int):
        """params -= (eta / n) grad: the paper's update on co_summed tendencies (nf_update)."""
        nf_update(self.h, grad, self.n_params, eta, n)

    def save(self, path: str):
        """Write the net (dims, activation spec, parameters) to a file (nf_save)."""
        nf_save(self.h, path)

    @classmethod
    def load(cls, path: str, stream=None, math: int | None = None):
        """A Net from a file written by save() (nf_load; with math: nf_load_as, which rejects a
        file of another precision)."""
        net = cls.__new__(cls)
        net.h = nf_load(path) if math is None else nf_load_as(path, math)
        with open(path) as f:
            f.readline(); f.readline()
            net.dims = [int(v) for v in f.readline().split()]
            net.activation = f.readline().strip()
        if stream is not None:
            nf_set_stream(net.h, stream)
        return net

    def loss(self, x, y) -> float:
        return nf_loss(self.h, x, y, x.shape[0])

    def accuracy(self, x, y) -> float:
        return nf_accuracy(self.h, x, y, x.shape[0])


def _empty_like_rows(x, n, w):
    shape = (n,) if w is None else (n, w)
    if hasattr(x, "data_ptr"):
        import torch
        return torch.empty(shape, dtype=torch.float32, device=x.device)
    return np.empty(shape, np.float32)
