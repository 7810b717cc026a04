"""Host -> device staging helpers (plumbing only; all compute is in libp3d.so)."""

from __future__ import annotations

import functools

import numpy as np
import torch

from . import _lib

DEV = "cuda"


def dev(x, dtype):
    """numpy / list / tensor -> contiguous CUDA tensor of `dtype` (copies only if needed)."""
    if isinstance(x, torch.Tensor):
        t = x
        if t.dtype != dtype:
            t = t.to(dtype)
        if not t.is_cuda:
            t = t.to(DEV)
        return t.contiguous()
    a = np.ascontiguousarray(np.asarray(x))
    if not a.flags.writeable:  # e.g. np.broadcast_to views
        a = a.copy()
    return torch.from_numpy(a).to(device=DEV, dtype=dtype).contiguous()


def f64(x):
    return dev(x, torch.float64)


def i32(x):
    return dev(x, torch.int32)


def u8(x):
    if isinstance(x, torch.Tensor):
        return x.to(device=DEV, dtype=torch.uint8).contiguous()
    return dev(np.asarray(x).astype(np.uint8), torch.uint8)


def stable_argsort(a):
    """np.argsort(a, kind="stable") of a 1-D integer array, computed on the
    device (host setup of the loop layouts: the stable order is unique, so
    the result is the same permutation)."""
    a = np.ascontiguousarray(np.asarray(a))
    if a.size < (1 << 16) or not torch.cuda.is_available():
        return np.argsort(a, kind="stable")
    t = torch.from_numpy(a).to(DEV)
    return torch.argsort(t, stable=True).cpu().numpy().astype(np.int64, copy=False)


def host(x):
    """Tensor -> numpy (for the reference-shaped return values of the loop driver)."""
    if isinstance(x, torch.Tensor):
        return x.detach().cpu().numpy()
    return np.asarray(x)


def zeros(n, dtype=torch.float64):
    return torch.zeros(int(max(n, 1)), dtype=dtype, device=DEV)


def scratch(n_doubles):
    """Zeroed reduction scratch (the C side resets its ticket counters)."""
    return torch.zeros(int(n_doubles), dtype=torch.float64, device=DEV)


def sync_scalar(t):
    return float(t.item())


class Keep:
    """Holds tensors alive for as long as a ctypes struct points at them."""

    def __init__(self):
        self.items = []

    def __call__(self, t):
        self.items.append(t)
        return _lib.ptr(t)


def _numpy_arg(a):
    if isinstance(a, (np.ndarray, list, tuple)):
        return True
    x = getattr(a, "x", None)  # a charge cloud of numpy arrays
    return isinstance(x, np.ndarray) and hasattr(a, "weight")


def _to_host(out):
    if isinstance(out, torch.Tensor):
        return out.detach().cpu().numpy()
    if isinstance(out, tuple):
        return tuple(_to_host(o) for o in out)
    if isinstance(out, list):
        return [_to_host(o) for o in out]
    return out


def numpy_io(*names):
    """Per-op drop-in convention: when the caller passes its data arrays (the
    arguments `names`) as numpy arrays, as the reference's callers do, the
    results come back as numpy arrays; CUDA tensors in, CUDA tensors out.  The
    computation is on the device either way."""
    import inspect

    def deco(fn):
        sig = inspect.signature(fn)

        @functools.wraps(fn)
        def wrapper(*args, **kw):
            out = fn(*args, **kw)
            b = sig.bind_partial(*args, **kw).arguments
            if any(_numpy_arg(b.get(n)) for n in names):
                return _to_host(out)
            return out

        return wrapper

    return deco
