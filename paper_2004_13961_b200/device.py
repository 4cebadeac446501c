"""Device-buffer plumbing (torch owns device memory and streams)."""

from __future__ import annotations

import numpy as np

from . import _lib


def torch():
    import torch as _t
    return _t


def is_device(a):
    t = torch()
    return isinstance(a, t.Tensor) and a.is_cuda


_PINNED = {}


def _pinned(n):
    """Cached page-locked staging buffer of n doubles (host side of the copies)."""
    t = torch()
    buf = _PINNED.get(n)
    if buf is None:
        if len(_PINNED) > 8:
            _PINNED.clear()
        buf = t.empty(n, dtype=t.float64, pin_memory=True)
        _PINNED[n] = buf
    return buf


def to_device(a):
    """float64 contiguous CUDA tensor holding `a` (numpy/torch) in memory order.
    Large host arrays go through a page-locked staging buffer (one DMA)."""
    t = torch()
    _lib.load()
    if isinstance(a, t.Tensor):
        return a.to(device="cuda", dtype=t.float64).contiguous()
    arr = np.ascontiguousarray(a, dtype=np.float64)
    if arr.size >= (1 << 16):
        st = _pinned(arr.size)
        st.numpy()[:] = arr.reshape(-1)
        out = st.to("cuda", non_blocking=True).reshape(arr.shape)
        t.cuda.current_stream().synchronize()   # the staging buffer is reused
        return out
    return t.from_numpy(arr).to("cuda", non_blocking=False)


def empty(n):
    t = torch()
    _lib.load()
    return t.empty(int(n), dtype=t.float64, device="cuda")


def ptr(tensor):
    return tensor.data_ptr() if tensor is not None else None


def host(tensor):
    return tensor.detach().cpu().numpy()


def fortran_flat(data):
    """K^d tensor (axis 0 = x) -> x-fastest flat layout (pcg.py:135)."""
    if is_device(data):
        d = data.dim()
        return data.permute(*reversed(range(d))).contiguous().reshape(-1)
    return np.asarray(data, dtype=float).flatten(order="F")


def from_fortran_flat(flat, K, d):
    """x-fastest flat vector -> K^d C-order ndarray / tensor with axis 0 = x."""
    if is_device(flat):
        v = flat.reshape((K,) * d)
        return v.permute(*reversed(range(d))).contiguous()
    return np.ascontiguousarray(np.asarray(flat).reshape((K,) * d, order="F"))
