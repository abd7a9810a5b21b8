"""Batched condensation log-determinant: one CTA per small matrix (K3).

No reference counterpart; its oracle is a loop of
mcnd.logdet_condensation (condense.py:134-160) over the batch, and the
pivots it takes are bitwise the reference's in the default mode.

``logdet_batched(a)`` takes a (B, n, n) float64 array (numpy: H2D inside the
call; CUDA torch tensor: used in place) with n <= 128 and returns
``(signs, log_abs)`` arrays of length B (numpy for numpy input, torch CUDA
tensors for torch input).  Singular matrices give sign 0 and -inf.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .condense import _is_torch_cuda


def logdet_batched(a, *, fast: bool = False, return_pivots: bool = False):
    lib = _lib.load()
    flags = _lib.FLAG_FAST if fast else 0
    if _is_torch_cuda(a):
        import torch

        if a.dim() != 3 or a.shape[1] != a.shape[2]:
            raise ValueError("expected a (B, n, n) batch of square matrices")
        a = a.to(torch.float64).contiguous()
        b, n, _ = a.shape
        signs = torch.empty(b, dtype=torch.int32, device=a.device)
        logs = torch.empty(b, dtype=torch.float64, device=a.device)
        piv = torch.empty((b, n), dtype=torch.float64, device=a.device) if return_pivots else None
        flag = torch.zeros(1, dtype=torch.int32, device=a.device)
        stream = torch.cuda.current_stream(a.device).cuda_stream
        rc = lib.mcnd_logdet_batched_dev(a.data_ptr(), b, n, n * n, flags, stream, signs.data_ptr(),
                                         logs.data_ptr(), piv.data_ptr() if piv is not None else None,
                                         flag.data_ptr())
        _lib.check(rc)
        if int(flag.item()):  # finiteness is checked on the device, fused into the load
            raise ValueError("matrix entries must be finite (no NaN/Inf)")
        return (signs, logs, piv) if return_pivots else (signs, logs)
    a = np.ascontiguousarray(a, dtype=np.float64)
    if a.ndim != 3 or a.shape[1] != a.shape[2]:
        raise ValueError("expected a (B, n, n) batch of square matrices")
    if a.shape[1] == 0:
        raise ValueError("matrix dimensions must be positive")
    b, n, _ = a.shape
    signs = np.zeros(b, dtype=np.int32)
    logs = np.zeros(b, dtype=np.float64)
    rc = lib.mcnd_logdet_batched(a.ctypes.data, b, n, n * n, flags, None, signs.ctypes.data, logs.ctypes.data)
    _lib.check(rc)
    return signs, logs
