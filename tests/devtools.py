"""Test-side device helpers (plain torch, no method arithmetic).

* dev_view(ptr, n, dtype): a torch CUDA tensor aliasing n elements at a raw
  device pointer handed out by the table hook (gbe_set_table_hook);
* mixsum(t, salt): the position-keyed checksum oracle.mixsum computes on the
  host (sum over i of mix(i * A + x_i + salt * C) mod 2^64), formed with
  int64 torch ops on whatever device t lives on, in chunks;
* near_tie_ok: the A10 reading for f64 argmin disagreements.
"""
from __future__ import annotations

import numpy as np
import torch

_A = 0x9E3779B97F4A7C15 - (1 << 64)
_B = 0xBF58476D1CE4E5B9 - (1 << 64)
_C = 0xD1B54A32D192ED03
_M64 = (1 << 64) - 1


def _s64(x: int) -> int:
    x &= _M64
    return x - (1 << 64) if x >= (1 << 63) else x


_TYPESTR = {torch.int32: "<i4", torch.uint8: "|u1", torch.float64: "<f8", torch.int64: "<i8"}


class _Cai:
    def __init__(self, ptr, n, dtype):
        self.__cuda_array_interface__ = {"shape": (int(n),), "typestr": _TYPESTR[dtype],
                                         "data": (int(ptr), False), "version": 3, "strides": None}


def dev_view(ptr, n, dtype) -> torch.Tensor:
    """n elements of `dtype` at device pointer ptr (no copy)."""
    if n == 0:
        return torch.empty(0, dtype=dtype, device="cuda")
    return torch.as_tensor(_Cai(ptr, n, dtype), device="cuda")


def _bits(t: torch.Tensor) -> torch.Tensor:
    if t.dtype == torch.uint8:
        return t.to(torch.int64)
    if t.dtype == torch.int32:
        return t.to(torch.int64) & 0xFFFFFFFF
    if t.dtype == torch.float64:
        return t.view(torch.int64)
    if t.dtype == torch.int64:
        return t
    raise TypeError(t.dtype)


def mixsum(t: torch.Tensor, salt: int, chunk: int = 1 << 27) -> int:
    """oracle.mixsum on a 1-D tensor (any device): returns an int in [0, 2^64)."""
    n = t.numel()
    t = t.reshape(-1)
    h = 0
    saltc = _s64(salt * _C)
    for s in range(0, n, chunk):
        x = _bits(t[s:s + chunk])
        i = torch.arange(s, s + x.numel(), dtype=torch.int64, device=t.device)
        z = i * _A + x + saltc
        z = (z ^ ((z >> 31) & ((1 << 33) - 1))) * _B
        z = z ^ ((z >> 29) & ((1 << 35) - 1))
        h = (h + int(z.sum().item())) & _M64
        del x, i, z
    return h


def mix_digest(out: torch.Tensor, arg: torch.Tensor) -> int:
    """Digest kind 1 of oracle.mix_digest: mixsum(out, 1) + mixsum(arg, 2)."""
    return (mixsum(out, 1) + mixsum(arg, 2)) & _M64


def near_tie_ok(sums: np.ndarray, a_gpu: np.ndarray, a_or: np.ndarray, rel=1e-9) -> np.ndarray:
    """Reading A10: an f64 argmin that differs from the oracle's is accepted
    only when the oracle's own sums of the two choices (sums[q, v], from
    oracle.bucket_row_sums) agree within rel (relative; absolute near 0)."""
    q = np.arange(len(a_gpu))
    sg = sums[q, a_gpu]
    so = sums[q, a_or]
    both_inf = np.isinf(sg) & np.isinf(so)
    return both_inf | (np.abs(sg - so) <= rel * np.maximum(1.0, np.maximum(np.abs(sg), np.abs(so))))
