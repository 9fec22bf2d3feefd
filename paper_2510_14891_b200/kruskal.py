"""Kruskal tensors: weights plus one row-major factor matrix per mode.

Container contract of cpkern.kruskal.KruskalTensor (pkg/src/cpkern/kruskal.py:
25-58): weights (R,) finite and >= 0, factors A_m (I_m, R) row-major float64.
Factors may be numpy arrays or CUDA torch tensors; kernels read cached device
copies.  Gram / Hadamard / norm run on the device through the C ABI.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from ._device import require_cuda, stream_ptr
from .errors import IndexRangeError, ShapeError


def _is_torch(x) -> bool:
    return isinstance(x, torch.Tensor)


def _as_factor(a, what="factor"):
    if _is_torch(a):
        a = a.detach()
        if a.dtype != torch.float64:
            a = a.to(torch.float64)
        if a.dim() != 2 or a.shape[0] < 1 or a.shape[1] < 1:
            raise ShapeError(f"{what} must be a 2-D matrix with at least one row and column")
        return a.contiguous()
    a = np.ascontiguousarray(a, dtype=np.float64)
    if a.ndim != 2 or a.shape[0] < 1 or a.shape[1] < 1:
        raise ShapeError(f"{what} must be a 2-D matrix with at least one row and column")
    return a


def _all_finite(x) -> bool:
    if _is_torch(x):
        return bool(torch.isfinite(x).all().item())
    return bool(np.all(np.isfinite(x)))


class KruskalTensor:
    """Rank-R factored tensor: weights (R,) and factors A_m (I_m, R)."""

    __slots__ = ("weights", "factors", "_dev")

    def __init__(self, weights, factors, validate=True):
        self.factors = [_as_factor(a, f"factor {m + 1}") for m, a in enumerate(factors)]
        if not self.factors:
            raise ShapeError("need at least one factor matrix")
        if _is_torch(weights):
            self.weights = weights.detach().to(torch.float64).reshape(-1).contiguous()
        else:
            self.weights = np.ascontiguousarray(weights, dtype=np.float64).ravel()
        self._dev = None
        if validate:
            r = self.factors[0].shape[1]
            for m, a in enumerate(self.factors):
                if a.shape[1] != r:
                    raise ShapeError(f"factor {m + 1} has {a.shape[1]} columns, expected {r}")
            if tuple(self.weights.shape) != (r,):
                raise ShapeError(f"weights must have shape ({r},), got {tuple(self.weights.shape)}")
            w = self.weights
            if not _all_finite(w) or bool((w < 0).any()):
                raise ShapeError("weights must be finite and nonnegative")
            for m, a in enumerate(self.factors):
                if not _all_finite(a):
                    raise ShapeError(f"factor {m + 1} has non-finite entries")

    @property
    def rank(self) -> int:
        return int(self.factors[0].shape[1])

    @property
    def ndim(self) -> int:
        return len(self.factors)

    @property
    def dims(self) -> tuple:
        return tuple(int(a.shape[0]) for a in self.factors)

    def device_factors(self, device=None):
        """Device copies (contiguous float64) of all factors.

        CUDA float64 factors are used in place.  Other torch factors are
        converted once and the copy is reused while the source tensor is the
        same object at the same address and version (no in-place write since);
        numpy factors are uploaded on every call -- they are I_m x R, and the
        reference packs them on every call too (`pack_factors`,
        _kernels.py:25-36) -- so reassigning `factors[k]` or writing into
        one is always seen."""
        dev = require_cuda(device)
        if self._dev is None or self._dev[0] != dev:
            self._dev = [dev, {}]
        cache = self._dev[1]
        return [self._device_copy(cache, ("A", m), a, dev) for m, a in enumerate(self.factors)]

    def device_weights(self, device=None):
        dev = require_cuda(device)
        if self._dev is None or self._dev[0] != dev:
            self._dev = [dev, {}]
        return self._device_copy(self._dev[1], "lam", self.weights, dev)

    @staticmethod
    def _device_copy(cache, slot, a, dev):
        if not _is_torch(a):
            cache.pop(slot, None)
            return _to_device(a, dev)
        key = (id(a), a.data_ptr(), a._version)
        hit = cache.get(slot)
        if hit is not None and hit[0] == key:
            return hit[1]
        t = _to_device(a, dev)
        cache[slot] = (key, t)
        return t

    def hadamard_gram(self, skip=None):
        """(*) of the factor Grams, optionally skipping one mode (kruskal.py:74-83)."""
        if skip is not None and not 0 <= int(skip) < self.ndim:
            raise IndexRangeError(f"mode {skip} out of range [0, {self.ndim - 1}]")
        dev = require_cuda()
        grams = [gram(a) for a in self.device_factors(dev)]
        return hadamard(grams, -1 if skip is None else int(skip))

    def norm_squared(self) -> float:
        """||M||_F^2 = lam^T (hadamard of all Grams) lam (kruskal.py:85-88)."""
        h = self.hadamard_gram()
        lam = self.device_weights()
        return float((lam @ h @ lam).item())

    def __repr__(self):
        return f"KruskalTensor(rank={self.rank}, dims={self.dims})"


def _to_device(x, dev) -> torch.Tensor:
    if _is_torch(x):
        return x.to(dev, dtype=torch.float64).contiguous()
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).to(dev)


def gram(a, out: torch.Tensor | None = None) -> torch.Tensor:
    """A^T A on the device, symmetrized exactly (kruskal.py:110-114)."""
    dev = require_cuda()
    a = _to_device(_as_factor(a), dev)
    r = a.shape[1]
    if out is None:
        out = torch.empty((r, r), dtype=torch.float64, device=dev)
    _lib.check(
        _lib.load().cpk_gram_f64(a.data_ptr(), a.shape[0], r, a.stride(0), out.data_ptr(), stream_ptr(dev)),
        "gram",
    )
    return out


def hadamard(grams, skip: int = -1, out: torch.Tensor | None = None) -> torch.Tensor:
    """Elementwise product of R x R device Grams in ascending mode order,
    skipping `skip` (cpals.py:129-132)."""
    dev = grams[0].device
    r = grams[0].shape[0]
    if out is None:
        out = torch.empty((r, r), dtype=torch.float64, device=dev)
    ptrs = _lib.ptr_array([g.data_ptr() if (g is not None and m != skip) else 0 for m, g in enumerate(grams)])
    _lib.check(
        _lib.load().cpk_hadamard_f64(ptrs, len(grams), int(skip), r, out.data_ptr(), stream_ptr(dev)),
        "hadamard",
    )
    return out
