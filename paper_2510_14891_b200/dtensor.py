"""Dense d-way tensors, flat float64 in first-mode-fastest (column-major) order.

Same layout contract as cpkern.dtensor (pkg/src/cpkern/dtensor.py:1-10,
226-278): element (i_0, ..., i_{d-1}) lives at sum_m i_m * prod_{l<m} I_l.
The payload may be a host numpy array (the reference's type) or a CUDA
torch tensor.  Kernels always read a device copy; a host payload is copied
to the device once and the copy is cached on the object (inputs are never
mutated, test_cpals.py:180-184), so repeated MTTKRPs in CP-ALS do not
re-stage the tensor.
"""

from __future__ import annotations

import numpy as np
import torch

from ._device import require_cuda
from .errors import IndexRangeError, ParameterError, ShapeError


def check_dims(dims) -> tuple:
    """Validate a shape and return it as a tuple of ints (dtensor.py:29-44)."""
    try:
        out = tuple(int(x) for x in dims)
    except (TypeError, ValueError) as exc:
        raise ShapeError(f"shape must be a sequence of integers, got {dims!r}") from exc
    if len(out) < 1:
        raise ShapeError("shape needs at least one mode")
    if any(x < 1 for x in out):
        raise ShapeError(f"every extent must be >= 1, got {out}")
    n = 1
    for x in out:
        n *= x
    if n >= 2 ** 63:
        raise ShapeError(f"volume {n} does not fit in a signed 64-bit index")
    return out


def num_elements(dims) -> int:
    n = 1
    for x in dims:
        n *= int(x)
    return n


def col_major_strides(dims) -> tuple:
    """Flat-index stride of each mode; stride of mode 0 is 1 (dtensor.py:54-61)."""
    strides = []
    s = 1
    for x in dims:
        strides.append(s)
        s *= int(x)
    return tuple(strides)


def _is_torch(x) -> bool:
    return isinstance(x, torch.Tensor)


def _payload_key(x):
    """Identity of a payload for cache validation: the object, its buffer
    address and (torch) its in-place version counter."""
    if _is_torch(x):
        return (id(x), x.data_ptr(), x._version)
    return (id(x), x.__array_interface__["data"][0])


class DenseTensor:
    """Dense tensor backed by one flat float64 buffer in first-mode-fastest order."""

    __slots__ = ("dims", "data", "_dev", "_landing", "_even", "_src")

    def __init__(self, dims, data, copy=False):
        self.dims = check_dims(dims)
        n = num_elements(self.dims)
        if _is_torch(data):
            arr = data.detach()
            if arr.dtype != torch.float64:
                arr = arr.to(torch.float64)
            arr = arr.reshape(-1)
            if not arr.is_contiguous():
                arr = arr.contiguous()
            if copy:
                arr = arr.clone()
        else:
            arr = np.asarray(data, dtype=np.float64)
            arr = (arr.copy() if copy else arr).ravel()
        size = arr.numel() if _is_torch(arr) else arr.size
        if size != n:
            raise ShapeError(f"data has {size} elements, shape {self.dims} needs {n}")
        self.data = arr
        self._dev = arr if (_is_torch(arr) and arr.is_cuda) else None
        self._landing = None  # (slab bounds, copy events) while a streamed upload is in flight
        self._even = None  # zero-padded copy with an even first extent (even_device_data)
        self._src = _payload_key(arr)  # which payload the cached device copies were made from

    @classmethod
    def zeros(cls, dims) -> "DenseTensor":
        dims = check_dims(dims)
        return cls(dims, np.zeros(num_elements(dims)))

    @classmethod
    def from_ndarray(cls, arr) -> "DenseTensor":
        """Copy a numpy array; axis 0 becomes the fastest-varying mode."""
        arr = np.asarray(arr, dtype=np.float64)
        return cls(arr.shape, arr.ravel(order="F"))

    @classmethod
    def uniform(cls, dims, seed: int = 0, device=None) -> "DenseTensor":
        """Synthetic U[0,1) tensor generated on the device by the counter-based
        generator of cpk_fill_uniform_f64 (CPU twin: oracle/gen.py), for
        shapes too large to stage through the host."""
        from . import _lib

        dims = check_dims(dims)
        dev = require_cuda(device)
        n = num_elements(dims)
        buf = torch.empty(n, dtype=torch.float64, device=dev)
        with torch.cuda.device(dev):
            from ._device import stream_ptr

            _lib.check(
                _lib.load().cpk_fill_uniform_f64(buf.data_ptr(), n, int(seed), 0, stream_ptr(dev)),
                "fill_uniform",
            )
        return cls(dims, buf)

    @property
    def ndim(self) -> int:
        return len(self.dims)

    @property
    def size(self) -> int:
        return num_elements(self.dims)

    @property
    def is_device(self) -> bool:
        return _is_torch(self.data) and self.data.is_cuda

    def _check_cache(self) -> None:
        """Drop the cached device copies when `data` is no longer the payload
        they were made from: reassigned, or (torch payloads) modified in
        place (tensor version counter).  An in-place write into a host
        *numpy* payload after the first GPU call cannot be seen; call
        `invalidate()` after one (the reference object holds no cache)."""
        key = _payload_key(self.data)
        if key != self._src:
            self.invalidate()
            self._src = key

    def invalidate(self) -> None:
        """Forget every device copy of a host payload (re-uploaded on next use)."""
        cuda_payload = _is_torch(self.data) and self.data.is_cuda
        self._dev = self.data.reshape(-1) if cuda_payload else None
        self._landing = None
        self._even = None

    def device_data(self, device=None, wait: bool = True) -> torch.Tensor:
        """The flat float64 payload on the CUDA device (cached H2D copy).

        While a streamed upload is in flight the current stream is made to
        wait for it (``wait=False``: the caller orders itself on the slab
        events)."""
        dev = require_cuda(device)
        self._check_cache()
        if self._dev is not None and self._dev.device == dev:
            if wait and self.landing is not None:
                torch.cuda.current_stream(dev).wait_event(self._landing[1][-1])
            return self._dev
        if _is_torch(self.data):
            t = self.data.to(dev, non_blocking=False)
        else:
            host = torch.from_numpy(np.ascontiguousarray(self.data))
            t = host.to(dev, non_blocking=False)
        self._dev = t
        return t

    def needs_upload(self, device=None) -> bool:
        """True when the payload lives on the host and no device copy is cached."""
        dev = require_cuda(device)
        self._check_cache()
        return not (self._dev is not None and self._dev.device == dev)

    def host_view(self) -> torch.Tensor:
        """The host payload as a flat float64 torch tensor (no copy when the
        payload is already contiguous; pinned if the caller pinned it)."""
        if _is_torch(self.data):
            return self.data.reshape(-1)
        return torch.from_numpy(np.ascontiguousarray(self.data).reshape(-1))

    def cache_device(self, t: torch.Tensor, landing=None) -> None:
        """Adopt `t` (flat float64 CUDA, same contents) as the device copy;
        `landing` = (slab bounds along the slowest mode, copy events) while
        the copy is still in flight."""
        self._dev = t
        self._landing = landing

    @property
    def landing(self):
        """(bounds, events) of an upload still in flight, else None."""
        if self._landing is not None and self._landing[1][-1].query():
            self._landing = None  # every slab has landed
        return self._landing

    def even_device_data(self, device=None) -> torch.Tensor:
        """A device copy with I_0 padded to I_0 + 1 by a zero slice (cached).

        The TMA kernels need 16-byte strides, i.e. an even I_0.  Zero
        elements contribute nothing to any MTTKRP, so the padded tensor
        gives the same G for every mode k > 0, and G's first I_0 rows for
        k = 0, with A_0 extended by any one row."""
        dev = require_cuda(device)
        self._check_cache()
        if self._even is None or self._even.device != dev:
            i0 = self.dims[0]
            src = self.device_data(dev).view(-1, i0)
            pad = torch.zeros((src.shape[0], i0 + 1), dtype=torch.float64, device=dev)
            pad[:, :i0] = src
            self._even = pad.view(-1)
        return self._even

    def to_ndarray(self) -> np.ndarray:
        """The data as a numpy array with axis 0 fastest (host copy if on device)."""
        host = self.data.detach().cpu().numpy() if _is_torch(self.data) else self.data
        return host.reshape(self.dims, order="F")

    def reshape(self, new_dims) -> "DenseTensor":
        new_dims = check_dims(new_dims)
        if num_elements(new_dims) != self.size:
            raise ShapeError(f"cannot reshape volume {self.size} to {new_dims}")
        return DenseTensor(new_dims, self.data)

    def copy(self) -> "DenseTensor":
        return DenseTensor(self.dims, self.data, copy=True)

    def norm(self) -> float:
        """Frobenius norm, computed on the device (deterministic reduction)."""
        from . import _lib
        from ._device import stream_ptr, workspace

        dev = require_cuda()
        x = self.device_data(dev)
        out = torch.empty(1, dtype=torch.float64, device=dev)
        work = workspace(dev, 8 * _lib.CPK_SUMSQ_PARTIALS, tag="sumsq")
        _lib.check(
            _lib.load().cpk_sumsq_f64(x.data_ptr(), x.numel(), work.data_ptr(), out.data_ptr(), stream_ptr(dev)),
            "sumsq",
        )
        return float(out.sqrt().item())

    def __repr__(self):
        where = "cuda" if self.is_device else "host"
        return f"DenseTensor(dims={self.dims}, {where})"


def check_mode(ndim: int, mode: int) -> int:
    mode = int(mode)
    if not 0 <= mode < ndim:
        raise IndexRangeError(f"mode {mode} out of range [0, {ndim - 1}]")
    return mode


# ------------------------------------------------------------------ DTEN v1
# dtensor.py:334-382: "DTEN", u32 version 1, u32 d, u64 dims[d], u32 element
# type 1 (float64), then the float64 payload first mode fastest.
DTEN_MAGIC = b"DTEN"
DTEN_VERSION = 1
DTEN_FLOAT64 = 1


def write_dten(path, t: DenseTensor) -> None:
    """Write a tensor as a DTEN v1 file (dtensor.py:334-340)."""
    import struct

    data = t.data.detach().cpu().numpy() if isinstance(t.data, torch.Tensor) else t.data
    with open(path, "wb") as f:
        f.write(struct.pack("<4sII", DTEN_MAGIC, DTEN_VERSION, t.ndim))
        f.write(struct.pack(f"<{t.ndim}Q", *t.dims))
        f.write(struct.pack("<I", DTEN_FLOAT64))
        f.write(np.ascontiguousarray(data, dtype="<f8").tobytes())


def read_dten_header(path) -> tuple:
    """Shape recorded in a DTEN file, without reading the payload
    (dtensor.py:343-347); parsed and validated by the native reader."""
    import ctypes

    from . import _lib

    d = ctypes.c_int(0)
    dims = (ctypes.c_int64 * _lib.CPK_DTEN_MAX_MODES)()
    _lib.check(_lib.load().cpk_dten_read_header(str(path).encode(), ctypes.byref(d), dims), "DTEN header")
    return tuple(int(dims[i]) for i in range(d.value))


def read_dten(path, device=None, mode: int = 0, lo: int | None = None, hi: int | None = None) -> DenseTensor:
    """Read a DTEN file (dtensor.py:350-357).

    ``device=None``: host payload, like the reference.  With a CUDA device
    the payload goes straight to HBM through the native loader
    (cpk_dten_load_slab_f64: threaded preads into pinned staging buffers,
    double-buffered async copies) and, with ``lo``/``hi``, only the slab
    [lo, hi) along ``mode`` is read -- one rank's shard of the sharded
    CP-ALS driver, as its own first-mode-fastest tensor.
    """
    from . import _lib
    from ._device import stream_ptr

    dims = read_dten_header(path)
    mode = check_mode(len(dims), mode)
    lo = 0 if lo is None else int(lo)
    hi = dims[mode] if hi is None else int(hi)
    if not 0 <= lo <= hi <= dims[mode]:
        raise IndexRangeError(f"slab [{lo}, {hi}) outside [0, {dims[mode]})")
    sub = tuple(hi - lo if m == mode else e for m, e in enumerate(dims))
    n = num_elements(sub) if hi > lo else 0
    if device is None:
        if (lo, hi) != (0, dims[mode]):
            raise ParameterError("host reads load the whole tensor; pass a CUDA device for a slab")
        off = 12 + 8 * len(dims) + 4
        data = np.fromfile(path, dtype="<f8", offset=off).astype(np.float64)
        if data.size != num_elements(dims):
            from .errors import FormatError

            raise FormatError(f"payload holds {8 * data.size} bytes, shape {dims} needs {8 * num_elements(dims)}")
        return DenseTensor(dims, data)
    dev = require_cuda(device)
    if n == 0:
        raise ShapeError(f"empty slab [{lo}, {hi}) of mode {mode}")
    buf = torch.empty(n, dtype=torch.float64, device=dev)
    with torch.cuda.device(dev):
        _lib.check(
            _lib.load().cpk_dten_load_slab_f64(str(path).encode(), mode, lo, hi, buf.data_ptr(), n, 0,
                                               stream_ptr(dev)),
            "DTEN load",
        )
    return DenseTensor(sub, buf)
