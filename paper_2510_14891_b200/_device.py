"""Device plumbing: CUDA availability, streams, workspaces, event timers.

PyTorch is used only for device memory (its caching allocator), streams and
events; all arithmetic on the hot path goes through the C ABI (_lib.py).
"""

from __future__ import annotations

import threading

import torch

from .errors import DeviceError

_ws_lock = threading.Lock()
_workspaces: dict = {}


def require_cuda(device=None) -> torch.device:
    if not torch.cuda.is_available():
        raise DeviceError("CUDA is not available: the B200 package has no CPU fallback")
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    dev = torch.device(device)
    if dev.type != "cuda":
        raise DeviceError(f"expected a CUDA device, got {dev}")
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    return dev


def stream_ptr(device: torch.device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def workspace(device: torch.device, nbytes: int, tag: str = "mttkrp") -> torch.Tensor:
    """Grow-only scratch buffer per (device, tag, current stream), float64.

    Keyed on the stream, so only calls ordered on one stream share a buffer:
    stream order serializes them, and calls on other streams (or threads
    using other streams) get buffers of their own.  A buffer is allocated
    while its stream is current, so when it grows the caching allocator
    recycles the old block in that same stream's order.
    """
    if nbytes <= 0:
        return None
    key = (device.index, tag, torch.cuda.current_stream(device).cuda_stream)
    with _ws_lock:
        buf = _workspaces.get(key)
        if buf is None or buf.numel() * 8 < nbytes:
            n = max(nbytes, int(buf.numel() * 8 * 1.25) if buf is not None else 0)
            buf = torch.empty((n + 7) // 8, dtype=torch.float64, device=device)
            _workspaces[key] = buf
        return buf


def release_workspaces() -> None:
    with _ws_lock:
        _workspaces.clear()


class EventTimer:
    """CUDA-event interval on the launching stream; reads lazily (one sync
    on first access), so timing never adds a host sync to the hot loop."""

    __slots__ = ("_start", "_end", "_seconds")

    def __init__(self, device: torch.device):
        self._start = torch.cuda.Event(enable_timing=True)
        self._end = torch.cuda.Event(enable_timing=True)
        self._start.record(torch.cuda.current_stream(device))
        self._seconds = None

    def stop(self, device: torch.device) -> "EventTimer":
        self._end.record(torch.cuda.current_stream(device))
        return self

    @property
    def seconds(self) -> float:
        if self._seconds is None:
            self._end.synchronize()
            self._seconds = self._start.elapsed_time(self._end) * 1e-3
        return self._seconds
