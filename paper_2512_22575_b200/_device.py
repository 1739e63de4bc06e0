"""Device plumbing: CUDA availability, current stream, raw pointers.

torch provides device memory and streams only; every computation on the hot
path is a libvpb200 kernel.  There is no CPU fallback: without a CUDA device
the product path raises.
"""

from __future__ import annotations

import ctypes

import torch

from ._lib import NativeError, load


def device(dev=None) -> torch.device:
    if not torch.cuda.is_available():
        raise NativeError("no CUDA device visible: the B200 path has no CPU fallback")
    load()
    if dev is None:
        return torch.device("cuda", torch.cuda.current_device())
    d = torch.device(dev)
    if d.type != "cuda":
        raise NativeError(f"device {d} is not a CUDA device (no CPU fallback)")
    return d


def stream(dev: torch.device | None = None) -> ctypes.c_void_p:
    s = torch.cuda.current_stream(dev)
    return ctypes.c_void_p(s.cuda_stream)


def ptr(t: torch.Tensor | None) -> ctypes.c_void_p | None:
    if t is None:
        return None
    if not t.is_cuda:
        raise NativeError("expected a CUDA tensor")
    if not t.is_contiguous():
        raise ValueError("expected a contiguous tensor")
    return ctypes.c_void_p(t.data_ptr())


def host_ptr(a) -> ctypes.c_void_p:
    return a.ctypes.data_as(ctypes.c_void_p)


class Workspace:
    """Grow-only scratch buffer per (device, tag); reused across calls so the
    hot path never allocates once warmed up."""

    _bufs: dict = {}

    @classmethod
    def get(cls, dev: torch.device, tag: str, nbytes: int, zeroed: bool = False) -> torch.Tensor:
        """``zeroed``: zero-filled when (re)allocated (buffers holding counters
        that the kernels return to zero themselves)."""
        key = (str(dev), tag)
        buf = cls._bufs.get(key)
        if buf is None or buf.numel() < nbytes:
            alloc = torch.zeros if zeroed else torch.empty
            buf = alloc(max(int(nbytes), 256), dtype=torch.uint8, device=dev)
            cls._bufs[key] = buf
        return buf
