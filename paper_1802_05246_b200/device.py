"""Device-memory plumbing (PyTorch is used only for allocation, copies and
streams; every numerical operation runs in libhermb200.so)."""

from __future__ import annotations

import warnings

import numpy as np

from ._lib import HermiteLibError
from .fields import is_device_array


def torch():
    import torch as _t

    return _t


def require_cuda():
    t = torch()
    if not t.cuda.is_available():
        raise HermiteLibError("a CUDA device is required: the Hermite hot path has no CPU fallback")
    return t


def stream_handle(device=None) -> int:
    t = torch()
    return t.cuda.current_stream(device).cuda_stream


def ptr(x) -> int:
    return int(x.data_ptr()) if x is not None else 0


class Staging:
    """Moves host (numpy) operands to the device and results back, keeping
    the caller's container kind (numpy in -> numpy out)."""

    def __init__(self, *arrays):
        t = require_cuda()
        self.host = not any(is_device_array(a) for a in arrays if a is not None)
        if self.host:
            self.device = t.device("cuda", t.cuda.current_device())
        else:
            dev = next(a.device for a in arrays if a is not None and is_device_array(a))
            if dev.type != "cuda":
                raise HermiteLibError("device-resident fields must be CUDA tensors")
            self.device = dev

    def to_dev(self, a):
        t = torch()
        if a is None:
            return None
        if is_device_array(a):
            if a.device != self.device:
                raise ValueError("all fields of one call must live on the same device")
            return a.contiguous() if not a.is_contiguous() else a
        a = np.ascontiguousarray(a, dtype=np.float64)
        if a.flags.writeable:
            host = t.from_numpy(a)
        else:
            # frozen Field values are read-only views; the tensor is only ever
            # a copy source, so wrapping it without a write flag is safe
            with warnings.catch_warnings():
                warnings.simplefilter("ignore", UserWarning)
                host = t.from_numpy(a)
        # pinned host memory (e.g. torch pin_memory buffers viewed as numpy)
        # copies asynchronously on the current stream; pageable memory is
        # staged by the driver and returns once copied
        return host.to(self.device, non_blocking=True)

    def empty(self, shape):
        return torch().empty(tuple(int(s) for s in shape), dtype=torch().float64, device=self.device)

    def out(self, d):
        """Device result -> caller's container.  Host results land in pinned
        memory from torch's caching host allocator (fast DMA, no page faults
        on reuse); the returned ndarray keeps that buffer alive."""
        if self.host:
            t = torch()
            h = t.empty(tuple(d.shape), dtype=d.dtype, pin_memory=True)
            h.copy_(d, non_blocking=True)
            t.cuda.current_stream(self.device).synchronize()
            return h.numpy()
        return d

    @property
    def stream(self) -> int:
        return stream_handle(self.device)
