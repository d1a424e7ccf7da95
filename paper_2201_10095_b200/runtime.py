"""Execution context: one ``rs_context`` (CUDA stream + scratch arena) per device.

By default the context runs on torch's current CUDA stream for the device, so
torch.cuda.Event timing and torch tensors interoperate with the C-ABI calls.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib

_contexts: dict = {}


class Context:
    def __init__(self, device: int = 0, stream=None):
        import torch

        if not torch.cuda.is_available():
            raise RuntimeError("paper_2201_10095_b200 needs a CUDA device (no CPU fallback)")
        self.device = device
        if stream is None:
            stream = torch.cuda.current_stream(device)
        self.torch_stream = stream
        h = C.c_void_p()
        _lib.check(_lib.lib().rs_context_create(device, C.c_void_p(stream.cuda_stream), 0,
                                                C.byref(h)))
        self.h = h

    def synchronize(self):
        _lib.check(_lib.lib().rs_context_synchronize(self.h))

    def close(self):
        if self.h:
            _lib.lib().rs_context_destroy(self.h)
            self.h = None

    def __del__(self):  # pragma: no cover - interpreter teardown
        try:
            self.close()
        except Exception:
            pass


def default_context(device: int = 0) -> Context:
    ctx = _contexts.get(device)
    if ctx is None:
        ctx = _contexts[device] = Context(device)
    return ctx


def ptr(a):
    """Device or host pointer of a torch tensor / numpy array (None passes through)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return C.c_void_p(a.ctypes.data)
    return C.c_void_p(a.data_ptr())


def is_device(a) -> bool:
    return not isinstance(a, np.ndarray) and getattr(a, "is_cuda", False)
