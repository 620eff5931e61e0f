"""Torch plumbing for the C ABI: device memory, streams, pointer arrays.

PyTorch is used only as an allocator / stream provider; every computation is a
libpearl_b200 kernel.  ``require_cuda`` raises when no CUDA device exists --
the product path has no CPU fallback.
"""

from __future__ import annotations

import threading
from typing import Sequence

import torch

from . import _lib
from .errors import DeviceError

_local = threading.local()


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise DeviceError("paper_2408_11850_b200 needs a CUDA (sm_100a) device; no CPU fallback exists")
    _lib.load()
    return torch.device("cuda", torch.cuda.current_device())


def stream_ptr(stream: torch.cuda.Stream | None = None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else int(t.data_ptr())


def row_ptrs(rows: Sequence[torch.Tensor], device) -> torch.Tensor:
    """Device int64 array holding the data pointers of ``rows``."""
    return torch.tensor([int(r.data_ptr()) for r in rows], dtype=torch.int64, device=device)


class Scratch:
    """Per-thread zero-initialised work buffers for the verify / pick kernels."""

    def __init__(self, device):
        self.device = device
        nbytes = int(_lib.load().pearl_verify_work_bytes(1024))
        self.verify_work = torch.zeros(nbytes, dtype=torch.uint8, device=device)
        self.sample_work = torch.zeros(nbytes, dtype=torch.uint8, device=device)
        self.result = torch.zeros(8, dtype=torch.int32, device=device)
        self.status = torch.zeros(1, dtype=torch.int32, device=device)
        self.cursor = torch.zeros(1, dtype=torch.int32, device=device)


def scratch() -> Scratch:
    dev = require_cuda()
    sc = getattr(_local, "scratch", None)
    if sc is None or sc.device != dev:
        sc = Scratch(dev)
        _local.scratch = sc
    return sc
