"""Device plumbing: torch owns every buffer, the C ABI only sees pointers.

Inputs may be numpy arrays (the reference's calling convention; copied to
the device per call, results copied back) or torch CUDA tensors (device
resident; results stay on the device).  Workspaces are cached per (thread,
device) so concurrent callers on different streams never share scratch.
"""

from __future__ import annotations

import threading
import warnings

import numpy as np
import torch

# read-only inputs (the reference's frozen core arrays) are only ever read
warnings.filterwarnings("ignore", message="The given NumPy array is not writable")

from .core import InputError

_tls = threading.local()


def cuda_device(like=None) -> torch.device:
    if isinstance(like, torch.Tensor) and like.is_cuda:
        return like.device
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2201_00701_b200 needs a CUDA device (B200); none is visible")
    return torch.device("cuda", torch.cuda.current_device())


def is_device_tensor(a) -> bool:
    return isinstance(a, torch.Tensor) and a.is_cuda


def to_f32(a, dev: torch.device) -> torch.Tensor:
    if isinstance(a, torch.Tensor):
        t = a.detach()
        if t.dtype != torch.float32:
            t = t.float()
        return t.to(dev).contiguous()
    arr = np.ascontiguousarray(a, dtype=np.float32)
    return torch.from_numpy(arr).to(dev)


def to_dev_async(arr: np.ndarray, dev: torch.device) -> torch.Tensor:
    """Small host array -> device without blocking the host: staged through
    page-locked memory (torch's caching host allocator keeps the staging
    buffer alive until the copy on the current stream has run)."""
    return torch.from_numpy(np.ascontiguousarray(arr)).pin_memory().to(dev, non_blocking=True)


def to_i32(a, dev: torch.device) -> torch.Tensor:
    if isinstance(a, torch.Tensor):
        return a.detach().to(device=dev, dtype=torch.int32).contiguous()
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.int32)).to(dev)


def to_f64(a, dev: torch.device) -> torch.Tensor:
    if isinstance(a, torch.Tensor):
        return a.detach().to(device=dev, dtype=torch.float64).contiguous()
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(dev)


def ptr(t) -> int:
    return 0 if t is None else int(t.data_ptr())


def stream_handle(dev: torch.device) -> int:
    return int(torch.cuda.current_stream(dev).cuda_stream)


def workspace(dev: torch.device, nbytes: int, slot: str = "main") -> torch.Tensor:
    cache = getattr(_tls, "ws", None)
    if cache is None:
        cache = _tls.ws = {}
    key = (dev.index, slot)
    buf = cache.get(key)
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=dev)
        cache[key] = buf
    return buf


def new_flag(dev: torch.device) -> torch.Tensor:
    return torch.zeros(1, dtype=torch.int32, device=dev)


def raise_if_nonfinite(flag: torch.Tensor) -> None:
    if int(flag.item()) != 0:  # the reference raises before compute (ref: knn.py:196-197)
        raise InputError("non-finite input")


def out_like(t: torch.Tensor, want_numpy: bool):
    return t.cpu().numpy() if want_numpy else t
