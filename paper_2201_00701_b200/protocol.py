"""FramePoints wire record packed on the device.

The reference server sends every frame as ``protocol.encode(FramePoints(
frame_id, positions, colors))`` (ref: protocol.py:205-210, 216-218):

    <u32 1 + len(payload)> <u8 TAG_FRAME_POINTS> <u32 frame_id> <u32 n>
    <n x 2 f32 little endian> <n u8>                     = 13 + 9n bytes

``encode_frame_points`` produces exactly those bytes with one kernel
(``esom_frame_points_pack``) that reads the device-resident positions and
colours and writes the record straight into a page-locked host buffer over
PCIe (mapped memory: no device staging buffer, no separate copy).
"""

from __future__ import annotations

import threading
from dataclasses import dataclass

import numpy as np
import torch

from . import _dev, _lib
from .core import ParameterError

TAG_FRAME_POINTS = 0x31  # ref: protocol.py:33


@dataclass(frozen=True)
class FramePoints:
    """ref: protocol.py FramePoints (frame_id, n×2 f32 positions, n u8 colours)."""

    frame_id: int
    positions: object
    colors: object


def frame_points_bytes(n: int) -> int:
    return 13 + 9 * int(n)


class FrameBuffer:
    """A reusable page-locked host buffer the pack kernel writes into."""

    def __init__(self, nbytes: int, device=None):
        self.device = device if device is not None else _dev.cuda_device()
        cap = max(int(nbytes), 16)
        self.host = torch.empty(cap, dtype=torch.uint8, pin_memory=True)
        dptr = _lib.load().esom_mapped_device_ptr(self.host.data_ptr())
        self.dev_ptr = int(dptr) if dptr else None
        # not mapped (should not happen with UVA): pack on the device, then copy
        self.staging = None if self.dev_ptr else torch.empty(cap, dtype=torch.uint8, device=self.device)
        self.event = torch.cuda.Event()

    @property
    def capacity(self) -> int:
        return self.host.numel()


def pack_frame_points(xy: torch.Tensor, colors: torch.Tensor, frame_id: int, buf: FrameBuffer) -> int:
    """Asynchronously pack one record into ``buf`` on the current stream;
    returns its length.  Wait on ``buf.event`` before reading ``buf.host``."""
    n = xy.shape[0]
    if xy.shape != (n, 2) or colors.shape != (n,):
        raise ParameterError("positions must be n x 2 and colors n")
    if not 0 <= int(frame_id) <= 0xFFFFFFFF:
        raise ParameterError(f"frame_id {frame_id} does not fit u32")  # struct.pack('<I') in the reference
    nbytes = frame_points_bytes(n)
    if nbytes > buf.capacity:
        raise ParameterError(f"frame buffer holds {buf.capacity} bytes, record needs {nbytes}")
    dev = xy.device
    st = _dev.stream_handle(dev)
    out = buf.dev_ptr if buf.dev_ptr else _dev.ptr(buf.staging)
    _lib.call("esom_frame_points_pack", _dev.ptr(xy), _dev.ptr(colors), n, int(frame_id), out, st)
    if buf.staging is not None:
        buf.host[:nbytes].copy_(buf.staging[:nbytes], non_blocking=True)
    buf.event.record(torch.cuda.current_stream(dev))
    return nbytes


_tls = threading.local()


def _cached_buffer(nbytes: int, dev) -> FrameBuffer:
    """Per-(thread, device) pinned buffer, grown on demand (page-locking is
    expensive; the synchronous encoder reuses it call after call)."""
    cache = getattr(_tls, "frames", None)
    if cache is None:
        cache = _tls.frames = {}
    key = dev.index if isinstance(dev, torch.device) else int(dev)
    buf = cache.get(key)
    if buf is None or buf.capacity < nbytes:
        buf = cache[key] = FrameBuffer(max(nbytes, 1 << 16), dev)
    return buf


def encode_frame_points(frame_id: int, positions, colors) -> bytes:
    """``protocol.encode(FramePoints(frame_id, positions, colors))`` computed on
    the device (ref: protocol.py:205-210, 216-218)."""
    dev = _dev.cuda_device(positions)
    with torch.cuda.device(dev):
        xy = _dev.to_f32(positions, dev)
        if isinstance(colors, torch.Tensor):
            col = colors.detach().to(device=dev, dtype=torch.uint8).contiguous()
        else:
            col = torch.from_numpy(np.ascontiguousarray(colors, dtype=np.uint8)).to(dev)
        buf = _cached_buffer(frame_points_bytes(xy.shape[0]), dev)
        nbytes = pack_frame_points(xy, col, frame_id, buf)
        buf.event.synchronize()
        return bytes(buf.host[:nbytes].numpy())

