"""FCS ingestion, per-dimension statistics and dataset transforms on the B200
(ref: io.py:72-229, core.py:44-69).

Only the byte-level work moves to the device: the DATA segment (n×d f32 in
either byte order) is copied once host -> HBM and decoded there
(``esom_fcs_decode``, with the finiteness check of ``Dataset.from_points``),
the column statistics (``esom_dim_stats``) and the transforms
(``esom_apply_transform``: minmax / zscore / affine in f64, rounded to f32)
run on the resident matrix, which then feeds the embed path directly.  The
HEADER and TEXT segments (a few KB of keywords) are parsed on the host with
the reference's rules and error messages.

Results are ``DeviceDataset`` objects: device points + names + DimStats
(numpy f64 arrays, like the reference's).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Sequence

import numpy as np
import torch

from . import _dev, _lib
from .core import InputError, ParameterError, ParseError

TRANSFORM_KINDS = ("none", "minmax", "zscore")  # ref: io.py:21
_KIND_CODE = {"none": 0, "minmax": 1, "zscore": 2}
_FCS_VERSIONS = (b"FCS3.0", b"FCS3.1")  # ref: io.py:18
_BYTEORD_BIG = {"1,2,3,4": 0, "4,3,2,1": 1}  # ref: io.py:19 ("<f4", ">f4")


@dataclass(frozen=True)
class DimStats:
    """ref: core.py:44-51 (population sd, divisor n)."""

    min: np.ndarray
    max: np.ndarray
    mean: np.ndarray
    sd: np.ndarray


@dataclass(frozen=True)
class DeviceDataset:
    """An HBM-resident n×d f32 matrix with the reference Dataset's metadata
    (ref: core.py:72-101)."""

    points: torch.Tensor
    dim_names: tuple
    dim_stats: DimStats

    @property
    def n(self) -> int:
        return self.points.shape[0]

    @property
    def d(self) -> int:
        return self.points.shape[1]

    @classmethod
    def from_points(cls, points, dim_names: Sequence[str] | None = None) -> "DeviceDataset":
        """Upload (if needed), check finiteness on the device, compute the
        statistics (ref: core.py:80-93)."""
        dev = _dev.cuda_device(points)
        with torch.cuda.device(dev):
            X = _dev.to_f32(points, dev)
            if X.ndim != 2:
                raise InputError(f"points must be a 2-d matrix, got shape {tuple(X.shape)}")
            if X.shape[0] < 1 or X.shape[1] < 1:
                raise InputError("empty dataset")
            if X.data_ptr() % 16:
                X = X.clone()  # the checking kernel streams 16-byte vectors
            flag = _dev.new_flag(dev)
            # little-endian "decode" in place = the finiteness scan (ref: core.py:38-40)
            _lib.call("esom_fcs_decode", _dev.ptr(X), X.numel(), 0, _dev.ptr(X), _dev.ptr(flag),
                      _dev.stream_handle(dev))
            if int(flag.item()):
                raise InputError("points contains non-finite values")
            return cls(points=X, dim_names=_names(dim_names, X.shape[1]), dim_stats=compute_dim_stats(X))


def _names(dim_names, d: int) -> tuple:
    if dim_names is None:
        return tuple(f"dim{i}" for i in range(d))
    names = tuple(str(s) for s in dim_names)
    if len(names) != d:
        raise InputError(f"got {len(names)} dimension names for {d} dimensions")
    return names


def compute_dim_stats(points) -> DimStats:
    """Column-wise f64 (min, max, mean, sd) on the device (ref: core.py:54-69).

    min/max are exact; mean/sd are deterministic blocked f64 sums (numpy sums
    each column sequentially; they agree to ~1e-15 relative)."""
    dev = _dev.cuda_device(points)
    with torch.cuda.device(dev):
        X = _dev.to_f32(points, dev)
        if X.ndim != 2 or X.shape[0] < 1 or X.shape[1] < 1:
            raise InputError("empty dataset")
        n, d = X.shape
        out = torch.empty((4, d), dtype=torch.float64, device=dev)
        ws = _dev.workspace(dev, _lib.load().esom_dim_stats_workspace_bytes(n, d), slot="stats")
        _lib.call("esom_dim_stats", _dev.ptr(X), n, d, _dev.ptr(out[0]), _dev.ptr(out[1]), _dev.ptr(out[2]),
                  _dev.ptr(out[3]), _dev.ptr(ws), ws.numel(), _dev.stream_handle(dev))
        h = out.cpu().numpy()
        return DimStats(min=h[0].copy(), max=h[1].copy(), mean=h[2].copy(), sd=h[3].copy())


@dataclass(frozen=True)
class TransformSpec:
    """Per-dimension transform: 'none' | 'minmax' | 'zscore' | ('affine', a, b)
    (ref: io.py:181-202)."""

    entries: tuple

    def __post_init__(self):
        for e in self.entries:
            ok = (e in TRANSFORM_KINDS) if isinstance(e, str) else (
                isinstance(e, tuple) and len(e) == 3 and e[0] == "affine")
            if not ok:
                raise ParameterError(f"unknown transform {e!r}")

    @classmethod
    def uniform(cls, kind: str, d: int) -> "TransformSpec":
        return cls(entries=tuple([kind] * d))


def apply_transform(dataset, spec: TransformSpec) -> DeviceDataset:
    """Scale every dimension on the device and rebuild the statistics
    (ref: io.py:205-229).  Bit-exact given the dataset's statistics."""
    if not isinstance(dataset, DeviceDataset):
        dataset = DeviceDataset.from_points(dataset.points, getattr(dataset, "dim_names", None))
    d = dataset.d
    if len(spec.entries) != d:
        raise ParameterError(f"transform has {len(spec.entries)} entries for {d} dimensions")
    X = dataset.points
    dev = X.device
    kind = np.zeros(d, np.int32)
    a = np.ones(d, np.float64)
    b = np.zeros(d, np.float64)
    for c, e in enumerate(spec.entries):
        if isinstance(e, str):
            kind[c] = _KIND_CODE[e]
        else:
            kind[c], a[c], b[c] = 3, float(e[1]), float(e[2])
    st = dataset.dim_stats
    with torch.cuda.device(dev):
        par = torch.from_numpy(np.stack([a, b, st.min, st.max, st.mean, st.sd]).astype(np.float64)).to(dev)
        kd = torch.from_numpy(kind).to(dev)
        out = torch.empty_like(X)
        flag = _dev.new_flag(dev)
        _lib.call("esom_apply_transform", _dev.ptr(X), X.shape[0], d, _dev.ptr(kd), _dev.ptr(par[0]),
                  _dev.ptr(par[1]), _dev.ptr(par[2]), _dev.ptr(par[3]), _dev.ptr(par[4]), _dev.ptr(par[5]),
                  _dev.ptr(out), _dev.ptr(flag), _dev.stream_handle(dev))
        if int(flag.item()):
            raise InputError("points contains non-finite values")
        return DeviceDataset(points=out, dim_names=dataset.dim_names, dim_stats=compute_dim_stats(out))


# ---------------------------------------------------------------------------
# FCS 3.0 / 3.1 list mode, $DATATYPE F, 32-bit parameters (ref: io.py:1-126)


def _offset(raw: bytes, lo: int, hi: int, label: str) -> int:
    field_ = raw[lo:hi].decode("ascii", errors="replace").strip()
    if not field_:
        return 0
    try:
        return int(field_)
    except ValueError:
        raise ParseError(f"malformed {label} offset at header bytes {lo}-{hi - 1}: {field_!r}") from None


def _keywords(seg: bytes) -> dict:
    """TEXT keyword/value pairs; the first byte is the delimiter and a doubled
    delimiter is a literal (ref: io.py:35-64)."""
    if not seg:
        raise ParseError("empty TEXT segment")
    delim = seg[:1]
    tokens, cur, p, end = [], [], 1, len(seg)
    while p < end:
        q = seg.find(delim, p)
        if q < 0:
            cur.append(seg[p:])
            break
        cur.append(seg[p:q])
        if seg[q + 1:q + 2] == delim:  # escaped delimiter
            cur.append(delim)
            p = q + 2
            continue
        tokens.append(b"".join(cur))
        cur, p = [], q + 1
    tail = b"".join(cur)
    if tail:
        tokens.append(tail)
    if tokens and tokens[-1] == b"":
        tokens.pop()
    if len(tokens) % 2:
        raise ParseError("TEXT segment has an unpaired keyword")
    return {tokens[i].decode("latin-1").strip().upper(): tokens[i + 1].decode("latin-1").strip()
            for i in range(0, len(tokens), 2)}


def _need(kw: dict, key: str) -> str:
    try:
        return kw[key]
    except KeyError:
        raise ParseError(f"missing required keyword {key}") from None


def _fcs_layout(data):
    """(n, d, big_endian, data_begin, names) with the reference's checks.
    ``data``: any byte buffer (bytes, memoryview, uint8 ndarray); only the
    header and TEXT slices are copied."""
    if len(data) < 42:
        raise ParseError("file shorter than the FCS header")
    head = bytes(data[:42])
    if head[:6] not in _FCS_VERSIONS:
        raise ParseError(f"unsupported version {head[:6]!r} (need FCS3.0 or FCS3.1)")
    t0, t1, d0, d1 = (_offset(head, lo, lo + 8, lab) for lo, lab in
                      ((10, "TEXT begin"), (18, "TEXT end"), (26, "DATA begin"), (34, "DATA end")))
    if t0 <= 0 or t1 < t0 or t1 >= len(data):
        raise ParseError(f"TEXT segment offsets {t0}-{t1} out of range")
    kw = _keywords(bytes(data[t0:t1 + 1]))
    n, d = int(_need(kw, "$TOT")), int(_need(kw, "$PAR"))
    for key, want, what in (("$DATATYPE", "F", "datatype $DATATYPE={!r} (only F)"),
                            ("$MODE", "L", "$MODE={!r} (only list mode L)")):
        v = _need(kw, key)
        if v != want:
            raise ParseError("unsupported " + what.format(v))
    byteord = _need(kw, "$BYTEORD")
    if byteord not in _BYTEORD_BIG:
        raise ParseError(f"unsupported $BYTEORD={byteord!r}")
    names = []
    for i in range(1, d + 1):
        bits = _need(kw, f"$P{i}B")
        if bits.strip() != "32":
            raise ParseError(f"unsupported $P{i}B={bits!r} (only 32)")
        names.append(kw.get(f"$P{i}N") or kw.get(f"$P{i}S") or f"P{i}")
    if d0 == 0 and d1 == 0:  # FCS3.1: offsets of large files live in TEXT
        d0, d1 = int(_need(kw, "$BEGINDATA")), int(_need(kw, "$ENDDATA"))
    need = 4 * n * d
    if d0 <= 0 or d0 + need - 1 > len(data) - 1:
        raise ParseError(f"truncated DATA segment: need {need} bytes at offset {d0}, file has {len(data)} bytes")
    if d1 and d1 - d0 + 1 < need:
        raise ParseError(f"truncated DATA segment: offsets {d0}-{d1} hold fewer than {need} bytes")
    return n, d, _BYTEORD_BIG[byteord], d0, names


def parse_fcs(data, device=None) -> DeviceDataset:
    """Parse an FCS 3.0/3.1 file image; the DATA segment is copied once to the
    device and decoded there (ref: io.py:72-126).  ``data``: bytes-like, or a
    (pinned) uint8 CPU tensor -- the latter is DMA'd at full PCIe rate."""
    if isinstance(data, torch.Tensor):
        tens = data.reshape(-1)
        view = tens.numpy()
    else:
        view = np.frombuffer(data, dtype=np.uint8)
        tens = torch.from_numpy(view) if view.flags.writeable else None
    n, d, big, d0, names = _fcs_layout(view)
    dev = device if device is not None else _dev.cuda_device()
    with torch.cuda.device(dev):
        if n * d == 0:
            raise InputError("empty dataset")
        nbytes = 4 * n * d
        stage = torch.empty(nbytes, dtype=torch.uint8, device=dev)
        src = tens[d0:d0 + nbytes] if tens is not None else torch.from_numpy(view[d0:d0 + nbytes].copy())
        stage.copy_(src, non_blocking=bool(src.is_pinned()))
        X = torch.empty((n, d), dtype=torch.float32, device=dev)
        flag = _dev.new_flag(dev)
        _lib.call("esom_fcs_decode", _dev.ptr(stage), n * d, big, _dev.ptr(X), _dev.ptr(flag),
                  _dev.stream_handle(dev))
        if int(flag.item()):
            raise InputError("points contains non-finite values")
        del stage
        return DeviceDataset(points=X, dim_names=tuple(names), dim_stats=compute_dim_stats(X))


def read_pinned(path: str) -> torch.Tensor:
    """The file's bytes in page-locked host memory (one read, no extra copy)."""
    import os

    size = os.path.getsize(path)
    buf = torch.empty(size, dtype=torch.uint8, pin_memory=True)
    with open(path, "rb", buffering=0) as fh:
        mv, got = memoryview(buf.numpy()), 0
        while got < size:
            r = fh.readinto(mv[got:])
            if not r:
                break
            got += r
    return buf[:got]


def load_fcs(path: str, transform: str | None = None, device=None) -> DeviceDataset:
    """``load_dataset(path, "fcs", transform)`` (ref: io.py:232-266): FCS with
    the default zscore transform, resident on the device."""
    ds = parse_fcs(read_pinned(path), device=device)
    tf = transform if transform is not None else "zscore"
    if tf != "none":
        ds = apply_transform(ds, TransformSpec.uniform(tf, ds.d))
    return ds
