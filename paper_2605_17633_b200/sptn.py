"""SPTN tensor files: the reference's golden-vector exchange format (tensor.py:65-116, grid.py:122-136).

Byte layout (little endian), identical to the reference so files round-trip between the two:

    offset 0   b"SPTN"
    offset 4   u8 version (1)
    offset 5   u8 dtype (0 = float32)
    offset 6   u8 rank (1..255)
    offset 7   3 zero bytes
    offset 10  rank x u64 extents (all > 0)
    then       prod(extents) float32, row-major, nothing after it

Errors follow the reference's classes (all ``ValueError`` subclasses, tensor.py:34-55) and
conditions: bad magic / version / dtype, a truncated header, dimension block or payload, and
a zero extent or trailing bytes (``SptnBadShape``).  Missing files raise ``OSError``.

B200 additions: ``tensor_read(..., device="cuda")`` lands the payload in pinned host memory and
copies it to the device asynchronously; ``tensor_write`` accepts device tensors (one D2H copy).
"""

from __future__ import annotations

import math
import os

import numpy as np

MAGIC = b"SPTN"
VERSION = 1
DTYPE_F32 = 0
PERM_INDEX_LIMIT = 1 << 24  # float32 represents every integer index below this exactly

_FIXED = np.dtype([("magic", "S4"), ("version", "u1"), ("dtype", "u1"), ("rank", "u1"), ("pad", "V3")])


class SptnError(ValueError):
    """Malformed SPTN file (base class)."""


class SptnBadMagic(SptnError):
    pass


class SptnBadVersion(SptnError):
    pass


class SptnBadDtype(SptnError):
    pass


class SptnTruncated(SptnError):
    pass


class SptnBadShape(SptnError):
    pass


def _host_f32(t) -> np.ndarray:
    if hasattr(t, "detach"):  # torch tensor (any device)
        import torch

        if t.dtype != torch.float32:
            raise TypeError(f"tensor must be float32, got {t.dtype}")
        return t.detach().contiguous().cpu().numpy()
    a = np.asarray(t)
    if a.dtype != np.float32:
        raise TypeError(f"tensor must be float32, got {a.dtype}")
    return np.ascontiguousarray(a)


def encode(t) -> bytes:
    """SPTN bytes of a float32 array / tensor."""
    a = _host_f32(t)
    if not 1 <= a.ndim <= 255:
        raise SptnBadShape(f"rank must be in [1, 255], got {a.ndim}")
    if min(a.shape) <= 0:
        raise SptnBadShape(f"extents must be positive, got {a.shape}")
    head = np.zeros((), _FIXED)
    head["magic"], head["version"], head["dtype"], head["rank"] = MAGIC, VERSION, DTYPE_F32, a.ndim
    return head.tobytes() + np.asarray(a.shape, "<u8").tobytes() + a.astype("<f4", copy=False).tobytes()


def decode_header(raw, name="<bytes>") -> tuple[tuple[int, ...], int]:
    """Validate the header of ``raw``; returns (shape, payload offset)."""
    if len(raw) < _FIXED.itemsize:
        raise SptnTruncated(f"{name}: header needs {_FIXED.itemsize} bytes, file has {len(raw)}")
    head = np.frombuffer(raw, _FIXED, count=1)[0]
    if bytes(head["magic"]) != MAGIC:
        raise SptnBadMagic(f"{name}: magic {bytes(raw[:4])!r} != {MAGIC!r}")
    if int(head["version"]) != VERSION:
        raise SptnBadVersion(f"{name}: version {int(head['version'])} unsupported")
    if int(head["dtype"]) != DTYPE_F32:
        raise SptnBadDtype(f"{name}: dtype code {int(head['dtype'])} unsupported")
    rank = int(head["rank"])
    if rank < 1:
        raise SptnBadShape(f"{name}: rank must be >= 1")
    off = _FIXED.itemsize + 8 * rank
    if len(raw) < off:
        raise SptnTruncated(f"{name}: truncated dimension block")
    shape = tuple(int(e) for e in np.frombuffer(raw, "<u8", count=rank, offset=_FIXED.itemsize))
    if min(shape) <= 0:
        raise SptnBadShape(f"{name}: extents must be positive, got {shape}")
    need = 4 * math.prod(shape)
    have = len(raw) - off
    if have < need:
        raise SptnTruncated(f"{name}: payload has {have} bytes, expected {need}")
    if have > need:
        raise SptnBadShape(f"{name}: {have - need} trailing bytes")
    return shape, off


def decode(raw, name="<bytes>") -> np.ndarray:
    shape, off = decode_header(raw, name)
    return np.frombuffer(raw, "<f4", count=math.prod(shape), offset=off).astype(np.float32).reshape(shape)


def tensor_write(t, path) -> None:
    """Write a float32 array (numpy, or a torch tensor on any device) as SPTN (tensor.py:65-84)."""
    data = encode(t)
    with open(path, "wb") as f:
        f.write(data)


def tensor_read(path, device=None):
    """Read an SPTN file (tensor.py:86-116).  ``device`` None -> numpy float32 array; otherwise a
    torch float32 tensor on ``device`` (payload staged in pinned memory, copied non-blocking)."""
    with open(os.fspath(path), "rb") as f:
        raw = f.read()
    if device is None:
        return decode(raw, str(path))
    import torch

    shape, off = decode_header(raw, str(path))
    host = torch.empty(shape, dtype=torch.float32, pin_memory=torch.cuda.is_available())
    host.numpy().reshape(-1)[:] = np.frombuffer(raw, "<f4", count=host.numel(), offset=off)
    return host.to(device, non_blocking=True)


def permutation_write(p, path) -> None:
    """Permutation as a rank-1 SPTN tensor of exact-integer float32 indices (grid.py:122-127)."""
    fwd = np.asarray(getattr(p, "forward", p), dtype=np.int64)
    if fwd.size > PERM_INDEX_LIMIT:
        raise ValueError(f"permutation longer than {PERM_INDEX_LIMIT} not serializable")
    tensor_write(fwd.astype(np.float32), path)


def permutation_read(path):
    """Inverse of :func:`permutation_write` (grid.py:130-136); returns an ``api.Permutation``."""
    from .api import Permutation

    vals = tensor_read(path)
    if vals.ndim != 1:
        raise ValueError(f"{path}: permutation tensor must be rank 1")
    idx = vals.astype(np.int64)
    if not np.array_equal(idx.astype(np.float32), vals):
        raise ValueError(f"{path}: permutation entries must be exact integers")
    return Permutation(idx)
