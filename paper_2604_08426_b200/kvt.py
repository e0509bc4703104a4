"""KVT1 tensor files and exported workloads (real-tensor import for the
decode path).

Same format and error conditions as the reference's ``write_kvt`` /
``read_kvt`` (numerics.py:151-190): magic ``KVT1``, u32 ndim, u64 extents,
little-endian float32 payload; ``KvtFormatError`` (a ``ValueError``) on bad
magic, truncation, an extent product above 2**32 or a payload whose size
does not match the extents. ``load_workload`` mirrors workload.py:110-119
(keys / values / queries + ``workload.json``).

B200 additions: ``read_kvt(..., pinned=True)`` reads the payload straight
into page-locked host memory (one ``readinto``, no intermediate numpy copy),
and ``to_device_tokens`` turns a reference-layout ``[H, n, D]`` tensor into
the store's token-major ``[1, n, H, D]`` device layout with one
pinned-to-HBM copy, so exported real K/V (KVT1 from a model dump) feed
``DeviceStore.build`` without staging through the CPU oracle.
"""

from __future__ import annotations

import json
import os
import struct
from dataclasses import dataclass

import numpy as np
import torch

KVT_MAGIC = b"KVT1"
_MAX_KVT_ELEMENTS = 1 << 32


class KvtFormatError(ValueError):
    """numerics.py:21-22: malformed KVT1 file."""


def write_kvt(path, arr) -> None:
    """numerics.py:151-162."""
    a = np.asarray(arr, dtype="<f4", order="C")
    with open(path, "wb") as f:
        f.write(KVT_MAGIC)
        f.write(struct.pack("<I", a.ndim))
        if a.ndim:
            f.write(struct.pack(f"<{a.ndim}Q", *a.shape))
        f.write(a.tobytes(order="C"))


def _header(f, size: int) -> tuple:
    head = f.read(8)
    if head[:4] != KVT_MAGIC:
        raise KvtFormatError(f"bad magic {head[:4]!r}, expected {KVT_MAGIC!r}")
    if len(head) < 8:
        raise KvtFormatError("truncated header")
    (ndim,) = struct.unpack_from("<I", head, 4)
    if size < 8 + 8 * ndim:
        raise KvtFormatError("truncated extent list")
    ext = struct.unpack(f"<{ndim}Q", f.read(8 * ndim)) if ndim else ()
    count = 1
    for e in ext:
        count *= e
    if count > _MAX_KVT_ELEMENTS:
        raise KvtFormatError(f"extent product {count} exceeds supported size")
    payload = size - 8 - 8 * ndim
    if payload != 4 * count:
        raise KvtFormatError(f"payload holds {payload} bytes, extents require {4 * count}")
    return tuple(int(e) for e in ext), count


def read_kvt(path, pinned: bool = False):
    """numerics.py:165-190. Returns a float32 numpy array, or with
    ``pinned=True`` a page-locked float32 torch tensor of the same shape."""
    size = os.path.getsize(path)
    with open(path, "rb") as f:
        ext, count = _header(f, size)
        if pinned:
            t = torch.empty(count, dtype=torch.float32, pin_memory=torch.cuda.is_available())
            if count:
                got = f.readinto(memoryview(t.numpy()).cast("B"))
                if got != 4 * count:
                    raise KvtFormatError("short read")
            return t.reshape(ext)
        arr = np.frombuffer(f.read(), dtype="<f4").astype(np.float32)
    return arr.reshape(ext)


def to_device_tokens(heads_major, dtype=torch.float32, device="cuda") -> torch.Tensor:
    """[H, n, D] (the reference layout) -> [1, n, H, D] contiguous on the
    device (the store layout), converting to ``dtype`` on the device."""
    t = heads_major if isinstance(heads_major, torch.Tensor) else torch.from_numpy(
        np.ascontiguousarray(heads_major, dtype=np.float32))
    if t.dim() == 2:
        t = t[None]
    if t.dim() != 3:
        raise ValueError(f"expected [H, n, D] or [n, D], got {tuple(t.shape)}")
    d = t.to(device, non_blocking=True)
    return d.permute(1, 0, 2).contiguous().to(dtype)[None]


@dataclass
class Workload:
    """workload.py:48-55 (GeneratedWorkload) for an exported instance."""

    spec: dict
    keys: np.ndarray      # [H, n, D]
    values: np.ndarray    # [H, n, D]
    queries: np.ndarray   # [steps, H, G, D]
    needle_ids: list


def save_workload(wl, directory) -> None:
    """workload.py:95-107."""
    os.makedirs(directory, exist_ok=True)
    write_kvt(os.path.join(directory, "keys.kvt"), wl.keys)
    write_kvt(os.path.join(directory, "values.kvt"), wl.values)
    write_kvt(os.path.join(directory, "queries.kvt"), wl.queries)
    spec = wl.spec if isinstance(wl.spec, dict) else dict(wl.spec.__dict__)
    meta = {"spec": spec, "needle_ids": [np.asarray(i).tolist() for i in wl.needle_ids]}
    with open(os.path.join(directory, "workload.json"), "w", encoding="utf-8") as f:
        json.dump(meta, f, indent=1, sort_keys=True)


def load_workload(directory) -> Workload:
    """workload.py:110-119."""
    with open(os.path.join(directory, "workload.json"), encoding="utf-8") as f:
        meta = json.load(f)
    return Workload(spec=meta["spec"],
                    keys=read_kvt(os.path.join(directory, "keys.kvt")),
                    values=read_kvt(os.path.join(directory, "values.kvt")),
                    queries=read_kvt(os.path.join(directory, "queries.kvt")),
                    needle_ids=[np.asarray(i, dtype=np.int64) for i in meta["needle_ids"]])
