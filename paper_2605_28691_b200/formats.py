"""On-disk formats of the reference, byte-compatible:
OSPT tensor files (gridseq.py:232-256) and padding-mask files (anyres.py:99-112).
Host I/O only: device tensors are copied to the host to be written."""

from __future__ import annotations

import struct

import numpy as np
import torch

from .gridseq import REAL, GridShape, SequenceTensor, default_device

OSPT_MAGIC = b"OSPT"
OSPT_VERSION = 1


def write_ospt(path, x: SequenceTensor) -> None:
    """magic "OSPT", version byte, batch/seq/chan as u32 LE, float64 LE payload."""
    if x.kind != REAL:
        raise ValueError("OSPT files store real-kind tensors")
    data = x.tensor.detach().to("cpu", torch.float64).contiguous().numpy()
    b, s, c = data.shape
    with open(path, "wb") as f:
        f.write(OSPT_MAGIC)
        f.write(bytes([OSPT_VERSION]))
        f.write(struct.pack("<III", b, s, c))
        f.write(data.astype("<f8").tobytes())


def read_ospt(path, device=None) -> SequenceTensor:
    with open(path, "rb") as f:
        magic = f.read(4)
        if magic != OSPT_MAGIC:
            raise ValueError(f"bad magic {magic!r}, expected {OSPT_MAGIC!r}")
        version = f.read(1)
        if version != bytes([OSPT_VERSION]):
            raise ValueError(f"unsupported OSPT version {version!r}")
        b, s, c = struct.unpack("<III", f.read(12))
        payload = f.read(8 * b * s * c)
    arr = np.frombuffer(payload, dtype="<f8").reshape(b, s, c).astype(np.float64)
    return SequenceTensor(torch.from_numpy(arr).to(device or default_device()))


def write_mask(path, pg) -> None:
    """Padded grid dims (t, h, w, k) as u32 LE, then one byte per flat padded token."""
    p = pg.padded
    with open(path, "wb") as f:
        f.write(struct.pack("<IIII", p.t, p.h, p.w, p.k))
        f.write(pg.mask.detach().to("cpu", torch.uint8).numpy().tobytes())


def read_mask(path) -> tuple[GridShape, torch.Tensor]:
    with open(path, "rb") as f:
        t, h, w, k = struct.unpack("<IIII", f.read(16))
        g = GridShape(t, h, w, k)
        mask = np.frombuffer(f.read(g.seq_len), dtype=np.uint8).astype(bool)
    return g, torch.from_numpy(mask.copy()).to(default_device())
