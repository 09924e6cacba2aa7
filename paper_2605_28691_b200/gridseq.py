"""(batch, seq, chan) tensors and lazy gather maps -- drop-in for osp.gridseq.

Mirrors reference gridseq.py: GridShape (41-76), SequenceTensor (79-116),
random_tensor (119-122), IndexMap (125-195), rearrange_map (198-229).

Differences by design (B200 path):
  * SequenceTensor wraps a torch tensor (normally CUDA, any dtype); numpy input
    is accepted and moved to the current CUDA device.  The reference coerces to
    float64 and freezes; here outputs are always fresh tensors (functional).
  * IndexMap is lazy: the six pattern maps are closed-form descriptors applied
    by the K1 kernel; `src` (the int64 gather table) is materialised on the GPU
    only when asked for, by pushing an iota through the same kernel.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Sequence

import numpy as np
import torch

from . import kernels
from .errors import CoordinateError, ShapeError

REAL = "real"
HIF8 = "hif8"

__all__ = ["GridShape", "SequenceTensor", "IndexMap", "random_tensor", "rearrange_map",
           "CoordinateError", "ShapeError", "REAL", "HIF8"]


def default_device() -> torch.device:
    return torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() \
        else torch.device("cpu")


@dataclass(frozen=True)
class GridShape:
    """A latent grid of t frames x h rows x w columns with sparse ratio k
    (gridseq.py:41-76)."""

    t: int
    h: int
    w: int
    k: int = 1

    def __post_init__(self) -> None:
        for name in ("t", "h", "w", "k"):
            v = getattr(self, name)
            if not isinstance(v, int) or isinstance(v, bool) or v < 1:
                raise ValueError(f"GridShape.{name} must be a positive integer, got {v!r}")

    @property
    def seq_len(self) -> int:
        return self.t * self.h * self.w

    def flatten_index(self, t: int, h: int, w: int) -> int:
        if not (0 <= t < self.t and 0 <= h < self.h and 0 <= w < self.w):
            raise CoordinateError(f"coordinate ({t}, {h}, {w}) outside grid "
                                  f"{self.t}x{self.h}x{self.w}")
        return (t * self.h + h) * self.w + w

    def unflatten_index(self, s: int) -> tuple[int, int, int]:
        if not 0 <= s < self.seq_len:
            raise CoordinateError(f"flat index {s} outside sequence of length {self.seq_len}")
        return s // (self.h * self.w), (s // self.w) % self.h, s % self.w


_DATA_MODE = ["torch"]


def set_data_mode(mode: str) -> str:
    """How `SequenceTensor.data` reads: "torch" (the device tensor, the default) or "numpy" (a
    host float64 / uint8 copy, what the reference's numpy callers expect, e.g. its checks and
    tests, gridseq.py:79-116).  The package itself always uses `SequenceTensor.tensor`.
    Returns the previous mode."""
    if mode not in ("torch", "numpy"):
        raise ValueError("data mode must be 'torch' or 'numpy'")
    prev = _DATA_MODE[0]
    _DATA_MODE[0] = mode
    return prev


class SequenceTensor:
    """(batch, seq, chan) tensor with a scalar kind ("real" or "hif8" codes)."""

    __slots__ = ("tensor", "kind")

    def __init__(self, data, kind: str = REAL):
        if kind not in (REAL, HIF8):
            raise ValueError(f"unknown scalar kind {kind!r}")
        if not isinstance(data, torch.Tensor):
            arr = np.asarray(data)
            if kind == HIF8:
                arr = arr.astype(np.uint8)
            elif not np.issubdtype(arr.dtype, np.floating):
                arr = arr.astype(np.float64)
            data = torch.from_numpy(np.ascontiguousarray(arr)).to(default_device())
        elif kind == HIF8 and data.dtype != torch.uint8:
            data = data.to(torch.uint8)
        if data.dim() != 3:
            raise ShapeError(f"SequenceTensor data must be (batch, seq, chan), got shape "
                             f"{tuple(data.shape)}")
        self.tensor = data
        self.kind = kind

    @property
    def data(self):
        """The (batch, seq, chan) values: the device tensor, or in numpy data mode a read-only
        host copy (float64 for real values, uint8 for HiF8 codes) as the reference returns."""
        if _DATA_MODE[0] == "numpy":
            return self.numpy()
        return self.tensor

    @property
    def batch(self) -> int:
        return self.tensor.shape[0]

    @property
    def seq(self) -> int:
        return self.tensor.shape[1]

    @property
    def chan(self) -> int:
        return self.tensor.shape[2]

    def with_data(self, data) -> "SequenceTensor":
        return SequenceTensor(data, kind=self.kind)

    def numpy(self) -> np.ndarray:
        t = self.tensor.detach()
        if self.kind == REAL and t.dtype != torch.float64:
            t = t.to(torch.float64)
        a = t.cpu().numpy()
        a.flags.writeable = False
        return a

    def __array__(self, dtype=None, copy=None):
        a = self.numpy()
        return a.astype(dtype) if dtype is not None else a

    @staticmethod
    def zeros(batch: int, seq: int, chan: int, kind: str = REAL, dtype=None,
              device=None) -> "SequenceTensor":
        dt = torch.uint8 if kind == HIF8 else (dtype or torch.float64)
        return SequenceTensor(torch.zeros((batch, seq, chan), dtype=dt,
                                          device=device or default_device()), kind=kind)


def random_tensor(batch: int, seq: int, chan: int, seed: int, dtype=torch.float64,
                  device=None) -> SequenceTensor:
    """Standard normal from a PCG64 stream in storage order (gridseq.py:119-122);
    identical values to the reference for the same seed (before any cast)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    arr = rng.standard_normal((batch, seq, chan))
    return SequenceTensor(torch.from_numpy(arr).to(device or default_device(), dtype))


# ----------------------------------------------------------------------------- IndexMap

class _MapApply(torch.autograd.Function):
    """Gather through a map; the backward applies the adjoint map (for the
    bijective pattern maps that is the inverse map; for the pad-fused maps it
    is the strip/pad dual)."""

    @staticmethod
    def forward(ctx, x, m):
        ctx.m = m
        return m._apply_raw(x)

    @staticmethod
    def backward(ctx, g):
        return ctx.m._adjoint()._apply_raw(g.contiguous()), None


class IndexMap:
    """Gather map: output address (b, s) reads input flat address src[b, s]
    (gridseq.py:125-195).

    Construct with an explicit table exactly like the reference
    (`IndexMap(in_batch, in_seq, out_batch, out_seq, src)`), or obtain a lazy
    closed-form map from the pattern builders in `skiparse`.
    """

    def __init__(self, in_batch: int, in_seq: int, out_batch: int, out_seq: int, src=None, *,
                 _spec: tuple | None = None):
        self.in_batch, self.in_seq = int(in_batch), int(in_seq)
        self.out_batch, self.out_seq = int(out_batch), int(out_seq)
        if self.in_batch * self.in_seq != self.out_batch * self.out_seq and _spec is None:
            raise ShapeError("IndexMap must preserve the total element count")
        self._spec = _spec
        self._src = None
        if _spec is None:
            if src is None:
                raise ValueError("IndexMap needs a src table")
            t = src if isinstance(src, torch.Tensor) else torch.from_numpy(
                np.ascontiguousarray(np.asarray(src, dtype=np.int64)))
            t = t.to(default_device(), torch.int64).contiguous()
            if tuple(t.shape) != (self.out_batch, self.out_seq):
                raise ShapeError(f"src shape {tuple(t.shape)} != ({self.out_batch}, {self.out_seq})")
            if t.numel() and (int(t.min()) < 0 or int(t.max()) >= self.total):
                raise ShapeError("source addresses out of range")
            self._src = t

    # -- closed-form constructors ------------------------------------------------
    @classmethod
    def _pattern(cls, name: str, g: GridShape, batch: int, h_orig: int | None = None,
                 w_orig: int | None = None) -> "IndexMap":
        h0 = g.h if h_orig is None else h_orig
        w0 = g.w if w_orig is None else w_orig
        S, S0, n = g.seq_len, g.t * h0 * w0, g.k * g.k
        shapes = {
            "identity": ((batch, S), (batch, S)),
            "orig_to_tsa": ((batch, S0), (n * batch, S // n)),
            "orig_to_gsa": ((batch, S0), (n * batch, S // n)),
            "tsa_to_orig": ((n * batch, S // n), (batch, S0)),
            "gsa_to_orig": ((n * batch, S // n), (batch, S0)),
            "tsa_to_gsa": ((n * batch, S // n), (n * batch, S // n)),
            "gsa_to_tsa": ((n * batch, S // n), (n * batch, S // n)),
        }
        (ib, is_), (ob, os_) = shapes[name]
        return cls(ib, is_, ob, os_, _spec=(name, g, batch, h0, w0))

    @staticmethod
    def identity(batch: int, seq: int) -> "IndexMap":
        return IndexMap._pattern("identity", GridShape(1, 1, seq, 1), batch)

    # -- properties ------------------------------------------------------------
    @property
    def total(self) -> int:
        return self.in_batch * self.in_seq

    @property
    def name(self) -> str:
        return self._spec[0] if self._spec else "table"

    @property
    def src(self) -> torch.Tensor:
        """The int64 gather table, computed on the GPU by the map's own kernel."""
        if self._src is None:
            iota = torch.arange(self.total, dtype=torch.int64, device=default_device())
            self._src = self._apply_raw(iota.view(self.in_batch, self.in_seq, 1)).view(
                self.out_batch, self.out_seq)
        return self._src

    def is_bijection(self) -> bool:
        if self.in_batch * self.in_seq != self.out_batch * self.out_seq:
            return False
        counts = torch.bincount(self.src.reshape(-1), minlength=self.total)
        return bool((counts == 1).all())

    # -- application -----------------------------------------------------------
    def _apply_raw(self, x: torch.Tensor) -> torch.Tensor:
        chan = x.shape[-1]
        if self._spec is not None:
            name, g, batch, h0, w0 = self._spec
            return kernels.rearrange(x, name, g.t, g.h, g.w, g.k, batch, h0, w0)
        out = kernels.gather_rows(x.reshape(-1, chan), self._src.reshape(-1),
                                  self.out_batch * self.out_seq)
        return out.view(self.out_batch, self.out_seq, chan)

    def _adjoint(self) -> "IndexMap":
        return self.invert()

    def apply(self, x):
        """Gather x through the map; channel vectors are copied verbatim.
        Accepts a SequenceTensor (returns one) or a (batch, seq, chan) tensor."""
        data = x.tensor if isinstance(x, SequenceTensor) else x
        if (data.shape[0], data.shape[1]) != (self.in_batch, self.in_seq):
            raise ShapeError(f"map expects input ({self.in_batch}, {self.in_seq}), got "
                             f"({data.shape[0]}, {data.shape[1]})")
        out = _MapApply.apply(data, self) if data.requires_grad else self._apply_raw(data)
        if isinstance(x, SequenceTensor):
            return SequenceTensor(out, kind=x.kind)
        return out

    def compose(self, inner: "IndexMap") -> "IndexMap":
        """Map equal to applying `inner` first, then this map (gridseq.py:171-177)."""
        if (self.in_batch, self.in_seq) != (inner.out_batch, inner.out_seq):
            raise ShapeError("composition shapes do not chain")
        src = kernels.gather_rows(inner.src.reshape(-1, 1), self.src.reshape(-1),
                                  self.out_batch * self.out_seq)
        return IndexMap(inner.in_batch, inner.in_seq, self.out_batch, self.out_seq,
                        src.view(self.out_batch, self.out_seq))

    def invert(self) -> "IndexMap":
        """Inverse map (gridseq.py:179-185).  Closed-form maps return their paired
        closed-form inverse; table maps are inverted on the GPU."""
        if self._spec is not None:
            name, g, batch, h0, w0 = self._spec
            pair = {"identity": "identity", "orig_to_tsa": "tsa_to_orig",
                    "tsa_to_orig": "orig_to_tsa", "orig_to_gsa": "gsa_to_orig",
                    "gsa_to_orig": "orig_to_gsa", "tsa_to_gsa": "gsa_to_tsa",
                    "gsa_to_tsa": "tsa_to_gsa"}[name]
            return IndexMap._pattern(pair, g, batch, h0, w0)
        if not self.is_bijection():
            raise ShapeError("only bijective maps can be inverted")
        inv = kernels.invert_index(self.src.reshape(-1))
        return IndexMap(self.out_batch, self.out_seq, self.in_batch, self.in_seq,
                        inv.view(self.in_batch, self.in_seq))

    def same_permutation(self, other: "IndexMap") -> bool:
        return (self.in_batch, self.in_seq, self.out_batch, self.out_seq) == \
            (other.in_batch, other.in_seq, other.out_batch, other.out_seq) and \
            bool(torch.equal(self.src, other.src))

    def __repr__(self) -> str:
        return (f"IndexMap({self.name}, in=({self.in_batch}, {self.in_seq}), "
                f"out=({self.out_batch}, {self.out_seq}))")


def rearrange_map(batch_axes: Sequence[tuple[str, int]], seq_axes: Sequence[tuple[str, int]],
                  out_batch: Sequence[str], out_seq: Sequence[str]) -> IndexMap:
    """Table map of a pure axis factorisation (gridseq.py:198-229); the table is
    built on the device (transpose of an iota) and applied by the gather kernel."""
    axes = list(batch_axes) + list(seq_axes)
    names = [n for n, _ in axes]
    sizes = dict(axes)
    if len(set(names)) != len(names):
        raise ValueError("duplicate axis names")
    out_names = list(out_batch) + list(out_seq)
    if sorted(out_names) != sorted(names):
        raise ValueError("output axes must be a permutation of input axes")
    prod = lambda xs: int(np.prod(xs, dtype=np.int64)) if xs else 1  # noqa: E731
    ib = prod([s for _, s in batch_axes])
    is_ = prod([s for _, s in seq_axes])
    ob = prod([sizes[n] for n in out_batch])
    os_ = prod([sizes[n] for n in out_seq])
    grid = torch.arange(ib * is_, dtype=torch.int64, device=default_device()).reshape(
        [s for _, s in axes])
    src = grid.permute([names.index(n) for n in out_names]).reshape(ob, os_).contiguous()
    return IndexMap(ib, is_, ob, os_, src)
