"""Any-resolution padding -- drop-in for osp.anyres (anyres.py:26-96).

Pad h, w up to multiples of k^2; the 1-D validity mask is evaluated from
coordinates on the GPU (K5) instead of being stored and permuted.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import torch

from . import kernels
from .errors import ShapeError
from .gridseq import GridShape, SequenceTensor, default_device
from .skiparse import SparsePattern, _require_gsa, _require_tsa

__all__ = ["PaddedGrid", "pad_grid", "pad_tensor", "strip_padding", "subsequence_mask"]


def _ceil_to(v: int, m: int) -> int:
    return -(-v // m) * m


@dataclass(frozen=True)
class PaddedGrid:
    """Original grid and its padded counterpart (anyres.py:26-54).  `mask` (flat
    padded validity) and `embedding` (padded positions of original tokens) are
    materialised lazily on the device."""

    original: GridShape
    padded: GridShape
    _cache: dict = field(default_factory=dict, compare=False, repr=False)

    @property
    def trivial(self) -> bool:
        return self.padded == self.original

    @property
    def mask(self) -> torch.Tensor:
        if "mask" not in self._cache:
            p = self.padded
            bits = kernels.pattern_mask_bits(1, p.t, p.h, p.w, p.k, "original", self.original.h,
                                             self.original.w, default_device())
            self._cache["mask"] = kernels.bits_to_bytes(bits, p.seq_len).view(-1)
        return self._cache["mask"]

    @property
    def embedding(self) -> torch.Tensor:
        if "embedding" not in self._cache:
            self._cache["embedding"] = torch.nonzero(self.mask).view(-1)
        return self._cache["embedding"]

    def mask_or_none(self):
        return None if self.trivial else self.mask

    def mask_bits(self, pattern: SparsePattern, batch: int = 1) -> torch.Tensor | None:
        """Bit-packed subsequence key mask for the attention kernel (K5), in the
        enlarged-batch order (pattern id, batch item); None when trivial."""
        if self.trivial:
            return None
        key = ("bits", pattern, batch)
        if key not in self._cache:
            p = self.padded
            self._cache[key] = kernels.pattern_mask_bits(batch, p.t, p.h, p.w, p.k, pattern.value,
                                                         self.original.h, self.original.w,
                                                         default_device())
        return self._cache[key]


    def compact_plan(self, pattern: SparsePattern, batch: int = 1, rows: tuple | None = None):
        """CompactPlan (compact.py) of the pattern layout's subsequences [rows[0], rows[1]) of
        the enlarged batch (all when None); None when the grid needs no padding."""
        if self.trivial:
            return None
        key = ("plan", pattern, batch, rows)
        if key not in self._cache:
            from .compact import compact_plan
            p = self.padded
            L = p.seq_len if pattern is SparsePattern.ORIGINAL else p.seq_len // (p.k * p.k)
            bits = self.mask_bits(pattern, batch)
            valid = kernels.bits_to_bytes(bits, L).view(-1, L).bool()
            if rows is not None:
                valid = valid[rows[0]:rows[1]]
            self._cache[key] = compact_plan(valid)
        return self._cache[key]


def pad_grid(g: GridShape) -> PaddedGrid:
    """Pad h and w to the nearest multiple of k^2; t is never padded (anyres.py:57-66)."""
    k2 = g.k * g.k
    return PaddedGrid(g, GridShape(g.t, _ceil_to(g.h, k2), _ceil_to(g.w, k2), g.k))


def pad_tensor(x, pg: PaddedGrid, pad_value: float = 0.0, pad_fill=None):
    """Embed an original-grid tensor into the padded grid (anyres.py:69-82):
    the K1 pad gather writes zeros to pad slots; a non-zero pad_value or the
    test-only pad_fill rows are then scattered into the pad slots."""
    data = x.tensor if isinstance(x, SequenceTensor) else x
    if data.shape[1] != pg.original.seq_len:
        raise ShapeError(f"expected seq {pg.original.seq_len}, got {data.shape[1]}")
    p = pg.padded
    out = kernels.rearrange(data, "pad", p.t, p.h, p.w, p.k, data.shape[0], pg.original.h,
                            pg.original.w)
    if pad_fill is not None or pad_value != 0.0:
        pads = ~pg.mask
        if pad_fill is not None:
            fill = torch.as_tensor(pad_fill, dtype=out.dtype, device=out.device)
            out[:, pads, :] = fill
        else:
            out[:, pads, :] = pad_value
    return SequenceTensor(out, kind=x.kind) if isinstance(x, SequenceTensor) else out


def strip_padding(x, pg: PaddedGrid):
    """Keep real tokens in original order (anyres.py:85-89)."""
    data = x.tensor if isinstance(x, SequenceTensor) else x
    if data.shape[1] != pg.padded.seq_len:
        raise ShapeError(f"expected padded seq {pg.padded.seq_len}, got {data.shape[1]}")
    p = pg.padded
    out = kernels.rearrange(data, "strip", p.t, p.h, p.w, p.k, data.shape[0], pg.original.h,
                            pg.original.w)
    return SequenceTensor(out, kind=x.kind) if isinstance(x, SequenceTensor) else out


def subsequence_mask(pg: PaddedGrid, pattern: SparsePattern) -> torch.Tensor:
    """(n_sub, L) validity of every (subsequence, position) slot (anyres.py:92-96)."""
    p = pg.padded
    if pattern is SparsePattern.TOKEN_WISE:
        _require_tsa(p)
    elif pattern is SparsePattern.GROUP_WISE:
        _require_gsa(p)
    n_sub = 1 if pattern is SparsePattern.ORIGINAL else p.k * p.k
    L = p.seq_len // n_sub
    bits = kernels.pattern_mask_bits(1, p.t, p.h, p.w, p.k, pattern.value, pg.original.h,
                                     pg.original.w, default_device())
    return kernels.bits_to_bytes(bits, L)
