"""Padding compaction for the attention (a B200-first restatement of the reference's masking).

On an any-resolution grid the reference pads H, W to multiples of k^2 and then *masks* the pad
tokens inside every subsequence (anyres.py:92-96, attention.py:121-130): pad keys weigh 0 and
pad queries output 0.  Computing those rows and then discarding them costs (S_pad / S_real)^2
of the attention work (1.14x at 720p, 45 -> 48 rows).  Here each subsequence's real rows are
gathered into a compact buffer (K1 table gather), attention runs with per-subsequence lengths
(K2/K3 `seq_lens`), and the outputs are scattered back with zero pad rows -- the same values the
masked computation produces, for ~12% less tensor work at 720p.  Both moves are exact
permutations whose adjoints are each other, so autograd is a gather with the other table.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import kernels
from .errors import ShapeError

__all__ = ["CompactPlan", "compact_plan", "compact_rows", "expand_rows", "RowMove", "row_move",
           "GatherPlan", "gather_plan", "ScatterPlan", "scatter_plan"]


@dataclass(frozen=True)
class CompactPlan:
    n_seq: int
    L: int                  # padded subsequence length
    cap: int                # longest compacted subsequence (buffer capacity)
    lens: torch.Tensor      # (n_seq,) int32 real rows per subsequence
    gather: torch.Tensor    # (n_seq*cap,) int64 padded row of each compact row, -1 = empty
    scatter: torch.Tensor   # (n_seq*L,) int64 compact row of each padded row, -1 = pad

    @property
    def real_rows(self) -> int:
        return int(self.lens.sum())


def compact_plan(valid: torch.Tensor) -> CompactPlan:
    """valid: (n_seq, L) bool on the device (True = real token)."""
    n_seq, L = valid.shape
    v = valid.to(torch.bool)
    lens = v.sum(dim=1)
    cap = max(int(lens.max().item()) if n_seq else 0, 1)
    j = torch.cumsum(v.to(torch.int64), dim=1) - 1
    s = torch.arange(n_seq, device=v.device, dtype=torch.int64)[:, None]
    pos = torch.arange(L, device=v.device, dtype=torch.int64)[None, :]
    scatter = torch.where(v, s * cap + j, torch.full_like(j, -1))
    gather = torch.full((n_seq * cap,), -1, dtype=torch.int64, device=v.device)
    gather[scatter[v]] = (s * L + pos).expand(n_seq, L)[v]
    return CompactPlan(n_seq, L, cap, lens.to(torch.int32).contiguous(), gather.contiguous(),
                       scatter.reshape(-1).contiguous())


def _move(x: torch.Tensor, index: torch.Tensor, n_rows: int, rows_per_seq: int) -> torch.Tensor:
    C = x.shape[-1]
    out = kernels.gather_rows(x.reshape(-1, C), index, n_rows)
    return out.view(n_rows // rows_per_seq, rows_per_seq, C)


class _Compact(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, plan):
        ctx.plan = plan
        return _move(x, plan.gather, plan.n_seq * plan.cap, plan.cap)

    @staticmethod
    def backward(ctx, g):
        p = ctx.plan
        return _move(g.contiguous(), p.scatter, p.n_seq * p.L, p.L), None


class _Expand(torch.autograd.Function):
    @staticmethod
    def forward(ctx, y, plan):
        ctx.plan = plan
        return _move(y, plan.scatter, plan.n_seq * plan.L, plan.L)

    @staticmethod
    def backward(ctx, g):
        p = ctx.plan
        return _move(g.contiguous(), p.gather, p.n_seq * p.cap, p.cap), None


def compact_rows(x: torch.Tensor, plan: CompactPlan) -> torch.Tensor:
    """(n_seq, L, C) padded pattern layout -> (n_seq, cap, C) real rows first."""
    return _Compact.apply(x, plan)


def expand_rows(y: torch.Tensor, plan: CompactPlan) -> torch.Tensor:
    """(n_seq, cap, C) -> (n_seq, L, C) with zero pad rows."""
    return _Expand.apply(y, plan)


@dataclass(frozen=True)
class RowMove:
    """An injective row move out[i] = in[src[i]] (src = -1 -> zero row) between two
    (n_seq, rows_per_seq, C) layouts, with its adjoint (the inverse table)."""

    src: torch.Tensor       # (n_out_seq*out_rows,) int64
    inv: torch.Tensor       # (n_in_seq*in_rows,) int64
    out_rows: int
    in_rows: int


def _check_table(tab: torch.Tensor, n_rows: int, what: str) -> torch.Tensor:
    """Range check of a row table once, when its plan is built (entries in [-1, n_rows)): the
    kernels index with it unchecked."""
    if tab.numel() and (int(tab.min()) < -1 or int(tab.max()) >= n_rows):
        raise ShapeError(f"{what}: row index out of range [-1, {n_rows})")
    return tab


def row_move(src: torch.Tensor, n_in_total: int, out_rows: int, in_rows: int) -> RowMove:
    src = _check_table(src.to(torch.int64).contiguous(), n_in_total, "row move")
    inv = torch.full((n_in_total,), -1, dtype=torch.int64, device=src.device)
    ok = src >= 0
    inv[src[ok]] = torch.nonzero(ok).view(-1)
    if int((inv >= 0).sum()) != int(ok.sum()):
        raise ShapeError("row move is not injective (its adjoint would be wrong)")
    return RowMove(src, inv, out_rows, in_rows)


class _Move(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, mv):
        ctx.mv = mv
        ctx.in_shape = x.shape
        return _move(x, mv.src, mv.src.numel(), mv.out_rows)

    @staticmethod
    def backward(ctx, g):
        mv = ctx.mv
        # returned in the input's own shape: a merely broadcast-compatible shape would make
        # autograd reduce it (sum_to_size), a full extra pass over the activation
        return _move(g.contiguous(), mv.inv, mv.inv.numel(), mv.in_rows).view(ctx.in_shape), None


def apply_move(x: torch.Tensor, mv: RowMove) -> torch.Tensor:
    return _Move.apply(x, mv)


@dataclass(frozen=True)
class ScatterPlan:
    """Output-side row table of the scatter-mode attention (K2 epilogue / K3 Delta pre-pass):
    row j of compact sequence s is stored to destination row out_index[s, j] (-1 = dropped);
    zero_rows are the destination rows no source lands on (zero-filled by the forward)."""

    out_index: torch.Tensor            # (n_seq, cap) int32
    zero_rows: torch.Tensor | None     # (n_zero,) int32
    n_out_rows: int
    out_shape: tuple                   # view of the (n_out_rows, C) output


def scatter_plan(out_index: torch.Tensor, n_seq: int, cap: int, n_out_rows: int,
                 out_shape: tuple) -> ScatterPlan:
    """out_index (n_seq*cap,) int64: destination row of every source row (-1 = none); the map
    must be injective."""
    oi = _check_table(out_index.to(torch.int64).reshape(-1), n_out_rows, "scatter plan")
    hit = torch.zeros(n_out_rows, dtype=torch.bool, device=oi.device)
    ok = oi >= 0
    hit[oi[ok]] = True
    if int(hit.sum()) != int(ok.sum()):
        raise ValueError("scatter plan is not injective")
    zero = torch.nonzero(~hit).view(-1).to(torch.int32).contiguous()
    return ScatterPlan(oi.view(n_seq, cap).to(torch.int32).contiguous(), zero if zero.numel() else None,
                       n_out_rows, tuple(out_shape))


@dataclass(frozen=True)
class GatherPlan:
    """Row table of the fused-rearrange attention (gather mode, K2/K3): subsequence s of a
    pattern is rows row_index[s, :lens[s]] of a token-major tensor (the original latent layout),
    so no rearranged copy is ever materialised."""

    row_index: torch.Tensor   # (n_seq, cap) int32, -1 beyond lens[s]; cap % 128 == 0
    lens: torch.Tensor        # (n_seq,) int32
    n_rows: int               # rows of the token-major tensors
    covers_all: bool          # every row belongs to some subsequence


def gather_plan(grid, pattern, batch: int = 1, pg=None, target: str = "original",
                rows: tuple | None = None) -> GatherPlan:
    """Table for `pattern` subsequences [rows) of `batch` items on the padded grid of `pg`
    (or `grid` when unpadded).  target "original": rows of the unpadded (batch, T*H0*W0) latent
    (pad tokens simply never appear); "padded": rows of the padded (batch, T*H*W) latent."""
    from .skiparse import SparsePattern, pattern_map
    from .gridseq import default_device
    padded = pg.padded if pg is not None else grid
    dev = default_device()
    S = padded.seq_len
    pat = SparsePattern(pattern)
    k2 = 1 if pat is SparsePattern.ORIGINAL else padded.k * padded.k
    L = S // k2
    if pat is SparsePattern.ORIGINAL:
        src = torch.arange(batch * S, device=dev, dtype=torch.int64).view(batch, S)
    else:
        src = pattern_map(padded, pat, batch).src.to(dev).view(batch * k2, L)   # -> b*S + token
    if pg is not None and not pg.trivial:
        mask = pg.mask.to(dev).bool()                                  # (S,) real tokens
        valid = mask[src % S]
    else:
        valid = torch.ones_like(src, dtype=torch.bool)
    if rows is not None:
        src, valid = src[rows[0]:rows[1]], valid[rows[0]:rows[1]]
    if target == "original" and pg is not None and not pg.trivial:
        real_idx = torch.cumsum(mask.to(torch.int64), 0) - 1          # padded token -> real index
        S_real = int(mask.sum())
        dest = (src // S) * S_real + real_idx[src % S]
        n_rows = batch * S_real
    else:
        dest = src
        n_rows = batch * S
    n_seq = src.shape[0]
    lens = valid.sum(dim=1)
    cap = max(int(lens.max().item()) if n_seq else 0, 1)
    cap = (cap + 127) // 128 * 128
    j = torch.cumsum(valid.to(torch.int64), dim=1) - 1
    table = torch.full((n_seq, cap), -1, dtype=torch.int64, device=dev)
    srow = torch.arange(n_seq, device=dev)[:, None].expand_as(j)
    table[srow[valid], j[valid]] = dest[valid]
    covered = int(lens.sum()) == n_rows
    return GatherPlan(table.to(torch.int32).contiguous(), lens.to(torch.int32).contiguous(), n_rows,
                      covered)
