"""Skiparse attention -- drop-in for osp.attention (attention.py:20-168).

dense_attention / skiparse_attention keep the reference signatures and
semantics (masked keys weigh 0, all-masked rows and pad queries output 0,
fixed seeded projections), extended with `heads` (per-head 1/sqrt(d) scale;
heads=1 is exactly the reference's single head over all channels).  The
per-subsequence attention runs on the K2/K3 tcgen05 kernels in bf16 with fp32
accumulation; the fixed q/k/v projection is one cuBLAS GEMM against the packed
[Wq | Wk | Wv] matrix, applied in the pattern layout (a token-wise op commutes
with the rearrange, so only x -- not q, k, v -- is rearranged).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch
import torch.nn.functional as F

from . import kernels
from .anyres import PaddedGrid
from .errors import ShapeError, UnsupportedError
from .gridseq import GridShape, SequenceTensor, default_device
from .skiparse import SparsePattern, assignment_of, inverse_pattern_map, pattern_map

__all__ = ["PROJECTION_SEED", "qkv_projections", "packed_projection", "project_qkv",
           "dense_attention", "skiparse_attention", "attention_packed", "attention_scatter",
           "masked_dense_attention",
           "pattern_allow_matrix", "skiparse_reference", "FlopReport",
           "flop_report"]

PROJECTION_SEED = 184594917  # attention.py:20
COMPUTE_DTYPE = torch.bfloat16


def qkv_projections(chan: int, seed: int = PROJECTION_SEED, device=None,
                    dtype=torch.float64) -> tuple[torch.Tensor, torch.Tensor, torch.Tensor]:
    """Three PCG64 standard-normal (chan x chan) draws scaled by 1/sqrt(chan)
    (attention.py:23-27); bit-identical to the reference in float64."""
    rng = np.random.Generator(np.random.PCG64(seed))
    s = 1.0 / np.sqrt(chan)
    mats = [rng.standard_normal((chan, chan)) * s for _ in range(3)]
    dev = device or default_device()
    return tuple(torch.from_numpy(m).to(dev, dtype) for m in mats)


_PACKED: dict = {}


def packed_projection(chan: int, dtype=COMPUTE_DTYPE, device=None,
                      seed: int = PROJECTION_SEED) -> torch.Tensor:
    """[Wq | Wk | Wv] as one (chan, 3*chan) matrix, cached per (chan, dtype, device)."""
    dev = device or default_device()
    key = (chan, dtype, str(dev), seed)
    if key not in _PACKED:
        wq, wk, wv = qkv_projections(chan, seed, dev)
        _PACKED[key] = torch.cat([wq, wk, wv], dim=1).to(dtype).contiguous()
    return _PACKED[key]


def project_qkv(x: SequenceTensor, seed: int = PROJECTION_SEED):
    """x @ Wq, x @ Wk, x @ Wv (attention.py:30-32)."""
    wq, wk, wv = qkv_projections(x.chan, seed, x.tensor.device, x.tensor.dtype)
    return x.with_data(x.tensor @ wq), x.with_data(x.tensor @ wk), x.with_data(x.tensor @ wv)


# ----------------------------------------------------------------------------- autograd ops

class _AttnPacked(torch.autograd.Function):
    """Attention over a packed (n_seq, L, 3*C) [q | k | v] tensor; the backward
    writes dq, dk, dv straight into one packed gradient buffer."""

    @staticmethod
    def forward(ctx, qkv, heads, d, bits, zero_q, scale, seq_lens=None):
        C = heads * d
        q, k, v = qkv[..., :C], qkv[..., C:2 * C], qkv[..., 2 * C:]
        o, lse = kernels.attn_fwd(q, k, v, heads, d, bits, zero_q, scale, seq_lens=seq_lens)
        ctx.save_for_backward(qkv, o, lse)
        ctx.cfg = (heads, d, bits, zero_q, scale, seq_lens)
        return o

    @staticmethod
    def backward(ctx, do):
        qkv, o, lse = ctx.saved_tensors
        heads, d, bits, zero_q, scale, seq_lens = ctx.cfg
        C = heads * d
        dqkv = torch.empty_like(qkv)
        kernels.attn_bwd(qkv[..., :C], qkv[..., C:2 * C], qkv[..., 2 * C:], o, do.contiguous(), lse,
                         heads, d, bits, zero_q, scale, dq=dqkv[..., :C], dk=dqkv[..., C:2 * C],
                         dv=dqkv[..., 2 * C:], seq_lens=seq_lens)
        return dqkv, None, None, None, None, None, None


class _Attn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, q, k, v, heads, d, bits, zero_q, scale, seq_lens=None):
        o, lse = kernels.attn_fwd(q, k, v, heads, d, bits, zero_q, scale, seq_lens=seq_lens)
        ctx.save_for_backward(q, k, v, o, lse)
        ctx.cfg = (heads, d, bits, zero_q, scale, seq_lens)
        return o

    @staticmethod
    def backward(ctx, do):
        q, k, v, o, lse = ctx.saved_tensors
        heads, d, bits, zero_q, scale, seq_lens = ctx.cfg
        dq, dk, dv = kernels.attn_bwd(q, k, v, o, do.contiguous(), lse, heads, d, bits, zero_q,
                                      scale, seq_lens=seq_lens)
        return dq, dk, dv, None, None, None, None, None, None


class _AttnGather(torch.autograd.Function):
    """Fused-rearrange attention over a token-major packed (n_rows, 3*C) [q | k | v]: the
    subsequences of a pattern are read and written through a GatherPlan row table (K2/K3
    gather mode); the result is token-major too."""

    @staticmethod
    def forward(ctx, qkv, heads, d, plan, scale):
        C = heads * d
        q, k, v = qkv[:, :C], qkv[:, C:2 * C], qkv[:, 2 * C:]
        out = None if plan.covers_all else torch.zeros((qkv.shape[0], C), dtype=qkv.dtype, device=qkv.device)
        o, lse = kernels.attn_fwd_gather(q, k, v, heads, d, plan.row_index, plan.lens, scale, out=out)
        ctx.save_for_backward(qkv, o, lse)
        ctx.cfg = (heads, d, plan, scale)
        return o

    @staticmethod
    def backward(ctx, do):
        qkv, o, lse = ctx.saved_tensors
        heads, d, plan, scale = ctx.cfg
        C = heads * d
        dqkv = torch.empty_like(qkv) if plan.covers_all else torch.zeros_like(qkv)
        kernels.attn_bwd_gather(qkv[:, :C], qkv[:, C:2 * C], qkv[:, 2 * C:], o, do.contiguous(), lse,
                                heads, d, plan.row_index, plan.lens, scale, dq=dqkv[:, :C],
                                dk=dqkv[:, C:2 * C], dv=dqkv[:, 2 * C:])
        return dqkv, None, None, None, None


class _AttnScatter(torch.autograd.Function):
    """Attention over a packed (n_seq, cap, 3*C) [q | k | v] whose output rows are STORED through
    a row table (compact.ScatterPlan): the rearrange / padding expansion that follows attention
    runs in the K2 epilogue, and the backward's Delta pre-pass gathers dO through the same table."""

    @staticmethod
    def forward(ctx, qkv, heads, d, lens, plan, scale):
        C = heads * d
        q, k, v = qkv[..., :C], qkv[..., C:2 * C], qkv[..., 2 * C:]
        out = torch.empty((plan.n_out_rows, C), dtype=qkv.dtype, device=qkv.device)
        lse = kernels.attn_fwd_scatter(q, k, v, heads, d, lens, plan.out_index, out, plan.zero_rows, scale)
        ctx.save_for_backward(qkv, out, lse)
        ctx.cfg = (heads, d, lens, plan, scale)
        return out.view(plan.out_shape)

    @staticmethod
    def backward(ctx, dout):
        qkv, out, lse = ctx.saved_tensors
        heads, d, lens, plan, scale = ctx.cfg
        C = heads * d
        dqkv = torch.empty_like(qkv)
        kernels.attn_bwd_scatter(qkv[..., :C], qkv[..., C:2 * C], qkv[..., 2 * C:], out,
                                 dout.reshape(-1, C), lse, heads, d, lens, plan.out_index, scale,
                                 dqkv[..., :C], dqkv[..., C:2 * C], dqkv[..., 2 * C:])
        return dqkv, None, None, None, None, None


def attention_scatter(qkv: torch.Tensor, heads: int, lens: torch.Tensor, plan,
                      scale: float | None = None) -> torch.Tensor:
    """Per-subsequence attention over packed bf16 [q | k | v] (n_seq, cap, 3*C) whose output is
    written straight into the next layout through plan (compact.ScatterPlan): returns a tensor of
    plan.out_shape.  head_dim 64 or 128."""
    C = qkv.shape[-1] // 3
    d = C // heads
    if heads * d != C or d not in (64, 128):
        raise UnsupportedError("scatter-mode attention runs head_dim 64 or 128")
    scale = 1.0 / math.sqrt(d) if scale is None else scale
    return _AttnScatter.apply(qkv.contiguous(), heads, d, lens, plan, scale)


def attention_gather(qkv: torch.Tensor, heads: int, plan, scale: float | None = None) -> torch.Tensor:
    """Skiparse attention with the rearrange fused into the kernels' TMA loads / stores:
    qkv (..., n_rows, 3*C) token-major bf16, plan = compact.GatherPlan.  head_dim 128."""
    shape = qkv.shape
    C = shape[-1] // 3
    d = C // heads
    if d != 128:
        raise UnsupportedError("gather-mode attention runs head_dim 128")
    scale = 1.0 / math.sqrt(d) if scale is None else scale
    o = _AttnGather.apply(qkv.reshape(-1, 3 * C).contiguous(), heads, d, plan, scale)
    return o.view(*shape[:-1], C)


def _pad_heads(t: torch.Tensor, heads: int, d: int, dp: int) -> torch.Tensor:
    n, L, _ = t.shape
    return F.pad(t.reshape(n, L, heads, d), (0, dp - d)).reshape(n, L, heads * dp)


def attention_packed(qkv: torch.Tensor, heads: int, bits=None, zero_invalid_queries=False,
                     scale: float | None = None, seq_lens: torch.Tensor | None = None) -> torch.Tensor:
    """Per-item attention over packed bf16 [q | k | v] (n_seq, L, 3*C) -> (n_seq, L, C).
    seq_lens (n_seq,) int32: item s uses only its first seq_lens[s] rows (compacted padding)."""
    C = qkv.shape[-1] // 3
    d = C // heads
    if heads * d != C:
        raise ShapeError(f"chan {C} not divisible by heads {heads}")
    scale = 1.0 / math.sqrt(d) if scale is None else scale
    dp = kernels._head_dim_plan(d)
    if dp == d:
        return _AttnPacked.apply(qkv.contiguous(), heads, d, bits, bool(zero_invalid_queries),
                                 scale, seq_lens)
    q, k, v = (_pad_heads(qkv[..., i * C:(i + 1) * C], heads, d, dp) for i in range(3))
    o = _Attn.apply(q.contiguous(), k.contiguous(), v.contiguous(), heads, dp, bits,
                    bool(zero_invalid_queries), scale, seq_lens)
    n, L, _ = o.shape
    return o.reshape(n, L, heads, dp)[..., :d].reshape(n, L, C)


def _attention(q, k, v, heads, bits, zero_q, scale):
    C = q.shape[-1]
    d = C // heads
    dp = kernels._head_dim_plan(d)
    if dp != d:
        q, k, v = (_pad_heads(t, heads, d, dp) for t in (q, k, v))
    o = _Attn.apply(q.contiguous(), k.contiguous(), v.contiguous(), heads, dp, bits, zero_q, scale)
    if dp != d:
        n, L, _ = o.shape
        o = o.reshape(n, L, heads, dp)[..., :d].reshape(n, L, C)
    return o


def _as_tensor(x):
    return x.tensor if isinstance(x, SequenceTensor) else x


def dense_attention(q, k, v, key_valid=None, heads: int = 1, scale: float | None = None):
    """Scaled dot-product attention per batch item (attention.py:47-67).
    key_valid: (batch, seq) or (seq,) flags; invalid keys are excluded and rows
    with no valid key output zeros.  Computed in bf16 on the B200 kernels; the
    result is returned in q's dtype."""
    qd, kd, vd = _as_tensor(q), _as_tensor(k), _as_tensor(v)
    if qd.shape != kd.shape or qd.shape != vd.shape:
        raise ShapeError("q, k, v must share (batch, seq, chan)")
    B, S, C = qd.shape
    if C % heads:
        raise ShapeError(f"chan {C} not divisible by heads {heads}")
    d = C // heads
    scale = 1.0 / math.sqrt(d) if scale is None else scale
    bits = None
    if key_valid is not None:
        kv = torch.as_tensor(np.asarray(key_valid) if not isinstance(key_valid, torch.Tensor)
                             else key_valid, device=qd.device).bool()
        if kv.dim() == 1:
            kv = kv.expand(B, S)
        if tuple(kv.shape) != (B, S):
            raise ShapeError(f"key_valid shape {tuple(kv.shape)} != ({B}, {S})")
        bits = kernels.bytes_to_bits(kv.contiguous())
    cast = (lambda t: t.to(COMPUTE_DTYPE)) if qd.dtype != COMPUTE_DTYPE else (lambda t: t)
    out = _attention(cast(qd), cast(kd), cast(vd), heads, bits, False, scale).to(qd.dtype)
    return SequenceTensor(out) if isinstance(q, SequenceTensor) else out


def skiparse_attention(x, g: GridShape, pattern: SparsePattern, pg: PaddedGrid | None = None,
                       heads: int = 1, weights: torch.Tensor | None = None):
    """Sparse attention (attention.py:97-131): rearrange to the pattern layout,
    dense attention per subsequence under the 1-D subsequence mask, zero pad-query
    rows, rearrange back.  With a PaddedGrid, x must already live on the padded
    grid.  `weights` optionally overrides the packed (C, 3C) projection."""
    xd = _as_tensor(x)
    grid = pg.padded if pg is not None else g
    if xd.shape[1] != grid.seq_len:
        raise ShapeError(f"expected seq {grid.seq_len}, got {xd.shape[1]}")
    B, S, C = xd.shape
    if C % heads:
        raise ShapeError(f"chan {C} not divisible by heads {heads}")
    W = weights if weights is not None else packed_projection(C, COMPUTE_DTYPE, xd.device)
    xb = xd.to(COMPUTE_DTYPE)
    if pattern is SparsePattern.ORIGINAL:
        xp = xb
    else:
        xp = pattern_map(grid, pattern, B).apply(xb)
    plan = pg.compact_plan(pattern, B) if pg is not None else None
    if plan is None:
        o = attention_packed(torch.matmul(xp, W), heads)
    else:
        # pad tokens are masked keys and zero-output queries (attention.py:121-130): run only the
        # real rows of each subsequence (compact.py) -- identical values, less work
        from .compact import compact_rows, expand_rows
        qkv = torch.matmul(compact_rows(xp, plan), W)
        o = expand_rows(attention_packed(qkv, heads, seq_lens=plan.lens), plan)
    if pattern is not SparsePattern.ORIGINAL:
        o = inverse_pattern_map(grid, pattern, B).apply(o)
    out = o.to(xd.dtype)
    return SequenceTensor(out) if isinstance(x, SequenceTensor) else out


def masked_dense_attention(q, k, v, allow):
    """Dense attention under an explicit 2-D (query, key) permission matrix
    (attention.py:70-82).  Like the reference this is the ORACLE route -- the production
    sparse path never builds a 2-D mask -- so it is plain fp64 torch on the device (O(S^2)
    memory), kept only so reference code that cross-checks skiparse_attention against it
    keeps running.  Queries with no allowed key output zeros."""
    qd, kd, vd = _as_tensor(q), _as_tensor(k), _as_tensor(v)
    a = torch.as_tensor(np.asarray(allow) if not isinstance(allow, torch.Tensor) else allow,
                        device=qd.device).bool()
    if a.dim() == 2:
        a = a.expand(qd.shape[0], qd.shape[1], qd.shape[1])
    qd, kd, vd = (t.to(torch.float64) for t in (qd, kd, vd))
    s = torch.einsum("bic,bjc->bij", qd, kd) / math.sqrt(qd.shape[-1])
    s = s.masked_fill(~a, float("-inf"))
    m = s.amax(-1, keepdim=True)
    m = torch.where(torch.isfinite(m), m, torch.zeros_like(m))
    w = torch.exp(s - m)
    den = w.sum(-1, keepdim=True)
    w = torch.where(den > 0, w / torch.where(den == 0, torch.ones_like(den), den), torch.zeros_like(w))
    out = torch.einsum("bij,bjc->bic", w, vd)
    return SequenceTensor(out) if isinstance(q, SequenceTensor) else out


def pattern_allow_matrix(g: GridShape, pattern: SparsePattern, pg: PaddedGrid | None = None):
    """(seq, seq) permission: u, v interact iff they share a subsequence under the pattern
    and, when padded, both are real tokens (attention.py:85-94)."""
    grid = pg.padded if pg is not None else g
    sub = assignment_of(grid, pattern).subseq
    allow = sub[:, None] == sub[None, :]
    if pg is not None:
        m = pg.mask.to(sub.device).bool()
        allow &= m[:, None] & m[None, :]
    return allow


def skiparse_reference(x, g: GridShape, pattern: SparsePattern, pg: PaddedGrid | None = None):
    """Oracle route (attention.py:134-143): dense attention over the original layout under
    the 2-D pattern mask, in fp64 with the reference's fp64 projections."""
    xd = _as_tensor(x)
    grid = pg.padded if pg is not None else g
    if xd.shape[1] != grid.seq_len:
        raise ShapeError(f"expected seq {grid.seq_len}, got {xd.shape[1]}")
    wq, wk, wv = qkv_projections(xd.shape[-1], device=xd.device)
    x64 = xd.to(torch.float64)
    out = masked_dense_attention(x64 @ wq, x64 @ wk, x64 @ wv, pattern_allow_matrix(g, pattern, pg))
    return SequenceTensor(out) if isinstance(x, SequenceTensor) else out


@dataclass(frozen=True)
class FlopReport:
    """Multiply-accumulate counts of one attention application over one batch
    item (attention.py:146-156)."""

    full_flops: int
    sparse_flops: int

    @property
    def ratio(self) -> float:
        return self.sparse_flops / self.full_flops


def flop_report(g: GridShape, pattern: SparsePattern, chan: int = 1) -> FlopReport:
    """Full attention costs 2*seq^2*chan MACs; a pattern runs k^2 subsequences
    of length seq/k^2 (attention.py:159-168)."""
    seq = g.seq_len
    full = 2 * seq * seq * chan
    if pattern is SparsePattern.ORIGINAL:
        return FlopReport(full, full)
    n_sub = g.k * g.k
    pattern_map(g, pattern)  # divisibility check, as the reference's map build does
    sub_len = seq // n_sub
    return FlopReport(full, n_sub * 2 * sub_len * sub_len * chan)
