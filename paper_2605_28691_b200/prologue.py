"""QKV projection + QK-RMSNorm + 3-D RoPE prologue, executed by the K6
tcgen05 GEMM (csrc/proj.cu) whose epilogue writes attention-ready q | k | v in the pattern layout.

With norm=None and rope=False this is exactly the reference's fixed projection
x @ [Wq | Wk | Wv] (attention.py:20-32, applied at attention.py:108) -- only in the pattern
layout, which is legal because a token-wise op commutes with the rearrange.  The norm / RoPE
options follow the Wan-style DiT attention the paper builds on (PAPER.md: Wan2.1-14B base):
QK-RMSNorm over all channels ("channel") or per head ("head"), and 3-D RoPE whose 64 rotation
pairs per 128-wide head split 22 / 21 / 21 over the (t, h, w) axes, positions being each token's
padded-grid coordinates (recovered on the device from its pattern-layout row).
"""

from __future__ import annotations

import numpy as np
import torch

from . import kernels
from .attention import PROJECTION_SEED, qkv_projections
from .gridseq import GridShape, default_device
from .skiparse import SparsePattern

__all__ = ["rope_table", "packed_projection_t", "qkv_project", "QKVPrologue", "ROPE_THETA"]

ROPE_THETA = 10000.0
_PATTERN_IDS = {SparsePattern.ORIGINAL: 0, SparsePattern.TOKEN_WISE: 1, SparsePattern.GROUP_WISE: 2}
_NORMS = {None: 0, "head": 1, "channel": 2}
_TABLES: dict = {}
_PACKED_T: dict = {}


def rope_axes(head_dim: int = 128) -> tuple[int, int, int]:
    """Channels per axis (t, h, w): d - 4*(d//6), 2*(d//6), 2*(d//6) (44, 42, 42 for d=128)."""
    return head_dim - 4 * (head_dim // 6), 2 * (head_dim // 6), 2 * (head_dim // 6)


def rope_table(grid: GridShape, head_dim: int = 128, theta: float = ROPE_THETA, device=None) -> torch.Tensor:
    """(t + h + w, 32, 2) fp32 (cos, sin): row a_off + pos, column = pair index within the
    axis, angle = pos * theta^(-2j / axis_dim) (computed in float64)."""
    dev = torch.device(device or default_device())
    key = (grid.t, grid.h, grid.w, head_dim, theta, str(dev))
    if key not in _TABLES:
        tab = np.zeros((grid.t + grid.h + grid.w, 32, 2))
        row = 0
        for n_pos, dim in zip((grid.t, grid.h, grid.w), rope_axes(head_dim)):
            freqs = theta ** (-np.arange(0, dim, 2, dtype=np.float64) / dim)
            ang = np.outer(np.arange(n_pos, dtype=np.float64), freqs)
            tab[row:row + n_pos, :dim // 2, 0] = np.cos(ang)
            tab[row:row + n_pos, :dim // 2, 1] = np.sin(ang)
            row += n_pos
        _TABLES[key] = torch.from_numpy(tab.astype(np.float32)).to(dev)
    return _TABLES[key]


def packed_projection_t(chan: int, device=None, seed: int = PROJECTION_SEED) -> torch.Tensor:
    """[Wq | Wk | Wv]^T as a (3*chan, chan) bf16 K-major matrix (the GEMM's B operand)."""
    dev = torch.device(device or default_device())
    key = (chan, str(dev), seed)
    if key not in _PACKED_T:
        wq, wk, wv = qkv_projections(chan, seed, dev)
        _PACKED_T[key] = torch.cat([wq, wk, wv], dim=1).t().contiguous().to(torch.bfloat16)
    return _PACKED_T[key]


def qkv_project(x: torch.Tensor, grid: GridShape, pattern: SparsePattern = SparsePattern.ORIGINAL,
                batch: int = 1, norm: str | None = None, gamma_q: torch.Tensor | None = None,
                gamma_k: torch.Tensor | None = None, eps: float = 1e-6, rope: bool = False,
                weight_t: torch.Tensor | None = None, theta: float = ROPE_THETA,
                row_offset: int = 0) -> torch.Tensor:
    """x: (rows, L, C) or (rows*L, C) bf16 in `pattern` layout on the padded `grid` with `batch`
    items.  Returns q | k | v as (..., 3C) bf16.  head_dim is 128 (C % 128 == 0)."""
    if norm not in _NORMS:
        raise ValueError(f"norm must be one of {sorted(k for k in _NORMS if k)} or None")
    shape = x.shape
    C = shape[-1]
    x2 = x.reshape(-1, C)
    if x2.dtype != torch.bfloat16:
        x2 = x2.to(torch.bfloat16)
    x2 = x2.contiguous()
    w_t = weight_t if weight_t is not None else packed_projection_t(C, x2.device)
    out = kernels.qkv_project(x2, w_t, _NORMS[norm], gamma_q, gamma_k, eps,
                              rope_table(grid, 128, theta, x2.device) if rope else None,
                              grid, _PATTERN_IDS[SparsePattern(pattern)], batch, row_offset)
    return out.view(*shape[:-1], 3 * C)


class QKVPrologue(torch.autograd.Function):
    """K6 forward; backward = one K6b kernel (inverse RoPE rotation + RMSNorm backward, in place
    on the bf16 gradient, fp32 math), then dx = d(pre-norm qkv) @ W^T.  Weights and gammas are
    fixed (no grad), like the reference's seeded projections."""

    @staticmethod
    def forward(ctx, x, grid, pattern, batch, norm, gamma_q, gamma_k, eps, rope, row_offset,
                weight_t=None):
        C = x.shape[-1]
        w_t = weight_t if weight_t is not None else packed_projection_t(C, x.device)
        out = qkv_project(x, grid, pattern, batch, norm, gamma_q, gamma_k, eps, rope,
                          weight_t=w_t, row_offset=row_offset)
        ctx.save_for_backward(x)
        ctx.cfg = (grid, pattern, batch, norm, gamma_q, gamma_k, eps, rope, row_offset, C, w_t)
        return out

    @staticmethod
    def backward(ctx, gout):
        (x,) = ctx.saved_tensors
        grid, pattern, batch, norm, gamma_q, gamma_k, eps, rope, row_offset, C, w_t = ctx.cfg
        shape = x.shape
        rows = x.numel() // C
        g = gout.reshape(rows, 3 * C).to(torch.bfloat16)
        if norm is not None or rope:
            # K6b, in place on a private copy of the incoming gradient: transpose RoPE rotation and
            # the RMSNorm backward against the recomputed pre-norm output
            g = g.clone() if g.data_ptr() == gout.data_ptr() else g.contiguous()
            y = qkv_project(x, grid, pattern, batch, weight_t=w_t).reshape(rows, 3 * C) if norm else None
            kernels.qk_norm_rope_bwd(g, y, _NORMS[norm], gamma_q, gamma_k, eps,
                                     rope_table(grid, 128, ROPE_THETA, x.device) if rope else None,
                                     grid, _PATTERN_IDS[SparsePattern(pattern)], batch, row_offset)
        dx = (g @ w_t).reshape(shape)
        return dx, None, None, None, None, None, None, None, None, None, None
