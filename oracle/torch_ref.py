"""Torch restatement of the reference attention for gradient parity.

TEST INFRASTRUCTURE ONLY (imported by tests/ and bench.py's CPU leg, never by
the product package).  The reference (attention.py:35-67) has no backward and
no multi-head notion; this restatement keeps its forward semantics exactly
(masked keys weigh 0, a row with no valid key outputs 0, pad-query rows zero)
so torch.autograd supplies the gradient oracle.  Its forward is asserted
against the numpy oracle (itself pinned to the reference) in
tests/test_torch_ref.py, and its gradients with torch.autograd.gradcheck.

`upcast=True` computes in float64 (the oracle); `upcast=False` mimics a plain
bf16 implementation (bf16 operands, fp32 softmax, bf16 probabilities and
outputs) and is used only to size the bf16 error budget.
"""

from __future__ import annotations

import math

import torch


def attention_ref(q, k, v, heads: int = 1, key_valid=None, zero_invalid_queries: bool = False,
                  scale: float | None = None, upcast: bool = True):
    """q, k, v: (n, L, C).  key_valid: (n, L) bool or None."""
    n, L, C = q.shape
    d = C // heads
    scale = 1.0 / math.sqrt(d) if scale is None else scale
    dt = torch.float64 if upcast else torch.float32
    qh = q.reshape(n, L, heads, d).transpose(1, 2)
    kh = k.reshape(n, L, heads, d).transpose(1, 2)
    vh = v.reshape(n, L, heads, d).transpose(1, 2)
    if upcast:
        qh, kh, vh = qh.to(dt), kh.to(dt), vh.to(dt)
        s = torch.matmul(qh, kh.transpose(-1, -2)) * scale
    else:
        s = torch.matmul(qh, kh.transpose(-1, -2)).to(dt) * scale
    if key_valid is not None:
        allowed = key_valid.bool()[:, None, None, :]
        s = s.masked_fill(~allowed, float("-inf"))
    mx = s.amax(dim=-1, keepdim=True)
    mx = torch.where(torch.isfinite(mx), mx, torch.zeros_like(mx))
    e = torch.exp(s - mx)
    z = e.sum(dim=-1, keepdim=True)
    p = torch.where(z > 0, e / torch.where(z == 0, torch.ones_like(z), z), torch.zeros_like(e))
    if upcast:
        out = torch.matmul(p, vh)
    else:
        out = torch.matmul(p.to(v.dtype), vh).to(dt)
    out = out.transpose(1, 2).reshape(n, L, C)
    if zero_invalid_queries and key_valid is not None:
        out = out * key_valid.to(out.dtype)[:, :, None]
    return out if upcast else out.to(q.dtype)


def pattern_positions(grid, pattern: str, batch: int):
    """(rows*L, 3) int64 padded-grid (t, h, w) of every pattern-layout row, from the oracle's
    map tables (osp_oracle.map_table, pinned to the reference) -- independent of the kernel's
    closed-form inverse."""
    import numpy as np

    from . import osp_oracle as O
    tab = O.map_table(O.PATTERN_FWD[pattern], grid, batch).reshape(-1) % grid.seq_len
    w = tab % grid.w
    h = (tab // grid.w) % grid.h
    t = tab // (grid.w * grid.h)
    return torch.from_numpy(np.stack([t, h, w], axis=1))


def qkv_prologue_ref(x, w, pos, norm=None, gamma_q=None, gamma_k=None, eps=1e-6, rope=False,
                     theta=10000.0, head_dim=128):
    """float64 reference of the sec. 8f row 2 prologue: y = x @ w (x, w as given -- pass the
    bf16-rounded operands the kernel sees); q/k: RMSNorm per head ("head") or over all channels
    of the bf16-rounded projection ("channel", Wan-style), times gamma, then 3-D RoPE on
    consecutive pairs with the (t, h, w) split d-4(d//6), 2(d//6), 2(d//6)."""
    x = x.double()
    y = x @ w.double()
    C = x.shape[-1]
    out = y.clone()
    dims = (head_dim - 4 * (head_dim // 6), 2 * (head_dim // 6), 2 * (head_dim // 6))
    freqs = [theta ** (-torch.arange(0, d, 2, dtype=torch.float64) / d) for d in dims]
    for which, gamma in ((0, gamma_q), (1, gamma_k)):
        z = y[:, which * C:(which + 1) * C]
        if norm == "channel":
            z = z.to(torch.bfloat16).double()
            z = z * torch.rsqrt((z * z).mean(-1, keepdim=True) + eps)
        elif norm == "head":
            zh = z.view(z.shape[0], -1, head_dim)
            z = (zh * torch.rsqrt((zh * zh).mean(-1, keepdim=True) + eps)).reshape(z.shape)
        if norm is not None and gamma is not None:
            z = z * gamma.double()
        if rope:
            ang = torch.cat([pos[:, a:a + 1].double() * freqs[a][None, :] for a in range(3)], dim=1)
            c, s = torch.cos(ang), torch.sin(ang)            # (rows, 64)
            zh = z.reshape(z.shape[0], -1, head_dim // 2, 2)
            x0, x1 = zh[..., 0], zh[..., 1]
            z = torch.stack([x0 * c[:, None, :] - x1 * s[:, None, :],
                             x0 * s[:, None, :] + x1 * c[:, None, :]], dim=-1).reshape(z.shape)
        out[:, which * C:(which + 1) * C] = z
    return out
