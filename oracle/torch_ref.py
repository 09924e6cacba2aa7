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
