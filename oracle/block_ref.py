"""Device restatement of one Skiparse-2D block, forward AND backward, for block-level parity at
the BASELINE sizes (cfg1-cfg3).  TEST INFRASTRUCTURE ONLY: imported by tests/ (never by the
product package or bench.py's timed path).

The block (paper_2605_28691_b200/block.py) is the reference operator skiparse_attention
(attention.py:97-131) applied with TOKEN_WISE and then GROUP_WISE, kept in the token-wise
pattern layout between blocks:

    qkv1 = x W1 ; o1 = attn(qkv1 | TSA subsequence mask) ; x2 = tsa_to_gsa(o1)
    qkv2 = x2 W2 ; o2 = attn(qkv2 | GSA subsequence mask) ; y = gsa_to_tsa(o2)

with the reference's masking rules (attention.py:35-44, 121-130): masked (pad) keys weigh 0, a row
with no valid key outputs 0, pad-query rows output 0.  The reference has no backward; the
gradient here is the hand-derived adjoint of exactly these formulas (softmax backward with
delta = rowsum(dO * O), pad-query rows' dO zeroed, permutations' adjoints are their inverses),
which tests/test_block_parity_gpu.py checks against torch.autograd of oracle/torch_ref.py at small
sizes (itself gradcheck'd in tests/test_torch_ref.py), and whose forward it checks against the
numpy oracle (pinned to the reference's own outputs).

Attention is evaluated one (subsequence, head) at a time with the L x L score matrix
materialised, so cfg3 (L = 20,160, 40 heads) fits in a few GB and runs in seconds in float64 on
a B200.  Two modes:
  "f64"  -- float64 everywhere: the oracle;
  "bf16" -- a plain bf16 implementation (bf16 operands and outputs, fp32 scores / softmax /
            accumulation, bf16 probabilities and dS for the matmuls), used only to size the error
            budget of the bf16 kernels (err <= 2 x err(plain bf16) + abs).
"""

from __future__ import annotations

import math

import torch


def _cast(mode):
    return torch.float64 if mode == "f64" else torch.float32


def _r(t, mode):
    """Round to the storage type of `mode` (bf16 for the plain-bf16 simulation)."""
    return t if mode == "f64" else t.to(torch.bfloat16).to(torch.float32)


def _probs(q, k, kv, scale, mode):
    s = torch.matmul(q, k.transpose(0, 1)) * scale
    if kv is not None:
        s.masked_fill_(~kv[None, :], float("-inf"))
    m = s.amax(dim=1, keepdim=True)
    m = torch.where(torch.isfinite(m), m, torch.zeros_like(m))
    s.sub_(m).exp_()
    z = s.sum(dim=1, keepdim=True)
    s.div_(torch.where(z == 0, torch.ones_like(z), z))
    return s


def attn_fwd(qkv: torch.Tensor, heads: int, valid: torch.Tensor | None, mode: str = "f64"):
    """qkv (n, L, 3C) -> o (n, L, C); valid (n, L) bool (keys and queries)."""
    n, L, C3 = qkv.shape
    C = C3 // 3
    d = C // heads
    scale = 1.0 / math.sqrt(d)
    dt = _cast(mode)
    o = torch.zeros(n, L, C, dtype=dt, device=qkv.device)
    for s in range(n):
        kv = None if valid is None else valid[s]
        for h in range(heads):
            q, k, v = (qkv[s, :, i * C + h * d: i * C + (h + 1) * d].to(dt) for i in range(3))
            p = _probs(q, k, kv, scale, mode)
            o[s, :, h * d:(h + 1) * d] = torch.matmul(_r(p, mode), v)
            del p
    if valid is not None:
        o.mul_(valid[..., None].to(dt))
    return _r(o, mode)


def attn_bwd(qkv: torch.Tensor, do: torch.Tensor, heads: int, valid: torch.Tensor | None,
             mode: str = "f64") -> torch.Tensor:
    """Adjoint of attn_fwd: returns dqkv (n, L, 3C)."""
    n, L, C3 = qkv.shape
    C = C3 // 3
    d = C // heads
    scale = 1.0 / math.sqrt(d)
    dt = _cast(mode)
    do = _r(do.to(dt), mode)
    if valid is not None:                        # pad-query outputs are constant zeros
        do = do * valid[..., None].to(dt)
    dqkv = torch.zeros(n, L, C3, dtype=dt, device=qkv.device)
    for s in range(n):
        kv = None if valid is None else valid[s]
        for h in range(heads):
            q, k, v = (qkv[s, :, i * C + h * d: i * C + (h + 1) * d].to(dt) for i in range(3))
            g = do[s, :, h * d:(h + 1) * d]
            p = _probs(q, k, kv, scale, mode)
            o = torch.matmul(_r(p, mode), v)
            delta = (g * _r(o, mode)).sum(dim=1, keepdim=True)
            dv = torch.matmul(_r(p, mode).transpose(0, 1), g)
            dp = torch.matmul(g, v.transpose(0, 1))
            dp.sub_(delta).mul_(p)               # dS = P * (dP - delta)
            del p
            ds = _r(dp, mode)
            dqkv[s, :, h * d:(h + 1) * d] = torch.matmul(ds, k) * scale
            dqkv[s, :, C + h * d:C + (h + 1) * d] = torch.matmul(ds.transpose(0, 1), q) * scale
            dqkv[s, :, 2 * C + h * d:2 * C + (h + 1) * d] = dv
            del dp, ds
    return _r(dqkv, mode)


class BlockRef:
    """x (n, L, C) in the padded token-wise layout -> y, same layout; dx from gy.

    t2g / g2t: flat padded-row maps with gsa_flat = tsa_flat[t2g], tsa_flat = gsa_flat[g2t]
    (oracle map tables, pinned to the reference); valid_tsa / valid_gsa: (n, L) real-token flags
    of each layout (None on an unpadded grid); W1, W2: the block's (C, 3C) projections."""

    def __init__(self, t2g, g2t, valid_tsa, valid_gsa, W1, W2, heads: int, mode: str = "f64"):
        self.t2g, self.g2t = t2g, g2t
        self.vt, self.vg = valid_tsa, valid_gsa
        dt = _cast(mode)
        self.W1, self.W2 = W1.to(dt), W2.to(dt)
        self.heads, self.mode = heads, mode

    def _proj(self, x, W):
        return _r(torch.matmul(x, W), self.mode)

    def forward(self, x: torch.Tensor):
        dt = _cast(self.mode)
        n, L, C = x.shape
        x = _r(x.to(dt), self.mode)
        qkv1 = self._proj(x, self.W1)
        o1 = attn_fwd(qkv1, self.heads, self.vt, self.mode)
        x2 = o1.reshape(n * L, C)[self.t2g].reshape(n, L, C)
        qkv2 = self._proj(x2, self.W2)
        o2 = attn_fwd(qkv2, self.heads, self.vg, self.mode)
        y = o2.reshape(n * L, C)[self.g2t].reshape(n, L, C)
        return y, (qkv1, qkv2)

    def backward(self, cache, gy: torch.Tensor) -> torch.Tensor:
        qkv1, qkv2 = cache
        dt = _cast(self.mode)
        n, L, C = gy.shape
        gy = _r(gy.to(dt), self.mode)
        do2 = gy.reshape(n * L, C)[self.t2g].reshape(n, L, C)
        dqkv2 = attn_bwd(qkv2, do2, self.heads, self.vg, self.mode)
        dx2 = _r(torch.matmul(dqkv2, self.W2.transpose(0, 1)), self.mode)
        do1 = dx2.reshape(n * L, C)[self.g2t].reshape(n, L, C)
        dqkv1 = attn_bwd(qkv1, do1, self.heads, self.vt, self.mode)
        return _r(torch.matmul(dqkv1, self.W1.transpose(0, 1)), self.mode)


def block_tables(grid, batch: int = 1):
    """(t2g, g2t) flat tables of the padded grid from the oracle's map tables."""
    import numpy as np

    from . import osp_oracle as O
    g = O.Grid(grid.t, grid.h, grid.w, grid.k)
    t2g = torch.from_numpy(np.ascontiguousarray(O.map_table("tsa_to_gsa", g, batch).reshape(-1)))
    g2t = torch.from_numpy(np.ascontiguousarray(O.map_table("gsa_to_tsa", g, batch).reshape(-1)))
    return t2g, g2t


def layout_valid(orig_grid, batch: int = 1):
    """(valid_tsa, valid_gsa) (k^2*batch, L) bool from the oracle's pad mask, or (None, None)."""
    import numpy as np

    from . import osp_oracle as O
    g = O.Grid(orig_grid.t, orig_grid.h, orig_grid.w, orig_grid.k)
    pg = O.padded_grid(g)
    if pg == g:
        return None, None
    out = []
    for pat in ("tsa", "gsa"):
        m = np.repeat(O.subseq_mask(g, pat), batch, axis=0)
        out.append(torch.from_numpy(np.ascontiguousarray(m)))
    return tuple(out)


def errors(got: torch.Tensor, want: torch.Tensor) -> dict:
    """max-abs and relative-L2 error of got against want (float64)."""
    g, w = got.double(), want.double()
    diff = g - w
    return {"max_abs": float(diff.abs().max()), "rel_l2": float(diff.norm() / w.norm().clamp_min(1e-300)),
            "ref_max_abs": float(w.abs().max())}
