"""Self-verification of the gradient oracles (CPU, float64).

The reference (attention.py:35-67) has no backward, so every gradient parity test in this repo is
pinned to two restatements: oracle/torch_ref.attention_ref (torch autograd supplies the gradient)
and oracle/block_ref (a hand-written adjoint used at the BASELINE sizes).  Here:
  * attention_ref's forward equals the reference's own dense_attention outputs (golden vectors
    written by the reference, tests/golden/attention.npz) to 1e-12, masks included;
  * attention_ref's gradients pass torch.autograd.gradcheck, with masked keys, all-masked rows
    and zeroed pad queries;
  * block_ref's hand-written attention backward equals autograd through attention_ref;
  * block_ref's whole block (TSA application -> switch -> GSA application -> switch) equals the
    numpy oracle's composition of skiparse_attention (pinned to the reference) forward, and
    torch.autograd through attention_ref backward, on padded and unpadded grids.
"""

import numpy as np
import pytest
import torch

from oracle import osp_oracle as O
from oracle.block_ref import BlockRef, attn_bwd, attn_fwd, block_tables, layout_valid
from oracle.torch_ref import attention_ref


def test_attention_ref_forward_matches_reference_goldens(golden, golden_meta):
    a = golden("attention")
    n = 0
    for m in golden_meta["attention"]:
        key = m["case"]
        if not key.startswith("dense"):
            continue
        q, k, v = (torch.from_numpy(a[f"{key}_{t}"]) for t in "qkv")
        kv = torch.from_numpy(a[f"{key}_valid"]) if f"{key}_valid" in a.files else None
        if kv is not None and kv.dim() == 1:
            kv = kv.expand(q.shape[0], q.shape[1])
        out = attention_ref(q, k, v, 1, kv)
        assert np.max(np.abs(out.numpy() - a[f"{key}_out"])) < 1e-12, key
        n += 1
    assert n >= 6


def _masked_inputs(seed, n=3, L=7, C=8):
    g = torch.Generator().manual_seed(seed)
    q, k, v = (torch.randn(n, L, C, dtype=torch.float64, generator=g) for _ in range(3))
    valid = torch.rand(n, L, generator=g) > 0.35
    valid[0] = True                      # unmasked sequence
    valid[1, :] = False                  # every key masked: rows output exactly 0
    valid[2, 0] = True                   # at least one valid key
    return q, k, v, valid


@pytest.mark.parametrize("zero_q", [False, True])
@pytest.mark.parametrize("heads", [1, 2])
def test_attention_ref_gradcheck_masked(zero_q, heads):
    q, k, v, valid = _masked_inputs(11 + heads)
    leaves = [t.clone().requires_grad_(True) for t in (q, k, v)]
    f = lambda a, b, c: attention_ref(a, b, c, heads, valid, zero_invalid_queries=zero_q)  # noqa: E731
    assert torch.autograd.gradcheck(f, leaves, eps=1e-6, atol=1e-7, rtol=1e-5)
    out = f(*leaves)
    assert torch.equal(out[1], torch.zeros_like(out[1]))   # all-masked rows (attention.py:35-44)


@pytest.mark.parametrize("heads", [1, 2])
def test_block_ref_attention_adjoint_equals_autograd(heads):
    q, k, v, valid = _masked_inputs(21 + heads, n=3, L=9, C=8)
    qkv = torch.cat([q, k, v], dim=-1)
    do = torch.randn(3, 9, 8, dtype=torch.float64, generator=torch.Generator().manual_seed(4))
    leaves = [t.clone().requires_grad_(True) for t in (q, k, v)]
    out = attention_ref(*leaves, heads, valid, zero_invalid_queries=True)
    assert torch.allclose(attn_fwd(qkv, heads, valid), out, atol=1e-13, rtol=0)
    out.backward(do)
    got = attn_bwd(qkv, do, heads, valid)
    want = torch.cat([t.grad for t in leaves], dim=-1)
    assert torch.allclose(got, want, atol=1e-12, rtol=0)


class _G:
    def __init__(self, t, h, w, k):
        self.t, self.h, self.w, self.k = t, h, w, k


@pytest.mark.parametrize("grid", [(2, 8, 8, 2), (2, 10, 12, 2), (1, 9, 9, 3)])
def test_block_ref_matches_oracle_composition_and_autograd(grid):
    og = O.Grid(*grid)
    pg = O.padded_grid(og)
    C, heads = 16, 2
    rng = np.random.default_rng(7)
    W1 = rng.standard_normal((C, 3 * C)) / np.sqrt(C)
    W2 = rng.standard_normal((C, 3 * C)) / np.sqrt(C)
    x_orig = O.pad(rng.standard_normal((1, og.seq_len, C)), og)        # zeros at pad tokens
    # numpy oracle (pinned to the reference): TSA then GSA in the original layout
    ws = lambda W: (W[:, :C], W[:, C:2 * C], W[:, 2 * C:])  # noqa: E731
    padded = pg != og
    y = O.skiparse_attention(x_orig, og, "tsa", padded=padded, heads=heads, weights=ws(W1))
    y = O.skiparse_attention(y, og, "gsa", padded=padded, heads=heads, weights=ws(W2))
    to_tsa = O.map_table("orig_to_tsa", pg, 1)
    want = O.apply_table(to_tsa, y)
    x_tsa = torch.from_numpy(O.apply_table(to_tsa, x_orig))
    t2g, g2t = block_tables(_G(pg.t, pg.h, pg.w, pg.k))
    vt, vg = layout_valid(_G(*grid))
    ref = BlockRef(t2g, g2t, vt, vg, torch.from_numpy(W1), torch.from_numpy(W2), heads)
    got, cache = ref.forward(x_tsa)
    assert np.max(np.abs(got.numpy() - want)) < 1e-12
    # backward: torch.autograd through attention_ref with the same tables and masks
    gy = torch.randn(got.shape, dtype=torch.float64, generator=torch.Generator().manual_seed(9))
    xl = x_tsa.clone().requires_grad_(True)
    n, L, _ = xl.shape
    W1t, W2t = torch.from_numpy(W1), torch.from_numpy(W2)

    def app(x, W, valid):
        qkv = x @ W
        return attention_ref(qkv[..., :C], qkv[..., C:2 * C], qkv[..., 2 * C:], heads, valid,
                             zero_invalid_queries=valid is not None)

    o1 = app(xl, W1t, vt)
    x2 = o1.reshape(n * L, C)[t2g].reshape(n, L, C)
    o2 = app(x2, W2t, vg)
    yy = o2.reshape(n * L, C)[g2t].reshape(n, L, C)
    assert torch.allclose(yy, got, atol=1e-13, rtol=0)
    yy.backward(gy)
    dx = ref.backward(cache, gy)
    assert torch.allclose(dx, xl.grad, atol=1e-12, rtol=0)
    if vt is not None:   # pad tokens neither attend nor are attended: zero gradient
        assert torch.equal(dx[~vt], torch.zeros_like(dx[~vt]))
