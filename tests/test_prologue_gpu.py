"""GPU parity of the K6 projection prologue (csrc/proj.cu) against the
float64 torch reference (oracle/torch_ref.qkv_prologue_ref).  Positions for RoPE come from the
oracle's reference-pinned map tables, independently of the kernel's closed-form inverse."""

import math

import pytest
import torch

from oracle import osp_oracle as O
from oracle import torch_ref as R

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P(lib):
    import paper_2605_28691_b200 as P
    return P


def _check(got, ref, C, what, roundings=1):
    got = got.double().cpu()
    ref = ref.cpu()
    # bf16 output: error within 2^-8 of the magnitude of the rotated pair (or element)
    pair = ref.view(ref.shape[0], -1, 2).norm(dim=-1, keepdim=True).expand(-1, -1, 2).reshape(ref.shape)
    err = (got - ref).abs()
    tol = roundings * 2.0 ** -8 * pair + 1e-4 * ref.abs().max()
    bad = err > tol
    assert not bad.any(), f"{what}: {int(bad.sum())} elements off, max err {float(err.max()):.3e}"


@pytest.mark.parametrize("grid,pattern,batch,C", [
    ((2, 8, 16, 2), "tsa", 1, 256), ((1, 16, 16, 2), "gsa", 2, 128), ((2, 4, 8, 2), "original", 1, 384),
    ((1, 16, 32, 4), "gsa", 1, 256), ((3, 8, 8, 2), "tsa", 1, 128)])
@pytest.mark.parametrize("norm,rope", [(None, False), ("head", True), ("channel", True), (None, True),
                                       ("head", False)])
def test_prologue_matches_float64_reference(P, grid, pattern, batch, C, norm, rope):
    from paper_2605_28691_b200.prologue import packed_projection_t, qkv_project
    g = P.GridShape(*grid)
    og = O.Grid(*grid)
    k2 = 1 if pattern == "original" else g.k * g.k
    rows = batch * g.seq_len
    torch.manual_seed(0)
    x = torch.randn(rows, C, device="cuda").to(torch.bfloat16)
    gq = torch.rand(C, device="cuda") + 0.5
    gk = torch.rand(C, device="cuda") + 0.5
    pat = {"tsa": P.SparsePattern.TOKEN_WISE, "gsa": P.SparsePattern.GROUP_WISE,
           "original": P.SparsePattern.ORIGINAL}[pattern]
    out = qkv_project(x.view(batch * k2, -1, C) if pattern != "original" else x.view(batch, -1, C), g,
                      pat, batch, norm=norm, gamma_q=gq if norm else None, gamma_k=gk if norm else None,
                      rope=rope)
    w_t = packed_projection_t(C, "cuda")
    pos = R.pattern_positions(og, pattern, batch)
    ref = R.qkv_prologue_ref(x.cpu(), w_t.t().cpu(), pos, norm, gq.cpu() if norm else None,
                             gk.cpu() if norm else None, rope=rope)
    # "channel" stores the projection in bf16 before normalising (Wan semantics): two roundings
    _check(out.view(rows, 3 * C), ref, C, f"{grid} {pattern} {norm} {rope}", 2 if norm == "channel" else 1)


def test_plain_projection_equals_reference_projection(P):
    """norm off, rope off == x @ [Wq|Wk|Wv] with the reference's seeded weights (attention.py:20-32)."""
    from paper_2605_28691_b200.prologue import qkv_project
    g = P.GridShape(1, 8, 8, 2)
    x = P.random_tensor(1, g.seq_len, 256, seed=3).data.cuda()
    out = qkv_project(x.to(torch.bfloat16), g).double().cpu()
    wq, wk, wv = O.qkv_weights(256)
    import numpy as np
    ref = torch.from_numpy(np.concatenate([x.to(torch.bfloat16).double().cpu().numpy()[0] @ w
                                           for w in (wq, wk, wv)], axis=1))
    assert ((out[0] - ref).abs() <= 2.0 ** -7 * ref.abs() + 0.02).all()


def test_prologue_errors(P):
    from paper_2605_28691_b200.prologue import qkv_project
    g = P.GridShape(1, 8, 8, 2)
    with pytest.raises(P.UnsupportedError):
        qkv_project(torch.zeros(64, 96, device="cuda", dtype=torch.bfloat16), g)
    with pytest.raises(ValueError):
        qkv_project(torch.zeros(64, 128, device="cuda", dtype=torch.bfloat16), g, norm="layer")


@pytest.mark.parametrize("norm,rope,pat", [(None, True, "tsa"), ("head", True, "tsa"), ("channel", True, "tsa"),
                                          ("head", False, "tsa"), ("head", True, "gsa"), ("channel", True, "gsa")])
def test_prologue_backward_matches_float64_autograd(P, norm, rope, pat):
    """QKVPrologue backward (K6b: inverse RoPE + RMSNorm backward; dx = dqkv W^T) vs float64
    autograd of the reference prologue."""
    from paper_2605_28691_b200.prologue import QKVPrologue, packed_projection_t
    g = P.GridShape(2, 8, 8, 2)
    og = O.Grid(2, 8, 8, 2)
    C = 256
    torch.manual_seed(1)
    x = torch.randn(4, g.seq_len // 4, C, device="cuda").to(torch.bfloat16).requires_grad_(True)
    gq = torch.rand(C, device="cuda") + 0.5
    gk = torch.rand(C, device="cuda") + 0.5
    w_t = packed_projection_t(C, "cuda")
    sp = P.SparsePattern.TOKEN_WISE if pat == "tsa" else P.SparsePattern.GROUP_WISE
    y = QKVPrologue.apply(x, g, sp, 1, norm, gq, gk, 1e-6, rope, 0, w_t)
    gy = torch.randn_like(y)
    y.backward(gy)
    xr = x.detach().double().cpu().reshape(-1, C).requires_grad_(True)
    pos = R.pattern_positions(og, pat, 1)
    ref = R.qkv_prologue_ref(xr, w_t.t().double().cpu(), pos, norm, gq.cpu(), gk.cpu(), rope=rope)
    ref.backward(gy.double().cpu().reshape(-1, 3 * C))
    got = x.grad.double().cpu().reshape(-1, C)
    err = (got - xr.grad).abs().max().item()
    assert err <= 2e-2 * xr.grad.abs().max().item(), err


def test_block_with_prologue_matches_float64_composition(P):
    """SkiparseBlock with QK-RMSNorm + RoPE equals the float64 composition: prologue_ref ->
    attention per subsequence -> TSA->GSA switch (oracle table) -> prologue_ref -> attention ->
    GSA->TSA switch."""
    from paper_2605_28691_b200.block import SkiparseBlock
    grid = (2, 8, 8, 2)
    g = P.GridShape(*grid)
    og = O.Grid(*grid)
    C, heads = 256, 2
    blk = SkiparseBlock(g, heads, C, qk_norm="head", rope=True)
    torch.manual_seed(2)
    x = torch.randn(blk.local_rows, blk.L, C, device="cuda").to(torch.bfloat16)
    y = blk(x).double().cpu()

    def app(xl, w_t, pattern):
        pos = R.pattern_positions(og, pattern, 1)
        qkv = R.qkv_prologue_ref(xl.reshape(-1, C), w_t.t().double().cpu(), pos, "head", None, None,
                                 rope=True).reshape(4, -1, 3 * C)
        return R.attention_ref(qkv[..., :C], qkv[..., C:2 * C], qkv[..., 2 * C:], heads)

    xd = x.double().cpu()
    o1 = app(xd, blk.W1t, "tsa")
    x2 = torch.from_numpy(O.apply_table(O.map_table("tsa_to_gsa", og, 1), o1.numpy()))
    o2 = app(x2, blk.W2t, "gsa")
    want = torch.from_numpy(O.apply_table(O.map_table("gsa_to_tsa", og, 1), o2.numpy()))
    err = (y - want).abs().max().item()
    assert err < 3e-2, err


def test_prologue_row_offset_matches_full_layout(P):
    """An SSP shard (rows [r0, r1) of the pattern layout) gets the same q|k|v (RoPE positions
    included) as the corresponding rows of the full-layout projection."""
    from paper_2605_28691_b200.prologue import qkv_project
    g = P.GridShape(2, 8, 16, 2)
    C = 256
    torch.manual_seed(5)
    x = torch.randn(4, g.seq_len // 4, C, device="cuda").to(torch.bfloat16)
    full = qkv_project(x, g, P.SparsePattern.GROUP_WISE, 1, norm="head", rope=True)
    L = g.seq_len // 4
    for r0, r1 in ((0, 2), (2, 4), (1, 3)):
        part = qkv_project(x[r0:r1], g, P.SparsePattern.GROUP_WISE, 1, norm="head", rope=True,
                           row_offset=r0 * L)
        assert torch.equal(part, full[r0:r1])


def test_attention_all_sequences_empty(lib):
    from paper_2605_28691_b200 import kernels
    q, k, v = (torch.randn(3, 256, 128, device="cuda").bfloat16() for _ in range(3))
    sl = torch.zeros(3, dtype=torch.int32, device="cuda")
    o, lse = kernels.attn_fwd(q, k, v, 1, 128, None, False, 0.1, seq_lens=sl)
    assert (o == 0).all() and torch.isinf(lse).all()
    dq, dk, dv = kernels.attn_bwd(q, k, v, o, torch.randn_like(o), lse, 1, 128, None, False, 0.1,
                                  seq_lens=sl)
    assert (dq == 0).all() and (dk == 0).all() and (dv == 0).all()
