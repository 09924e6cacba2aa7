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
