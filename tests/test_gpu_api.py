"""GPU parity of the drop-in API (reference names/signatures) against the
reference's own outputs (tests/golden) and the CPU oracle, mirroring the
reference test suite (pkg/tests/test_{gridseq,skiparse,anyres,attention,ssp}.py)."""

import math

import numpy as np
import pytest
import torch

from oracle import osp_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P(lib):
    import paper_2605_28691_b200 as P
    return P


def test_pattern_maps_src_equals_reference(P, golden, golden_meta):
    maps = golden("maps")
    for m in golden_meta["maps"]:
        if "key" not in m or m["map"] not in ("orig_to_tsa", "tsa_to_gsa", "gsa_to_orig"):
            continue
        g = P.GridShape(*m["grid"])
        im = getattr(P, m["map"])(g, m["batch"])
        assert (im.in_batch, im.in_seq) == tuple(m["in"])
        assert (im.out_batch, im.out_seq) == tuple(m["out"])
        assert np.array_equal(im.src.cpu().numpy(), maps[m["key"]])


def test_roundtrips_coherence_bijection(P):
    # test_skiparse.py:77-121, test_acceptance.py:46-56
    for grid in [(1, 4, 4, 2), (2, 8, 8, 2), (1, 9, 9, 3), (2, 16, 16, 4)]:
        g = P.GridShape(*grid)
        x = P.random_tensor(2, g.seq_len, 3, seed=g.seq_len)
        to_t, to_g = P.orig_to_tsa(g, 2), P.orig_to_gsa(g, 2)
        assert torch.equal(P.tsa_to_orig(g, 2).apply(to_t.apply(x)).data, x.data)
        assert torch.equal(P.gsa_to_orig(g, 2).apply(to_g.apply(x)).data, x.data)
        assert P.tsa_to_gsa(g, 2).compose(to_t).same_permutation(to_g)
        assert P.gsa_to_tsa(g, 2).compose(to_g).same_permutation(to_t)
        for b in (P.orig_to_tsa, P.tsa_to_orig, P.orig_to_gsa, P.gsa_to_orig, P.tsa_to_gsa,
                  P.gsa_to_tsa):
            assert b(g, 2).is_bijection()
        assert P.tsa_to_orig(g, 3).same_permutation(P.orig_to_tsa(g, 3).invert())


def test_frozen_classes_and_k1_identity(P):
    a = P.assignment_of(P.GridShape(1, 4, 4, 2), P.SparsePattern.TOKEN_WISE)
    assert sorted(torch.nonzero(a.subseq == 0).view(-1).tolist()) == [0, 2, 8, 10]
    a = P.assignment_of(P.GridShape(1, 4, 4, 2), P.SparsePattern.GROUP_WISE)
    assert sorted(torch.nonzero(a.subseq == 3).view(-1).tolist()) == [10, 11, 14, 15]
    g = P.GridShape(2, 3, 5, 1)
    x = P.random_tensor(1, g.seq_len, 2, seed=1)
    for b in (P.orig_to_tsa, P.orig_to_gsa, P.tsa_to_gsa, P.gsa_to_tsa):
        assert torch.equal(b(g).apply(x).data, x.data)


def test_table_indexmap_semantics(P):
    # test_gridseq.py:55-101
    swap = P.IndexMap(1, 2, 1, 2, np.array([[1, 0]]))
    out = swap.apply(P.SequenceTensor(np.array([[[1.0], [2.0]]])))
    assert out.data[0, :, 0].tolist() == [2.0, 1.0]
    rng = np.random.default_rng(7)
    m1 = P.IndexMap(3, 5, 3, 5, rng.permutation(15).reshape(3, 5))
    m2 = P.IndexMap(3, 5, 3, 5, rng.permutation(15).reshape(3, 5))
    x = P.random_tensor(3, 5, 2, seed=2)
    assert torch.equal(m2.apply(m1.apply(x)).data, m2.compose(m1).apply(x).data)
    assert torch.equal(m1.invert().apply(m1.apply(x)).data, x.data)
    assert m1.invert().compose(m1).same_permutation(P.IndexMap.identity(3, 5))
    with pytest.raises(P.ShapeError):
        P.IndexMap.identity(2, 4).apply(P.random_tensor(2, 5, 1, seed=0))
    rm = P.rearrange_map([("b", 1)], [("x", 2), ("y", 3)], ["b"], ["y", "x"])
    xs = P.SequenceTensor(np.arange(6, dtype=float).reshape(1, 6, 1))
    assert rm.apply(xs).data[0, :, 0].tolist() == [0, 3, 1, 4, 2, 5]
    codes = P.SequenceTensor(np.arange(12, dtype=np.uint8).reshape(1, 6, 2), kind="hif8")
    back = rm.invert().apply(rm.apply(codes))
    assert back.kind == "hif8" and torch.equal(back.data, codes.data)


def test_anyres_api(P, golden, golden_meta):
    pad = golden("pad")
    for m in golden_meta["pad"]:
        g = P.GridShape(*m["grid"])
        pg = P.pad_grid(g)
        assert [pg.padded.t, pg.padded.h, pg.padded.w] == m["padded"]
        assert pg.trivial == m["trivial"]
        assert np.array_equal(pg.mask.cpu().numpy(), pad[f"mask_{m['key']}"])
        assert np.array_equal(pg.embedding.cpu().numpy(), pad[f"embed_{m['key']}"])
        x = P.SequenceTensor(pad[f"x_{m['key']}"])
        xp = P.pad_tensor(x, pg)
        assert np.array_equal(xp.numpy(), pad[f"padded_{m['key']}"])
        assert torch.equal(P.strip_padding(xp, pg).data, x.data)
        for pat in ("tsa", "gsa"):
            key = f"submask_{pat}_{m['key']}"
            if key in pad.files:
                got = P.subsequence_mask(pg, P.SparsePattern(pat)).cpu().numpy()
                assert np.array_equal(got, pad[key])
    pg = P.pad_grid(P.GridShape(1, 5, 6, 2))
    x = P.random_tensor(1, 30, 2, seed=1)
    junk = np.full((34, 2), 7.0)
    assert (P.pad_tensor(x, pg, pad_fill=junk).data[:, ~pg.mask, :] == 7.0).all()
    assert (P.pad_tensor(x, pg, pad_value=-1.0).data[:, ~pg.mask, :] == -1.0).all()


def _bf16_budget(got, want):
    return float(np.max(np.abs(got - want)))


def test_skiparse_attention_matches_reference_goldens(P, golden, golden_meta):
    """Reference skiparse_attention outputs (single head of chan) vs the B200 path
    (bf16 compute).  Tolerance: err <= 2 * err(plain bf16 simulation: x, weights,
    q/k/v and outputs rounded to bf16, float64 otherwise) + 1e-2, both measured
    against the reference's float64 output."""
    a = golden("attention")
    for m in golden_meta["attention"]:
        if "pattern" not in m:
            continue
        key = m["case"]
        g = P.GridShape(*m["grid"])
        pg = P.pad_grid(g) if m["padded"] else None
        x = a[f"{key}_x"]
        xb = O.bf16_round(x)
        out = P.skiparse_attention(P.SequenceTensor(xb), g, P.SparsePattern(m["pattern"]), pg)
        got = out.numpy()
        ref = a[f"{key}_out"]
        err = _bf16_budget(got, ref)
        sim = O.skiparse_attention(x, O.Grid(*m["grid"]), m["pattern"], padded=m["padded"],
                                   round_fn=O.bf16_round)
        budget = 2 * _bf16_budget(sim, ref) + 1e-2
        print(f"{key}: max|err| {err:.3e} (bf16 simulation {budget:.3e} budget)")
        assert err <= budget, (key, err, budget)
        if m["padded"]:
            real = O.pad_mask(O.Grid(*m["grid"]))
            assert (got[:, ~real] == 0).all(), key


def test_skiparse_attention_multihead_vs_oracle(P):
    for grid, padded, pat in [((2, 10, 12, 2), True, "tsa"), ((2, 16, 16, 2), False, "gsa"),
                              ((1, 45, 80, 2), True, "gsa"), ((3, 8, 8, 2), False, "original")]:
        g = P.GridShape(*grid)
        og = O.Grid(*grid)
        S = (O.padded_grid(og) if padded else og).seq_len
        rng = np.random.default_rng(S)
        x = O.bf16_round(rng.standard_normal((2, S, 256)))
        if padded:
            x[:, ~O.pad_mask(og), :] = 0.0
        pg = P.pad_grid(g) if padded else None
        got = P.skiparse_attention(torch.from_numpy(x).cuda(), g, P.SparsePattern(pat), pg,
                                   heads=2).cpu().numpy()
        want = O.skiparse_attention(x, og, pat, padded=padded, heads=2)
        sim = O.skiparse_attention(x, og, pat, padded=padded, heads=2, round_fn=O.bf16_round)
        err = np.max(np.abs(got - want))
        budget = 2 * np.max(np.abs(sim - want)) + 1e-2
        print(f"skiparse heads=2 {grid} {pat} padded={padded}: max|err| {err:.3e} budget {budget:.3e}")
        assert err <= budget


def test_pad_content_never_leaks(P):
    # test_attention.py:129-137 with 1e4 junk (bf16 range)
    g = P.GridShape(1, 10, 12, 2)
    pg = P.pad_grid(g)
    x = P.random_tensor(1, g.seq_len, 64, seed=13, dtype=torch.bfloat16)
    junk = np.random.default_rng(99).standard_normal((int((~pg.mask).sum()), 64)) * 1e4
    clean = P.skiparse_attention(P.pad_tensor(x, pg), g, P.SparsePattern.TOKEN_WISE, pg)
    dirty = P.skiparse_attention(P.pad_tensor(x, pg, pad_fill=junk), g, P.SparsePattern.TOKEN_WISE, pg)
    m = pg.mask
    assert torch.equal(clean.data[:, m], dirty.data[:, m])


def test_dense_attention_api(P, golden, golden_meta):
    a = golden("attention")
    for m in golden_meta["attention"]:
        key = m["case"]
        if not key.startswith("dense"):
            continue
        q, k, v = (O.bf16_round(a[f"{key}_{n}"]) for n in "qkv")
        kv = a[f"{key}_valid"] if f"{key}_valid" in a.files else None
        got = P.dense_attention(P.SequenceTensor(q), P.SequenceTensor(k), P.SequenceTensor(v),
                                key_valid=kv).numpy()
        want = O.dense_attention(q, k, v, kv)
        assert np.max(np.abs(got - want)) < 3e-2, key
        if m["mask"] == "none":
            assert (got == 0).all()


def test_skiparse_attention_gradient_vs_autograd(P):
    from oracle.torch_ref import attention_ref
    g = P.GridShape(2, 12, 16, 2)
    og = O.Grid(2, 12, 16, 2)
    rng = np.random.default_rng(3)
    C, heads = 256, 2
    x = O.bf16_round(rng.standard_normal((1, g.seq_len, C)))
    W = P.packed_projection(C)
    xt = torch.from_numpy(x).cuda().to(torch.bfloat16).requires_grad_(True)
    out = P.skiparse_attention(xt, g, P.SparsePattern.GROUP_WISE, heads=heads)
    gy = torch.from_numpy(O.bf16_round(rng.standard_normal(out.shape))).cuda().to(torch.bfloat16)
    out.backward(gy)
    # fp64 reference: same bf16 weights, gather with the oracle table
    tab = torch.from_numpy(O.map_table("orig_to_gsa", og, 1).reshape(-1))
    x64 = torch.from_numpy(x).requires_grad_(True)
    W64 = W.double().cpu()
    xp = x64.reshape(-1, C)[tab].reshape(4, -1, C)
    qkv = xp @ W64
    o = attention_ref(qkv[..., :C], qkv[..., C:2 * C], qkv[..., 2 * C:], heads)
    inv = torch.from_numpy(O.map_table("gsa_to_orig", og, 1).reshape(-1))
    y = o.reshape(-1, C)[inv].reshape(1, -1, C)
    y.backward(gy.double().cpu())
    e = (xt.grad.double().cpu() - x64.grad).abs().max().item()
    rel = e / x64.grad.abs().max().item()
    print(f"skiparse_attention dx: max|err| {e:.3e} rel {rel:.3e}")
    assert rel < 3e-2


def test_ssp_inprocess_matches_reference(P, golden, golden_meta):
    s = golden("ssp")
    for m in golden_meta["ssp"]:
        key = m["case"]
        g = P.GridShape(*m["grid"])
        log = P.CommLog()
        group = P.shard_pattern_layout(P.SequenceTensor(s[f"{key}_in"]), m["n"], log)
        out = P.ssp_pattern_switch(group, g)
        got = np.stack([sh.tensor.numpy() for sh in out.shards])
        assert np.array_equal(got, s[f"{key}_out"]), key
        assert log.count("all_to_all") == 1 and log.count("all_gather") == 0
        assert log.events[0].payload_per_rank == group.local_elements
        back = P.ssp_pattern_switch(out, g)
        assert np.array_equal(np.stack([sh.tensor.numpy() for sh in back.shards]), s[f"{key}_in"].reshape(got.shape))


def test_ssp_errors(P, golden_meta):
    g = P.GridShape(1, 4, 4, 2)
    x = P.orig_to_tsa(g, 3).apply(P.random_tensor(3, 16, 4, seed=0))
    with pytest.raises(P.ShardingError):
        P.ssp_pattern_switch(P.shard_pattern_layout(x, 3), g)
    with pytest.raises(P.ShardingError):
        P.shard_pattern_layout(P.orig_to_tsa(g).apply(P.random_tensor(1, 16, 4, seed=0)), 3)
    with pytest.raises(P.CollectiveError):
        P.all_to_all([torch.zeros(3, 1, device="cuda"), torch.zeros(3, 1, device="cuda")], P.CommLog())


def test_ssp_channel_split_composability(P):
    # test_ssp.py:167-178
    g = P.GridShape(1, 8, 8, 2)
    x = P.orig_to_tsa(g).apply(P.random_tensor(1, 64, 8, seed=8))
    whole = P.ssp_pattern_switch(P.shard_pattern_layout(x, 4), g)
    parts = [P.ssp_pattern_switch(P.shard_pattern_layout(P.SequenceTensor(x.data[:, :, h * 4:(h + 1) * 4]), 4), g)
             for h in range(2)]
    for r in range(4):
        merged = torch.cat([p.shards[r].tensor.data for p in parts], dim=2)
        assert torch.equal(merged, whole.shards[r].tensor.data)


@pytest.mark.parametrize("grid", [(2, 10, 12, 2), (1, 10, 12, 3), (1, 17, 20, 4), (2, 16, 16, 4)])
def test_block_matches_composed_applications(P, grid):
    """SkiparseBlock (steady-state TSA layout) equals two reference-style
    applications composed through the original layout (k = 2, 3, 4; padded and not)."""
    from paper_2605_28691_b200.block import SkiparseBlock
    g = P.GridShape(*grid)
    pg = P.pad_grid(g)
    C, heads = 256, 2
    blk = SkiparseBlock(g, heads, C)
    x0 = P.random_tensor(1, g.seq_len, C, seed=5, dtype=torch.bfloat16).data
    xt = blk.to_local_tsa(x0)
    y = blk(xt)
    xp = P.pad_tensor(x0, pg)
    y1 = P.skiparse_attention(xp, g, P.SparsePattern.TOKEN_WISE, pg, heads=heads, weights=blk.W1)
    y2 = P.skiparse_attention(y1, g, P.SparsePattern.GROUP_WISE, pg, heads=heads, weights=blk.W2)
    want = P.orig_to_tsa(pg.padded).apply(y2)
    err = (y.float() - want.float()).abs().max().item()
    assert err < 2e-2, err


@pytest.mark.parametrize("grid,padded", [((2, 12, 16, 2), False), ((2, 10, 12, 2), True)])
def test_hybrid_stack_matches_layerwise_oracle(P, grid, padded):
    """HybridStack (FULL, TSA, GSA, TSA, FULL, all in the token-wise layout) equals the
    reference-semantics composition of skiparse_attention layers in the original layout
    (ORIGINAL pattern for FULL layers), with the stack's own weights."""
    from paper_2605_28691_b200.skiparse import LayerKind
    from paper_2605_28691_b200.stack import HybridStack
    g = P.GridShape(*grid)
    og = O.Grid(*grid)
    C, heads = 256, 2
    sched = [LayerKind.FULL, LayerKind.TSA, LayerKind.GSA, LayerKind.TSA, LayerKind.FULL]
    st = HybridStack(g, heads, C, schedule=sched)
    pgr = O.padded_grid(og)
    rng = np.random.default_rng(4)
    x0 = O.bf16_round(rng.standard_normal((1, og.seq_len, C)))
    x_orig = torch.from_numpy(x0).cuda().to(torch.bfloat16)
    xt = st.pg.padded  # noqa: F841
    x_tsa = kernels_rearrange(x_orig, pgr, og)
    y = st(x_tsa).float().cpu().numpy()
    # oracle: layer by layer in the original (padded) layout
    xp = O.pad(x0, og)
    pat = {LayerKind.FULL: "original", LayerKind.TSA: "tsa", LayerKind.GSA: "gsa"}
    sim = xp.copy()
    for kind, W in zip(sched, st.weights):
        Wd = W.double().cpu().numpy()
        C_ = W.shape[0]
        ws = (Wd[:, :C_], Wd[:, C_:2 * C_], Wd[:, 2 * C_:])
        xp = O.skiparse_attention(xp, og, pat[kind], padded=True, heads=heads, weights=ws)
        sim = O.skiparse_attention(sim, og, pat[kind], padded=True, heads=heads, weights=ws,
                                   round_fn=O.bf16_round)
    tab = O.map_table("orig_to_tsa", pgr, 1)
    want = O.apply_table(tab, xp)
    want_sim = O.apply_table(tab, sim)
    err = np.max(np.abs(y - want))
    budget = 2 * np.max(np.abs(want_sim - want)) + 1e-2
    print(f"hybrid stack {grid} padded={padded}: max|err| {err:.3e} budget {budget:.3e}")
    assert err <= budget


def kernels_rearrange(x_orig, pgr, og):
    from paper_2605_28691_b200 import kernels
    return kernels.rearrange(x_orig, "orig_to_tsa", pgr.t, pgr.h, pgr.w, pgr.k, 1, og.h, og.w)


def test_hybrid_stack_backward_runs(P):
    from paper_2605_28691_b200.stack import HybridStack
    g = P.GridShape(2, 10, 12, 2)
    st = HybridStack(g, 2, 256, num_layers=4, n_full=2)
    x = torch.randn(st.local_rows, st.L, 256, device="cuda").bfloat16().requires_grad_(True)
    y = st(x)
    y.float().sum().backward()
    assert x.grad is not None and torch.isfinite(x.grad).all()


def test_block_compaction_paths_agree_fwd_bwd(P):
    """Padded grid: the compacted block (fused row moves on one GPU) and the masked block give the
    same outputs and input gradients."""
    from paper_2605_28691_b200.block import SkiparseBlock
    g = P.GridShape(2, 10, 12, 2)
    C, heads = 256, 2
    a = SkiparseBlock(g, heads, C)
    b = SkiparseBlock(g, heads, C, compact=False)
    assert a._scatter is not None and b.plan_tsa is None
    torch.manual_seed(3)
    x = torch.randn(a.local_rows, a.L, C, device="cuda").to(torch.bfloat16)
    xa, xb = x.clone().requires_grad_(True), x.clone().requires_grad_(True)
    ya, yb = a(xa), b(xb)
    assert (ya.float() - yb.float()).abs().max().item() < 2e-2
    gy = torch.randn_like(ya)
    ya.backward(gy)
    yb.backward(gy)
    real = P.pad_grid(g).compact_plan(P.SparsePattern.TOKEN_WISE, 1).scatter.view(a.local_rows, a.L) >= 0
    ga, gb = xa.grad.float(), xb.grad.float()
    assert (ga[~real] == 0).all()
    rel = (ga - gb).abs().max().item() / gb.abs().max().item()
    assert rel < 2e-2, rel


@pytest.mark.parametrize("method", ["forward_original", "forward_original_gather"])
@pytest.mark.parametrize("grid", [(2, 10, 12, 2), (2, 8, 16, 2)])
def test_block_forward_original_matches_pattern_layout_block(P, grid, method):
    """Original-layout block (scatter mode: rearranges in the attention epilogues; gather mode:
    in the TMA loads) equals the pattern-layout block composed with explicit rearranges, fwd and
    input grad."""
    from paper_2605_28691_b200.block import SkiparseBlock
    g = P.GridShape(*grid)
    pg = P.pad_grid(g)
    C, heads = 256, 2
    blk = SkiparseBlock(g, heads, C)
    assert blk.gather is not None
    torch.manual_seed(4)
    x = torch.randn(1, g.seq_len, C, device="cuda").to(torch.bfloat16)
    xa = x.clone().requires_grad_(True)
    ya = getattr(blk, method)(xa)
    xt = blk.to_local_tsa(x).detach().requires_grad_(True)
    yt = blk(xt)
    p = pg.padded
    yb = P.kernels.rearrange(yt.detach(), "tsa_to_orig", p.t, p.h, p.w, p.k, 1, g.h, g.w)
    assert (ya.float() - yb.float()).abs().max().item() < 2e-2
    gy = torch.randn_like(ya)
    ya.backward(gy)
    # the maps are permutations with zero pad rows: push gy into the TSA layout, pull back
    yt.backward(P.kernels.rearrange(gy, "orig_to_tsa", p.t, p.h, p.w, p.k, 1, g.h, g.w))
    gb = P.kernels.rearrange(xt.grad, "tsa_to_orig", p.t, p.h, p.w, p.k, 1, g.h, g.w)
    rel = (xa.grad.float() - gb.float()).abs().max().item() / gb.float().abs().max().item()
    assert rel < 2e-2, rel


def test_block_forward_original_with_prologue(P):
    from paper_2605_28691_b200.block import SkiparseBlock
    g = P.GridShape(2, 10, 12, 2)
    blk = SkiparseBlock(g, 2, 256, qk_norm="head", rope=True)
    x = torch.randn(1, g.seq_len, 256, device="cuda").to(torch.bfloat16).requires_grad_(True)
    y = blk.forward_original_gather(x)
    y.float().sum().backward()
    assert torch.isfinite(y).all() and torch.isfinite(x.grad).all()


def test_block_head_dim_64_compaction_paths_agree(P):
    """head_dim 64 (the v1 backward kernel) with padding compaction vs the masked block."""
    from paper_2605_28691_b200.block import SkiparseBlock
    g = P.GridShape(2, 10, 12, 2)
    C, heads = 256, 4
    a = SkiparseBlock(g, heads, C)
    b = SkiparseBlock(g, heads, C, compact=False)
    torch.manual_seed(6)
    x = torch.randn(a.local_rows, a.L, C, device="cuda").to(torch.bfloat16)
    xa, xb = x.clone().requires_grad_(True), x.clone().requires_grad_(True)
    ya, yb = a(xa), b(xb)
    assert (ya.float() - yb.float()).abs().max().item() < 2e-2
    gy = torch.randn_like(ya)
    ya.backward(gy)
    yb.backward(gy)
    rel = (xa.grad.float() - xb.grad.float()).abs().max().item() / xb.grad.float().abs().max().item()
    assert rel < 2e-2, rel
