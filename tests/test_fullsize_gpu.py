"""Parity at BASELINE.json's full cfg3 size (Wan-14B shape, 720p latent 21x45x80 padded to
21x48x80, k=2, 40 heads x 128), through properties that do not need a full float64 oracle:
bit-exact rearrange / switch round trips, and attention rows, key-gradient and query-gradient
rows sampled from the full-length subsequences, each recomputed in float64 on the device from
the same bf16 inputs."""

import math

import pytest
import torch

pytestmark = pytest.mark.gpu

T, H, W, K, HEADS, D = 21, 45, 80, 2, 40, 128
C = HEADS * D


@pytest.fixture(scope="module")
def P(lib):
    import paper_2605_28691_b200 as P
    return P


def test_cfg3_rearrange_and_switch_round_trips_bit_exact(P):
    from paper_2605_28691_b200 import kernels, ssp
    g = P.GridShape(T, H, W, K)
    pg = P.pad_grid(g)
    p = pg.padded
    torch.manual_seed(0)
    x = torch.randn(1, g.seq_len, C, device="cuda").to(torch.bfloat16)
    xt = kernels.rearrange(x, "orig_to_tsa", p.t, p.h, p.w, p.k, 1, g.h, g.w)      # fused pad
    xg = kernels.rearrange(xt, "tsa_to_gsa", p.t, p.h, p.w, p.k, 1)
    back = kernels.rearrange(kernels.rearrange(xg, "gsa_to_tsa", p.t, p.h, p.w, p.k, 1),
                             "tsa_to_orig", p.t, p.h, p.w, p.k, 1, g.h, g.w)      # fused strip
    assert torch.equal(back, x)
    # direct TSA->GSA equals orig->GSA of the padded latent (coherence, skiparse.py:117-128)
    assert torch.equal(xg, kernels.rearrange(x, "orig_to_gsa", p.t, p.h, p.w, p.k, 1, g.h, g.w))
    # SSP switch over N in-process ranks: TSA -> GSA equals the direct map, and is self-inverse
    for n in (2, 4):
        grp = ssp.shard_pattern_layout(xt, n)
        sw = ssp.ssp_pattern_switch(grp, p)
        assert torch.equal(ssp.gather_shards(sw).data, xg)
        assert torch.equal(ssp.gather_shards(ssp.ssp_pattern_switch(sw, p)).data, xt)


def _attention_inputs(P, pattern):
    from paper_2605_28691_b200.compact import compact_rows
    g = P.GridShape(T, H, W, K)
    pg = P.pad_grid(g)
    plan = pg.compact_plan(pattern, 1)
    torch.manual_seed(1)
    L = plan.L
    qkv = torch.randn(K * K, L, 3 * C, device="cuda").to(torch.bfloat16)
    return plan, compact_rows(qkv, plan).contiguous()


@pytest.mark.parametrize("pattern_name", ["TOKEN_WISE", "GROUP_WISE"])
def test_cfg3_attention_rows_and_gradients_sampled(P, pattern_name):
    from paper_2605_28691_b200 import kernels
    plan, qkv = _attention_inputs(P, getattr(P.SparsePattern, pattern_name))
    scale = 1 / math.sqrt(D)
    q, k, v = qkv[..., :C], qkv[..., C:2 * C], qkv[..., 2 * C:]
    o, lse = kernels.attn_fwd(q, k, v, HEADS, D, None, False, scale, seq_lens=plan.lens)
    torch.manual_seed(2)
    do = torch.randn(o.shape, device="cuda").to(torch.bfloat16)
    dq, dk, dv = kernels.attn_bwd(q, k, v, o, do, lse, HEADS, D, None, False, scale,
                                  seq_lens=plan.lens)
    gen = torch.Generator(device="cuda").manual_seed(3)
    for s in (0, plan.n_seq - 1):
        n = int(plan.lens[s])
        for h in (0, HEADS - 1):
            sl = slice(h * D, (h + 1) * D)
            Q, Kk, V, dO = (t[s, :n, sl].double() for t in (q, k, v, do))
            O = o[s, :n, sl].double()
            rows = torch.randint(0, n, (48,), generator=gen, device="cuda")
            # forward rows and lse
            S = (Q[rows] @ Kk.T) * scale
            Pm = torch.softmax(S, dim=-1)
            ref_o = Pm @ V
            err = (o[s, rows, sl].double() - ref_o).abs().max().item()
            assert err < 2e-2 * ref_o.abs().max().item() + 2e-3, ("o", s, h, err)
            assert (lse[s, h, rows].double() - torch.logsumexp(S, -1)).abs().max().item() < 1e-2
            # dq rows: scale * sum_k P (dP - delta) K, delta from the kernel's bf16 O (as K3 does)
            dP = dO[rows] @ V.T
            delta = (dO[rows] * O[rows]).sum(-1, keepdim=True)
            ref_dq = scale * (Pm * (dP - delta)) @ Kk
            err = (dq[s, rows, sl].double() - ref_dq).abs().max().item()
            assert err < 3e-2 * ref_dq.abs().max().item() + 2e-3, ("dq", s, h, err)
            # dk / dv rows: full columns of P over all queries of the subsequence
            keys = torch.randint(0, n, (32,), generator=gen, device="cuda")
            Sc = (Q @ Kk[keys].T) * scale                                   # (n, 32)
            lse_all = torch.logsumexp((Q @ Kk.T) * scale, dim=-1, keepdim=True)
            Pc = torch.exp(Sc - lse_all)
            ref_dv = Pc.T @ dO
            dPc = dO @ V[keys].T
            delta_all = (dO * O).sum(-1, keepdim=True)
            ref_dk = scale * (Pc * (dPc - delta_all)).T @ Q
            e_dv = (dv[s, keys, sl].double() - ref_dv).abs().max().item()
            e_dk = (dk[s, keys, sl].double() - ref_dk).abs().max().item()
            assert e_dv < 3e-2 * ref_dv.abs().max().item() + 2e-3, ("dv", s, h, e_dv)
            assert e_dk < 3e-2 * ref_dk.abs().max().item() + 2e-3, ("dk", s, h, e_dk)
