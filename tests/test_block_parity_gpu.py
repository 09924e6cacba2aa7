"""Block-level parity of the EXACT benched path at the BASELINE configs.

SkiparseBlock.__call__ on one GPU is what bench.py times: padding compaction, the row moves
fused into the attention epilogue / backward prologue, the projection GEMMs and the K2/K3
tcgen05 kernels, forward and backward.  Here its output y and input gradient dx are compared,
WHOLE (no sampling), with a float64 recomputation of the same block on the device
(oracle/block_ref.py: per (subsequence, head) exact softmax attention with the reference's
masking rules and the hand-derived adjoint, pinned in tests/test_torch_ref.py), and at cfg1
additionally with the numpy oracle's composition of skiparse_attention (pinned to the
reference's own outputs).

Tolerance rule, per tensor T in {y, dx}:
    max|T_kernel - T_f64| <= 2 * max|T_plainbf16 - T_f64| + 1e-3 * max|T_f64|
    relL2(T_kernel)       <= 2 * relL2(T_plainbf16) + 1e-3
where T_plainbf16 is the same block computed as a plain bf16 implementation would (bf16 operands
and outputs, fp32 softmax / accumulation, bf16 P and dS).  Inputs x, gy are bf16 N(0,1).
Errors are recorded (conftest parity_record -> $OSP_PARITY_OUT, committed as
profiles/r02_parity.json).
"""

import numpy as np
import pytest
import torch

from oracle import osp_oracle as O
from oracle.block_ref import BlockRef, block_tables, errors, layout_valid

pytestmark = pytest.mark.gpu

CASES = {
    # name: (T, H, W, k, heads, head_dim) -- BASELINE.json configs 1-3
    "cfg1": (4, 16, 16, 2, 4, 64),
    "cfg2": (21, 30, 52, 2, 12, 128),
    "cfg3": (21, 45, 80, 2, 40, 128),
}


def _run(name):
    import paper_2605_28691_b200 as P
    from paper_2605_28691_b200.block import SkiparseBlock
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.set_float32_matmul_precision("highest")
    T, H, W, k, heads, d = CASES[name]
    g = P.GridShape(T, H, W, k)
    C = heads * d
    blk = SkiparseBlock(g, heads, C)
    gen = torch.Generator(device="cuda").manual_seed(2024)
    x = torch.randn(blk.local_rows, blk.L, C, generator=gen, device="cuda").to(torch.bfloat16)
    gy = torch.randn(blk.local_rows, blk.L, C, generator=gen, device="cuda").to(torch.bfloat16)
    xk = x.clone().requires_grad_(True)
    y = blk(xk)
    y.backward(gy)
    torch.cuda.synchronize()
    t2g, g2t = block_tables(blk.grid)
    vt, vg = layout_valid(g)
    dev = torch.device("cuda")
    vt = None if vt is None else vt.to(dev)
    vg = None if vg is None else vg.to(dev)
    res = {}
    for mode in ("f64", "bf16"):
        ref = BlockRef(t2g.to(dev), g2t.to(dev), vt, vg, blk.W1.double(), blk.W2.double(), heads, mode)
        yr, cache = ref.forward(x)
        dxr = ref.backward(cache, gy)
        del cache
        res[mode] = (yr, dxr)
    return blk, x, y.detach(), xk.grad, res


def _check(name, got, f64, sim, parity_record, extra=None):
    entry = {}
    ok = True
    for t, a, w, s in (("y", got[0], f64[0], sim[0]), ("dx", got[1], f64[1], sim[1])):
        e, es = errors(a, w), errors(s, w)
        budget_abs = 2 * es["max_abs"] + 1e-3 * e["ref_max_abs"]
        budget_rel = 2 * es["rel_l2"] + 1e-3
        entry[t] = {"max_abs": e["max_abs"], "rel_l2": e["rel_l2"], "ref_max_abs": e["ref_max_abs"],
                    "plain_bf16_max_abs": es["max_abs"], "plain_bf16_rel_l2": es["rel_l2"],
                    "budget_max_abs": budget_abs, "budget_rel_l2": budget_rel,
                    "pass": e["max_abs"] <= budget_abs and e["rel_l2"] <= budget_rel}
        ok &= entry[t]["pass"]
        print(f"{name} {t}: max|err| {e['max_abs']:.3e} (budget {budget_abs:.3e}, plain bf16 "
              f"{es['max_abs']:.3e}), relL2 {e['rel_l2']:.3e} (budget {budget_rel:.3e})")
    entry["rule"] = ("max|err| <= 2*max|err_plain_bf16| + 1e-3*max|ref|; relL2 <= 2*relL2_plain_bf16 + 1e-3; "
                     "ref = float64 block recomputed on the device (oracle/block_ref.py)")
    if extra:
        entry.update(extra)
    parity_record(f"block_{name}", entry)
    assert ok, entry


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3"])
def test_block_fwd_bwd_matches_f64(lib, name, parity_record):
    blk, x, y, dx, res = _run(name)
    T, H, W, k, heads, d = CASES[name]
    extra = {"config": {"grid": [T, H, W], "k": k, "heads": heads, "head_dim": d,
                        "padded_grid": [blk.grid.t, blk.grid.h, blk.grid.w], "subseq_len": blk.L},
             "path": "SkiparseBlock.__call__ (the benched N=1 path), whole tensors, no sampling"}
    if name == "cfg1":
        # the reference's own CPU path: skiparse_attention TSA then GSA (numpy oracle, pinned to
        # the reference) in the original layout with the block's bf16 weights, mapped to TSA
        og = O.Grid(T, H, W, k)
        C = heads * d
        x_orig = O.apply_table(O.map_table("tsa_to_orig", og, 1), x.double().cpu().numpy())
        W1, W2 = blk.W1.double().cpu().numpy(), blk.W2.double().cpu().numpy()
        ws = lambda Wm: (Wm[:, :C], Wm[:, C:2 * C], Wm[:, 2 * C:])  # noqa: E731
        yo = O.skiparse_attention(x_orig, og, "tsa", heads=heads, weights=ws(W1))
        yo = O.skiparse_attention(yo, og, "gsa", heads=heads, weights=ws(W2))
        want = O.apply_table(O.map_table("orig_to_tsa", og, 1), yo)
        assert np.max(np.abs(res["f64"][0].cpu().numpy() - want)) < 1e-10   # oracle == block_ref
        e = errors(y.cpu(), torch.from_numpy(want))
        extra["y_vs_numpy_oracle"] = e
    _check(name, (y, dx), res["f64"], res["bf16"], parity_record, extra)


def _orig_tables(g):
    """(o2t flat table of the padded grid, pad mask flat) from the oracle (reference-pinned)."""
    og = O.Grid(g.t, g.h, g.w, g.k)
    pg = O.padded_grid(og)
    o2t = torch.from_numpy(np.ascontiguousarray(O.map_table("orig_to_tsa", pg, 1).reshape(-1)))
    mask = torch.from_numpy(np.ascontiguousarray(O.pad_mask(og).reshape(-1))) if pg != og else \
        torch.ones(og.seq_len, dtype=torch.bool)
    return o2t, mask


EXTRA = {
    # odd, padded and k = 3 / 4 grids through the same benched path (not BASELINE configs)
    "k3_pad": (2, 20, 30, 3, 2, 64),     # H, W -> 27, 36
    "k4_pad": (3, 30, 20, 4, 2, 128),    # H, W -> 32, 32
    "k2_odd": (1, 13, 17, 2, 1, 64),     # H, W -> 16, 20
    "k2_T5": (5, 8, 12, 2, 4, 64),       # no padding, T > 1
    "cfg3k4": (21, 45, 80, 4, 40, 128),  # the cfg3 shape at k = 4 (bench --config cfg3k4)
    "cfg5k2": (33, 45, 80, 2, 40, 128),  # BASELINE config 5, 129 frames (bench --config cfg5k2)
    "cfg5k4": (33, 45, 80, 4, 40, 128),  # BASELINE config 5 at k = 4
}


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3", *EXTRA])
def test_block_original_layout_fwd_bwd_matches_f64(lib, name, parity_record):
    """SkiparseBlock.forward_original -- what bench.py times at N=1 (orig -> TSA -> GSA -> orig:
    one K1 gather into compact TSA rows, both rearranges after the attention applications stored
    by the attention epilogues, dO gathered in the backward's Delta pre-pass) -- whole output and
    input gradient against the float64 block on the oracle's pad + orig_to_tsa tables."""
    import paper_2605_28691_b200 as P
    from paper_2605_28691_b200.block import SkiparseBlock
    torch.backends.cuda.matmul.allow_tf32 = False
    T, H, W, k, heads, d = CASES[name] if name in CASES else EXTRA[name]
    g = P.GridShape(T, H, W, k)
    C = heads * d
    blk = SkiparseBlock(g, heads, C)
    S = T * H * W
    gen = torch.Generator(device="cuda").manual_seed(77)
    x = torch.randn(1, S, C, generator=gen, device="cuda").to(torch.bfloat16)
    gy = torch.randn(1, S, C, generator=gen, device="cuda").to(torch.bfloat16)
    xk = x.clone().requires_grad_(True)
    y = blk.forward_original(xk)
    y.backward(gy)
    torch.cuda.synchronize()
    dev = torch.device("cuda")
    o2t, mask = (t.to(dev) for t in _orig_tables(g))
    Sp = o2t.numel()

    def to_tsa(t):                       # (1, S, C) unpadded -> (k^2, L, C) token-wise, pads 0
        pad = torch.zeros(Sp, C, dtype=t.dtype, device=dev)
        pad[mask] = t.reshape(S, C)
        return pad[o2t].view(blk.local_rows, blk.L, C)

    def to_orig(t):                      # adjoint / inverse of to_tsa on the real rows
        pad = torch.empty(Sp, C, dtype=t.dtype, device=dev)
        pad[o2t] = t.reshape(Sp, C)
        return pad[mask].view(1, S, C)

    t2g, g2t = block_tables(blk.grid)
    vt, vg = layout_valid(g)
    vt = None if vt is None else vt.to(dev)
    vg = None if vg is None else vg.to(dev)
    res = {}
    for mode in ("f64", "bf16"):
        ref = BlockRef(t2g.to(dev), g2t.to(dev), vt, vg, blk.W1.double(), blk.W2.double(), heads, mode)
        yr, cache = ref.forward(to_tsa(x))
        dxr = ref.backward(cache, to_tsa(gy))
        del cache
        res[mode] = (to_orig(yr), to_orig(dxr))
    extra = {"config": {"grid": [T, H, W], "k": k, "heads": heads, "head_dim": d,
                        "padded_grid": [blk.grid.t, blk.grid.h, blk.grid.w], "subseq_len": blk.L},
             "path": "SkiparseBlock.forward_original (the benched N=1 step, orig -> orig), whole tensors"}
    _check(name + "_orig", (y.detach(), xk.grad), res["f64"], res["bf16"], parity_record, extra)
