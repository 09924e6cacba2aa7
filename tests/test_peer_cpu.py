"""Host logic of the peer-memory switch (peer.py, K7): the cross-rank tables must equal the
composition the N-GPU block performs around each NCCL switch -- expand the compacted attention
output, switch the pattern over the whole grid, compact for the next attention -- and their
inverse tables must be the exact adjoint.  The oracle supplies the maps and the pad masks; the
kernel's semantics (row table[i] % stride of source table[i] // stride, -1 = zero row) are
simulated with indexing."""

import numpy as np
import pytest
import torch

from oracle import osp_oracle as O


def _pull(srcs, table, stride):
    C = srcs[0].shape[-1]
    flat = torch.zeros(len(srcs) * stride + 1, C, dtype=srcs[0].dtype)
    for j, s in enumerate(srcs):
        flat[j * stride: j * stride + s.shape[0]] = s
    idx = torch.where(table >= 0, table, torch.full_like(table, len(srcs) * stride))
    return flat[idx]


@pytest.mark.parametrize("grid,world,batch", [((2, 10, 12, 2), 2, 1), ((2, 10, 12, 2), 4, 1),
                                              ((1, 8, 16, 2), 2, 1), ((2, 9, 17, 3), 3, 1),
                                              ((2, 10, 12, 2), 4, 2), ((1, 9, 17, 3), 9, 2)])
@pytest.mark.parametrize("padded_gsa", [False, True])
def test_block_switch_tables_equal_expand_switch_compact(grid, world, batch, padded_gsa):
    from paper_2605_28691_b200.compact import compact_plan
    from paper_2605_28691_b200.peer import block_switch_moves
    og = O.Grid(*grid)
    pgr = O.padded_grid(og)
    k2 = og.k * og.k
    S = pgr.seq_len
    L = S // k2
    local = k2 * batch // world
    LR = local * L
    mask = O.pad_mask(og)

    def valid(name):   # validity of every (subsequence, position) slot, rows nested (pattern, b)
        tab = O.map_table(name, pgr, batch)
        return torch.from_numpy(mask[tab.reshape(-1) % S].reshape(k2 * batch, L))

    vt, vg = valid("orig_to_tsa"), valid("orig_to_gsa")
    pts = [compact_plan(vt[j * local:(j + 1) * local]) for j in range(world)]
    pgs = [compact_plan(vg[j * local:(j + 1) * local]) for j in range(world)]
    t2g = torch.from_numpy(O.map_table("tsa_to_gsa", pgr, batch).reshape(-1))
    g2t = torch.from_numpy(O.map_table("gsa_to_tsa", pgr, batch).reshape(-1))
    C = 5
    gen = torch.Generator().manual_seed(7)
    # compact attention outputs, junk beyond each subsequence's length: it must never be read
    o1 = [torch.randn(p.n_seq * p.cap, C, generator=gen, dtype=torch.float64) for p in pts]
    o2 = [torch.randn(p.n_seq * p.cap, C, generator=gen, dtype=torch.float64) for p in pgs]

    def expand(y, p):
        out = torch.zeros(p.n_seq * p.L, C, dtype=y.dtype)
        ok = p.scatter >= 0
        out[ok] = y[p.scatter[ok]]
        return out

    def compact(x, p):
        out = torch.zeros(p.n_seq * p.cap, C, dtype=x.dtype)
        ok = p.gather >= 0
        out[ok] = x[p.gather[ok]]
        return out

    glob_t = torch.cat([expand(o1[j], pts[j]) for j in range(world)])       # padded TSA, all ranks
    glob_g = glob_t[t2g]                                                   # switch (whole grid)
    glob_g2 = torch.cat([expand(o2[j], pgs[j]) for j in range(world)])
    glob_t2 = glob_g2[g2t]
    moves = [block_switch_moves(world, r, local, L, t2g, g2t, pts, pgs, padded_gsa)
             for r in range(world)]
    for r, (A, B) in enumerate(moves):
        mine = glob_g[r * LR:(r + 1) * LR]
        want_a = mine if padded_gsa else compact(mine, pgs[r])
        assert torch.equal(_pull(o1, A.table, A.stride), want_a)
        assert torch.equal(_pull(o2, B.table, B.stride), glob_t2[r * LR:(r + 1) * LR])
        assert A.out_rows == (L if padded_gsa else pgs[r].cap) and B.out_rows == L
        assert A.in_rows == pts[r].cap and B.in_rows == pgs[r].cap
    # adjoint: pulling gradients with the inverse tables == scatter of the forward tables
    for which in (0, 1):
        dst_g = [torch.randn(m[which].table.numel(), C, generator=gen, dtype=torch.float64)
                 for m in moves]
        src_rows = [p.n_seq * p.cap for p in (pts if which == 0 else pgs)]
        stride = moves[0][which].stride
        for j in range(world):
            mv = moves[j][which]
            got = _pull(dst_g, mv.inv, mv.inv_stride)
            want = torch.zeros(src_rows[j], C, dtype=torch.float64)
            for r in range(world):
                t = moves[r][which].table
                hit = (t >= 0) & (t // stride == j)
                want.index_add_(0, t[hit] % stride, dst_g[r][hit])
            assert torch.equal(got, want)
    # only real tokens cross: every real row of every rank is pulled exactly once per switch
    real_t = sum(int(p.lens.sum()) for p in pts)
    assert sum(int((m[1].table >= 0).sum()) for m in moves) == sum(int(p.lens.sum()) for p in pgs)
    if not padded_gsa:
        assert sum(int((m[0].table >= 0).sum()) for m in moves) == real_t
