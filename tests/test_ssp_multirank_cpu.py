"""Multi-process SSP host logic on CPU: world_size 2 and 4 over gloo.

The device pack/unpack kernels need a GPU, so here they are replaced (test-only
monkeypatch) by the oracle's restatement of Alg. 1 steps 1 and 3-4; everything
else is the product's distributed path (`ssp.ssp_switch` / `SSPSwitch`:
guards, one all_to_all_single per switch, ledger, autograd backward)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import osp_oracle as O


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, grid, batch, pattern, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2605_28691_b200 import GridShape, kernels, ssp

        og = O.Grid(*grid)

        def pack(x, n, t, h, w, k):
            return torch.from_numpy(O.ssp_pack(x.detach().numpy(), n, O.Grid(t, h, w, k)))

        def unpack(recv, n, local_batch, t, h, w, k, out=None):
            return torch.from_numpy(O.ssp_unpack(recv.numpy(), n, local_batch, O.Grid(t, h, w, k)))

        kernels.ssp_pack = pack
        kernels.ssp_unpack = unpack
        rng = np.random.default_rng(11)
        x_orig = rng.standard_normal((batch, og.seq_len, 3))
        layout = O.apply_table(O.map_table(O.PATTERN_FWD[pattern], og, batch), x_orig)
        shards = O.shard(layout, world)
        want = O.ssp_switch(shards, og)[rank]
        log = ssp.CommLog()
        x = torch.from_numpy(shards[rank].copy()).requires_grad_(True)
        y = ssp.ssp_switch(x, GridShape(*grid), None, log)
        ok_fwd = np.array_equal(y.detach().numpy(), want)
        gy = torch.from_numpy(rng.standard_normal(y.shape))
        y.backward(gy)
        # backward = the same self-inverse switch applied to the gradient
        gshards = [None] * world
        dist.all_gather_object(gshards, gy.numpy())
        want_grad = O.ssp_switch(gshards, og)[rank]
        ok_bwd = np.allclose(x.grad.numpy(), want_grad)
        q.put((rank, ok_fwd, ok_bwd, log.count("all_to_all"), log.events[0].payload_per_rank,
               shards[rank].size))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - surfaced by the parent
        q.put((rank, repr(e)))


@pytest.mark.parametrize("grid,world,batch,pattern", [
    ((1, 8, 8, 2), 2, 1, "tsa"), ((2, 8, 12, 2), 4, 1, "gsa"), ((1, 8, 8, 2), 2, 3, "gsa"),
    ((1, 16, 16, 4), 4, 1, "tsa")])
def test_ssp_switch_over_gloo(grid, world, batch, pattern):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, grid, batch, pattern, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for r in res:
        assert len(r) == 6, r
        _, ok_fwd, ok_bwd, n_a2a, payload, local = r
        assert ok_fwd and ok_bwd
        assert n_a2a == 2  # one forward switch + one backward switch
        assert payload == local  # ledger counts the whole per-rank buffer (ssp.py:135)


def test_plan_parallel():
    from paper_2605_28691_b200.block import plan_parallel
    assert plan_parallel(1, 2) == (1, 1)
    assert plan_parallel(2, 2) == (2, 1)
    assert plan_parallel(4, 2) == (4, 1)
    assert plan_parallel(8, 2) == (4, 2)   # SSP4 x DP2
    assert plan_parallel(8, 4) == (8, 1)   # k=4: 16 subsequences over 8 ranks
    with pytest.raises(ValueError):
        plan_parallel(3, 2)
    from paper_2605_28691_b200.block import plan_parallel_3d
    assert plan_parallel_3d(1, 2, 40, 252) == (1, 1, 1)
    assert plan_parallel_3d(4, 2, 40, 252) == (4, 1, 1)
    assert plan_parallel_3d(8, 2, 40, 252) == (4, 2, 1)     # SSP4 x Ulysses2 (paper setting)
    assert plan_parallel_3d(8, 2, 40, 251) == (4, 1, 2)     # txh odd: SSP4 x DP2
    assert plan_parallel_3d(8, 2, 3, 252) == (4, 1, 2)      # heads not divisible
    assert plan_parallel_3d(8, 4, 40, 63) == (8, 1, 1)      # k=4: plain SSP8


def test_check_switch_guards():
    from paper_2605_28691_b200 import GridShape, ProtocolError, ShardingError
    from paper_2605_28691_b200.ssp import check_switch
    g = GridShape(1, 8, 8, 2)
    assert check_switch(2, 2, 16, g) == (2, 1)
    with pytest.raises(ShardingError):
        check_switch(3, 4, 16, g)
    with pytest.raises(ProtocolError):
        check_switch(2, 3, 16, g)
    with pytest.raises(ProtocolError):
        check_switch(2, 2, 15, g)


def _ulysses_worker(rank, world, port, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2605_28691_b200 import kernels
        from paper_2605_28691_b200.stack import _UlyssesOut, _UlyssesQKV

        def gather_chunks(src, dst, index, n_out, n_in, nc, cc, srs, scs, drs, dcs):
            # test-side restatement of the K1 chunked gather's element-stride contract
            s, d = src.reshape(-1), dst.reshape(-1)
            for r in range(n_out):
                for c in range(nc):
                    o = c * dcs + r * drs
                    if index[r] < 0:
                        d[o:o + cc] = 0
                    else:
                        i = c * scs + int(index[r]) * srs
                        d[o:o + cc] = s[i:i + cc]
            return dst

        kernels.gather_chunks = gather_chunks
        kernels._cuda = lambda t, name: None
        R, L, C = 3, 5, 8
        torch.manual_seed(0)
        full = torch.randn(world * R, L, 3 * C, dtype=torch.float64)   # all rows, all heads
        mine = full[rank * R:(rank + 1) * R].clone().requires_grad_(True)
        heads = _UlyssesQKV.apply(mine, world, None, None)
        Cn = C // world
        want = full.view(world * R, L, 3, world, Cn)[:, :, :, rank, :].reshape(world * R, L, 3 * Cn)
        ok_fwd = torch.equal(heads, want)
        # adjoint check <f(x), y> == <x, f^T(y)>
        torch.manual_seed(100 + rank)
        yb = torch.randn_like(heads)
        (heads * yb).sum().backward()
        lhs = torch.tensor([(heads * yb).sum().item()], dtype=torch.float64)
        rhs = torch.tensor([(mine * mine.grad).sum().item()], dtype=torch.float64)
        dist.all_reduce(lhs)
        dist.all_reduce(rhs)
        ok_adj = torch.allclose(lhs, rhs)
        # output direction: rows of my heads -> my rows of all heads
        torch.manual_seed(7)
        o_all = torch.randn(world * R, L, C, dtype=torch.float64)      # identical on all ranks
        o_mine_heads = o_all.view(world * R, L, world, Cn)[:, :, rank, :].contiguous().requires_grad_(True)
        back = _UlyssesOut.apply(o_mine_heads, world, None, None)
        ok_out = torch.equal(back, o_all[rank * R:(rank + 1) * R])
        yo = torch.randn_like(back)
        (back * yo).sum().backward()
        l2 = torch.tensor([(back * yo).sum().item()], dtype=torch.float64)
        r2 = torch.tensor([(o_mine_heads * o_mine_heads.grad).sum().item()], dtype=torch.float64)
        dist.all_reduce(l2)
        dist.all_reduce(r2)
        q.put((rank, ok_fwd, ok_adj, ok_out, bool(torch.allclose(l2, r2))))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e)))


@pytest.mark.parametrize("world", [2, 4])
def test_ulysses_all_to_all_over_gloo(world):
    """Head-parallel redistribution used by FULL blocks of the hybrid stack: forward
    gathers all rows for this rank's heads; the backward is the exact adjoint."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ulysses_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for r in res:
        assert len(r) == 5 and all(r[1:]), r


def test_switch_on_position_blocks_equals_restriction_of_full_switch():
    """SSP x Ulysses premise: a contiguous block of the txh = t*H/k^2 + h/k^2 axis is a run of
    whole rows in both pattern layouts, and the SSP switch of that block on the sub-grid
    (1, txh_block*k^2, W, k) equals the full-grid switch restricted to the block."""
    for grid, n, U in [((2, 8, 16, 2), 2, 2), ((3, 8, 8, 2), 4, 2), ((1, 16, 16, 2), 2, 4),
                       ((2, 16, 32, 4), 4, 2)]:
        g = O.Grid(*grid)
        k2 = g.k * g.k
        txh = g.t * g.h // k2
        L = g.seq_len // k2
        Lu = L // U
        rng = np.random.default_rng(sum(grid))
        x = rng.standard_normal((k2, L, 3))
        full = O.ssp_switch(O.shard(x, n), g)
        sub = O.Grid(1, txh // U * k2, g.w, g.k)
        for u in range(U):
            blk = O.ssp_switch(O.shard(np.ascontiguousarray(x[:, u * Lu:(u + 1) * Lu]), n), sub)
            for r in range(n):
                assert np.array_equal(blk[r], full[r][:, u * Lu:(u + 1) * Lu]), (grid, n, U, u, r)
