"""K7 peer-memory switch kernels on one GPU.  The gather kernel reads from any set of device
addresses, so N ranks' source buffers are simulated by N local buffers (no kernel waits on
another); the barrier is checked with the other ranks' arrivals pre-published.  The N-process
block over CUDA IPC is in test_multirank_gpu.py (p2p transport)."""

import socket

import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("chan,dtype", [(5120, torch.bfloat16), (64, torch.bfloat16), (5, torch.bfloat16),
                                        (3, torch.float32), (7, torch.uint8)])
@pytest.mark.parametrize("n", [1, 3, 8])
def test_peer_gather_matches_indexing(lib, chan, dtype, n):
    from paper_2605_28691_b200 import kernels
    gen = torch.Generator(device="cuda").manual_seed(n * 31 + chan)
    rows = [int(r) for r in torch.randint(1, 300, (n,), generator=gen, device="cuda")]
    stride = max(rows)
    if dtype is torch.uint8:
        srcs = [torch.randint(0, 255, (r, chan), generator=gen, device="cuda", dtype=torch.int32).to(dtype)
                for r in rows]
    else:
        srcs = [torch.randn(r, chan, generator=gen, device="cuda").to(dtype) for r in rows]
    n_out = 517
    j = torch.randint(0, n, (n_out,), generator=gen, device="cuda")
    lim = torch.tensor(rows, device="cuda")[j]
    s = (torch.rand(n_out, generator=gen, device="cuda") * lim).long()
    table = j * stride + s
    table[::7] = -1
    out = torch.full((n_out, chan), 3, dtype=dtype, device="cuda")
    kernels.peer_gather([t.data_ptr() for t in srcs], stride, table, out)
    flat = torch.zeros(n * stride + 1, chan, dtype=dtype, device="cuda")
    for i, t in enumerate(srcs):
        flat[i * stride: i * stride + rows[i]] = t
    want = flat[torch.where(table >= 0, table, torch.full_like(table, n * stride))]
    assert torch.equal(out, want)


def test_peer_barrier_publishes_and_passes(lib):
    from paper_2605_28691_b200 import kernels
    n, rank = 4, 2
    blocks = [torch.zeros(n, dtype=torch.int32, device="cuda") for _ in range(n)]
    for epoch in (1, 2, 3):
        for t in range(n):          # the other ranks have already arrived
            if t != rank:
                blocks[rank][t] = epoch
        kernels.peer_barrier([b.data_ptr() for b in blocks], rank, epoch)
        torch.cuda.synchronize()
        for t in range(n):
            assert int(blocks[t][rank]) == epoch        # published to every peer's block


def test_peer_arena_single_rank_round_trip(lib):
    import torch.distributed as dist
    from paper_2605_28691_b200.peer import PeerArena, peer_move
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        g = dist.new_group([0])
        for host_sync in (False, True):
            arena = PeerArena(g, 1 << 16, host_sync=host_sync)
            perm = torch.randperm(96, device="cuda")
            mv = peer_move([perm], [96], 0, 32, 32)
            x = torch.randn(3, 32, 40, device="cuda").to(torch.bfloat16)
            for _ in range(3):           # slots alternate, epochs advance
                y = arena.move(x, mv.table, mv.stride, mv.out_rows)
                assert torch.equal(y.view(96, 40), x.view(96, 40)[perm])
                back = arena.move(y, mv.inv, mv.inv_stride, mv.in_rows)
                assert torch.equal(back, x)
            arena.close()
    finally:
        dist.destroy_process_group()
