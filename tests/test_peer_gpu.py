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
            old = arena.slot_bytes
            arena.ensure(4 * old)        # grows in place: old mappings released, same object
            assert arena.slot_bytes >= 4 * old
            y = arena.move(x, mv.table, mv.stride, mv.out_rows)
            assert torch.equal(y.view(96, 40), x.view(96, 40)[perm])
            arena.status[0] = 2          # as written by a timed-out device barrier
            from paper_2605_28691_b200.errors import CollectiveError
            with pytest.raises(CollectiveError):
                arena.check()
            arena.status[0] = 0
            arena.close()
    finally:
        dist.destroy_process_group()


def test_peer_barrier_two_ranks_on_two_streams(lib):
    """The device barrier protocol with both ranks live: rank r's copy -> barrier -> pull runs on
    its own stream of one GPU, so rank 0's barrier kernel really spins until rank 1's publishes
    (no host_sync).  A lost rank would end in the bounded timeout, not a hang."""
    from paper_2605_28691_b200 import kernels
    n, rows, chan = 2, 300, 256
    flags = [torch.zeros(n, dtype=torch.int32, device="cuda") for _ in range(n)]
    slots = [torch.zeros(rows, chan, dtype=torch.bfloat16, device="cuda") for _ in range(n)]
    status = torch.zeros(1, dtype=torch.int32, pin_memory=True)
    streams = [torch.cuda.Stream() for _ in range(n)]
    gen = torch.Generator(device="cuda").manual_seed(5)
    tables = [torch.randint(0, n * rows, (rows,), generator=gen, device="cuda") for _ in range(n)]
    torch.cuda.synchronize()
    for epoch in (1, 2, 3):
        src = [torch.randn(rows, chan, generator=gen, device="cuda").to(torch.bfloat16) for _ in range(n)]
        outs = [torch.empty(rows, chan, dtype=torch.bfloat16, device="cuda") for _ in range(n)]
        torch.cuda.synchronize()
        for r in range(n):        # rank 0's barrier is enqueued before rank 1 has arrived
            with torch.cuda.stream(streams[r]):
                slots[r].copy_(src[r])
                kernels.peer_barrier([f.data_ptr() for f in flags], r, epoch, timeout_ms=20000,
                                     status=status)
                kernels.peer_gather([s.data_ptr() for s in slots], rows, tables[r], outs[r])
        torch.cuda.synchronize()
        assert int(status[0]) == 0
        flat = torch.cat(src)
        for r in range(n):
            assert torch.equal(outs[r], flat[tables[r]])
            for j in range(n):
                assert int(flags[j][r]) == epoch


def test_peer_barrier_timeout_reports_missing_rank(lib):
    """A rank that never arrives: the barrier exits after the timeout with 1 + that rank in the
    status word (no __trap, the context stays usable) and PeerArena.check raises."""
    from paper_2605_28691_b200 import kernels
    n, rank = 3, 0
    flags = [torch.zeros(n, dtype=torch.int32, device="cuda") for _ in range(n)]
    flags[rank][1] = 1                 # rank 1 arrived, rank 2 never does
    status = torch.zeros(1, dtype=torch.int32, pin_memory=True)
    kernels.peer_barrier([f.data_ptr() for f in flags], rank, 1, timeout_ms=200, status=status)
    torch.cuda.synchronize()
    assert int(status[0]) == 1 + 2
    x = torch.ones(4, device="cuda")
    assert float((x * 2).sum()) == 8.0   # context still alive
