"""The SSP block with its pattern switches overlapped with attention (north star (3)).

The reference switch (ssp.py:139-180, Alg. 1) is pack -> one all-to-all ->
unpack between two attention applications.  On N GPUs this module runs a block as

    compact TSA rows x --GEMM--> qkv1 --attn(head chunk c) --epilogue store--> send1[c] ==a2a==> recv1[c]
    recv1 --(unpack o compact, one K1 gather)--> x2 --GEMM--> qkv2 --attn(c)--> send2[c] ==a2a==> recv2[c]
    recv2 --(unpack, one K1 gather)--> y (this rank's padded token-wise shard)

* The attention of each head chunk stores its rows straight into the SSP send layout through a
  row table (scatter mode: padding expansion + Alg. 1 step 1 "pack" in the K2 epilogue).
* The all-to-all of chunk c runs on a communication stream while the attention of chunk c+1
  computes, so only the last chunk's transfer is exposed.  Chunking the switch by channels is
  exact by the reference's channel-split identity (pkg/tests/test_ssp.py:167-178); attention is
  per head, so the chunked block equals the whole one bit for bit.
* The receive side's unpack (Alg. 1 steps 3-4) and the next application's compaction are one K1
  gather over all chunks.
* Backward mirrors it: the output gradient is packed into per-chunk send blocks (one K1 gather),
  the all-to-all of chunk c+1 overlaps the attention backward of chunk c (whose Delta pre-pass
  reads O and dO through the forward's store table), and so on.

Per switch this moves the shard once over the fabric (one all-to-all in total, as Alg. 1) with
one local K1 pass, against pack + unpack + expand + compact (four passes) of the unfused path.
"""

from __future__ import annotations

import math

import torch

from . import kernels
from .compact import scatter_plan


def _iota_map(fn, rows: int, L: int, dev) -> torch.Tensor:
    """A closed-form K1 row map as an int64 table: run it on an iota payload."""
    iota = torch.arange(rows * L, dtype=torch.int64, device=dev).view(rows, L, 1)
    return fn(iota).reshape(-1).contiguous()


def _inverse(tab: torch.Tensor, n: int) -> torch.Tensor:
    inv = torch.full((n,), -1, dtype=torch.int64, device=tab.device)
    ok = tab >= 0
    inv[tab[ok]] = torch.nonzero(ok).view(-1)
    return inv


class SSPOverlapPlan:
    """Per-rank tables of the overlapped SSP block (built once per block)."""

    def __init__(self, blk, n_chunks: int):
        from .ssp import check_switch
        g = blk.sub_grid
        dev = blk.W1.device
        n, R, L, C = blk.world, blk.local_rows, blk.L, blk.chan
        check_switch(n, R, L, g)
        if blk.heads % n_chunks:
            raise ValueError(f"{blk.heads} heads do not split into {n_chunks} switch chunks")
        self.n, self.R, self.L, self.C = n, R, L, C
        self.nc = n_chunks
        self.hc = blk.heads // n_chunks
        self.cc = C // n_chunks
        rows = R * L
        # send row d <- local row pack_src[d] (Alg. 1 step 1); unpacked row x <- recv row unpack_src[x]
        pack_src = _iota_map(lambda t: kernels.ssp_pack(t, n, g.t, g.h, g.w, g.k), R, L, dev)
        unpack_src = _iota_map(lambda t: kernels.ssp_unpack(t, n, R, g.t, g.h, g.w, g.k), R, L, dev)
        pack_dst = _inverse(pack_src, rows)
        pt, pgs = blk.plan_tsa, blk.plan_gsa

        def through(tab, idx):
            return torch.where(idx >= 0, tab[idx.clamp(min=0)], torch.full_like(idx, -1))

        self.pt, self.pgs = pt, pgs
        # application 1 stores compact TSA row i at send row pack_dst[padded TSA row]
        self.A1 = scatter_plan(through(pack_dst, pt.gather), pt.n_seq, pt.cap, rows, (rows, self.cc))
        # x2 (compact GSA) row j <- recv1 row unpack_src[padded GSA row]
        self.G1 = through(unpack_src, pgs.gather).contiguous()
        self.G1_inv = _inverse(self.G1, rows)
        self.A2 = scatter_plan(through(pack_dst, pgs.gather), pgs.n_seq, pgs.cap, rows, (rows, self.cc))
        # y (padded TSA) row x <- recv2 row unpack_src[x]; its adjoint pulls gy row unpack_dst[m]
        self.Y = unpack_src
        self.Y_inv = _inverse(unpack_src, rows)
        self.stream = torch.cuda.Stream(device=dev)


def _a2a(recv: torch.Tensor, send: torch.Tensor, group) -> None:
    import torch.distributed as dist
    dist.all_to_all_single(recv, send, group=group)


def _chunk_qkv(qkv: torch.Tensor, c: int, cc: int, C: int):
    return (qkv[..., c * cc:(c + 1) * cc], qkv[..., C + c * cc:C + (c + 1) * cc],
            qkv[..., 2 * C + c * cc:2 * C + (c + 1) * cc])


def _attn_chunks_then_a2a(qkv, plan: SSPOverlapPlan, lens, A, group, d, scale, log, label):
    """Attention per head chunk, each chunk's output stored into its send block and its
    all-to-all issued on the comm stream as soon as the chunk is done."""
    S = torch.cuda.current_stream()
    M = plan.stream
    rows = plan.R * plan.L
    send = torch.empty((plan.nc, rows, plan.cc), dtype=qkv.dtype, device=qkv.device)
    recv = torch.empty_like(send)
    lses = []
    for c in range(plan.nc):
        q, k, v = _chunk_qkv(qkv, c, plan.cc, plan.C)
        lses.append(kernels.attn_fwd_scatter(q, k, v, plan.hc, d, lens, A.out_index, send[c], A.zero_rows, scale))
        ev = torch.cuda.Event()
        ev.record(S)
        with torch.cuda.stream(M):
            M.wait_event(ev)
            tok = log.time_start(M) if log is not None else None
            _a2a(recv[c], send[c], group)
            if log is not None:
                log.time_end(tok, label)
    S.wait_stream(M)
    if log is not None:
        log.record("all_to_all", send.numel(), label, send.numel() * send.element_size())
    return send, recv, lses


def _a2a_chunks_then_attn_bwd(g_recv, qkv, send, lses, plan: SSPOverlapPlan, lens, A, group, d,
                              scale, log, label):
    """Backward of _attn_chunks_then_a2a: the all-to-all of each gradient chunk on the comm
    stream, the attention backward of chunk c as soon as its chunk has arrived."""
    S = torch.cuda.current_stream()
    M = plan.stream
    g_send = torch.empty_like(g_recv)
    M.wait_stream(S)
    evs = []
    with torch.cuda.stream(M):
        for c in range(plan.nc):
            tok = log.time_start(M) if log is not None else None
            _a2a(g_send[c], g_recv[c], group)
            if log is not None:
                log.time_end(tok, label + "-bwd")
            ev = torch.cuda.Event()
            ev.record(M)
            evs.append(ev)
    if log is not None:
        log.record("all_to_all", g_recv.numel(), label, g_recv.numel() * g_recv.element_size())
    dqkv = torch.empty_like(qkv)
    for c in range(plan.nc):
        S.wait_event(evs[c])
        q, k, v = _chunk_qkv(qkv, c, plan.cc, plan.C)
        dq, dk, dv = _chunk_qkv(dqkv, c, plan.cc, plan.C)
        kernels.attn_bwd_scatter(q, k, v, send[c], g_send[c], lses[c], plan.hc, d, lens, A.out_index,
                                 scale, dq, dk, dv)
    g_recv.record_stream(M)
    g_send.record_stream(M)
    return dqkv


class SSPOverlapBlock(torch.autograd.Function):
    """compact TSA rows (n_seq, cap, C) of this rank -> padded token-wise shard (R, L, C)."""

    @staticmethod
    def forward(ctx, x1c, blk):
        plan: SSPOverlapPlan = blk._overlap
        d = blk.chan // blk.heads
        scale = 1.0 / math.sqrt(d)
        pt, pgs = plan.pt, plan.pgs
        rows = plan.R * plan.L
        qkv1 = torch.matmul(x1c, blk.W1)
        send1, recv1, lse1 = _attn_chunks_then_a2a(qkv1, plan, pt.lens, plan.A1, blk.group, d, scale,
                                                   blk.log, "pattern-switch")
        x2 = kernels.gather_rows_chunked(recv1, plan.G1, pgs.n_seq * pgs.cap, plan.nc, True, False)
        qkv2 = torch.matmul(x2.view(pgs.n_seq, pgs.cap, plan.C), blk.W2)
        send2, recv2, lse2 = _attn_chunks_then_a2a(qkv2, plan, pgs.lens, plan.A2, blk.group, d, scale,
                                                   blk.log, "pattern-switch")
        y = kernels.gather_rows_chunked(recv2, plan.Y, rows, plan.nc, True, False)
        ctx.blk = blk
        ctx.saved = (qkv1, send1, lse1, qkv2, send2, lse2)
        return y.view(plan.R, plan.L, plan.C)

    @staticmethod
    def backward(ctx, gy):
        blk = ctx.blk
        plan: SSPOverlapPlan = blk._overlap
        qkv1, send1, lse1, qkv2, send2, lse2 = ctx.saved
        d = blk.chan // blk.heads
        scale = 1.0 / math.sqrt(d)
        pt, pgs = plan.pt, plan.pgs
        rows = plan.R * plan.L
        g_recv2 = kernels.gather_rows_chunked(gy.contiguous().view(rows, plan.C), plan.Y_inv, rows, plan.nc,
                                              False, True)
        dqkv2 = _a2a_chunks_then_attn_bwd(g_recv2, qkv2, send2, lse2, plan, pgs.lens, plan.A2, blk.group, d,
                                          scale, blk.log, "pattern-switch")
        dx2 = torch.matmul(dqkv2, blk.W2.t())
        g_recv1 = kernels.gather_rows_chunked(dx2.view(-1, plan.C), plan.G1_inv, rows, plan.nc, False, True)
        dqkv1 = _a2a_chunks_then_attn_bwd(g_recv1, qkv1, send1, lse1, plan, pt.lens, plan.A1, blk.group, d,
                                          scale, blk.log, "pattern-switch")
        dx1 = torch.matmul(dqkv1, blk.W1.t())
        ctx.saved = None
        return dx1, None
