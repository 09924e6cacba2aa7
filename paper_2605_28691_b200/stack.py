"""Hybrid Skiparse DiT attention stack: full-attention blocks at
both ends, alternating token-wise / group-wise Skiparse blocks in the middle
(`build_layer_schedule`, skiparse.py:221-237).

Layout: the hidden states live in a pattern layout (token-wise or group-wise) for the whole
stack.  Attention is permutation-equivariant (test_attention.py:140-149), so a FULL block runs
directly on that layout: per batch item it attends over all k^2 subsequences concatenated,
keyed by the concatenated subsequence masks.  No rearrange is needed at Full<->Skiparse
boundaries; TSA<->GSA transitions are one `tsa_to_gsa` / `gsa_to_tsa` map (N=1) or one SSP
all-to-all (N>1).

Multi-GPU: Skiparse blocks use SSP (whole subsequences per rank, no communication inside
attention).  FULL blocks use Ulysses head parallelism: one all-to-all turns
the packed [q|k|v] of this rank's subsequences (all heads) into all subsequences for
heads/N heads, and one all-to-all returns the output -- the Ulysses four-collective volume
(ssp.py:183-191) in two calls.
"""

from __future__ import annotations

import torch

from . import kernels
from .anyres import pad_grid
from .attention import COMPUTE_DTYPE, PROJECTION_SEED, attention_packed, packed_projection
from .gridseq import GridShape, IndexMap
from .skiparse import LayerKind, SparsePattern, build_layer_schedule
from .ssp import CommLog, ssp_switch

__all__ = ["HybridStack", "full_sequence_bits", "ulysses_qkv_to_heads", "ulysses_out_to_rows"]


def full_sequence_bits(sub_bits: torch.Tensor, n_sub: int, batch: int, L: int) -> torch.Tensor:
    """Key-validity bits of each batch item's full sequence in a pattern layout: the k^2
    subsequence masks (rows nested (pattern id, batch item)) concatenated in pattern order."""
    valid = kernels.bits_to_bytes(sub_bits, L).view(n_sub, batch, L)
    full = valid.permute(1, 0, 2).reshape(batch, n_sub * L).contiguous()
    return kernels.bytes_to_bits(full)


def ulysses_qkv_to_heads(qkv_local: torch.Tensor, n: int, group=None, log: CommLog | None = None):
    """(R, L, 3C) packed q|k|v of this rank's R pattern rows, all heads  ->  (N*R, L, 3C/N) of
    all rows for this rank's C/N channels (heads), via one all_to_all_single."""
    import torch.distributed as dist
    R, L, C3 = qkv_local.shape
    C = C3 // 3
    send = kernels.ulysses_pack_qkv(qkv_local, n)           # (n, R*L, 3C/n), K1 chunked gathers
    recv = torch.empty_like(send)
    tok = log.time_start() if log is not None else None
    dist.all_to_all_single(recv, send, group=group)
    if log is not None:
        log.time_end(tok, "ulysses-qkv")
        log.record("all_to_all", send.numel(), "ulysses-qkv", send.numel() * send.element_size())
    return recv.view(n * R, L, 3 * (C // n))


def ulysses_out_to_rows(o_heads: torch.Tensor, n: int, group=None, log: CommLog | None = None):
    """(N*R, L, C/N) output for this rank's heads -> (R, L, C) this rank's rows, all heads."""
    import torch.distributed as dist
    NR, L, Cn = o_heads.shape
    R = NR // n
    recv = torch.empty_like(o_heads)
    tok = log.time_start() if log is not None else None
    dist.all_to_all_single(recv, o_heads.contiguous(), group=group)
    if log is not None:
        log.time_end(tok, "ulysses-out")
        log.record("all_to_all", o_heads.numel(), "ulysses-out", o_heads.numel() * o_heads.element_size())
    # (n, R*L, C/n) head blocks -> (R*L, C) rows: one K1 chunked gather
    out = kernels.gather_rows_chunked(recv.view(n, R * L, Cn), kernels.iota_index(R * L, recv.device), R * L, n,
                                      True, False)
    return out.view(R, L, n * Cn)


class _UlyssesQKV(torch.autograd.Function):
    @staticmethod
    def forward(ctx, qkv, n, group, log):
        ctx.n, ctx.group, ctx.log = n, group, log
        return ulysses_qkv_to_heads(qkv, n, group, log)

    @staticmethod
    def backward(ctx, g):
        # adjoint of the row->head redistribution: send each head block back to its rows
        import torch.distributed as dist
        n = ctx.n
        NR, L, C3n = g.shape
        R = NR // n
        recv = torch.empty_like(g)
        dist.all_to_all_single(recv, g.contiguous(), group=ctx.group)
        if ctx.log is not None:
            ctx.log.record("all_to_all", g.numel(), "ulysses-qkv-bwd", g.numel() * g.element_size())
        out = kernels.ulysses_unpack_qkv(recv.view(n, R * L, C3n), n)
        return out.view(R, L, -1), None, None, None


class _UlyssesOut(torch.autograd.Function):
    @staticmethod
    def forward(ctx, o, n, group, log):
        ctx.n, ctx.group, ctx.log = n, group, log
        return ulysses_out_to_rows(o, n, group, log)

    @staticmethod
    def backward(ctx, g):
        import torch.distributed as dist
        n = ctx.n
        R, L, C = g.shape
        send = kernels.gather_rows_chunked(g.reshape(R * L, C), kernels.iota_index(R * L, g.device), R * L, n,
                                           False, True)
        recv = torch.empty_like(send)
        dist.all_to_all_single(recv, send, group=ctx.group)
        if ctx.log is not None:
            ctx.log.record("all_to_all", send.numel(), "ulysses-out-bwd", send.numel() * send.element_size())
        return recv.view(n * R, L, C // n), None, None, None


class HybridStack:
    """A stack of attention layers following `schedule` (LayerKind FULL / TSA / GSA) on one
    latent grid `g` (padded internally as anyres.py:57-66).  Input and output: this rank's
    token-wise shard (G*B, L, C) bf16."""

    def __init__(self, g: GridShape, heads: int, chan: int, schedule=None, num_layers: int = 6,
                 n_full: int = 2, batch: int = 1, group=None, log: CommLog | None = None,
                 device=None, seed: int = PROJECTION_SEED, transport: str = "native"):
        import torch.distributed as dist
        self.schedule = list(schedule) if schedule is not None else build_layer_schedule(num_layers, n_full)
        self.g, self.pg = g, pad_grid(g)
        self.grid = self.pg.padded
        self.heads, self.chan, self.batch = heads, chan, batch
        self.group, self.log = group, log
        self.world = dist.get_world_size(group) if (group is not None or (
            dist.is_available() and dist.is_initialized())) else 1
        self.rank = dist.get_rank(group) if self.world > 1 else 0
        k2 = g.k * g.k
        if (k2 * batch) % self.world:
            raise ValueError(f"{k2 * batch} subsequences do not shard over {self.world} ranks")
        if any(s is LayerKind.FULL for s in self.schedule) and heads % self.world:
            raise ValueError(f"full-attention blocks need heads ({heads}) divisible by {self.world}")
        self.n_sub, self.L = k2, self.grid.seq_len // k2
        self.local_rows = k2 * batch // self.world
        dev = device or torch.device("cuda", torch.cuda.current_device())
        self.weights = [packed_projection(chan, COMPUTE_DTYPE, dev, seed + i)
                        for i in range(len(self.schedule))]
        r0 = self.rank * self.local_rows
        self.bits = {}
        self.full_bits = {}
        for pat in (SparsePattern.TOKEN_WISE, SparsePattern.GROUP_WISE):
            b = self.pg.mask_bits(pat, batch)
            self.bits[pat] = None if b is None else b[r0:r0 + self.local_rows].contiguous()
            self.full_bits[pat] = None if b is None else full_sequence_bits(b, k2, batch, self.L)
        # padding compaction (compact.py): attention over real rows only, for both block kinds
        from .compact import compact_plan
        self.plans = {pat: self.pg.compact_plan(pat, batch, (r0, r0 + self.local_rows))
                      for pat in (SparsePattern.TOKEN_WISE, SparsePattern.GROUP_WISE)}
        self.full_plans = {pat: None if fb is None else
                           compact_plan(kernels.bits_to_bytes(fb, k2 * self.L).view(batch, -1))
                           for pat, fb in self.full_bits.items()}
        self._t2g = IndexMap._pattern("tsa_to_gsa", self.grid, batch)
        self._g2t = IndexMap._pattern("gsa_to_tsa", self.grid, batch)
        # transport "p2p": each switch is one pull over peer memory (K7, peer.py)
        self.transport = transport
        self._peer = None
        if transport == "p2p" and self.world > 1:
            from .peer import padded_switch_moves, shared_arena
            self._peer = padded_switch_moves(self.world, self.rank, self.local_rows, self.L,
                                             self._t2g.src.reshape(-1).to(dev),
                                             self._g2t.src.reshape(-1).to(dev))
            row_bytes = chan * torch.finfo(COMPUTE_DTYPE).bits // 8
            self.arena = shared_arena(group, self.local_rows * self.L * row_bytes)
        elif transport not in ("native", "hif8", "p2p"):
            raise ValueError(f"unknown transport {transport!r}")

    # ------------------------------------------------------------------ pieces
    def _switch(self, x, to: SparsePattern):
        if self.world == 1:
            return (self._t2g if to is SparsePattern.GROUP_WISE else self._g2t).apply(x)
        if self._peer is not None:
            from .peer import peer_switch
            return peer_switch(x, self._peer[0 if to is SparsePattern.GROUP_WISE else 1], self.arena,
                               self.log)
        return ssp_switch(x, self.grid, self.group, self.log,
                          "hif8" if self.transport == "hif8" else "native")

    def _skiparse(self, x, W, pat):
        from .compact import compact_rows, expand_rows
        plan = self.plans[pat]
        if plan is not None:
            qkv = torch.matmul(compact_rows(x, plan), W)
            return expand_rows(attention_packed(qkv, self.heads, seq_lens=plan.lens), plan)
        return attention_packed(torch.matmul(x, W), self.heads)

    def _full(self, x, W, pat):
        """Full attention over each batch item's whole (padded) sequence, computed in the
        current pattern layout."""
        qkv = torch.matmul(x, W)                                  # (R, L, 3C)
        bits = self.full_bits[pat]
        n = self.world
        if n > 1:
            qkv = _UlyssesQKV.apply(qkv, n, self.group, self.log)  # (k2*B, L, 3C/n)
        rows, L, C3 = qkv.shape
        B = self.batch
        # rows are nested (pattern id, batch item): regroup to one sequence per batch item
        seq = qkv.view(self.n_sub, B, L, C3).transpose(0, 1).reshape(B, self.n_sub * L, C3)
        plan = self.full_plans[pat]
        if plan is not None:
            from .compact import compact_rows, expand_rows
            o = expand_rows(attention_packed(compact_rows(seq, plan), self.heads // n,
                                             seq_lens=plan.lens), plan)
        else:
            o = attention_packed(seq, self.heads // n, bits, zero_invalid_queries=bits is not None)
        o = o.view(B, self.n_sub, L, C3 // 3).transpose(0, 1).reshape(rows, L, C3 // 3)
        if n > 1:
            o = _UlyssesOut.apply(o, n, self.group, self.log)
        return o

    def __call__(self, x_tsa: torch.Tensor) -> torch.Tensor:
        x, layout = x_tsa, SparsePattern.TOKEN_WISE
        for kind, W in zip(self.schedule, self.weights):
            if kind is LayerKind.FULL:
                x = self._full(x, W, layout)
                continue
            want = SparsePattern.TOKEN_WISE if kind is LayerKind.TSA else SparsePattern.GROUP_WISE
            if want is not layout:
                x = self._switch(x, want)
                layout = want
            x = self._skiparse(x, W, layout)
        if layout is not SparsePattern.TOKEN_WISE:
            x = self._switch(x, SparsePattern.TOKEN_WISE)
        return x

    def flops(self) -> dict:
        """Executed attention FLOPs (real-token interactions when the grid is padded)."""
        d = self.chan // self.heads

        def sq(plan, default):
            if plan is None:
                return default
            lens = plan.lens.to(torch.int64)
            return int((lens * lens).sum())

        sk = 4 * d * self.heads * sq(self.plans[SparsePattern.TOKEN_WISE],
                                     self.local_rows * self.L * self.L)
        S = self.n_sub * self.L
        full = 4 * d * self.heads * sq(self.full_plans[SparsePattern.TOKEN_WISE],
                                       self.batch * S * S) // self.world
        n_full = sum(1 for s in self.schedule if s is LayerKind.FULL)
        n_sk = len(self.schedule) - n_full
        return {"attention_fwd": n_full * full + n_sk * sk,
                "attention_fwd_bwd": 3.5 * (n_full * full + n_sk * sk)}
