"""One Skiparse-2D attention block (token-wise application, then group-wise
application) in the steady-state layout of a Skiparse DiT, single GPU or SSP.

The reference operator is skiparse_attention (attention.py:97-131) applied
with TOKEN_WISE and then GROUP_WISE; in a model the hidden states stay in a
pattern layout between blocks, so the block maps a
token-wise input to a token-wise output:

    qkv1 = x W1 ; o1 = attn_tsa(qkv1)          (per subsequence, 1-D mask)
    x2   = switch(o1)                           tsa_to_gsa (N=1) | SSP all-to-all
    qkv2 = x2 W2 ; o2 = attn_gsa(qkv2)
    y    = switch(o2)                           gsa_to_tsa (N=1) | SSP all-to-all

Under SSP each rank holds G = k^2/N whole subsequences (ssp.py:91-106) and the
switch is one NCCL all-to-all (ssp.py:139-180); attention needs no
communication.  W1, W2 are the reference's fixed seeded projections
(attention.py:20-32) in bf16; they are constants, so the backward produces the
input gradient only.
"""

from __future__ import annotations

import torch

from . import kernels
from .anyres import PaddedGrid, pad_grid
from .attention import COMPUTE_DTYPE, PROJECTION_SEED, attention_packed, packed_projection
from .gridseq import GridShape, IndexMap
from .skiparse import SparsePattern
from .ssp import CommLog, ssp_switch


def plan_parallel(world: int, k: int) -> tuple[int, int]:
    """(SSP group size, data-parallel replicas) for `world` GPUs.  SSP shards the
    k^2 subsequences of one latent over N ranks when N | k^2 (ssp.py:147-148);
    otherwise (e.g. k=2 on 8 GPUs) groups of k^2 ranks run SSP and the groups
    take different latents (SURVEY.md sec. 8e option 2)."""
    k2 = k * k
    if world < 1:
        raise ValueError("world size must be positive")
    if k2 % world == 0:
        return world, 1
    if world % k2 == 0:
        return k2, world // k2
    raise ValueError(f"cannot shard k^2={k2} subsequences over {world} ranks")


def plan_parallel_3d(world: int, k: int, heads: int, txh: int) -> tuple[int, int, int]:
    """(SSP size, Ulysses size, data-parallel replicas).  When N > k^2 the paper's 8-GPU setting
    composes SSP with Ulysses (SURVEY.md sec. 8e option 1): the k^2 subsequences
    shard over k^2 SSP ranks and each subsequence's positions split over U Ulysses ranks along
    the (t, h/k^2) "txh" axis -- the slowest index of both pattern layouts, so a position block
    is a whole run of minimal repeatable units and the SSP switch acts on it independently.
    Falls back to SSP x DP when heads or txh do not divide."""
    k2 = k * k
    if world <= k2 or world % k2:
        s, dp = plan_parallel(world, k)
        return s, 1, dp
    u = world // k2
    if heads % u == 0 and txh % u == 0:
        return k2, u, 1
    return k2, 1, u


class SkiparseBlock:
    def __init__(self, g: GridShape, heads: int, chan: int, batch: int = 1, group=None,
                 log: CommLog | None = None, device=None, seeds=(PROJECTION_SEED, PROJECTION_SEED + 1),
                 transport: str = "native", qk_norm: str | None = None, rope: bool = False,
                 eps: float = 1e-6, compact: bool = True, ulysses_group=None, switch_chunks: int | None = None):
        import torch.distributed as dist
        self.g = g
        self.pg: PaddedGrid = pad_grid(g)
        self.grid = self.pg.padded
        self.heads, self.chan, self.batch = heads, chan, batch
        self.group = group
        self.world = dist.get_world_size(group) if (group is not None or (
            dist.is_available() and dist.is_initialized())) else 1
        self.rank = dist.get_rank(group) if self.world > 1 else 0
        self.log = log
        self.transport = transport
        # sec. 8f row 2: QK-RMSNorm ("head" | "channel") and 3-D RoPE fused into the projection
        # (K6); off = the reference's plain fixed projection (cuBLAS GEMM)
        self.qk_norm, self.rope, self.eps = qk_norm, rope, eps
        n_sub = g.k * g.k
        if (n_sub * batch) % self.world:
            raise ValueError(f"{n_sub * batch} subsequences do not shard over {self.world} ranks")
        self.local_rows = n_sub * batch // self.world
        self.L = self.grid.seq_len // n_sub
        # SSP x Ulysses: this rank holds position block u of its subsequences (a txh range)
        self.uly_group = ulysses_group
        self.uly = dist.get_world_size(ulysses_group) if ulysses_group is not None else 1
        self.uly_rank = dist.get_rank(ulysses_group) if ulysses_group is not None else 0
        if self.uly > 1:
            txh = self.grid.t * self.grid.h // n_sub
            if qk_norm is not None or rope:
                raise ValueError("SSP x Ulysses does not support the projection prologue")
            if heads % self.uly or txh % self.uly:
                raise ValueError(f"Ulysses size {self.uly} must divide heads ({heads}) and txh ({txh})")
            self.L_local = self.L // self.uly
            # the switch acts on one position block as on a grid of txh/U frames-rows
            self.sub_grid = GridShape(1, txh // self.uly * n_sub, self.grid.w, g.k)
        else:
            self.L_local = self.L
            self.sub_grid = self.grid
        dev = device or torch.device("cuda", torch.cuda.current_device())
        self.W1 = packed_projection(chan, COMPUTE_DTYPE, dev, seeds[0])
        self.W2 = packed_projection(chan, COMPUTE_DTYPE, dev, seeds[1])
        self.prologue = qk_norm is not None or rope
        if self.prologue:
            from .prologue import packed_projection_t
            self.W1t = packed_projection_t(chan, dev, seeds[0])
            self.W2t = packed_projection_t(chan, dev, seeds[1])
            self.gamma_q = torch.ones(chan, device=dev)
            self.gamma_k = torch.ones(chan, device=dev)
        r0, r1 = self.rank * self.local_rows, (self.rank + 1) * self.local_rows
        bt = self.pg.mask_bits(SparsePattern.TOKEN_WISE, batch)
        bg = self.pg.mask_bits(SparsePattern.GROUP_WISE, batch)
        self.bits_tsa = None if bt is None else bt[r0:r1].contiguous()
        self.bits_gsa = None if bg is None else bg[r0:r1].contiguous()
        # padding compaction (compact.py): attention over each subsequence's real rows only
        self.plan_tsa = self.pg.compact_plan(SparsePattern.TOKEN_WISE, batch, (r0, r1)) if compact else None
        self.plan_gsa = self.pg.compact_plan(SparsePattern.GROUP_WISE, batch, (r0, r1)) if compact else None
        self._t2g = IndexMap._pattern("tsa_to_gsa", self.grid, batch)
        self._g2t = IndexMap._pattern("gsa_to_tsa", self.grid, batch)
        # one GPU, head_dim 128: the rearranges can also be fused into the attention kernels' TMA
        # LOADS (gather mode, forward_original_gather) -- exact but slower
        self.gather = None
        if self.world == 1 and chan // heads == 128:
            from .compact import gather_plan
            self.gather = (gather_plan(g, SparsePattern.TOKEN_WISE, batch, self.pg, "original"),
                           gather_plan(g, SparsePattern.GROUP_WISE, batch, self.pg, "original"))
        # one GPU (the benched path): every rearrange that follows an attention application runs
        # in its epilogue (scatter mode): application 1 stores its compact TSA rows straight into
        # the compact GSA layout application 2 projects, application 2 stores into the block's
        # output layout; the backward's Delta pre-pass gathers dO through the same tables.  On an
        # unpadded grid the "compact" plans are the identity plans (every row real).
        self._scatter = None
        self._fused = None
        self._orig = None
        d = chan // heads
        if self.world == 1 and compact and not self.prologue and d in (64, 128):
            from .compact import compact_plan, scatter_plan
            if self.plan_tsa is None:   # trivial grid: identity plans
                full = compact_plan(torch.ones(self.local_rows, self.L, dtype=torch.bool, device=dev))
                self.plan_tsa = self.plan_gsa = full
            pt, pgs = self.plan_tsa, self.plan_gsa
            t2g = self._t2g.src.reshape(-1).to(dev)          # padded GSA row x holds TSA row t2g[x]
            g2t = self._g2t.src.reshape(-1).to(dev)          # padded TSA row y holds GSA row g2t[y]
            pgt = pt.gather                                   # compact TSA row -> padded TSA row
            a = torch.where(pgt >= 0, pgs.scatter[g2t[pgt.clamp(min=0)]], torch.full_like(pgt, -1))
            pgg = pgs.gather                                  # compact GSA row -> padded GSA row
            b = torch.where(pgg >= 0, t2g[pgg.clamp(min=0)], torch.full_like(pgg, -1))
            self._scatter = (
                scatter_plan(a, pt.n_seq, pt.cap, pgs.n_seq * pgs.cap, (pgs.n_seq, pgs.cap, chan)),
                scatter_plan(b, pgs.n_seq, pgs.cap, self.local_rows * self.L, (self.local_rows, self.L, chan)))
        elif self.world == 1 and self.plan_tsa is not None and not self.prologue:
            # other head dims: fold expand -> pattern switch -> compact into one K1 row move each way
            from .compact import row_move
            pt, pgs = self.plan_tsa, self.plan_gsa
            t2g = self._t2g.src.reshape(-1)                 # padded GSA row <- padded TSA row
            g2t = self._g2t.src.reshape(-1)
            gp = pgs.gather                                  # compact GSA row -> padded GSA row
            a = torch.where(gp >= 0, pt.scatter[t2g[gp.clamp(min=0)]], torch.full_like(gp, -1))
            b = pgs.scatter[g2t]                             # padded TSA row <- compact GSA row
            self._fused = (row_move(a, pt.n_seq * pt.cap, pgs.cap, pt.cap),
                           row_move(b, pgs.n_seq * pgs.cap, pt.L, pgs.cap))

        # N GPUs, NCCL transport: the switches run per head chunk on a communication stream,
        # overlapped with the attention of the next chunk (ssp_overlap.py); switch_chunks=1 keeps
        # one all-to-all per switch without overlap, 0 the unfused reference-shaped path
        self._overlap = None
        if switch_chunks is None:
            switch_chunks = next(c for c in (4, 2, 1) if heads % c == 0)
        if (self.world > 1 and self.uly == 1 and transport == "native" and compact and not self.prologue
                and d in (64, 128) and switch_chunks >= 1):
            from .compact import compact_plan
            from .ssp_overlap import SSPOverlapPlan
            if self.plan_tsa is None:   # trivial grid: identity plans
                full = compact_plan(torch.ones(self.local_rows, self.L, dtype=torch.bool, device=dev))
                self.plan_tsa = self.plan_gsa = full
            self._overlap = SSPOverlapPlan(self, switch_chunks)

        # N GPUs, transport "p2p": each switch is one pull over peer memory (K7, peer.py) whose
        # table folds expand -> switch -> compact; every rank builds every rank's plans
        self._peer = None
        if transport == "p2p":
            if self.world == 1:
                pass
            elif self.uly > 1 or not compact:
                raise ValueError("the p2p switch needs compaction and no Ulysses group")
            else:
                from .peer import same_host
                if not same_host(group):
                    raise ValueError("the p2p switch maps peers' memory through CUDA IPC: every "
                                     "rank of the SSP group must be on one host")
                from .compact import compact_plan
                from .peer import block_switch_moves, shared_arena
                rng = [(j * self.local_rows, (j + 1) * self.local_rows) for j in range(self.world)]
                if self.pg.trivial:   # no pad tokens: identity plans (every row real)
                    full = compact_plan(torch.ones(self.local_rows, self.L, dtype=torch.bool, device=dev))
                    pts = pgs = [full] * self.world
                    self.plan_tsa = self.plan_gsa = full
                else:
                    pts = [self.pg.compact_plan(SparsePattern.TOKEN_WISE, batch, r) for r in rng]
                    pgs = [self.pg.compact_plan(SparsePattern.GROUP_WISE, batch, r) for r in rng]
                A, B = block_switch_moves(self.world, self.rank, self.local_rows, self.L,
                                          self._t2g.src.reshape(-1).to(dev),
                                          self._g2t.src.reshape(-1).to(dev), pts, pgs,
                                          padded_gsa=self.prologue)
                self._peer = (A, B)
                row_bytes = chan * torch.finfo(COMPUTE_DTYPE).bits // 8
                slot_rows = max(max(p.n_seq * p.cap for p in pts), max(p.n_seq * p.cap for p in pgs),
                                self.local_rows * self.L)
                self.arena = shared_arena(self.group, slot_rows * row_bytes)

    # ------------------------------------------------------------------ pieces
    def switch_to_gsa(self, x):
        if self.world == 1:
            return self._t2g.apply(x)
        return ssp_switch(x, self.sub_grid, self.group, self.log, self.transport)

    def switch_to_tsa(self, x):
        if self.world == 1:
            return self._g2t.apply(x)
        return ssp_switch(x, self.sub_grid, self.group, self.log, self.transport)

    def _uly_moves(self, R: int):
        """K1 row moves between Ulysses position blocks and whole subsequences: (n*R, L/U, X) with
        rows (block j, subsequence r) <-> (R, L, X) with the U blocks of r concatenated."""
        key = ("uly", R)
        if key not in self.__dict__.setdefault("_moves", {}):
            from .compact import row_move
            n, Lu = self.uly, self.L_local
            dev = self.W1.device
            r = torch.arange(R, device=dev).view(R, 1, 1)
            j = torch.arange(n, device=dev).view(1, n, 1)
            p = torch.arange(Lu, device=dev).view(1, 1, Lu)
            src = ((j * R + r) * Lu + p).reshape(-1)          # dst row (r, j, p) <- src (j, r, p)
            gather = row_move(src, n * R * Lu, self.L, Lu)
            scatter = row_move(gather.inv, R * self.L, Lu, self.L)
            self._moves[key] = (gather, scatter)
        return self._moves[key]

    def _ulysses_in(self, qkv):
        """(R, L/U, 3C) position block, all heads -> (R, L, 3C/U) all positions, my heads."""
        from .compact import apply_move
        from .stack import _UlyssesQKV
        n = self.uly
        h = _UlyssesQKV.apply(qkv, n, self.uly_group, self.log)            # (n*R, L/U, 3C/n)
        return apply_move(h, self._uly_moves(qkv.shape[0])[0])

    def _ulysses_out(self, o):
        """(R, L, C/U) my heads -> (R, L/U, C) my position block, all heads."""
        from .compact import apply_move
        from .stack import _UlyssesOut
        rows = apply_move(o, self._uly_moves(o.shape[0])[1])               # (n*R, L/U, C/n)
        return _UlyssesOut.apply(rows, self.uly, self.uly_group, self.log)

    def attend(self, x, W, bits, pattern=SparsePattern.TOKEN_WISE, compact_in=False, expand=True):
        """One attention application on this rank's shard.  compact_in: x already holds the
        compacted rows; expand=False: return the compacted output (the peer switch moves
        compact rows directly)."""
        from .compact import compact_rows, expand_rows
        plan = self.plan_tsa if pattern is SparsePattern.TOKEN_WISE else self.plan_gsa
        if self.uly > 1:
            # projection on my position block, Ulysses all-to-all to whole subsequences with
            # H/U heads, compacted attention, and back
            qkv = self._ulysses_in(torch.matmul(x, W))
            heads = self.heads // self.uly
            if plan is not None:
                o = expand_rows(attention_packed(compact_rows(qkv, plan), heads, seq_lens=plan.lens), plan)
            else:
                o = attention_packed(qkv, heads, bits, zero_invalid_queries=bits is not None)
            return self._ulysses_out(o)
        if self.prologue:
            from .prologue import QKVPrologue
            Wt = self.W1t if W is self.W1 else self.W2t
            # RoPE positions come from padded-layout rows: project first, then compact
            qkv = QKVPrologue.apply(x, self.grid, pattern, self.batch, self.qk_norm, self.gamma_q,
                                    self.gamma_k, self.eps, self.rope,
                                    self.rank * self.local_rows * self.L, Wt)
            if plan is not None:
                qkv = compact_rows(qkv, plan)
        elif plan is not None:
            qkv = torch.matmul(x if compact_in else compact_rows(x, plan), W)
        else:
            qkv = torch.matmul(x, W)
        if plan is not None:
            o = attention_packed(qkv, self.heads, seq_lens=plan.lens)
            return expand_rows(o, plan) if expand else o
        return attention_packed(qkv, self.heads, bits, zero_invalid_queries=bits is not None)

    def _orig_plans(self):
        """Tables of the original-layout step (orig -> TSA -> GSA -> orig): the
        K1 gather of the unpadded latent into compact TSA rows, and application 2's scatter
        straight into the unpadded latent (every real token is one compact GSA row)."""
        if self._orig is None:
            from .compact import row_move, scatter_plan
            dev = self.W1.device
            p, B = self.grid, self.batch
            S = p.seq_len
            mask = self.pg.mask.to(dev).bool() if not self.pg.trivial else torch.ones(S, dtype=torch.bool, device=dev)
            real_idx = torch.cumsum(mask.to(torch.int64), 0) - 1
            S_real = int(mask.sum())

            def real_row(src):        # padded (batch, token) flat index -> unpadded latent row
                return (src // S) * S_real + real_idx[src % S]

            o2t = IndexMap._pattern("orig_to_tsa", p, B).src.reshape(-1).to(dev)
            o2g = IndexMap._pattern("orig_to_gsa", p, B).src.reshape(-1).to(dev)
            pt, pgs = self.plan_tsa, self.plan_gsa
            tin = torch.where(pt.gather >= 0, real_row(o2t[pt.gather.clamp(min=0)]), torch.full_like(pt.gather, -1))
            bo = torch.where(pgs.gather >= 0, real_row(o2g[pgs.gather.clamp(min=0)]), torch.full_like(pgs.gather, -1))
            self._orig = (row_move(tin, B * S_real, pt.cap, S_real),
                          scatter_plan(bo, pgs.n_seq, pgs.cap, B * S_real, (B, S_real, self.chan)))
        return self._orig

    def forward_original(self, x: torch.Tensor) -> torch.Tensor:
        """One GPU: the block on the original (unpadded) latent layout (B, T*H0*W0, C) ->
        same layout.  One K1 row gather brings the latent into compact TSA rows for the first
        projection GEMM; every later rearrange runs in an attention epilogue (application 1 ->
        compact GSA rows, application 2 -> the unpadded latent), and their backward adjoints in
        the attention backward's Delta pre-pass."""
        if self._scatter is None:
            raise ValueError("forward_original needs one GPU, head_dim 64/128 and no projection prologue")
        from .attention import attention_scatter
        from .compact import apply_move
        tin, bo = self._orig_plans()
        pt, pgs = self.plan_tsa, self.plan_gsa
        x1 = apply_move(x.reshape(-1, self.chan), tin)
        x2 = attention_scatter(torch.matmul(x1, self.W1), self.heads, pt.lens, self._scatter[0])
        return attention_scatter(torch.matmul(x2, self.W2), self.heads, pgs.lens, bo)

    def forward_original_gather(self, x: torch.Tensor) -> torch.Tensor:
        """One GPU: the block on the original (unpadded) latent layout (B, T*H0*W0, C) -- TSA
        application then GSA application with no rearranged copy in HBM (gather-mode kernels)."""
        if self.gather is None:
            raise ValueError("forward_original_gather needs one GPU and head_dim 128")
        from .attention import attention_gather
        for W, Wt, plan, pat in ((self.W1, getattr(self, "W1t", None), self.gather[0], SparsePattern.TOKEN_WISE),
                                 (self.W2, getattr(self, "W2t", None), self.gather[1], SparsePattern.GROUP_WISE)):
            if self.prologue:
                from .prologue import QKVPrologue
                qkv = QKVPrologue.apply(x, self.g, SparsePattern.ORIGINAL, self.batch, self.qk_norm,
                                        self.gamma_q, self.gamma_k, self.eps, self.rope, 0, Wt)
            else:
                qkv = torch.matmul(x, W)
            x = attention_gather(qkv, self.heads, plan)
        return x

    def _call_scatter(self, x_tsa):
        from .attention import attention_scatter
        from .compact import compact_rows
        pt, pgs = self.plan_tsa, self.plan_gsa
        a, b = self._scatter
        x2 = attention_scatter(torch.matmul(compact_rows(x_tsa, pt), self.W1), self.heads, pt.lens, a)
        return attention_scatter(torch.matmul(x2, self.W2), self.heads, pgs.lens, b)

    def _call_fused(self, x_tsa):
        from .compact import apply_move, compact_rows
        pt, pgs = self.plan_tsa, self.plan_gsa
        o1 = attention_packed(torch.matmul(compact_rows(x_tsa, pt), self.W1), self.heads, seq_lens=pt.lens)
        x2 = apply_move(o1, self._fused[0])
        o2 = attention_packed(torch.matmul(x2, self.W2), self.heads, seq_lens=pgs.lens)
        return apply_move(o2, self._fused[1])

    def _call_peer(self, x_tsa):
        from .peer import peer_switch
        A, B = self._peer
        o1 = self.attend(x_tsa, self.W1, self.bits_tsa, expand=False)
        x2 = peer_switch(o1, A, self.arena, self.log)
        o2 = self.attend(x2, self.W2, self.bits_gsa, SparsePattern.GROUP_WISE,
                         compact_in=not self.prologue, expand=False)
        return peer_switch(o2, B, self.arena, self.log)

    def __call__(self, x_tsa: torch.Tensor) -> torch.Tensor:
        """x_tsa: this rank's (G*B, L, C) bf16 shard in the token-wise layout."""
        if self._scatter is not None:
            return self._call_scatter(x_tsa)
        if self._overlap is not None:
            from .compact import compact_rows
            from .ssp_overlap import SSPOverlapBlock
            return SSPOverlapBlock.apply(compact_rows(x_tsa, self.plan_tsa), self)
        if self._fused is not None:
            return self._call_fused(x_tsa)
        if self._peer is not None:
            return self._call_peer(x_tsa)
        o1 = self.attend(x_tsa, self.W1, self.bits_tsa)
        x2 = self.switch_to_gsa(o1)
        o2 = self.attend(x2, self.W2, self.bits_gsa, SparsePattern.GROUP_WISE)
        return self.switch_to_tsa(o2)

    # ------------------------------------------------------------------ layouts
    def to_local_tsa(self, x_orig: torch.Tensor) -> torch.Tensor:
        """(B, T*H0*W0, C) unpadded original layout -> this rank's token-wise shard
        (fused pad + orig_to_tsa, K1)."""
        p = self.grid
        full = kernels.rearrange(x_orig, "orig_to_tsa", p.t, p.h, p.w, p.k, self.batch,
                                 self.g.h, self.g.w)
        r0 = self.rank * self.local_rows
        mine = full[r0:r0 + self.local_rows]
        if self.uly > 1:   # this rank's position block (txh range) of its subsequences
            mine = mine[:, self.uly_rank * self.L_local:(self.uly_rank + 1) * self.L_local]
        return mine.contiguous()

    def flops(self) -> dict:
        """Tensor FLOPs of one block fwd+bwd for this rank.  `attention_fwd_per_app` counts the
        padded grid as the reference's flop_report does (checks.py:144-146); the `executed`
        counts are what the kernels run -- with padding compaction exactly the real-token
        ("useful") interactions."""
        d = self.chan // self.heads
        att_fwd = 4 * self.local_rows * self.L * self.L * d * self.heads  # per application
        rows = self.local_rows * self.L

        def executed(plan):
            if plan is None:
                return att_fwd, rows
            lens = plan.lens.to(torch.int64)
            return int((lens * lens).sum()) * 4 * d * self.heads, int(lens.sum())

        (f1, r1), (f2, r2) = executed(self.plan_tsa), executed(self.plan_gsa)
        proj = 2 * self.chan * 3 * self.chan  # per row: x @ [Wq|Wk|Wv]
        proj_rows = 2 * rows if self.prologue or self.plan_tsa is None else r1 + r2
        if self.uly > 1:   # H/U heads over whole subsequences; projection on the position block
            f1, f2 = f1 // self.uly, f2 // self.uly
            proj_rows = 2 * self.local_rows * self.L_local
        return {
            "attention_fwd_per_app": att_fwd,
            "attention_fwd_executed": f1 + f2,           # both applications
            "attention_fwd_bwd": 3.5 * (f1 + f2),
            "projection_fwd_bwd": 2 * proj * proj_rows,  # fwd GEMM + input-gradient GEMM
            "total": 3.5 * (f1 + f2) + 2 * proj * proj_rows,
        }
