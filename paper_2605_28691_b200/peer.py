"""SSP pattern switch as one pull over peer memory (K7, csrc/peer.cu).

The reference switch (ssp.py:139-180, Alg. 1) is pack -> one all-to-all -> unpack.  On an
NVSwitch node every GPU can load from every peer's HBM at full fabric bandwidth, so the switch
needs neither the pack nor the unpack pass nor a staging buffer: each rank copies its source
rows into a CUDA-IPC buffer (its "arena" slot), one flag barrier proves every rank's rows are
there, and each rank gathers its destination rows straight from its peers' slots with one
kernel.  The gather table composes the whole move the block needs around a switch -- expand the
compacted attention output, switch the pattern, compact for the next attention -- so only real
tokens cross the fabric.

`PeerMove` tables are exact injective row maps; the backward of a move is the pull with the
inverse table (the adjoint of a permutation is its inverse, as for RowMove in compact.py), so the
autograd switch runs the same kernel both ways.

Arena slots alternate, so the barrier in front of switch i+1 also proves every rank finished
pulling from switch i-1's slot: one barrier per switch.  `host_sync` (env OSP_PEER_HOST_SYNC=1)
replaces the device barrier with synchronize + group barrier: the test mode in which several
ranks share one GPU and no rank's kernel may wait on another's.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import torch

from . import _lib, kernels

__all__ = ["PeerArena", "PeerMove", "peer_move", "shared_arena", "close_arenas", "same_host", "peer_switch",
           "block_switch_moves", "padded_switch_moves"]


class _Mem:
    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False),
                                         "strides": None, "version": 3, "stream": None}


def _round(n: int, a: int = 256) -> int:
    return (n + a - 1) // a * a


def _timeout_ms() -> int:
    return int(float(os.environ.get("OSP_PEER_TIMEOUT_S", "60")) * 1000)


def same_host(group) -> bool:
    """True when every rank of `group` runs on this host (CUDA-IPC handles only open locally).
    Collective over `group`."""
    import socket

    import torch.distributed as dist
    names = [None] * dist.get_world_size(group)
    dist.all_gather_object(names, socket.gethostname(), group=group)
    return len(set(names)) == 1


class PeerArena:
    """One CUDA-IPC buffer per rank of `group`: a flag block (uint32 per rank) followed by
    `slots` source slots of `slot_bytes`; every rank holds every peer's base address.

    The device barrier is bounded by OSP_PEER_TIMEOUT_S (default 60 s): a rank that never
    arrives is reported through a pinned host status word (no __trap, the context survives) and
    the next barrier / close() raises CollectiveError naming it."""

    def __init__(self, group, slot_bytes: int, slots: int = 2, host_sync: bool | None = None):
        import torch.distributed as dist
        self.group = group
        self.n = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.host_sync = (os.environ.get("OSP_PEER_HOST_SYNC") == "1") if host_sync is None else host_sync
        self.flag_bytes = _round(4 * self.n)
        self.slots = slots
        self.device = torch.device("cuda", torch.cuda.current_device())
        self.status = torch.zeros(1, dtype=torch.int32, pin_memory=True)
        self.timeout_ms = _timeout_ms()
        self._own = None
        self._imported = []
        self._map(slot_bytes)

    def _map(self, slot_bytes: int) -> None:
        """Collective: allocate, export and import every rank's buffer."""
        import torch.distributed as dist
        L = _lib.lib()
        self.slot_bytes = _round(max(slot_bytes, 1))
        total = self.flag_bytes + self.slots * self.slot_bytes
        base = ctypes.c_void_p()
        _lib.check(L.osp_peer_alloc(total, ctypes.byref(base)))
        self._own = base.value
        handle = (ctypes.c_uint8 * 64)()
        _lib.check(L.osp_peer_export(ctypes.c_void_p(self._own), handle))
        handles = [None] * self.n
        dist.all_gather_object(handles, bytes(handle), group=self.group)
        self._imported = []
        self.bases = []
        for j, h in enumerate(handles):
            if j == self.rank:
                self.bases.append(self._own)
                continue
            p = ctypes.c_void_p()
            _lib.check(L.osp_peer_import((ctypes.c_uint8 * 64).from_buffer_copy(h), ctypes.byref(p)))
            self._imported.append(p.value)
            self.bases.append(p.value)
        self.epoch = 0
        self.turn = 0
        self._views = [torch.as_tensor(_Mem(self._own + self.flag_bytes + s * self.slot_bytes,
                                            self.slot_bytes), device=self.device)
                       for s in range(self.slots)]

    def ensure(self, slot_bytes: int) -> "PeerArena":
        """Collective: grow the slots in place (old mappings are released first), so every block
        sharing this arena sees the larger buffer and nothing leaks."""
        if self._own is None or self.slot_bytes < slot_bytes:
            self._unmap()
            self._map(slot_bytes)
        return self

    # ------------------------------------------------------------------ pieces
    def slot_ptrs(self, s: int) -> list[int]:
        return [b + self.flag_bytes + s * self.slot_bytes for b in self.bases]

    def check(self) -> None:
        """Raise CollectiveError if an earlier device barrier timed out (reads the pinned
        status word the barrier kernel writes; no device synchronisation)."""
        v = int(self.status[0])
        if v:
            from .errors import CollectiveError
            raise CollectiveError(f"peer barrier: rank {v - 1} of {self.n} did not arrive within "
                                  f"{self.timeout_ms / 1000:g} s (OSP_PEER_TIMEOUT_S)")

    def barrier(self) -> None:
        if self.host_sync:
            import torch.distributed as dist
            torch.cuda.synchronize()
            dist.barrier(group=self.group)
            return
        self.check()
        self.epoch += 1
        kernels.peer_barrier(self.bases, self.rank, self.epoch, self.device, self.timeout_ms,
                             self.status)

    def move(self, x: torch.Tensor, table: torch.Tensor, stride: int, out_rows: int,
             col0: int = 0, out: torch.Tensor | None = None) -> torch.Tensor:
        """Publish x's rows in the next slot, barrier, pull `table` from every rank's slot."""
        C = x.shape[-1]
        nb = x.numel() * x.element_size()
        if nb > self.slot_bytes:
            raise ValueError(f"source of {nb} bytes exceeds the arena slot ({self.slot_bytes})")
        s = self.turn
        self.turn = (self.turn + 1) % self.slots
        self._views[s][:nb].view(x.dtype).view(x.shape).copy_(x)
        self.barrier()
        if out is None:
            out = torch.empty((table.numel(), C), dtype=x.dtype, device=x.device)
        kernels.peer_gather(self.slot_ptrs(s), stride, table, out)
        return out.view(table.numel() // out_rows, out_rows, C)

    def _unmap(self) -> None:
        if self._own is None:
            return
        import torch.distributed as dist
        L = _lib.lib()
        torch.cuda.synchronize()
        for p in self._imported:
            L.osp_peer_close(ctypes.c_void_p(p))
        dist.barrier(group=self.group)
        L.osp_peer_free(ctypes.c_void_p(self._own))
        self._own, self._imported, self._views = None, [], []

    def close(self) -> None:
        """Collective: unmap the peers' buffers, wait until every rank has, then free our own."""
        if self._own is None:
            return
        self._unmap()
        self.check()


_ARENAS: dict = {}


def shared_arena(group, slot_bytes: int) -> PeerArena:
    """One arena per group, shared by every block (the same shapes repeat down a stack); a block
    that needs larger slots grows the shared arena in place.  Collective: every rank must call
    it with the same slot_bytes."""
    key = group   # the group object itself (held), so a recycled id() can never alias it
    a = _ARENAS.get(key)
    host_sync = os.environ.get("OSP_PEER_HOST_SYNC") == "1"
    if a is not None and a.host_sync != host_sync:
        a.close()
        a = None
    if a is None:
        a = PeerArena(group, slot_bytes)
        _ARENAS[key] = a
    return a.ensure(slot_bytes)


def close_arenas() -> None:
    """Collective teardown of every shared arena (call before destroy_process_group)."""
    while _ARENAS:
        _, a = _ARENAS.popitem()
        a.close()


@dataclass(frozen=True)
class PeerMove:
    """This rank's side of a cross-rank injective row move.  Forward: dst row i <- row
    table[i] % stride of rank table[i] // stride (-1 = zero).  Backward: source row s <-
    row inv[s] % inv_stride of rank inv[s] // inv_stride."""

    table: torch.Tensor
    stride: int
    out_rows: int          # output rows per sequence (view)
    inv: torch.Tensor
    inv_stride: int
    in_rows: int           # input rows per sequence (view of the gradient)
    remote_rows: int       # rows of `table` pulled from other ranks
    remote_rows_bwd: int


def peer_move(dst_src: list, src_rows: list, rank: int, out_rows: int, in_rows: int) -> PeerMove:
    """dst_src[r] = (n_dst_r,) int64 global source rows of rank r's destination rows, encoded
    j * max(src_rows) + s (-1 = zero row); every rank passes the same lists."""
    stride = max(max(src_rows), 1)
    dstride = max(max(int(t.numel()) for t in dst_src), 1)
    dev = dst_src[0].device
    inv_all = torch.full((len(dst_src) * stride,), -1, dtype=torch.int64, device=dev)
    for r, t in enumerate(dst_src):
        ok = t >= 0
        inv_all[t[ok]] = r * dstride + torch.nonzero(ok).view(-1)
    inv = inv_all[rank * stride: rank * stride + src_rows[rank]].contiguous()
    tab = dst_src[rank].contiguous()
    remote = int(((tab >= 0) & (tab // stride != rank)).sum())
    remote_b = int(((inv >= 0) & (inv // dstride != rank)).sum())
    return PeerMove(tab, stride, out_rows, inv, dstride, in_rows, remote, remote_b)


def block_switch_moves(world: int, rank: int, local_rows: int, L: int, t2g: torch.Tensor,
                       g2t: torch.Tensor, plans_tsa: list, plans_gsa: list,
                       padded_gsa: bool = False) -> tuple[PeerMove, PeerMove]:
    """The two moves of an SSP block (SkiparseBlock.__call__) as cross-rank tables.
    A: compact TSA attention output of every rank -> this rank's compact GSA rows (padded GSA
       rows when padded_gsa, for the projection prologue), i.e. expand -> switch -> compact.
    B: compact GSA attention output of every rank -> this rank's padded TSA rows (zero pads),
       i.e. expand -> switch back.
    t2g / g2t: global padded-row maps (gsa[x] = tsa[t2g[x]], tsa[y] = gsa[g2t[y]]); plans_* the
    CompactPlan of each rank's subsequence range."""
    LR = local_rows * L
    dev = t2g.device

    def encoded_scatter(plans):
        stride = max(p.n_seq * p.cap for p in plans)
        enc = torch.cat([torch.where(p.scatter >= 0, j * stride + p.scatter, torch.full_like(p.scatter, -1))
                         for j, p in enumerate(plans)])
        return enc, [p.n_seq * p.cap for p in plans]

    enc_t, rows_t = encoded_scatter(plans_tsa)
    enc_g, rows_g = encoded_scatter(plans_gsa)
    a_dst = []
    for r in range(world):
        if padded_gsa:
            lg = torch.arange(LR, device=dev, dtype=torch.int64)
        else:
            lg = plans_gsa[r].gather
        src = enc_t[t2g[(r * LR + lg).clamp(min=0)]]
        a_dst.append(torch.where(lg >= 0, src, torch.full_like(src, -1)))
    ar = plans_gsa[rank].cap if not padded_gsa else L
    A = peer_move(a_dst, rows_t, rank, ar, plans_tsa[rank].cap)
    b_dst = [enc_g[g2t[r * LR + torch.arange(LR, device=dev, dtype=torch.int64)]] for r in range(world)]
    B = peer_move(b_dst, rows_g, rank, L, plans_gsa[rank].cap)
    return A, B


def padded_switch_moves(world: int, rank: int, local_rows: int, L: int, t2g: torch.Tensor,
                        g2t: torch.Tensor) -> tuple[PeerMove, PeerMove]:
    """Plain switches between padded layouts (HybridStack): (TSA -> GSA, GSA -> TSA)."""
    from .compact import compact_plan
    full = compact_plan(torch.ones(local_rows, L, dtype=torch.bool, device=t2g.device))
    plans = [full] * world
    to_gsa, to_tsa = block_switch_moves(world, rank, local_rows, L, t2g, g2t, plans, plans,
                                        padded_gsa=True)
    return to_gsa, to_tsa


class _PeerSwitch(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, mv, arena, log):
        ctx.mv, ctx.arena, ctx.log = mv, arena, log
        if log is not None:
            log.record("peer_pull", x.numel(), "pattern-switch-p2p",
                       mv.remote_rows * x.shape[-1] * x.element_size())
        return arena.move(x.contiguous(), mv.table, mv.stride, mv.out_rows)

    @staticmethod
    def backward(ctx, g):
        mv, log = ctx.mv, ctx.log
        if log is not None:
            log.record("peer_pull", g.numel(), "pattern-switch-p2p",
                       mv.remote_rows_bwd * g.shape[-1] * g.element_size())
        return ctx.arena.move(g.contiguous(), mv.inv, mv.inv_stride, mv.in_rows), None, None, None


def peer_switch(x: torch.Tensor, mv: PeerMove, arena: PeerArena, log=None) -> torch.Tensor:
    """Apply a cross-rank move (autograd: the backward pulls with the inverse table)."""
    return _PeerSwitch.apply(x, mv, arena, log)
