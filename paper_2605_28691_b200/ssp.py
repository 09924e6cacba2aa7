"""Sparse Sequence Parallelism -- drop-in for osp.ssp (ssp.py:45-239) plus the
real multi-GPU switch.

Two front ends share the same K4 pack/unpack kernels:

* the reference's in-process API (`ProcessGroup` of `RankShard`s,
  `shard_pattern_layout`, `all_to_all`, `ssp_pattern_switch`, `gather_shards`),
  where the all-to-all is a device-side chunk transpose and the ledger counts
  elements exactly like the reference;
* `SSPSwitch` / `ssp_switch`: one rank's shard per process, the all-to-all
  being a single NCCL `all_to_all_single` over NVLink (torch.distributed,
  one process per GPU).  It is an autograd op whose backward is the same
  self-inverse switch.

Alg. 1: 1. pack = token-wise split on the reduced grid,
2. one all-to-all, 3.+4. unpack = chunk permutation fused with the token-wise
merge.  Volume per switch = the local shard; Ulysses needs four (q, k, v, out).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import torch

from . import kernels
from .errors import CollectiveError, ProtocolError, ShardingError
from .gridseq import GridShape, SequenceTensor

__all__ = ["CommEvent", "CommLog", "RankShard", "ProcessGroup", "shard_pattern_layout",
           "gather_shards", "all_to_all", "ssp_pattern_switch", "ulysses_block_comm",
           "naive_switch_comm", "comm_comparison", "ssp_switch", "SSPSwitch", "check_switch",
           "ShardingError", "CollectiveError", "ProtocolError"]


@dataclass(frozen=True)
class CommEvent:
    kind: str
    payload_per_rank: int
    label: str = ""
    bytes_per_rank: int = 0


@dataclass
class CommLog:
    """Collective ledger (ssp.py:45-63); additionally records bytes."""

    events: list = field(default_factory=list)
    # device timing of the collectives (CUDA event pairs on the stream each runs on), enabled by
    # the benchmark for its timed region; read with collective_ms() after a synchronize
    timing: bool = False
    timed: list = field(default_factory=list)

    def record(self, kind: str, payload_per_rank: int, label: str = "",
               bytes_per_rank: int = 0) -> None:
        self.events.append(CommEvent(kind, int(payload_per_rank), label, int(bytes_per_rank)))

    def time_start(self, stream=None):
        """Event pair around one collective issued on `stream` (default: the current stream);
        None when timing is off."""
        if not self.timing:
            return None
        import torch
        stream = stream if stream is not None else torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        return (e0, e1, stream)

    def time_end(self, tok, label: str) -> None:
        if tok is not None:
            tok[1].record(tok[2])
            self.timed.append((label, tok[0], tok[1]))

    def collective_ms(self) -> dict:
        """Summed device time of the timed collectives per label (ms)."""
        out: dict = {}
        for label, e0, e1 in self.timed:
            out[label] = out.get(label, 0.0) + e0.elapsed_time(e1)
        return out

    def count(self, kind: str | None = None) -> int:
        return sum(1 for e in self.events if kind is None or e.kind == kind)

    def total_payload(self, kind: str | None = None) -> int:
        return sum(e.payload_per_rank for e in self.events if kind is None or e.kind == kind)

    def total_bytes(self, kind: str | None = None) -> int:
        return sum(e.bytes_per_rank for e in self.events if kind is None or e.kind == kind)


@dataclass(frozen=True)
class RankShard:
    rank: int
    tensor: SequenceTensor


@dataclass(frozen=True)
class ProcessGroup:
    """In-process group of equal-shape rank shards (ssp.py:66-88)."""

    shards: tuple
    log: CommLog

    def __post_init__(self) -> None:
        shapes = {tuple(s.tensor.tensor.shape) for s in self.shards}
        if len(shapes) > 1:
            raise ShardingError(f"ranks hold unequal shapes: {sorted(shapes)}")

    @property
    def size(self) -> int:
        return len(self.shards)

    @property
    def local_elements(self) -> int:
        return self.shards[0].tensor.tensor.numel()


def shard_pattern_layout(x_pattern, group_size: int, log: CommLog | None = None) -> ProcessGroup:
    """Contiguous enlarged-batch blocks: rank r holds rows [r*B/N, (r+1)*B/N)
    (ssp.py:91-106); each row is one whole subsequence."""
    xs = x_pattern if isinstance(x_pattern, SequenceTensor) else SequenceTensor(x_pattern)
    if xs.batch % group_size:
        raise ShardingError(f"batch {xs.batch} not divisible by group size {group_size}")
    per = xs.batch // group_size
    shards = tuple(RankShard(r, xs.with_data(xs.tensor[r * per:(r + 1) * per]))
                   for r in range(group_size))
    return ProcessGroup(shards, log if log is not None else CommLog())


def gather_shards(group: ProcessGroup) -> SequenceTensor:
    """Concatenate shards along the batch axis; verification helper (ssp.py:109-113)."""
    return SequenceTensor(torch.cat([s.tensor.tensor for s in group.shards], dim=0),
                          kind=group.shards[0].tensor.kind)


def all_to_all(send: list, log: CommLog, label: str = "") -> list:
    """In-process transpose collective (ssp.py:116-136): received[r] concatenates
    chunk r of every rank's send buffer.  Logs the whole per-rank buffer."""
    n = len(send)
    shapes = {tuple(b.shape) for b in send}
    if len(shapes) > 1:
        raise CollectiveError(f"ranks send unequal shapes: {sorted(shapes)}")
    lead = send[0].shape[0]
    if lead % n:
        raise CollectiveError(f"leading axis {lead} not divisible into {n} chunks")
    per = lead // n
    recv = [torch.cat([send[j][r * per:(r + 1) * per] for j in range(n)], dim=0)
            for r in range(n)]
    log.record("all_to_all", send[0].numel(), label, send[0].numel() * send[0].element_size())
    return recv


def check_switch(group_size: int, local_batch: int, seq: int, g: GridShape) -> tuple[int, int]:
    """Guards of ssp.py:145-160; returns (G, b)."""
    k2 = g.k * g.k
    if k2 % group_size:
        raise ShardingError(f"k^2={k2} not divisible by group size {group_size}")
    G = k2 // group_size
    if local_batch % G:
        raise ProtocolError(f"local batch {local_batch} not divisible by G={G}")
    L = g.seq_len // k2
    if seq != L:
        raise ProtocolError(f"shard seq {seq} != subsequence length {L}")
    return G, local_batch // G


def ssp_pattern_switch(group: ProcessGroup, g: GridShape) -> ProcessGroup:
    """Switch every rank between token-wise and group-wise layouts with exactly
    one all-to-all (ssp.py:139-180).  Self-inverse."""
    n = group.size
    first = group.shards[0].tensor
    check_switch(n, first.batch, first.seq, g)
    send = [kernels.ssp_pack(s.tensor.tensor, n, g.t, g.h, g.w, g.k) for s in group.shards]
    recv = all_to_all(send, group.log, label="pattern-switch")
    out = tuple(RankShard(r, SequenceTensor(
        kernels.ssp_unpack(buf, n, first.batch, g.t, g.h, g.w, g.k), kind=group.shards[r].tensor.kind))
        for r, buf in enumerate(recv))
    return ProcessGroup(out, group.log)


def ulysses_block_comm(group_size: int, per_rank_elements: int, blocks: int = 1) -> CommLog:
    """Ulysses: four all-to-alls per block (q, k, v, out) (ssp.py:183-191)."""
    log = CommLog()
    for b in range(blocks):
        for name in ("query", "key", "value", "attn_out"):
            log.record("all_to_all", per_rank_elements, f"block{b}:{name}")
    return log


def naive_switch_comm(group_size: int, per_rank_elements: int):
    """Gather-rearrange-reshard baseline (ssp.py:194-205)."""
    n, s = group_size, per_rank_elements
    log = CommLog()
    log.record("all_gather", (n - 1) * s, "gather-rearrange-reshard")
    return log, {"events": 1, "recv_per_rank": (n - 1) * s, "global_traffic": n * (n - 1) * s}


def comm_comparison(group_size: int, per_rank_elements: int, blocks: int = 1,
                    growth_sizes: tuple = (2, 4, 8)) -> dict:
    """SSP vs Ulysses vs naive accounting (ssp.py:208-239)."""
    n, s = group_size, per_rank_elements
    ssp_total, uly_total = blocks * s, 4 * blocks * s
    return {
        "group_size": n, "per_rank_elements": s, "blocks": blocks,
        "ssp_events": blocks, "ulysses_events": 4 * blocks,
        "ssp_total_per_rank": ssp_total, "ulysses_total_per_rank": uly_total,
        "volume_ratio": ssp_total / uly_total,
        "volume_reduction_percent": 100.0 * (1.0 - ssp_total / uly_total),
        "ssp_global_per_switch": (n - 1) * s,
        "naive_global_per_switch": n * (n - 1) * s,
        "naive_over_ssp": n,
        "growth_table": [{"group_size": m, "ssp_global": (m - 1) * s,
                          "naive_global": m * (m - 1) * s, "naive_over_ssp": m}
                         for m in growth_sizes],
    }


# ----------------------------------------------------------------------------- multi-process

def _dist_switch(x: torch.Tensor, g: GridShape, group, log: CommLog | None,
                 transport: str = "native", mode: str = "forward") -> torch.Tensor:
    import torch.distributed as dist
    n = dist.get_world_size(group)
    local_batch, seq, chan = x.shape
    check_switch(n, local_batch, seq, g)
    send = kernels.ssp_pack(x, n, g.t, g.h, g.w, g.k)
    if transport == "hif8":
        # 8-bit transport: per-rank current scaling of the send
        # buffer (hif8.py:223-246), one all-to-all of codes, every rank's scale all-gathered,
        # each received chunk decoded with its source rank's scale.
        from .hif8 import BACKWARD_MAX, DEFAULT_EPS, DEFAULT_SPEC, FORWARD_MAX
        table = DEFAULT_SPEC.device_table(x.device)
        amax = kernels.absmax(send)
        scale = kernels.hif8_scale(amax, FORWARD_MAX if mode == "forward" else BACKWARD_MAX,
                                   DEFAULT_EPS)
        codes = kernels.hif8_encode(send, table, scale, check_finite=False)
        scales = torch.empty(n, dtype=scale.dtype, device=scale.device)
        rcodes = torch.empty_like(codes)
        if n == 1:
            scales.copy_(scale)
            rcodes = codes
        else:
            dist.all_gather_into_tensor(scales, scale, group=group)
            dist.all_to_all_single(rcodes, codes, group=group)
        if log is not None:
            log.record("all_to_all", codes.numel(), "pattern-switch-hif8", codes.numel())
        recv = kernels.hif8_decode(rcodes, table, send.dtype, scales, codes.numel() // n)
    elif transport == "native":
        recv = torch.empty_like(send)
        if n == 1:
            recv = send
        else:
            tok = log.time_start() if log is not None else None
            dist.all_to_all_single(recv, send, group=group)
            if log is not None:
                log.time_end(tok, "pattern-switch-" + mode)
        if log is not None:
            log.record("all_to_all", send.numel(), "pattern-switch", send.numel() * send.element_size())
    else:
        raise ValueError(f"unknown transport {transport!r}")
    return kernels.ssp_unpack(recv, n, local_batch, g.t, g.h, g.w, g.k)


class SSPSwitch(torch.autograd.Function):
    """One rank's TSA<->GSA switch over a torch.distributed group; the backward
    is the same switch (the routine is its own inverse, ssp.py:142-144).  With the
    HiF8 transport the forward uses forward-mode scaling and the backward
    backward-mode scaling (hif8.py:47-52)."""

    @staticmethod
    def forward(ctx, x, g, group, log, transport):
        ctx.g, ctx.group, ctx.log, ctx.transport = g, group, log, transport
        return _dist_switch(x.contiguous(), g, group, log, transport, "forward")

    @staticmethod
    def backward(ctx, gy):
        return (_dist_switch(gy.contiguous(), ctx.g, ctx.group, ctx.log, ctx.transport, "backward"),
                None, None, None, None)


def ssp_switch(x: torch.Tensor, g: GridShape, group=None, log: CommLog | None = None,
               transport: str = "native") -> torch.Tensor:
    """Switch this rank's (G*b, L, C) shard between token-wise and group-wise
    layouts with one NCCL all-to-all (g = padded global grid).  transport="hif8"
    moves 8-bit HiF8 codes instead of the native dtype (half of bf16's bytes)."""
    return SSPSwitch.apply(x, g, group, log, transport)
