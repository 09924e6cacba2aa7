"""Torch-tensor wrappers over the C ABI (one function per exported kernel).

Tensors must be CUDA tensors; shapes/strides are checked here, semantics in the
kernels.  These are the only functions that call into libosp_skiparse.so.
"""

from __future__ import annotations

import math

import torch

from . import _lib
from .errors import ShapeError, UnsupportedError

MAP_IDS = {"identity": 0, "orig_to_tsa": 1, "tsa_to_orig": 2, "orig_to_gsa": 3, "gsa_to_orig": 4,
           "tsa_to_gsa": 5, "gsa_to_tsa": 6, "pad": 7, "strip": 8}
PATTERN_IDS = {"original": 0, "tsa": 1, "gsa": 2}


class LaunchStats:
    """Counts this library's kernel launches and optionally brackets each C-ABI
    call with CUDA events on the launching stream (bench.py uses both)."""

    def __init__(self):
        self.launches = 0
        self.timing = False
        self.events: dict = {}

    def reset(self, timing: bool = False):
        self.launches = 0
        self.timing = timing
        self.events = {}

    def run(self, name: str, n_kernels: int, fn):
        if self.timing:
            s = torch.cuda.Event(enable_timing=True)
            e = torch.cuda.Event(enable_timing=True)
            s.record()
            rc = fn()
            e.record()
            self.events.setdefault(name, []).append((s, e))
        else:
            rc = fn()
        self.launches += n_kernels
        return rc

    def elapsed_ms(self) -> dict:
        return {k: [s.elapsed_time(e) for s, e in v] for k, v in self.events.items()}


STATS = LaunchStats()


def _cuda(t: torch.Tensor, name: str) -> torch.Tensor:
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (the B200 path has no CPU fallback)")
    return t


def rearrange(x: torch.Tensor, map_name: str, t: int, h: int, w: int, k: int, batch: int,
              h_orig: int | None = None, w_orig: int | None = None,
              out: torch.Tensor | None = None) -> torch.Tensor:
    """Apply one closed-form map to a (rows, seq, chan)-shaped tensor.  (t,h,w,k)
    is the padded grid; output shape follows the map."""
    L = _lib.lib()
    _cuda(x, "x")
    x = x.contiguous()
    h0 = h if h_orig is None else h_orig
    w0 = w if w_orig is None else w_orig
    chan = x.shape[-1]
    S, S0 = t * h * w, t * h0 * w0
    n_sub = k * k
    if map_name in ("orig_to_tsa", "orig_to_gsa"):
        in_shape, out_shape = (batch, S0), (n_sub * batch, S // n_sub)
    elif map_name in ("tsa_to_orig", "gsa_to_orig"):
        in_shape, out_shape = (n_sub * batch, S // n_sub), (batch, S0)
    elif map_name in ("tsa_to_gsa", "gsa_to_tsa"):
        in_shape = out_shape = (n_sub * batch, S // n_sub)
    elif map_name == "pad":
        in_shape, out_shape = (batch, S0), (batch, S)
    elif map_name == "strip":
        in_shape, out_shape = (batch, S), (batch, S0)
    elif map_name == "identity":
        in_shape = out_shape = (batch, S)
    else:
        raise ValueError(f"unknown map {map_name!r}")
    if x.numel() != in_shape[0] * in_shape[1] * chan:
        raise ShapeError(f"map expects input ({in_shape[0]}, {in_shape[1]}, {chan}), got "
                         f"{tuple(x.shape)}")
    if out is None:
        out = torch.empty((out_shape[0], out_shape[1], chan), dtype=x.dtype, device=x.device)
    _lib.check(STATS.run('rearrange', 1, lambda: L.osp_rearrange(x.data_ptr(), out.data_ptr(), x.element_size(), chan, batch, t, h,
                               w, k, MAP_IDS[map_name], h0, w0, _lib.stream_ptr(x.device))))
    return out


def gather_rows(x: torch.Tensor, index: torch.Tensor, n_out_rows: int) -> torch.Tensor:
    """dst row i = src row index[i] (rows = leading (batch, seq) addresses)."""
    L = _lib.lib()
    _cuda(x, "x")
    x = x.contiguous()
    index = index.to(device=x.device, dtype=torch.int64).contiguous()
    chan = x.shape[-1]
    n_in = x.numel() // max(chan, 1) if chan else 0
    out = torch.empty((n_out_rows, chan), dtype=x.dtype, device=x.device)
    _lib.check(STATS.run('gather_rows', 1, lambda: L.osp_gather_rows(x.data_ptr(), out.data_ptr(), index.data_ptr(), n_out_rows, n_in,
                                 chan * x.element_size(), _lib.stream_ptr(x.device))))
    return out


def gather_chunks(src: torch.Tensor, dst: torch.Tensor, index: torch.Tensor, n_out_rows: int, n_in_rows: int,
                  n_chunks: int, chunk_elems: int, src_row_stride: int, src_chunk_stride: int,
                  dst_row_stride: int, dst_chunk_stride: int) -> torch.Tensor:
    """Raw chunked row gather (element strides from the tensors' data pointers, which may be views):
    for r < n_out_rows, c < n_chunks: dst[c*dcs + r*drs : +chunk] = src[c*scs + index[r]*srs : +chunk]
    (index[r] < 0 -> zeros)."""
    L = _lib.lib()
    _cuda(src, "src")
    _cuda(dst, "dst")
    if src.dtype != dst.dtype:
        raise ShapeError("src and dst dtypes differ")
    es = src.element_size()
    index = index.to(device=src.device, dtype=torch.int64).contiguous()
    _lib.check(STATS.run('gather_rows', 1, lambda: L.osp_gather_rows_chunked(
        src.data_ptr(), dst.data_ptr(), index.data_ptr(), n_out_rows, n_in_rows, n_chunks, chunk_elems * es,
        src_row_stride * es, src_chunk_stride * es, dst_row_stride * es, dst_chunk_stride * es,
        _lib.stream_ptr(src.device))))
    return dst


def gather_rows_chunked(src: torch.Tensor, index: torch.Tensor, n_out_rows: int, n_chunks: int,
                        src_chunked: bool, dst_chunked: bool, out: torch.Tensor | None = None) -> torch.Tensor:
    """Row gather between channel-chunked layouts.  A plain layout is (rows, C); a chunked one is
    (n_chunks, rows, C / n_chunks) (every chunk a contiguous block).  dst row r = src row index[r]
    (-1 = zeros), chunk by chunk; returns dst in the requested layout."""
    _cuda(src, "src")
    src = src.contiguous()
    if src_chunked:
        nc, n_in, cc = src.shape
        C = nc * cc
    else:
        n_in, C = src.reshape(-1, src.shape[-1]).shape
        cc = C // n_chunks
        nc = n_chunks
    if nc != n_chunks or cc * nc != C:
        raise ShapeError(f"channels {C} do not split into {n_chunks} chunks")
    if out is None:
        shape = (nc, n_out_rows, cc) if dst_chunked else (n_out_rows, C)
        out = torch.empty(shape, dtype=src.dtype, device=src.device)
    s_rs, s_cs = (cc, n_in * cc) if src_chunked else (C, cc)
    d_rs, d_cs = (cc, n_out_rows * cc) if dst_chunked else (C, cc)
    return gather_chunks(src, out, index, n_out_rows, n_in, nc, cc, s_rs, s_cs, d_rs, d_cs)


_IOTA: dict = {}


def iota_index(n: int, device) -> torch.Tensor:
    key = (n, str(device))
    if key not in _IOTA:
        _IOTA[key] = torch.arange(n, dtype=torch.int64, device=device)
    return _IOTA[key]


def ulysses_pack_qkv(qkv: torch.Tensor, n: int) -> torch.Tensor:
    """(R, L, 3C) packed [q|k|v], all heads -> (n, R*L, 3C/n) send blocks: block j holds peer j's
    channel slice of q, k and v (three K1 chunked gathers; replaces view/permute/contiguous)."""
    R, L, C3 = qkv.shape
    C = C3 // 3
    Cn = C // n
    rows = R * L
    src = qkv.contiguous()
    out = torch.empty((n, rows, 3 * Cn), dtype=qkv.dtype, device=qkv.device)
    idx = iota_index(rows, qkv.device)
    for t in range(3):     # q, k, v part: src chunk j = columns t*C + j*Cn, dst chunk j = block j, cols t*Cn
        gather_chunks(src.view(-1)[t * C:], out.view(-1)[t * Cn:], idx, rows, rows, n, Cn, C3, Cn,
                      3 * Cn, rows * 3 * Cn)
    return out


def ulysses_unpack_qkv(blocks: torch.Tensor, n: int) -> torch.Tensor:
    """Adjoint of ulysses_pack_qkv: (n, R*L, 3C/n) -> (R*L, 3C)."""
    _, rows, C3n = blocks.shape
    Cn = C3n // 3
    C = n * Cn
    src = blocks.contiguous()
    out = torch.empty((rows, 3 * C), dtype=blocks.dtype, device=blocks.device)
    idx = iota_index(rows, blocks.device)
    for t in range(3):
        gather_chunks(src.view(-1)[t * Cn:], out.view(-1)[t * C:], idx, rows, rows, n, Cn, 3 * Cn, rows * 3 * Cn,
                      3 * C, Cn)
    return out


def _ptr_array(ptrs) -> "ctypes.Array":
    import ctypes
    return (ctypes.c_void_p * len(ptrs))(*[int(p) for p in ptrs])


def peer_gather(src_ptrs, stride_rows: int, table: torch.Tensor, out: torch.Tensor) -> torch.Tensor:
    """K7: out row i = row (table[i] % stride) of source buffer src_ptrs[table[i] // stride]
    (device addresses, local or peer-mapped); table[i] < 0 -> zero row."""
    L = _lib.lib()
    _cuda(out, "out")
    if not out.is_contiguous():
        raise ShapeError("peer_gather output must be contiguous")
    table = table.to(device=out.device, dtype=torch.int64).contiguous()
    n_rows = table.numel()
    row_bytes = out.numel() // max(n_rows, 1) * out.element_size() if n_rows else 0
    if n_rows and out.numel() % n_rows:
        raise ShapeError("output does not split into table rows")
    arr = _ptr_array(src_ptrs)
    _lib.check(STATS.run('peer_gather', 1, lambda: L.osp_peer_gather(
        arr, len(src_ptrs), stride_rows, table.data_ptr(), n_rows, out.data_ptr(), row_bytes,
        _lib.stream_ptr(out.device))))
    return out


def peer_barrier(flag_ptrs, rank: int, epoch: int, device=None, timeout_ms: int = 0,
                 status: torch.Tensor | None = None) -> None:
    """K7: device-side flag barrier over the peers' flag blocks (see include/osp_skiparse.h).
    status: pinned host int32 word the kernel sets to 1 + the missing rank on timeout."""
    L = _lib.lib()
    arr = _ptr_array(flag_ptrs)
    _lib.check(STATS.run('peer_barrier', 1, lambda: L.osp_peer_barrier(
        arr, rank, len(flag_ptrs), epoch & 0xFFFFFFFF, int(timeout_ms), _lib.ptr(status),
        _lib.stream_ptr(device))))


def invert_index(index: torch.Tensor) -> torch.Tensor:
    L = _lib.lib()
    _cuda(index, "index")
    index = index.contiguous().to(torch.int64)
    inv = torch.full_like(index, -1)
    _lib.check(STATS.run('invert_index', 1, lambda: L.osp_invert_index(index.data_ptr(), inv.data_ptr(), index.numel(),
                                  _lib.stream_ptr(index.device))))
    return inv


def pattern_mask_bits(batch: int, t: int, h: int, w: int, k: int, pattern: str, h_orig: int,
                      w_orig: int, device) -> torch.Tensor:
    """(rows, ceil(L/32)) int32 bit words of the 1-D validity mask."""
    L = _lib.lib()
    n_sub = 1 if pattern == "original" else k * k
    Ls = t * h * w // n_sub
    bits = torch.empty((n_sub * batch, (Ls + 31) // 32), dtype=torch.int32, device=device)
    _lib.check(STATS.run('mask_bits', 1, lambda: L.osp_pattern_mask_bits(bits.data_ptr(), batch, t, h, w, k, PATTERN_IDS[pattern],
                                       h_orig, w_orig, _lib.stream_ptr(device))))
    return bits


def bytes_to_bits(valid: torch.Tensor) -> torch.Tensor:
    L = _lib.lib()
    _cuda(valid, "valid")
    v = valid.to(torch.uint8).contiguous()
    rows, n = v.shape
    bits = torch.empty((rows, (n + 31) // 32), dtype=torch.int32, device=v.device)
    _lib.check(STATS.run('mask_bits', 1, lambda: L.osp_mask_bytes_to_bits(v.data_ptr(), bits.data_ptr(), rows, n,
                                        _lib.stream_ptr(v.device))))
    return bits


def bits_to_bytes(bits: torch.Tensor, n: int) -> torch.Tensor:
    L = _lib.lib()
    rows = bits.shape[0]
    out = torch.empty((rows, n), dtype=torch.uint8, device=bits.device)
    _lib.check(STATS.run('mask_bits', 1, lambda: L.osp_mask_bits_to_bytes(bits.data_ptr(), out.data_ptr(), rows, n,
                                        _lib.stream_ptr(bits.device))))
    return out.bool()


def _head_dim_plan(d: int) -> int:
    if d in (64, 128):
        return d
    if 0 < d < 64:
        return 64
    if 64 < d < 128:
        return 128
    raise UnsupportedError(f"head_dim {d} > 128 is not supported by the B200 attention kernels")


def _lens(seq_lens, n_seq, seq_len):
    if seq_lens is None:
        return None
    _cuda(seq_lens, "seq_lens")
    if seq_lens.dtype != torch.int32 or seq_lens.numel() != n_seq:
        raise ShapeError(f"seq_lens must be ({n_seq},) int32")
    return seq_lens.contiguous()


def attn_fwd(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, heads: int, head_dim: int,
             valid_bits: torch.Tensor | None, zero_invalid_queries: bool, scale: float,
             out: torch.Tensor | None = None, seq_lens: torch.Tensor | None = None):
    """q, k, v: (n_seq, L, >= heads*head_dim) bf16 views with unit column stride.
    Returns (o (n_seq, L, heads*head_dim) bf16, lse (n_seq, heads, L) fp32).  seq_lens
    (n_seq,) int32: per-sequence lengths <= L (rows beyond are ignored and not written)."""
    L = _lib.lib()
    for name, t in (("q", q), ("k", k), ("v", v)):
        _cuda(t, name)
        if t.dtype != torch.bfloat16:
            raise UnsupportedError(f"{name} must be bfloat16, got {t.dtype}")
        if t.stride(-1) != 1 or t.stride(0) != t.shape[1] * t.stride(1):
            raise ShapeError(f"{name} needs unit column stride and dense rows")
    n_seq, seq_len = q.shape[0], q.shape[1]
    if out is None:
        out = torch.empty((n_seq, seq_len, heads * head_dim), dtype=torch.bfloat16, device=q.device)
    lse = torch.empty((n_seq, heads, seq_len), dtype=torch.float32, device=q.device)
    lens = _lens(seq_lens, n_seq, seq_len)
    _lib.check(STATS.run('attn_fwd', 1, lambda: L.osp_attn_fwd(q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(),
                              lse.data_ptr(), n_seq, seq_len, heads, head_dim, q.stride(1),
                              k.stride(1), v.stride(1), out.stride(1), _lib.ptr(valid_bits),
                              _lib.ptr(lens), int(zero_invalid_queries), float(scale),
                              _lib.stream_ptr(q.device))))
    return out, lse


def attn_bwd(q, k, v, o, do, lse, heads: int, head_dim: int, valid_bits, zero_invalid_queries: bool,
             scale: float, dq=None, dk=None, dv=None, seq_lens=None):
    L = _lib.lib()
    n_seq, seq_len = q.shape[0], q.shape[1]
    C = heads * head_dim
    dev = q.device
    if do.stride(-1) != 1 or do.stride(0) != do.shape[1] * do.stride(1):
        do = do.contiguous()
    if dq is None:
        dq = torch.empty((n_seq, seq_len, C), dtype=torch.bfloat16, device=dev)
    if dk is None:
        dk = torch.empty((n_seq, seq_len, C), dtype=torch.bfloat16, device=dev)
    if dv is None:
        dv = torch.empty((n_seq, seq_len, C), dtype=torch.bfloat16, device=dev)
    ws_bytes = L.osp_attn_bwd_workspace_bytes(n_seq, seq_len, heads, head_dim)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    lens = _lens(seq_lens, n_seq, seq_len)
    _lib.check(STATS.run('attn_bwd', 3, lambda: L.osp_attn_bwd(q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(), do.data_ptr(),
                              lse.data_ptr(), dq.data_ptr(), dk.data_ptr(), dv.data_ptr(), n_seq,
                              seq_len, heads, head_dim, q.stride(1), k.stride(1), v.stride(1),
                              o.stride(1), do.stride(1), dq.stride(1), dk.stride(1), dv.stride(1),
                              _lib.ptr(valid_bits), _lib.ptr(lens), int(zero_invalid_queries),
                              float(scale), ws.data_ptr(), ws_bytes, _lib.stream_ptr(dev))))
    return dq, dk, dv


def attn_fwd_gather(q, k, v, heads: int, head_dim: int, row_index: torch.Tensor,
                    seq_lens: torch.Tensor, scale: float, out: torch.Tensor | None = None):
    """Gather-mode attention: q, k, v (n_rows, >= C) in any token layout; subsequence s is rows
    row_index[s, :seq_lens[s]] ((n_seq, capacity) int32, -1 padded).  Returns (o (n_rows, C)
    with only the indexed rows written, lse (n_seq, heads, capacity))."""
    L = _lib.lib()
    for name, t in (("q", q), ("k", k), ("v", v)):
        _cuda(t, name)
        if t.dtype != torch.bfloat16 or t.stride(-1) != 1:
            raise UnsupportedError(f"{name} must be bf16 with unit column stride")
    n_rows = q.shape[0]
    n_seq, cap = row_index.shape
    if out is None:
        out = torch.empty((n_rows, heads * head_dim), dtype=torch.bfloat16, device=q.device)
    lse = torch.empty((n_seq, heads, cap), dtype=torch.float32, device=q.device)
    ri = row_index.to(torch.int32).contiguous()
    sl = _lens(seq_lens, n_seq, cap)
    _lib.check(STATS.run('attn_fwd', 1, lambda: L.osp_attn_fwd_gather(
        q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(), lse.data_ptr(), n_rows, ri.data_ptr(),
        sl.data_ptr(), n_seq, cap, heads, head_dim, q.stride(0), k.stride(0), v.stride(0), out.stride(0),
        float(scale), _lib.stream_ptr(q.device))))
    return out, lse


def attn_bwd_gather(q, k, v, o, do, lse, heads: int, head_dim: int, row_index, seq_lens, scale: float,
                    dq=None, dk=None, dv=None):
    L = _lib.lib()
    n_rows = q.shape[0]
    n_seq, cap = row_index.shape
    C = heads * head_dim
    dev = q.device
    if do.stride(-1) != 1:
        do = do.contiguous()
    dq = dq if dq is not None else torch.empty((n_rows, C), dtype=torch.bfloat16, device=dev)
    dk = dk if dk is not None else torch.empty((n_rows, C), dtype=torch.bfloat16, device=dev)
    dv = dv if dv is not None else torch.empty((n_rows, C), dtype=torch.bfloat16, device=dev)
    ws_bytes = L.osp_attn_bwd_workspace_bytes(n_seq, cap, heads, head_dim)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    ri = row_index.to(torch.int32).contiguous()
    sl = _lens(seq_lens, n_seq, cap)
    _lib.check(STATS.run('attn_bwd', 3, lambda: L.osp_attn_bwd_gather(
        q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(), do.data_ptr(), lse.data_ptr(),
        dq.data_ptr(), dk.data_ptr(), dv.data_ptr(), n_rows, ri.data_ptr(), sl.data_ptr(), n_seq, cap,
        heads, head_dim, q.stride(0), k.stride(0), v.stride(0), o.stride(0), do.stride(0), dq.stride(0),
        dk.stride(0), dv.stride(0), float(scale), ws.data_ptr(), ws_bytes, _lib.stream_ptr(dev))))
    return dq, dk, dv


def attn_fwd_scatter(q, k, v, heads: int, head_dim: int, seq_lens: torch.Tensor, out_index: torch.Tensor,
                     out: torch.Tensor, zero_rows: torch.Tensor | None, scale: float):
    """Scatter-mode attention: q, k, v (n_seq, cap, >= C) contiguous per-sequence rows as in
    attn_fwd; output row j of sequence s is stored to row out_index[s, j] of `out` (n_out_rows, C)
    (-1 = not stored) and the rows listed in zero_rows are zero-filled.  Returns lse
    (n_seq, heads, cap)."""
    L = _lib.lib()
    for name, t in (("q", q), ("k", k), ("v", v)):
        _cuda(t, name)
        if t.dtype != torch.bfloat16:
            raise UnsupportedError(f"{name} must be bfloat16, got {t.dtype}")
        if t.stride(-1) != 1 or t.stride(0) != t.shape[1] * t.stride(1):
            raise ShapeError(f"{name} needs unit column stride and dense rows")
    n_seq, cap = q.shape[0], q.shape[1]
    if tuple(out_index.shape) != (n_seq, cap) or out_index.dtype != torch.int32:
        raise ShapeError(f"out_index must be ({n_seq}, {cap}) int32")
    if out.dim() != 2 or out.stride(1) != 1:
        raise ShapeError("out must be a (rows, C) tensor with unit column stride")
    lse = torch.empty((n_seq, heads, cap), dtype=torch.float32, device=q.device)
    lens = _lens(seq_lens, n_seq, cap)
    nz = 0 if zero_rows is None else zero_rows.numel()
    _lib.check(STATS.run('attn_fwd', 1, lambda: L.osp_attn_fwd_scatter(
        q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(), lse.data_ptr(), n_seq, cap, heads,
        head_dim, q.stride(1), k.stride(1), v.stride(1), out.stride(0), lens.data_ptr(),
        out_index.data_ptr(), out.shape[0], _lib.ptr(zero_rows) if nz else 0, nz, float(scale),
        _lib.stream_ptr(q.device))))
    return lse


def attn_bwd_scatter(q, k, v, out, dout, lse, heads: int, head_dim: int, seq_lens, out_index,
                     scale: float, dq, dk, dv):
    """Backward of attn_fwd_scatter: out / dout are the scattered (n_out_rows, C) output and its
    gradient (read through out_index); dq, dk, dv are contiguous (n_seq, cap, C) views."""
    L = _lib.lib()
    n_seq, cap = q.shape[0], q.shape[1]
    dev = q.device
    if dout.stride(-1) != 1:
        dout = dout.contiguous()
    ws_bytes = L.osp_attn_bwd_scatter_workspace_bytes(n_seq, cap, heads, head_dim)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    lens = _lens(seq_lens, n_seq, cap)
    _lib.check(STATS.run('attn_bwd', 3, lambda: L.osp_attn_bwd_scatter(
        q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(), dout.data_ptr(), lse.data_ptr(),
        dq.data_ptr(), dk.data_ptr(), dv.data_ptr(), n_seq, cap, heads, head_dim, q.stride(1),
        k.stride(1), v.stride(1), out.stride(0), dout.stride(0), dq.stride(1), dk.stride(1),
        dv.stride(1), lens.data_ptr(), out_index.data_ptr(), out.shape[0], float(scale), ws.data_ptr(),
        ws_bytes, _lib.stream_ptr(dev))))
    return dq, dk, dv


def ssp_pack(x: torch.Tensor, group_size: int, t: int, h: int, w: int, k: int) -> torch.Tensor:
    L = _lib.lib()
    _cuda(x, "x")
    x = x.contiguous()
    local_batch, seq, chan = x.shape
    out = torch.empty((k * k * local_batch, seq // (k * k), chan), dtype=x.dtype, device=x.device)
    _lib.check(STATS.run('ssp_pack', 1, lambda: L.osp_ssp_pack(x.data_ptr(), out.data_ptr(), x.element_size(), chan, group_size,
                              local_batch, t, h, w, k, _lib.stream_ptr(x.device))))
    return out


def ssp_unpack(recv: torch.Tensor, group_size: int, local_batch: int, t: int, h: int, w: int,
               k: int, out: torch.Tensor | None = None) -> torch.Tensor:
    L = _lib.lib()
    _cuda(recv, "recv")
    recv = recv.contiguous()
    chan = recv.shape[-1]
    seq = t * h * w // (k * k)
    if out is None:
        out = torch.empty((local_batch, seq, chan), dtype=recv.dtype, device=recv.device)
    _lib.check(STATS.run('ssp_unpack', 1, lambda: L.osp_ssp_unpack(recv.data_ptr(), out.data_ptr(), recv.element_size(), chan,
                                group_size, local_batch, t, h, w, k, _lib.stream_ptr(recv.device))))
    return out


def debug_mma(a: torch.Tensor, b: torch.Tensor, v: torch.Tensor):
    L = _lib.lib()
    d = a.shape[1]
    s = torch.empty((128, 128), dtype=torch.float32, device=a.device)
    o = torch.empty((128, d), dtype=torch.float32, device=a.device)
    _lib.check(L.osp_debug_mma(a.data_ptr(), b.data_ptr(), v.data_ptr(), s.data_ptr(), o.data_ptr(),
                               d, _lib.stream_ptr(a.device)))
    return s, o


def softmax_scale(d: int) -> float:
    return 1.0 / math.sqrt(d)


# ----------------------------------------------------------------------------- HiF8
DTYPE_IDS = {torch.bfloat16: 0, torch.float32: 1, torch.float64: 2}


def absmax(x: torch.Tensor) -> torch.Tensor:
    """max |x| as a 1-element float64 device tensor (no host sync)."""
    L = _lib.lib()
    _cuda(x, "x")
    x = x.contiguous()
    out = torch.empty(1, dtype=torch.float64, device=x.device)
    _lib.check(STATS.run("hif8", 1, lambda: L.osp_absmax(x.data_ptr(), DTYPE_IDS[x.dtype], x.numel(),
                                                          out.data_ptr(), _lib.stream_ptr(x.device))))
    return out


def hif8_scale(amax: torch.Tensor, target: float, eps: float) -> torch.Tensor:
    L = _lib.lib()
    scale = torch.empty_like(amax)
    _lib.check(STATS.run("hif8", 1, lambda: L.osp_hif8_scale(amax.data_ptr(), amax.numel(), target, eps,
                                                              scale.data_ptr(), _lib.stream_ptr(amax.device))))
    return scale


def hif8_encode(x: torch.Tensor, table: torch.Tensor, scale: torch.Tensor | None = None,
                scale_group: int = 0, check_finite: bool = True) -> torch.Tensor:
    L = _lib.lib()
    _cuda(x, "x")
    x = x.contiguous()
    if x.dtype not in DTYPE_IDS:
        raise UnsupportedError(f"hif8 encode supports bf16/fp32/fp64, got {x.dtype}")
    codes = torch.empty(x.shape, dtype=torch.uint8, device=x.device)
    flag = torch.zeros(1, dtype=torch.int32, device=x.device) if check_finite else None
    _lib.check(STATS.run("hif8", 1, lambda: L.osp_hif8_encode(
        x.data_ptr(), DTYPE_IDS[x.dtype], x.numel(), _lib.ptr(scale), scale_group, table.data_ptr(),
        codes.data_ptr(), _lib.ptr(flag), _lib.stream_ptr(x.device))))
    if check_finite and int(flag.item()):
        from .hif8 import EncodeError
        raise EncodeError("cannot encode non-finite values")
    return codes


def hif8_decode(codes: torch.Tensor, table: torch.Tensor, dtype=torch.float64,
                scale: torch.Tensor | None = None, scale_group: int = 0) -> torch.Tensor:
    L = _lib.lib()
    _cuda(codes, "codes")
    codes = codes.contiguous()
    out = torch.empty(codes.shape, dtype=dtype, device=codes.device)
    _lib.check(STATS.run("hif8", 1, lambda: L.osp_hif8_decode(
        codes.data_ptr(), codes.numel(), _lib.ptr(scale), scale_group, table.data_ptr(), out.data_ptr(),
        DTYPE_IDS[dtype], _lib.stream_ptr(codes.device))))
    return out


def qk_norm_rope_bwd(g: torch.Tensor, y: torch.Tensor | None, norm: int, gamma_q, gamma_k, eps: float,
                     rope_tab, grid, pattern: int, batch: int, row_offset: int = 0) -> torch.Tensor:
    """Backward of K6's q/k epilogue, in place on g (rows, >= 2C) bf16: transpose RoPE rotation,
    then the RMSNorm backward against the pre-norm output y (rows, >= 2C) bf16."""
    L = _lib.lib()
    _cuda(g, "g")
    if g.dtype != torch.bfloat16 or (y is not None and y.dtype != torch.bfloat16):
        raise UnsupportedError("qk_norm_rope_bwd runs bf16 g and y")
    rows, W3 = g.shape
    C = W3 // 3
    gq = None if gamma_q is None else gamma_q.to(device=g.device, dtype=torch.float32).contiguous()
    gk = None if gamma_k is None else gamma_k.to(device=g.device, dtype=torch.float32).contiguous()
    _lib.check(STATS.run("qk_norm_rope_bwd", 1, lambda: L.osp_qk_norm_rope_bwd(
        g.data_ptr(), g.stride(0), _lib.ptr(y), y.stride(0) if y is not None else 0, rows, C, norm,
        _lib.ptr(gq), _lib.ptr(gk), float(eps), _lib.ptr(rope_tab), grid.t, grid.h, grid.w, grid.k,
        pattern, batch, row_offset, _lib.stream_ptr(g.device))))
    return g


def qkv_project(x: torch.Tensor, w_t: torch.Tensor, norm: int, gamma_q, gamma_k, eps: float,
                rope_tab, grid, pattern: int, batch: int, row_offset: int = 0) -> torch.Tensor:
    """K6: (rows, C) bf16 @ w_t^T (w_t (3C, C) bf16) with the q/k norm + RoPE epilogue."""
    L = _lib.lib()
    _cuda(x, "x")
    _cuda(w_t, "w_t")
    if x.dtype != torch.bfloat16 or w_t.dtype != torch.bfloat16:
        raise UnsupportedError("qkv_project runs bf16 x and weights")
    rows, C = x.shape
    if tuple(w_t.shape) != (3 * C, C):
        raise ShapeError(f"w_t must be (3C, C) = ({3 * C}, {C}), got {tuple(w_t.shape)}")
    out = torch.empty((rows, 3 * C), dtype=torch.bfloat16, device=x.device)
    gq = None if gamma_q is None else gamma_q.to(device=x.device, dtype=torch.float32).contiguous()
    gk = None if gamma_k is None else gamma_k.to(device=x.device, dtype=torch.float32).contiguous()
    ws = torch.empty((rows, 2), dtype=torch.float32, device=x.device) if norm == 2 else None
    _lib.check(STATS.run("qkv_project", 2 if norm == 2 else 1, lambda: L.osp_qkv_project(
        x.data_ptr(), w_t.data_ptr(), out.data_ptr(), rows, C, 3 * C, norm, _lib.ptr(gq), _lib.ptr(gk),
        float(eps), _lib.ptr(ws), _lib.ptr(rope_tab), grid.t, grid.h, grid.w, grid.k, pattern, batch,
        row_offset, _lib.stream_ptr(x.device))))
    return out
