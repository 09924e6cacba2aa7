"""ctypes binding of libosp_skiparse.so (C ABI in include/osp_skiparse.h).

There is no fallback: if the library or a CUDA device is missing, every
operator raises.  Status codes map 1:1 to the reference's exception classes.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

from . import errors

_PATH = Path(os.environ["OSP_LIB"]) if os.environ.get("OSP_LIB") else \
    Path(__file__).resolve().with_name("libosp_skiparse.so")
_LIB = None

c_i64 = ctypes.c_int64
c_int = ctypes.c_int
c_vp = ctypes.c_void_p
c_f = ctypes.c_float

_SIGS = {
    "osp_last_error": ([], ctypes.c_char_p),
    "osp_abi_version": ([], c_int),
    "osp_device_check": ([], c_int),
    "osp_rearrange": ([c_vp, c_vp, c_i64, c_i64, c_i64, c_i64, c_i64, c_i64, c_i64, c_int, c_i64,
                       c_i64, c_vp], c_int),
    "osp_gather_rows": ([c_vp, c_vp, c_vp, c_i64, c_i64, c_i64, c_vp], c_int),
    "osp_gather_rows_chunked": ([c_vp, c_vp, c_vp, c_i64, c_i64, c_i64, c_i64, c_i64, c_i64, c_i64, c_i64,
                                 c_vp], c_int),
    "osp_invert_index": ([c_vp, c_vp, c_i64, c_vp], c_int),
    "osp_pattern_mask_bits": ([c_vp, c_i64, c_i64, c_i64, c_i64, c_i64, c_int, c_i64, c_i64, c_vp],
                              c_int),
    "osp_mask_bytes_to_bits": ([c_vp, c_vp, c_i64, c_i64, c_vp], c_int),
    "osp_mask_bits_to_bytes": ([c_vp, c_vp, c_i64, c_i64, c_vp], c_int),
    "osp_attn_fwd": ([c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_i64, c_i64, c_i64, c_i64, c_i64,
                      c_i64, c_vp, c_vp, c_int, c_f, c_vp], c_int),
    "osp_attn_bwd_workspace_bytes": ([c_i64, c_i64, c_i64, c_i64], ctypes.c_size_t),
    "osp_attn_bwd": ([c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_i64,
                      c_i64, c_i64, c_i64, c_i64, c_i64, c_i64, c_i64, c_i64, c_i64, c_vp, c_vp,
                      c_int, c_f, c_vp, ctypes.c_size_t, c_vp], c_int),
    "osp_attn_fwd_gather": ([c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, c_i64, c_i64, c_i64,
                             c_i64, c_i64, c_i64, c_i64, c_i64, c_f, c_vp], c_int),
    "osp_attn_bwd_gather": ([c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_vp, c_vp,
                             c_i64, c_i64, c_i64, c_i64, c_i64, c_i64, c_i64, c_i64, c_i64, c_i64,
                             c_i64, c_i64, c_f, c_vp, ctypes.c_size_t, c_vp], c_int),
    "osp_attn_fwd_scatter": ([c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_i64, c_i64, c_i64, c_i64,
                              c_i64, c_i64, c_vp, c_vp, c_i64, c_vp, c_i64, c_f, c_vp], c_int),
    "osp_attn_bwd_scatter_workspace_bytes": ([c_i64, c_i64, c_i64, c_i64], ctypes.c_size_t),
    "osp_attn_bwd_scatter": ([c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_i64,
                              c_i64, c_i64, c_i64, c_i64, c_i64, c_i64, c_i64, c_i64, c_i64, c_vp, c_vp,
                              c_i64, c_f, c_vp, ctypes.c_size_t, c_vp], c_int),
    "osp_ssp_pack": ([c_vp, c_vp, c_i64, c_i64, c_i64, c_i64, c_i64, c_i64, c_i64, c_i64, c_vp],
                     c_int),
    "osp_ssp_unpack": ([c_vp, c_vp, c_i64, c_i64, c_i64, c_i64, c_i64, c_i64, c_i64, c_i64, c_vp],
                       c_int),
    "osp_qkv_project": ([c_vp, c_vp, c_vp, c_i64, c_i64, c_i64, c_int, c_vp, c_vp, c_f, c_vp, c_vp,
                         c_i64, c_i64, c_i64, c_i64, c_int, c_i64, c_i64, c_vp], c_int),
    "osp_qk_norm_rope_bwd": ([c_vp, c_i64, c_vp, c_i64, c_i64, c_i64, c_int, c_vp, c_vp, c_f, c_vp,
                              c_i64, c_i64, c_i64, c_i64, c_int, c_i64, c_i64, c_vp], c_int),
    "osp_absmax": ([c_vp, c_int, c_i64, c_vp, c_vp], c_int),
    "osp_hif8_scale": ([c_vp, c_i64, ctypes.c_double, ctypes.c_double, c_vp, c_vp], c_int),
    "osp_hif8_encode": ([c_vp, c_int, c_i64, c_vp, c_i64, c_vp, c_vp, c_vp, c_vp], c_int),
    "osp_hif8_decode": ([c_vp, c_i64, c_vp, c_i64, c_vp, c_vp, c_int, c_vp], c_int),
    "osp_peer_alloc": ([c_i64, c_vp], c_int),
    "osp_peer_free": ([c_vp], c_int),
    "osp_peer_export": ([c_vp, c_vp], c_int),
    "osp_peer_import": ([c_vp, c_vp], c_int),
    "osp_peer_close": ([c_vp], c_int),
    "osp_peer_barrier": ([c_vp, c_int, c_int, ctypes.c_uint32, c_i64, c_vp, c_vp], c_int),
    "osp_peer_gather": ([c_vp, c_int, c_i64, c_vp, c_i64, c_vp, c_i64, c_vp], c_int),
    "osp_debug_counters": ([c_vp, c_int, c_int], c_int),
    "osp_debug_counters_bwd": ([c_vp, c_int, c_int], c_int),
    "osp_debug_mma": ([c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_vp], c_int),
}

EXPORTS = tuple(_SIGS)


def load_library(path: str | os.PathLike | None = None) -> ctypes.CDLL:
    """Load the shared library and declare every exported signature.  Works
    without a GPU (no CUDA call is made at load time)."""
    p = Path(path) if path else _PATH
    if not p.exists():
        raise RuntimeError(
            f"{p} is missing; build it with `python -m paper_2605_28691_b200.build` "
            "(no CPU fallback exists)")
    lib_ = ctypes.CDLL(str(p))
    for name, (args, res) in _SIGS.items():
        fn = getattr(lib_, name)
        fn.argtypes = args
        fn.restype = res
    return lib_


_CHECKED = False


def lib() -> ctypes.CDLL:
    global _LIB, _CHECKED
    if _LIB is None:
        _LIB = load_library()
    if not _CHECKED:
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2605_28691_b200 needs a CUDA B200 device; none is visible")
        torch.cuda.init()
        rc = _LIB.osp_device_check()
        if rc != 0:
            raise errors.from_status(rc, _LIB.osp_last_error().decode())
        _CHECKED = True
    return _LIB


def check(rc: int) -> None:
    if rc != 0:
        raise errors.from_status(rc, _LIB.osp_last_error().decode())


def stream_ptr(device=None) -> int:
    import torch
    return torch.cuda.current_stream(device).cuda_stream


def ptr(t) -> int:
    return t.data_ptr() if t is not None else 0
