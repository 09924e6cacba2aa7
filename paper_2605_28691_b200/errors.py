"""Exception classes of the reference (all ValueError subclasses), shared by
the shim modules and mapped from C-ABI status codes.

Reference: gridseq.py:33-38, skiparse.py:33-38, ssp.py:33-42.
"""


class CoordinateError(ValueError):
    """A (t, h, w) coordinate lies outside its grid."""


class ShapeError(ValueError):
    """Tensor and map shapes do not agree."""


class PatternError(ValueError):
    """The grid does not satisfy the pattern's divisibility requirement."""


class ScheduleError(ValueError):
    """Invalid layer-schedule parameters."""


class ShardingError(ValueError):
    """Shard counts do not divide evenly."""


class CollectiveError(ValueError):
    """Send buffers cannot be chunked equally."""


class ProtocolError(ValueError):
    """Rank shards are inconsistent with the declared grid."""


class UnsupportedError(ValueError):
    """Dtype or head_dim outside what the B200 kernels implement (no fallback)."""


_BY_CODE = {
    1: PatternError,
    2: ShapeError,
    3: CoordinateError,
    4: ShardingError,
    5: CollectiveError,
    6: ProtocolError,
    7: ValueError,
    8: UnsupportedError,
}


def from_status(code: int, message: str) -> Exception:
    cls = _BY_CODE.get(code)
    if cls is None:
        return RuntimeError(f"libosp_skiparse: {message} (status {code})")
    return cls(message)
