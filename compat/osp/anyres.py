"""osp.anyres -> paper_2605_28691_b200.anyres (numpy data mode, see osp/__init__.py)."""
from paper_2605_28691_b200 import anyres as _m

from ._conv import export as _export

_export(_m, globals())
from paper_2605_28691_b200 import formats as _f  # noqa: E402

_export(_f, globals(), {"read_mask", "write_mask"})
