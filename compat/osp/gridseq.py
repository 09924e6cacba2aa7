"""osp.gridseq -> paper_2605_28691_b200.gridseq (numpy data mode, see osp/__init__.py)."""
from paper_2605_28691_b200 import gridseq as _m

from ._conv import export as _export

_export(_m, globals())
from paper_2605_28691_b200 import formats as _f  # noqa: E402
from paper_2605_28691_b200.errors import CoordinateError, ShapeError  # noqa: E402,F401

_export(_f, globals(), {"OSPT_MAGIC", "read_ospt", "write_ospt"})
