"""osp.skiparse -> paper_2605_28691_b200.skiparse (numpy data mode, see osp/__init__.py)."""
from paper_2605_28691_b200 import skiparse as _m

from ._conv import export as _export

_export(_m, globals())
