"""Import shim: `import osp` -> this package, for reference-style numpy callers (the reference's
own tests and checks, pkg/src/osp/__init__.py:4-15).  Importing it switches
`SequenceTensor.data` to numpy data mode (host float64 / uint8 copies), and the shim modules
convert the few torch results the reference returns as numpy arrays.  The kernels run on the GPU
exactly as through `paper_2605_28691_b200`; only the host-facing values are converted."""

import paper_2605_28691_b200 as _p
from paper_2605_28691_b200.gridseq import set_data_mode as _set_mode

_set_mode("numpy")

from paper_2605_28691_b200 import *  # noqa: E402,F401,F403
from . import anyres, attention, gridseq, skiparse, ssp  # noqa: E402,F401

__version__ = _p.__version__
