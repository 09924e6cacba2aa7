"""osp.ssp -> paper_2605_28691_b200.ssp (numpy data mode, see osp/__init__.py)."""
from paper_2605_28691_b200 import ssp as _m

from ._conv import export as _export

_export(_m, globals())


def all_to_all(send, log, label=""):  # noqa: F811
    """The reference's in-process transpose over numpy (or torch) per-rank buffers."""
    import numpy as np
    import torch

    from paper_2605_28691_b200.gridseq import default_device
    dev = default_device()
    t = [b if isinstance(b, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(b)).to(dev) for b in send]
    out = _m.all_to_all(t, log, label)
    return [o.cpu().numpy() for o in out]
