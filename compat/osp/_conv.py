"""Host-facing conversions of the `osp` shim (compatibility / test infrastructure): torch results
become numpy, and the package's PaddedGrid / PatternAssignment are presented through a proxy whose
tensor attributes read as numpy; arguments are unwrapped before the package sees them."""
import numpy as np
import torch

from paper_2605_28691_b200.anyres import PaddedGrid
from paper_2605_28691_b200.skiparse import PatternAssignment

_PROXIED = (PaddedGrid, PatternAssignment)


class Proxy:
    __slots__ = ("_obj",)

    def __init__(self, obj):
        object.__setattr__(self, "_obj", obj)

    def __getattr__(self, name):
        v = getattr(self._obj, name)
        return wrap(v) if callable(v) else to_np(v)

    def __eq__(self, other):
        return self._obj == unwrap(other)

    def __hash__(self):
        return hash(self._obj)

    def __repr__(self):
        return repr(self._obj)


def to_np(x):
    if isinstance(x, torch.Tensor):
        t = x.detach()
        if t.is_floating_point() and t.dtype != torch.float64:
            t = t.to(torch.float64)
        return t.cpu().numpy()
    if isinstance(x, _PROXIED):
        return Proxy(x)
    if isinstance(x, tuple):
        return tuple(to_np(v) for v in x)
    if isinstance(x, list):
        return [to_np(v) for v in x]
    return x


def unwrap(x):
    if isinstance(x, Proxy):
        return x._obj
    if isinstance(x, tuple):
        return tuple(unwrap(v) for v in x)
    if isinstance(x, list):
        return [unwrap(v) for v in x]
    return x


def wrap(fn):
    def f(*a, **k):
        return to_np(fn(*unwrap(a), **{n: unwrap(v) for n, v in k.items()}))
    f.__name__ = getattr(fn, "__name__", "f")
    f.__doc__ = getattr(fn, "__doc__", None)
    return f


def export(module, namespace, names=None):
    """Copy `module`'s public names into `namespace`, wrapping its plain functions."""
    import inspect
    for k, v in vars(module).items():
        if k.startswith("_") or (names is not None and k not in names):
            continue
        namespace[k] = wrap(v) if inspect.isfunction(v) else v
