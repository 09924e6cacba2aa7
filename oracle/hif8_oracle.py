"""CPU oracle for the HiF8 codec and per-tensor current-scaling quantizer.

TEST INFRASTRUCTURE ONLY (see oracle/osp_oracle.py).  Restates the reference
hif8.py (value table hif8.py:77-134, encode_array 171-186, decode_array
189-193, quantize_tensor 223-246) from its published algorithm: 256 codes in
ascending value order, code 127 remapped to zero, nearest-value encoding with
ties to the even code and saturation, scale = target / (amax + eps) with
target 15 (forward) or 224 (backward).  Pinned to the reference's own outputs
in tests/test_oracle_golden.py.
"""

from __future__ import annotations

import numpy as np

EXP_MIN, EXP_MAX = -22, 15
TARGET = {"forward": 15.0, "backward": 224.0}
EPS = 1e-12


def default_widths() -> dict:
    w = {}
    for e in range(EXP_MIN, EXP_MAX + 1):
        w[e] = 3 if -3 <= e <= 3 else (2 if e in (-5, -4, 4, 5, 6) else 1)
    return w


def value_table(widths=None) -> np.ndarray:
    widths = widths or default_widths()
    mags = np.array([(1.0 + f / (1 << widths[e])) * 2.0 ** e
                     for e in range(EXP_MIN, EXP_MAX + 1) for f in range(1 << widths[e])])
    vals = np.concatenate([-mags[::-1], mags])
    vals[127] = 0.0
    return vals


def encode(x, vals=None) -> np.ndarray:
    """Nearest value; a tie (x exactly at a midpoint) takes the even code; saturating."""
    vals = value_table() if vals is None else vals
    x = np.asarray(x, dtype=np.float64)
    if not np.isfinite(x).all():
        raise ValueError("cannot encode non-finite values")
    mids = (vals[:-1] + vals[1:]) / 2.0          # exact: <= 5 significant bits
    c = np.searchsorted(mids, x, side="left")     # number of midpoints < x
    tie = np.zeros(x.shape, dtype=bool)
    inside = c < mids.size
    tie[inside] = mids[c[inside]] == x[inside]
    code = np.where(tie & (c % 2 == 1), c + 1, c)
    return code.astype(np.uint8)


def decode(codes, vals=None) -> np.ndarray:
    vals = value_table() if vals is None else vals
    return vals[np.asarray(codes).astype(np.int64)]


def quantize(x, mode: str):
    amax = float(np.max(np.abs(x))) if np.asarray(x).size else 0.0
    scale = TARGET[mode] / (amax + EPS)
    return encode(np.asarray(x, dtype=np.float64) * scale), scale, amax
