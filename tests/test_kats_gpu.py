"""The reference tests' known-answer values for the device-side API: the maps and
masks computed by the kernels."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def test_rearrange_map_simple_transpose(lib):
    # test_gridseq.py:115-120: splitting seq (2, 3) and swapping the factors is a transpose
    from paper_2605_28691_b200.gridseq import SequenceTensor, rearrange_map
    m = rearrange_map([("b", 1)], [("x", 2), ("y", 3)], ["b"], ["y", "x"])
    x = SequenceTensor(torch.arange(6, dtype=torch.float64, device="cuda").reshape(1, 6, 1))
    assert m.apply(x).data[0, :, 0].tolist() == [0, 3, 1, 4, 2, 5]


def test_tsa_on_2x2_grid_gives_singleton_subsequences(lib):
    # test_skiparse.py:50-57
    from paper_2605_28691_b200 import GridShape
    from paper_2605_28691_b200.gridseq import random_tensor
    from paper_2605_28691_b200.skiparse import orig_to_tsa
    x = random_tensor(1, 4, 1, seed=0)
    out = orig_to_tsa(GridShape(1, 2, 2, 2)).apply(x)
    assert (out.batch, out.seq) == (4, 1)
    assert torch.equal(out.data[:, 0, 0], x.data[0, :, 0])


def test_tsa_gsa_frozen_subsequences(lib):
    # test_skiparse.py:39-47: TSA subsequence 0 of a 4x4 grid is {0,2,8,10}; GSA subsequence 0 is
    # {0,1,4,5} and subsequence 3 is {10,11,14,15}
    from paper_2605_28691_b200 import GridShape
    from paper_2605_28691_b200.skiparse import assignment_of, SparsePattern
    g = GridShape(1, 4, 4, 2)
    sub = assignment_of(g, SparsePattern.TOKEN_WISE).subseq.cpu().numpy()
    assert sorted(np.flatnonzero(sub == 0)) == [0, 2, 8, 10]
    sub = assignment_of(g, SparsePattern.GROUP_WISE).subseq.cpu().numpy()
    assert sorted(np.flatnonzero(sub == 0)) == [0, 1, 4, 5]
    assert sorted(np.flatnonzero(sub == 3)) == [10, 11, 14, 15]


def test_pad_and_subsequence_mask_counts(lib):
    # test_anyres.py:18-29, 74-81
    from paper_2605_28691_b200 import GridShape, SparsePattern
    from paper_2605_28691_b200.anyres import pad_grid, subsequence_mask
    pg = pad_grid(GridShape(1, 5, 6, 2))
    assert int(pg.mask.sum()) == 30 and pg.mask.numel() == 64
    for pat in (SparsePattern.TOKEN_WISE, SparsePattern.GROUP_WISE):
        sm = subsequence_mask(pg, pat)
        assert tuple(sm.shape) == (4, 16) and int(sm.sum()) == 30
    pg = pad_grid(GridShape(2, 45, 80, 2))
    assert int(pg.mask.sum()) == 2 * 45 * 80
    assert pad_grid(GridShape(1, 8, 8, 2)).mask_or_none() is None
