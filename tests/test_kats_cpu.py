"""The reference tests' known-answer values, restated against the oracle and the
product's host-side API (the parts that run without a GPU).  GPU-side KATs (maps, masks) are in
test_kats_gpu.py."""

import numpy as np
import pytest
import torch

from oracle import osp_oracle as O


def test_tsa_on_2x2_grid_gives_singletons_oracle():
    # test_skiparse.py:50-57: a 2x2 grid at k=2 -> four singleton subsequences in (p, q) order
    g = O.Grid(1, 2, 2, 2)
    x = np.arange(4, dtype=np.float64).reshape(1, 4, 1)
    out = O.apply_table(O.map_table("orig_to_tsa", g, 1), x)
    assert out.shape == (4, 1, 1)
    assert np.array_equal(out[:, 0, 0], x[0, :, 0])


def test_pad_grid_kats():
    # test_anyres.py:18-29
    from paper_2605_28691_b200 import GridShape
    from paper_2605_28691_b200.anyres import pad_grid
    p = pad_grid(GridShape(1, 5, 6, 2)).padded
    assert (p.h, p.w) == (8, 8)
    assert int(O.pad_mask(O.Grid(1, 5, 6, 2)).sum()) == 30 and O.pad_mask(O.Grid(1, 5, 6, 2)).size == 64
    p = pad_grid(GridShape(2, 45, 80, 2)).padded
    assert (p.t, p.h, p.w) == (2, 48, 80)
    assert int(O.pad_mask(O.Grid(2, 45, 80, 2)).sum()) == 2 * 45 * 80
    # test_anyres.py:74-81: the subsequence mask keeps every real token
    for pat in ("tsa", "gsa"):
        sm = O.subseq_mask(O.Grid(1, 5, 6, 2), pat)
        assert sm.shape == (4, 16) and int(sm.sum()) == 30


def test_flop_report_kats():
    # test_attention.py:152-158
    from paper_2605_28691_b200 import GridShape, SparsePattern
    from paper_2605_28691_b200.attention import flop_report
    assert flop_report(GridShape(1, 4, 4, 1), SparsePattern.TOKEN_WISE).ratio == 1.0
    rep = flop_report(GridShape(1, 8, 8, 2), SparsePattern.TOKEN_WISE, chan=16)
    assert rep.full_flops == 2 * 64 * 64 * 16
    assert rep.sparse_flops == 4 * 2 * 16 * 16 * 16
    assert rep.ratio == 0.25
    assert flop_report(GridShape(1, 9, 9, 3), SparsePattern.GROUP_WISE).ratio == pytest.approx(1 / 9)


def test_all_to_all_two_rank_transpose():
    # test_ssp.py:48-55: send[0] = [A, B], send[1] = [C, D] -> recv[0] = [A, C], recv[1] = [B, D]
    from paper_2605_28691_b200 import ssp
    a, b, c, d = (torch.full((1, 2), v, dtype=torch.float64) for v in (1.0, 2.0, 3.0, 4.0))
    log = ssp.CommLog()
    out = ssp.all_to_all([torch.cat([a, b]), torch.cat([c, d])], log)
    assert torch.equal(out[0], torch.cat([a, c])) and torch.equal(out[1], torch.cat([b, d]))
    assert log.events[0].payload_per_rank == 4
    ref = O.transpose_all_to_all([np.concatenate([x.numpy() for x in (a, b)]),
                                  np.concatenate([x.numpy() for x in (c, d)])])
    assert np.array_equal(ref[0], out[0].numpy()) and np.array_equal(ref[1], out[1].numpy())


def test_comm_ledger_kats():
    # test_ssp.py:181-215
    from paper_2605_28691_b200 import ssp
    log = ssp.ulysses_block_comm(8, 1000)
    assert log.count("all_to_all") == 4 and log.total_payload() == 4000
    assert ssp.ulysses_block_comm(2, 0).total_payload() == 0
    assert ssp.ulysses_block_comm(8, 4096).total_payload() == 16384
    assert ssp.naive_switch_comm(1, 100)[1]["global_traffic"] == 0
    _, rep = ssp.naive_switch_comm(4, 100)
    assert rep["global_traffic"] == 1200 and rep["recv_per_rank"] == 300
    assert ssp.naive_switch_comm(8, 100)[1]["global_traffic"] == 5600
    rep = ssp.comm_comparison(4, 1000, blocks=3)
    assert (rep["ssp_events"], rep["ulysses_events"]) == (3, 12)
    assert rep["volume_ratio"] == 0.25 and rep["volume_reduction_percent"] == 75.0
    assert rep["ssp_global_per_switch"] == 3000 and rep["naive_global_per_switch"] == 12000
    rows = ssp.comm_comparison(4, 100)["growth_table"]
    assert [r["group_size"] for r in rows] == [2, 4, 8]
    assert all(r["naive_global"] == r["group_size"] * r["ssp_global"] for r in rows)
