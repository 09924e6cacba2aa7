"""Pin the CPU oracle to golden vectors produced by the reference itself
(tests/golden, made by oracle/make_golden.py) and to the reference tests'
known-answer values (cited per test).  CPU only."""

import numpy as np
import pytest

from oracle import osp_oracle as O


def test_maps_match_reference_tables(golden, golden_meta):
    maps = golden("maps")
    n = 0
    for m in golden_meta["maps"]:
        g = O.Grid(*m["grid"])
        if m.get("error") == "PatternError":
            with pytest.raises(O.PatternError):
                O.map_table(m["map"], g, m["batch"])
            continue
        if m.get("ok_only"):
            O.map_table(m["map"], g, m["batch"])
            continue
        tab = O.map_table(m["map"], g, m["batch"])
        assert np.array_equal(tab, maps[m["key"]]), m["key"]
        n += 1
    assert n > 100


def test_assignments_match_reference(golden, golden_meta):
    maps = golden("maps")
    for key in maps.files:
        if not key.startswith("assign_") or not key.endswith("_subseq"):
            continue
        _, pat, dims, kk, _ = key.split("_")
        t, h, w = map(int, dims.split("x"))
        sub, pos = O.assignment(O.Grid(t, h, w, int(kk[1:])), pat)
        assert np.array_equal(sub, maps[key])
        assert np.array_equal(pos, maps[key.replace("_subseq", "_pos")])


def test_frozen_kats():
    # test_skiparse.py:39-47 / SPEC.md:114,122-123
    sub, _ = O.assignment(O.Grid(1, 4, 4, 2), "tsa")
    assert sorted(np.flatnonzero(sub == 0)) == [0, 2, 8, 10]
    sub, _ = O.assignment(O.Grid(1, 4, 4, 2), "gsa")
    assert sorted(np.flatnonzero(sub == 0)) == [0, 1, 4, 5]
    assert sorted(np.flatnonzero(sub == 3)) == [10, 11, 14, 15]
    # flatten KATs test_gridseq.py:10-18
    g = O.Grid(2, 4, 4)
    assert O.flat(g, 0, 2, 0) == 8 and O.flat(g, 1, 0, 0) == 16


def test_roundtrips_and_coherence():
    for grid in [(1, 8, 8, 2), (2, 8, 12, 2), (1, 9, 9, 3), (2, 16, 16, 4)]:
        g = O.Grid(*grid)
        for b in (1, 3):
            t = O.map_table("orig_to_tsa", g, b)
            gg = O.map_table("orig_to_gsa", g, b)
            assert np.array_equal(O.compose_tables(O.map_table("tsa_to_orig", g, b), t),
                                  np.arange(t.size).reshape(b, -1))
            assert np.array_equal(O.compose_tables(O.map_table("tsa_to_gsa", g, b), t), gg)
            assert np.array_equal(O.compose_tables(O.map_table("gsa_to_tsa", g, b), gg), t)
            assert np.array_equal(O.invert_table(t, b, g.seq_len), O.map_table("tsa_to_orig", g, b))


def test_pad_matches_reference(golden, golden_meta):
    pad = golden("pad")
    for m in golden_meta["pad"]:
        g = O.Grid(*m["grid"])
        key = m["key"]
        assert np.array_equal(O.pad_mask(g), pad[f"mask_{key}"])
        assert np.array_equal(O.pad_embedding(g), pad[f"embed_{key}"])
        pgrid = O.padded_grid(g)
        assert [pgrid.t, pgrid.h, pgrid.w] == m["padded"]
        assert np.array_equal(O.pad(pad[f"x_{key}"], g), pad[f"padded_{key}"])
        assert np.array_equal(O.strip(pad[f"padded_{key}"], g), pad[f"x_{key}"])
        for pat in ("tsa", "gsa"):
            if f"submask_{pat}_{key}" in pad.files:
                assert np.array_equal(O.subseq_mask(g, pat), pad[f"submask_{pat}_{key}"])
    # 720p-style KAT test_anyres.py:25-29
    pg = O.padded_grid(O.Grid(2, 45, 80, 2))
    assert (pg.t, pg.h, pg.w) == (2, 48, 80)


def test_dense_attention_matches_reference(golden, golden_meta):
    a = golden("attention")
    for m in golden_meta["attention"]:
        key = m["case"]
        if not key.startswith("dense"):
            continue
        kv = a[f"{key}_valid"] if f"{key}_valid" in a.files else None
        out = O.dense_attention(a[f"{key}_q"], a[f"{key}_k"], a[f"{key}_v"], kv)
        assert np.max(np.abs(out - a[f"{key}_out"])) < 1e-12, key


def test_projections_bitwise(golden):
    a = golden("attention")
    for c in (4, 6, 8, 16):
        wq, wk, wv = O.qkv_weights(c)
        assert np.array_equal(wq, a[f"proj{c}_q"])
        assert np.array_equal(wk, a[f"proj{c}_k"])
        assert np.array_equal(wv, a[f"proj{c}_v"])


def test_skiparse_attention_matches_reference(golden, golden_meta):
    a = golden("attention")
    for m in golden_meta["attention"]:
        if "pattern" not in m:
            continue
        key = m["case"]
        g = O.Grid(*m["grid"])
        out = O.skiparse_attention(a[f"{key}_x"], g, m["pattern"], padded=m["padded"])
        assert np.max(np.abs(out - a[f"{key}_out"])) < 1e-12, key


def test_skiparse_equals_dense_2d_mask_oracle():
    # test_attention.py:93-100 shape of check, on the restatement itself
    for grid, padded in [((1, 8, 8, 2), False), ((1, 5, 6, 2), True)]:
        g = O.Grid(*grid)
        S = (O.padded_grid(g) if padded else g).seq_len
        x = O.random_normal((2, S, 8), 11)
        for pat in ("tsa", "gsa"):
            a = O.skiparse_attention(x, g, pat, padded=padded, heads=2)
            b = O.skiparse_dense_reference(x, g, pat, padded=padded, heads=2)
            if padded:
                m = O.pad_mask(g)
                assert np.max(np.abs(a[:, m] - b[:, m])) < 1e-10
                assert (a[:, ~m] == 0).all()
            else:
                assert np.max(np.abs(a - b)) < 1e-10


def test_flops_match_reference(golden_meta):
    for f in golden_meta["flops"]:
        full, sparse = O.flop_macs(O.Grid(*f["grid"]), f["pattern"], f["chan"])
        assert (full, sparse) == (f["full"], f["sparse"])


def test_ssp_switch_matches_reference(golden, golden_meta):
    s = golden("ssp")
    for m in golden_meta["ssp"]:
        key = m["case"]
        g = O.Grid(*m["grid"])
        shards = O.shard(s[f"{key}_in"], m["n"])
        out = O.ssp_switch(shards, g)
        assert np.array_equal(np.stack(out), s[f"{key}_out"]), key
        direction = "t2g" if m["pattern"] == "tsa" else "g2t"
        alt = O.ssp_switch_by_gather(shards, g, direction)
        assert np.array_equal(np.stack(alt), s[f"{key}_out"]), key
        assert m["a2a"] == 1 and m["payload"] == shards[0].size


def test_ssp_errors_match_reference(golden_meta):
    for e in golden_meta["errors"]:
        g = O.Grid(*e["grid"])
        x = np.zeros((g.k * g.k * e["batch"], g.seq_len // (g.k * g.k), 2))
        with pytest.raises(O.ShardingError):
            O.ssp_switch(O.shard(x, e["n"]), g)


def test_comm_accounting_matches_reference(golden_meta):
    for ref in golden_meta["comm"]:
        got = O.comm_comparison(ref["group_size"], ref["per_rank_elements"], ref["blocks"])
        assert got == ref


def test_bf16_round():
    x = np.array([1.0, 1.0 + 2 ** -8, 1.0 + 3 * 2 ** -9, -3.14159, 1e-30])
    r = O.bf16_round(x)
    import torch
    want = torch.tensor(x, dtype=torch.float64).to(torch.bfloat16).to(torch.float64).numpy()
    assert np.array_equal(r, want)


def test_hif8_oracle_matches_reference(golden):
    from oracle import hif8_oracle as H
    h = golden("hif8")
    vals = H.value_table()
    assert np.array_equal(vals, h["values"])
    assert len(set(vals.tolist())) == 256 and vals[127] == 0.0
    assert np.array_equal(H.encode(h["x"]), h["codes"])
    assert np.array_equal(H.decode(np.arange(256)), h["decoded"])
    for mode in ("forward", "backward"):
        codes, scale, amax = H.quantize(h["q_x"], mode)
        assert np.array_equal(codes, h[f"q_{mode}_codes"])
        assert (scale, amax) == tuple(h[f"q_{mode}_scale"])
        assert np.array_equal(H.decode(codes) / scale, h[f"q_{mode}_deq"])
    with pytest.raises(ValueError):
        H.encode(np.array([np.inf]))
