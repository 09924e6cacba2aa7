"""Generate tests/golden/ fixtures by running the REFERENCE `osp` package.

TEST INFRASTRUCTURE ONLY.  Run in the build container, where the reference is
mounted read-only:

    PYTHONDONTWRITEBYTECODE=1 python oracle/make_golden.py [report]

It imports /root/reference/pkg/src/osp (never copied into this repo), calls
its public functions on small seeded inputs and stores inputs + outputs as
compressed .npz / .json under tests/golden/.  The GPU box never needs the
reference: tests read only these committed fixtures.

Cases follow the reference's own test grids (pkg/tests/test_skiparse.py:9-15,
test_ssp.py:79-83, test_anyres.py:18-29, test_attention.py:79-137) plus the
larger cases SURVEY.md sec. 8c lists as unpinned (k=4, T>1, B>1, N=8).
"""

from __future__ import annotations

import json
import os
import sys
from pathlib import Path

import numpy as np

sys.dont_write_bytecode = True
REF = Path(os.environ.get("OSP_REFERENCE", "/root/reference/pkg/src"))
sys.path.insert(0, str(REF))

import osp  # noqa: E402  (reference package)
from osp import anyres, attention, gridseq, skiparse, ssp  # noqa: E402

OUT = Path(__file__).resolve().parent.parent / "tests" / "golden"

MAP_GRIDS = [(1, 4, 4, 2), (2, 4, 4, 2), (1, 8, 8, 2), (2, 8, 8, 2), (1, 9, 9, 3),
             (3, 8, 12, 2), (2, 16, 16, 4), (1, 2, 2, 2), (2, 3, 5, 1)]
MAP_BATCHES = [1, 2, 3]
BUILDERS = ["orig_to_tsa", "tsa_to_orig", "orig_to_gsa", "gsa_to_orig", "tsa_to_gsa",
            "gsa_to_tsa"]
PAD_GRIDS = [(1, 5, 6, 2), (2, 45, 80, 2), (2, 5, 6, 2), (1, 7, 10, 3), (2, 30, 52, 2),
             (1, 4, 4, 2), (1, 13, 9, 4)]


def maps_golden():
    arrays, meta = {}, []
    for (t, h, w, k) in MAP_GRIDS:
        g = gridseq.GridShape(t, h, w, k)
        for name in BUILDERS:
            for b in MAP_BATCHES:
                try:
                    m = getattr(skiparse, name)(g, b)
                except skiparse.PatternError:
                    meta.append({"grid": [t, h, w, k], "map": name, "batch": b,
                                 "error": "PatternError"})
                    continue
                key = f"{name}_{t}x{h}x{w}_k{k}_b{b}"
                arrays[key] = m.src
                meta.append({"grid": [t, h, w, k], "map": name, "batch": b, "key": key,
                             "in": [m.in_batch, m.in_seq], "out": [m.out_batch, m.out_seq]})
        for pat in ("tsa", "gsa"):
            try:
                a = skiparse.assignment_of(g, skiparse.SparsePattern(pat))
            except skiparse.PatternError:
                continue
            arrays[f"assign_{pat}_{t}x{h}x{w}_k{k}_subseq"] = a.subseq
            arrays[f"assign_{pat}_{t}x{h}x{w}_k{k}_pos"] = a.position
    # divisibility failures the reference raises on (test_skiparse.py:124-132)
    for (t, h, w, k) in [(1, 5, 6, 2), (1, 6, 6, 2)]:
        g = gridseq.GridShape(t, h, w, k)
        for name in BUILDERS:
            try:
                getattr(skiparse, name)(g, 1)
                meta.append({"grid": [t, h, w, k], "map": name, "batch": 1, "error": None,
                             "ok_only": True})
            except skiparse.PatternError:
                meta.append({"grid": [t, h, w, k], "map": name, "batch": 1,
                             "error": "PatternError"})
    # rearrange_map transpose KAT (test_gridseq.py:117-122)
    rm = gridseq.rearrange_map([("b", 1)], [("x", 2), ("y", 3)], ["b"], ["y", "x"])
    arrays["kat_transpose"] = rm.src
    return arrays, meta


def pad_golden():
    arrays, meta = {}, []
    for (t, h, w, k) in PAD_GRIDS:
        g = gridseq.GridShape(t, h, w, k)
        pg = anyres.pad_grid(g)
        key = f"{t}x{h}x{w}_k{k}"
        arrays[f"mask_{key}"] = pg.mask
        arrays[f"embed_{key}"] = pg.embedding
        x = gridseq.random_tensor(2, g.seq_len, 3, seed=t * 100 + h)
        arrays[f"x_{key}"] = x.data
        arrays[f"padded_{key}"] = anyres.pad_tensor(x, pg).data
        for pat in ("tsa", "gsa"):
            try:
                arrays[f"submask_{pat}_{key}"] = anyres.subsequence_mask(
                    pg, skiparse.SparsePattern(pat))
            except skiparse.PatternError:
                pass
        meta.append({"grid": [t, h, w, k], "key": key,
                     "padded": [pg.padded.t, pg.padded.h, pg.padded.w],
                     "trivial": pg.trivial, "real": int(pg.mask.sum())})
    return arrays, meta


def attention_golden():
    arrays, meta = {}, []
    # dense_attention cases (test_attention.py:33-66)
    for i, (b, s, c, mask) in enumerate([(1, 4, 2, None), (2, 5, 3, None), (1, 6, 4, "some"),
                                         (1, 3, 2, "none"), (2, 64, 8, "some"),
                                         (3, 130, 16, "some")]):
        q = gridseq.random_tensor(b, s, c, 3 + i)
        k = gridseq.random_tensor(b, s, c, 4 + i)
        v = gridseq.random_tensor(b, s, c, 5 + i)
        kv = None
        if mask == "some":
            kv = np.random.Generator(np.random.PCG64(77 + i)).random((b, s)) > 0.3
        elif mask == "none":
            kv = np.zeros(s, dtype=bool)
        out = attention.dense_attention(q, k, v, key_valid=kv)
        key = f"dense{i}"
        arrays[f"{key}_q"], arrays[f"{key}_k"], arrays[f"{key}_v"] = q.data, k.data, v.data
        if kv is not None:
            arrays[f"{key}_valid"] = np.broadcast_to(kv, (b, s)).copy()
        arrays[f"{key}_out"] = out.data
        meta.append({"case": key, "shape": [b, s, c], "mask": mask})
    # skiparse_attention cases (test_attention.py:69-137), single head of chan
    cases = [((1, 4, 4, 2), 1, 4, False), ((2, 4, 4, 2), 2, 6, False),
             ((1, 8, 8, 2), 2, 6, False), ((1, 9, 9, 3), 2, 6, False),
             ((1, 5, 6, 2), 1, 4, True), ((1, 5, 6, 2), 3, 4, True),
             ((2, 6, 10, 2), 1, 8, True), ((1, 16, 16, 2), 1, 16, False)]
    for i, (grid, b, c, padded) in enumerate(cases):
        g = gridseq.GridShape(*grid)
        pg = anyres.pad_grid(g) if padded else None
        for pat in ("original", "tsa", "gsa"):
            x = gridseq.random_tensor(b, g.seq_len, c, seed=10 + i)
            xin = anyres.pad_tensor(x, pg) if padded else x
            out = attention.skiparse_attention(xin, g, skiparse.SparsePattern(pat), pg)
            key = f"skip{i}_{pat}"
            arrays[f"{key}_x"] = xin.data
            arrays[f"{key}_out"] = out.data
            meta.append({"case": key, "grid": list(grid), "batch": b, "chan": c,
                         "padded": padded, "pattern": pat})
    # fixed projections (attention.py:20-27)
    for c in (4, 6, 8, 16):
        wq, wk, wv = attention.qkv_projections(c)
        arrays[f"proj{c}_q"], arrays[f"proj{c}_k"], arrays[f"proj{c}_v"] = wq, wk, wv
    flops = []
    for grid, pat, chan in [((1, 8, 8, 2), "tsa", 16), ((1, 4, 4, 1), "tsa", 1),
                            ((1, 9, 9, 3), "gsa", 1), ((1, 8, 8, 2), "original", 1),
                            ((21, 48, 80, 2), "tsa", 5120), ((21, 32, 52, 2), "gsa", 1536)]:
        rep = attention.flop_report(gridseq.GridShape(*grid), skiparse.SparsePattern(pat), chan)
        flops.append({"grid": list(grid), "pattern": pat, "chan": chan,
                      "full": rep.full_flops, "sparse": rep.sparse_flops, "ratio": rep.ratio})
    return arrays, meta, flops


def ssp_golden():
    arrays, meta = {}, []
    cases = [((1, 4, 4, 2), 4, 1), ((1, 8, 8, 2), 2, 1), ((1, 8, 8, 2), 4, 1),
             ((1, 8, 8, 2), 2, 3), ((1, 8, 8, 2), 1, 1), ((2, 8, 8, 2), 4, 2),
             ((1, 16, 16, 4), 8, 1), ((2, 16, 16, 4), 4, 1), ((1, 16, 16, 4), 16, 2),
             ((1, 18, 18, 3), 9, 1), ((1, 18, 18, 3), 3, 2)]
    for i, (grid, n, b) in enumerate(cases):
        g = gridseq.GridShape(*grid)
        for pat in ("tsa", "gsa"):
            x = gridseq.random_tensor(b, g.seq_len, 4, seed=50 + i)
            layout = skiparse.pattern_map(g, skiparse.SparsePattern(pat), b).apply(x)
            log = ssp.CommLog()
            group = ssp.shard_pattern_layout(layout, n, log)
            out = ssp.ssp_pattern_switch(group, g)
            key = f"ssp{i}_{pat}"
            arrays[f"{key}_in"] = layout.data
            arrays[f"{key}_out"] = np.stack([s.tensor.data for s in out.shards])
            meta.append({"case": key, "grid": list(grid), "n": n, "batch": b, "pattern": pat,
                         "a2a": log.count("all_to_all"), "payload": log.events[0].payload_per_rank})
    errors = []
    g = gridseq.GridShape(1, 4, 4, 2)
    x = skiparse.pattern_map(g, skiparse.SparsePattern.TOKEN_WISE, 3).apply(
        gridseq.random_tensor(3, 16, 4, 0))
    try:
        ssp.ssp_pattern_switch(ssp.shard_pattern_layout(x, 3), g)
    except ssp.ShardingError:
        errors.append({"grid": [1, 4, 4, 2], "n": 3, "batch": 3, "error": "ShardingError"})
    # k=2 cannot shard over 8 ranks even with B=2 (SURVEY.md sec. 7 hard part 3)
    g = gridseq.GridShape(1, 8, 8, 2)
    x = skiparse.pattern_map(g, skiparse.SparsePattern.TOKEN_WISE, 2).apply(
        gridseq.random_tensor(2, 64, 4, 0))
    try:
        ssp.ssp_pattern_switch(ssp.shard_pattern_layout(x, 8), g)
    except ssp.ShardingError:
        errors.append({"grid": [1, 8, 8, 2], "n": 8, "batch": 2, "error": "ShardingError"})
    comm = [ssp.comm_comparison(n, s, blocks=bl) for n, s, bl in
            [(4, 1000, 3), (2, 64, 1), (8, 4096, 1), (4, 100, 1)]]
    uly = [{"n": n, "s": s, "payload": ssp.ulysses_block_comm(n, s).total_payload(),
            "events": ssp.ulysses_block_comm(n, s).count("all_to_all")}
           for n, s in [(8, 1000), (2, 0), (8, 4096)]]
    naive = [{"n": n, "s": s, **ssp.naive_switch_comm(n, s)[1]} for n, s in
             [(1, 100), (4, 100), (8, 100)]]
    return arrays, meta, {"errors": errors, "comm": comm, "ulysses": uly, "naive": naive}


def formats_golden():
    """Byte-exact reference files: OSPT tensor (gridseq.py:232-256) and mask file
    (anyres.py:99-112)."""
    x = gridseq.random_tensor(2, 7, 3, seed=9)
    gridseq.write_ospt(OUT / "ref_x.ospt", x)
    pg = anyres.pad_grid(gridseq.GridShape(1, 5, 6, 2))
    anyres.write_mask(OUT / "ref_mask_1x5x6_k2.bin", pg)


def hif8_golden():
    """HiF8 codec (hif8.py:77-193) and quantizer (hif8.py:223-246) outputs."""
    from osp import hif8
    spec = hif8.DEFAULT_SPEC
    rng = np.random.Generator(np.random.PCG64(8))
    vals = spec.values
    mids = (vals[:-1] + vals[1:]) / 2
    x = np.concatenate([
        rng.standard_normal(4000) * 3, rng.standard_normal(2000) * 1e-5,
        np.geomspace(2.0 ** -24, 1.2 * spec.max_value, 600), -np.geomspace(2.0 ** -24, 1.2 * spec.max_value, 600),
        vals, mids, np.nextafter(mids, np.inf), np.nextafter(mids, -np.inf), [0.0, -0.0]])
    arrays = {"values": vals, "x": x, "codes": hif8.encode_array(x), "decoded": hif8.decode_array(np.arange(256))}
    qx = gridseq.random_tensor(2, 33, 5, seed=3)
    for mode in ("forward", "backward"):
        q = hif8.quantize_tensor(qx, mode)
        arrays[f"q_{mode}_codes"] = q.codes.data
        arrays[f"q_{mode}_scale"] = np.array([q.scale, q.amax])
        arrays[f"q_{mode}_deq"] = hif8.dequantize(q).data
    arrays["q_x"] = qx.data
    np.savez_compressed(OUT / "hif8.npz", **arrays)


def report_golden():
    """The reference's `report-all` document for seed 0 (cli.py:279-325), which
    paper_2605_28691_b200.report reproduces section by section on the device."""
    from osp.cli import build_full_report
    text = json.dumps(build_full_report(0), indent=2, sort_keys=True) + "\n"
    (OUT / "report_all_seed0.json").write_text(text)


def main():
    OUT.mkdir(parents=True, exist_ok=True)
    if sys.argv[1:] == ["report"]:      # only the report-all document
        report_golden()
        return
    report_golden()
    formats_golden()
    hif8_golden()
    a_maps, m_maps = maps_golden()
    np.savez_compressed(OUT / "maps.npz", **a_maps)
    a_pad, m_pad = pad_golden()
    np.savez_compressed(OUT / "pad.npz", **a_pad)
    a_att, m_att, flops = attention_golden()
    np.savez_compressed(OUT / "attention.npz", **a_att)
    a_ssp, m_ssp, extra = ssp_golden()
    np.savez_compressed(OUT / "ssp.npz", **a_ssp)
    meta = {"reference_version": osp.__version__, "numpy": np.__version__,
            "maps": m_maps, "pad": m_pad, "attention": m_att, "flops": flops,
            "ssp": m_ssp, **extra}
    (OUT / "golden.json").write_text(json.dumps(meta, indent=1, sort_keys=True))
    for f in sorted(OUT.iterdir()):
        print(f"{f.name}: {f.stat().st_size} bytes")


if __name__ == "__main__":
    main()
