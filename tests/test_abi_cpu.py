"""CPU-only checks of the C-ABI library: it loads without a GPU and exports
every symbol include/osp_skiparse.h declares; host-side API logic."""

import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def _header_functions():
    text = (ROOT / "include" / "osp_skiparse.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(osp_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def cdll():
    from paper_2605_28691_b200 import build
    build.build()
    from paper_2605_28691_b200 import _lib
    return _lib.load_library()


def test_header_and_binding_agree():
    from paper_2605_28691_b200 import _lib
    assert _header_functions() == sorted(_lib.EXPORTS)


def test_library_exports_every_symbol(cdll):
    for name in _header_functions():
        assert hasattr(cdll, name), name
    assert cdll.osp_abi_version() == 2


def test_library_is_sm100a_only(cdll):
    import subprocess
    from paper_2605_28691_b200 import _lib
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(_lib._PATH)],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(8|9)\d", out)


def test_sass_has_tcgen05_and_tma(cdll):
    import subprocess
    from paper_2605_28691_b200 import _lib
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", str(_lib._PATH)],
                          capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass or "UTCMMA" in sass  # tcgen05.mma
    assert "UTMALDG" in sass                     # TMA tensor loads
    assert "LDTM" in sass and "STTM" in sass     # TMEM ld/st
    assert " HMMA" not in sass                   # no legacy mma.sync path


def test_argument_errors_without_gpu(cdll):
    # validation happens before any CUDA call, so these run on CPU
    rc = cdll.osp_rearrange(None, None, 2, 8, 1, 1, 5, 6, 2, 1, 0, 0, None)
    assert rc == 1  # PatternError: 5x6 not divisible by k=2
    assert b"token-wise" in cdll.osp_last_error()
    rc = cdll.osp_rearrange(None, None, 2, 8, 1, 1, 6, 6, 2, 3, 0, 0, None)
    assert rc == 1  # group-wise needs k^2
    rc = cdll.osp_ssp_pack(None, None, 2, 8, 3, 4, 1, 4, 4, 2, None)
    assert rc == 4  # ShardingError k^2 % N
    rc = cdll.osp_ssp_pack(None, None, 2, 8, 2, 3, 1, 4, 4, 2, None)
    assert rc == 6  # ProtocolError local batch % G
    rc = cdll.osp_attn_fwd(None, None, None, None, None, 1, 128, 1, 96, 96, 96, 96, 96, None, None,
                           0, 1.0, None)
    assert rc == 8  # unsupported head_dim


def test_error_mapping():
    from paper_2605_28691_b200 import errors
    assert isinstance(errors.from_status(1, "x"), errors.PatternError)
    assert isinstance(errors.from_status(4, "x"), errors.ShardingError)
    assert isinstance(errors.from_status(9, "x"), RuntimeError)
    for cls in (errors.PatternError, errors.ShapeError, errors.ShardingError,
                errors.ProtocolError, errors.CollectiveError, errors.CoordinateError):
        assert issubclass(cls, ValueError)


def test_host_logic_mirrors_reference():
    from paper_2605_28691_b200 import (GridShape, LayerKind, PatternError, SparsePattern,
                                       build_layer_schedule, comm_comparison, flop_report,
                                       naive_switch_comm, orig_to_gsa, orig_to_tsa,
                                       ulysses_block_comm)
    from paper_2605_28691_b200.errors import CoordinateError, ScheduleError
    g = GridShape(2, 4, 4)
    assert g.flatten_index(1, 0, 0) == 16 and g.unflatten_index(8) == (0, 2, 0)
    with pytest.raises(CoordinateError):
        g.flatten_index(2, 0, 0)
    with pytest.raises(ValueError):
        GridShape(0, 4, 4)
    with pytest.raises(PatternError):
        orig_to_tsa(GridShape(1, 5, 6, 2))
    with pytest.raises(PatternError):
        orig_to_gsa(GridShape(1, 6, 6, 2))
    m = orig_to_tsa(GridShape(1, 8, 8, 2), 3)
    assert (m.in_batch, m.in_seq, m.out_batch, m.out_seq) == (3, 64, 12, 16)
    s = build_layer_schedule(40, 8)
    assert s[:4] == [LayerKind.FULL] * 4 and s[4:8] == [LayerKind.TSA, LayerKind.GSA] * 2
    with pytest.raises(ScheduleError):
        build_layer_schedule(10, 3)
    rep = flop_report(GridShape(1, 8, 8, 2), SparsePattern.TOKEN_WISE, chan=16)
    assert (rep.full_flops, rep.sparse_flops, rep.ratio) == (2 * 64 * 64 * 16, 4 * 2 * 16 * 16 * 16, 0.25)
    assert ulysses_block_comm(8, 1000).total_payload() == 4000
    assert naive_switch_comm(4, 100)[1]["global_traffic"] == 1200
    c = comm_comparison(4, 1000, blocks=3)
    assert c["volume_ratio"] == 0.25 and c["ulysses_events"] == 12


def test_comm_comparison_matches_reference_golden(golden_meta):
    from paper_2605_28691_b200 import comm_comparison
    for ref in golden_meta["comm"]:
        assert comm_comparison(ref["group_size"], ref["per_rank_elements"], ref["blocks"]) == ref


def test_ospt_and_mask_formats_byte_exact(tmp_path):
    """OSPT (gridseq.py:232-256) and mask files (anyres.py:99-112) against files the
    reference wrote (tests/golden/ref_*, made by oracle/make_golden.py)."""
    import numpy as np
    import torch
    from paper_2605_28691_b200 import SequenceTensor, read_ospt, write_ospt
    from paper_2605_28691_b200 import formats
    golden = ROOT / "tests" / "golden"
    x = read_ospt(golden / "ref_x.ospt", device="cpu")
    want = np.random.Generator(np.random.PCG64(9)).standard_normal((2, 7, 3))
    assert np.array_equal(x.data.numpy(), want)
    write_ospt(tmp_path / "x.ospt", x)
    assert (tmp_path / "x.ospt").read_bytes() == (golden / "ref_x.ospt").read_bytes()
    with pytest.raises(ValueError):
        (tmp_path / "bad.ospt").write_bytes(b"NOPE" + bytes(20))
        read_ospt(tmp_path / "bad.ospt", device="cpu")
    g, mask = formats.read_mask(golden / "ref_mask_1x5x6_k2.bin")
    assert (g.t, g.h, g.w, g.k) == (1, 8, 8, 2) and int(mask.sum()) == 30

    class _PG:  # a PaddedGrid-shaped stand-in (the product PaddedGrid needs a GPU mask)
        padded = g
    _PG.mask = mask.cpu()
    formats.write_mask(tmp_path / "m.bin", _PG)
    assert (tmp_path / "m.bin").read_bytes() == (golden / "ref_mask_1x5x6_k2.bin").read_bytes()


def test_integration_stub_matches_abi():
    """The ctypes stub shown in INTEGRATION.md binds the same signatures as the package."""
    import ctypes
    import re
    from pathlib import Path

    from paper_2605_28691_b200 import _lib
    text = (Path(__file__).resolve().parent.parent / "INTEGRATION.md").read_text()
    env = {"vp": ctypes.c_void_p, "i64": ctypes.c_int64, "c_int": ctypes.c_int, "c_f": ctypes.c_float,
           "ctypes": ctypes}
    found = 0
    for name, args in re.findall(r"_lib\.(osp_\w+)\.argtypes = \[([^\]]*)\]", text):
        got = [eval(a.strip(), env) for a in args.split(",")]
        assert got == _lib._SIGS[name][0], name
        found += 1
    assert found >= 4
