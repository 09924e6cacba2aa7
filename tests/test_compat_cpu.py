"""The `osp` import shim (compat/osp) exposes the reference's hot-path module layout and names,
and numpy data mode is switchable.  The shim's numerical behaviour is exercised on the GPU by
the reference's own tests (tools/run_reference_tests.sh, profiles/r02_reference_tests_via_shim.txt)."""

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent

# hot-path names the reference's tests import from each osp module (pkg/tests/test_*.py)
NAMES = {
    "gridseq": ["GridShape", "SequenceTensor", "IndexMap", "random_tensor", "rearrange_map", "read_ospt",
                "write_ospt", "OSPT_MAGIC", "CoordinateError", "ShapeError"],
    "skiparse": ["SparsePattern", "LayerKind", "PatternError", "ScheduleError", "assignment_of",
                 "build_layer_schedule", "orig_to_tsa", "tsa_to_orig", "orig_to_gsa", "gsa_to_orig",
                 "tsa_to_gsa", "gsa_to_tsa", "pattern_map", "reachability_hops"],
    "anyres": ["pad_grid", "pad_tensor", "strip_padding", "subsequence_mask", "read_mask", "write_mask"],
    "attention": ["dense_attention", "skiparse_attention", "flop_report", "project_qkv",
                  "masked_dense_attention", "pattern_allow_matrix", "skiparse_reference"],
    "ssp": ["CommLog", "ProcessGroup", "RankShard", "ShardingError", "CollectiveError", "ProtocolError",
            "shard_pattern_layout", "all_to_all", "ssp_pattern_switch", "gather_shards",
            "comm_comparison", "naive_switch_comm", "ulysses_block_comm"],
}


def test_shim_layout_and_data_mode():
    import importlib

    from paper_2605_28691_b200.gridseq import SequenceTensor, set_data_mode
    sys.path.insert(0, str(ROOT / "compat"))
    try:
        osp = importlib.import_module("osp")
        for mod, names in NAMES.items():
            m = importlib.import_module(f"osp.{mod}")
            missing = [n for n in names if not hasattr(m, n)]
            assert not missing, (mod, missing)
        assert set_data_mode("torch") == "numpy"        # importing the shim selected numpy mode
        x = SequenceTensor(np.zeros((1, 2, 3)))         # (built on CPU here: no GPU needed)
        assert set_data_mode("numpy") == "torch"
        assert isinstance(x.data, np.ndarray) and x.data.dtype == np.float64
        assert not x.data.flags.writeable
        assert osp.__version__
    finally:
        set_data_mode("torch")
        sys.path.remove(str(ROOT / "compat"))
