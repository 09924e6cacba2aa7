"""report-all: the reference-written document and the comparator that
holds this package's device-side report to it (the GPU run is tests/test_report_gpu.py)."""
import copy
import json
from pathlib import Path

from paper_2605_28691_b200 import report

GOLDEN = Path(__file__).resolve().parent / "golden" / "report_all_seed0.json"


def _golden():
    return json.loads(GOLDEN.read_text())


def test_golden_is_the_reference_layout_and_passes():
    text = GOLDEN.read_text()
    ref = json.loads(text)
    assert report.dumps(ref) == text          # two-space indent, sorted keys (cli.py:75-76)
    assert ref["pass"] and ref["seed"] == 0
    assert all(s["pass"] for s in ref["sections"].values())


def test_report_runs_on_the_reference_grids():
    ref = _golden()
    grids = [(*c["grid"], c["k"]) for c in ref["sections"]["rearrange"]["grids"]]
    assert grids == list(report.REPORT_GRIDS)


def test_comparator_accepts_itself_and_names_differences():
    ref = _golden()
    assert report.diff_against_reference(ref, ref) == []
    bad = copy.deepcopy(ref)
    bad["sections"]["rearrange"]["grids"][1]["subseq_len"] += 1
    bad["sections"]["hif8_format"]["max_rel_over_bound"] *= 1.001
    bad["sections"]["ssp"]["cases"][0]["checks"]["zero_all_gathers"] = False
    del bad["sections"]["flops"]["note"]
    diffs = report.diff_against_reference(bad, ref)
    assert any("rearrange.grids[1].subseq_len" in d for d in diffs)
    assert any("hif8_format.max_rel_over_bound" in d for d in diffs)
    assert any("zero_all_gathers" in d for d in diffs)
    assert any("flops" in d and "missing" in d for d in diffs)
    # bf16 attention errors and probe outputs are compared by structure only
    ok = copy.deepcopy(ref)
    ok["sections"]["attention"]["cases"][0]["max_abs_err"] = 3e-3
    ok["sections"]["attention"]["cases"][0]["tolerance"] = 2 * report.ATTN_TOLERANCE_BF16
    ok["sections"]["quantized_attention_probe"]["reports"]["tsa"]["output"]["max_abs"] = 0.5
    assert report.diff_against_reference(ok, ref) == []
