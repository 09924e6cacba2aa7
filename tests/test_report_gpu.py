"""The package's report-all document, computed on the device, against the one the reference
wrote (tests/golden/report_all_seed0.json, oracle/make_golden.py)."""
import json
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

GOLDEN = Path(__file__).resolve().parent / "golden" / "report_all_seed0.json"


def test_report_all_matches_reference_document():
    from paper_2605_28691_b200 import report
    mine = report.report_all(0)
    ref = json.loads(GOLDEN.read_text())
    assert report.diff_against_reference(mine, ref) == []
    assert mine["pass"] is True
    for case in mine["sections"]["attention"]["cases"]:
        assert 0.0 < case["max_abs_err"] <= case["tolerance"]
    # deterministic: the same document twice
    assert report.dumps(report.report_all(0)) == report.dumps(mine)


def test_report_cli_writes_the_document(tmp_path):
    from paper_2605_28691_b200 import report
    out = tmp_path / "r.json"
    assert report.main(["--seed", "0", "--out", str(out)]) == 0
    assert json.loads(out.read_text())["pass"] is True
