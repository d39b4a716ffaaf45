"""sembench-1 report rows (paper_2005_13425_b200.report) against text the
reference's own report module emitted (tests/golden/make_golden.py): parsing
the reference's CSV / JSON and re-emitting must reproduce it byte for byte,
so B200 rows interoperate with the reference's tooling and plots."""

import dataclasses

import numpy as np
import pytest

from paper_2005_13425_b200 import report as R


def _text(golden, fmt):
    return bytes(np.asarray(golden[f"report/{fmt}"], dtype=np.uint8)).decode()


def test_csv_roundtrip_matches_reference(golden):
    ref_csv = _text(golden, "csv")
    rows = R.parse_csv(ref_csv)
    assert len(rows) == 5 and rows[1].include_dssum is True and rows[0].include_dssum is False
    assert R.emit_csv(rows) == ref_csv
    assert R.parse_csv(R.emit_csv(rows)) == rows


def test_json_and_gnuplot_match_reference(golden):
    rows = R.parse_csv(_text(golden, "csv"))
    assert R.emit_json(rows) == _text(golden, "json")
    assert R.parse_json(_text(golden, "json")) == rows
    assert R.emit_gnuplot(rows) == _text(golden, "gnuplot")


def test_schema_and_validation(golden):
    rows = R.parse_csv(_text(golden, "csv"))
    assert [f.name for f in dataclasses.fields(R.PerfReport)][0] == "schema_version"
    assert len(dataclasses.fields(R.PerfReport)) == 26
    assert all(r.schema_version == R.SCHEMA_VERSION == "sembench-1" for r in rows)
    with pytest.raises(ValueError):
        dataclasses.replace(rows[0], achieved_gflops=float("nan"))
    with pytest.raises(ValueError):
        R.parse_csv("not,a,header\n1,2,3\n")
    assert R.parse_csv(R.emit_csv([])) == []
