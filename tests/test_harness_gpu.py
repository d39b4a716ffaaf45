"""The reference benchmark protocol on the GPU (paper_2005_13425_b200.harness,
contract of sembench/bench.py) and the device bandwidth probe (perf.py:162-203).

Timings are machine-dependent; the deterministic parts are pinned to the
reference's own rows (tests/golden/make_golden.py): box, dofs, the model
inventory and the instrumented traffic / flop counters of every variant."""

import numpy as np
import pytest

import paper_2005_13425_b200 as sb
from paper_2005_13425_b200 import perf

pytestmark = pytest.mark.gpu


def _csv(golden, key):
    return bytes(np.asarray(golden[key], dtype=np.uint8)).decode().split(",")


def test_measure_bandwidth(cuda):
    bw = sb.measure_bandwidth(4096 * 1000)  # 983 MB payload, well above L2
    assert 2e12 < bw < 2e13, bw
    with pytest.raises(ValueError):
        sb.measure_bandwidth(4096 * 1000, repetitions=5)
    with pytest.warns(RuntimeWarning):
        sb.measure_bandwidth(64 * 1000)  # 15 MB: fits in L2


def test_run_bench_matches_reference_inventory(cuda, golden):
    rows = sb.run_bench(sb.BenchConfig(elements=64, iterations=10, variant="all"))
    fields = _csv(golden, "bench64/int_fields")
    assert [r.variant for r in rows] == _csv(golden, "bench64/variants")
    ref = golden["bench64/values"]
    for row, want in zip(rows, ref):
        assert [getattr(row, k) for k in fields] == [int(v) for v in want], row.variant
        assert row.box == "4x4x4" and row.workers > 0 and row.total_seconds > 0
        assert row.achieved_gflops > 0 and row.roofline_peak_gflops > 0
        assert row.ax_seconds > 0 and row.dssum_seconds > 0
        assert "probe-under-llc" in row.flags.split(";")
    assert sb.parse_csv(sb.emit_csv(rows)) == rows
    assert "phase-shares-fused" in rows[2].flags
    assert rows[2].ax_seconds + rows[2].dssum_seconds < rows[2].total_seconds


def test_run_roofline_and_sweep(cuda, golden):
    d = sb.run_roofline(sb.BenchConfig(elements=4096))
    assert list(d.keys()) == _csv(golden, "bench64/roofline_keys")
    assert d["flags"] == "" and d["dofs"] == 4_096_000
    assert d["roofline_peak_gflops"] == pytest.approx(perf.roofline_peak(d["measured_bandwidth"], 10) / 1e9)
    rows = sb.run_sweep(sb.BenchConfig(sweep=(64, 512), iterations=5, variant="layered"))
    assert [(r.elements, r.box) for r in rows] == [(64, "4x4x4"), (512, "8x8x8")]
    with pytest.raises(ValueError):
        sb.run_bench(sb.BenchConfig(sweep=(64,)))
