"""CPU tests of bench.py's host-side measurement logic (no GPU): the clock
summary is restricted to the timed window, throttle reasons are parsed, the
max-over-ranks helper is a no-op without a process group, and the work
accounting matches the reference's cost model (sembench/kernels.py:121-125)."""

import importlib.util
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def bench():
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def _row(sm, power, cap="Not Active", thermal="Not Active"):
    # clocks.sm, clocks.max.sm, power.draw, reasons.active, hw_slowdown,
    # hw_thermal_slowdown, sw_thermal_slowdown, sw_power_cap
    return [str(sm), "1965", str(power), "0x0", "Not Active", "Not Active", thermal, cap]


def test_clock_summary_uses_only_the_timed_window(bench):
    c = bench.ClockSampler(0)
    c.rows = [(0.0, _row(120, 90)),                     # idle, before the window
              (1.00, _row(1965, 600)), (1.05, _row(1965, 640)),
              (2.0, _row(300, 100))]                     # after the window
    c.mark(0.98, 1.06)
    s = c.summary()
    assert s["samples"] == 2 and s["sm_mhz"] == 1965.0 and s["reasons"] == []
    assert s["power_w_max"] == 640.0


def test_clock_summary_reports_power_cap_and_thermal(bench):
    c = bench.ClockSampler(0)
    c.rows = [(1.0, _row(1650, 1000, cap="Active")),
              (1.05, _row(1600, 1001, cap="Active", thermal="Active"))]
    c.mark(0.9, 1.1)
    s = c.summary()
    assert s["reasons"] == ["sw_power_cap", "sw_thermal_slowdown"]


def test_clock_summary_without_samples(bench):
    c = bench.ClockSampler(0)
    assert c.summary()["reasons"] == ["unsampled"]
    c.rows = [(5.0, _row(1965, 500))]
    c.mark(0.0, 1.0)  # no sample inside the window: the last one stands in
    assert c.summary()["samples"] == 1


def test_max_over_ranks_without_process_group(bench):
    assert bench.max_over_ranks(1.25, None) == 1.25


def test_work_accounting(bench):
    assert bench.ax_flops(4096, 10) == 4096 * 1000 * 135      # 552,960,000 flop
    assert bench.ax_bytes(4096, 10) == 262_144_000            # u 8 + g 48 + w 8 B/point
