"""bench.py's clock sampler: only samples stamped inside the timed region count, a region shorter
than the sampling interval takes the first sample after it starts, throttle reasons are collected
(CPU test: synthetic nvidia-smi lines)."""
import datetime
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def _line(t, mhz, power_cap=False, thermal=False):
    ts = datetime.datetime.fromtimestamp(t).strftime("%Y/%m/%d %H:%M:%S.%f")[:-3]
    act = lambda b: "Active" if b else "Not Active"
    return f"{ts}, 0, {mhz}, 1965, 900.0, 0x0, {act(False)}, {act(thermal)}, {act(False)}, {act(power_cap)}"


def test_samples_inside_region_only():
    t0 = 1_700_000_000.0
    lines = [_line(t0 - 0.5, 1965), _line(t0 + 0.1, 1600, power_cap=True), _line(t0 + 0.2, 1700),
             _line(t0 + 0.3, 1650), _line(t0 + 5.0, 1965, thermal=True)]
    out = bench.Clocks.parse(lines, t0, t0 + 1.0)
    assert out["samples"] == 3 and out["sm_mhz"] == 1650 and out["sm_max_mhz"] == 1965
    assert out["reasons"] == ["sw_power_cap"]  # the thermal sample lies after the region


def test_short_region_takes_first_sample_after_start():
    t0 = 1_700_000_000.0
    lines = [_line(t0 - 0.05, 1965), _line(t0 + 0.03, 1800), "garbage", _line(t0 + 0.05, 1700)]
    out = bench.Clocks.parse(lines, t0, t0 + 0.01)
    assert out["samples"] == 1 and out["sm_mhz"] == 1800


def test_no_samples():
    out = bench.Clocks.parse([], 0.0, 1.0)
    assert out["samples"] == 0 and out["sm_mhz"] is None and out["reasons"] == []
