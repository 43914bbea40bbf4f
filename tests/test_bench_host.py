"""Host-side logic of bench.py (no GPU): the clock summary the driver checks for throttling, the
peak choice, and the reference arm's JSON line shape."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def _sampler(rows, source="nvml, 5 ms"):
    c = bench.ClockSampler(0)
    c.rows = rows
    c.source = source
    return c.summary()


def test_clock_summary_reports_median_min_and_cap_fraction():
    rows = [(1965.0, 1965.0, [])] * 6 + [(1470.0, 1965.0, ["sw_power_cap"])] * 4
    s = _sampler(rows)
    assert s["sm_mhz"] == 1965.0 and s["sm_min_mhz"] == 1470.0 and s["sm_max_mhz"] == 1965.0
    assert s["reasons"] == ["sw_power_cap"] and s["samples"] == 10
    assert abs(s["sw_power_cap_frac"] - 0.4) < 1e-12


def test_clock_summary_lists_every_throttle_reason_once():
    rows = [(1800.0, 1965.0, ["hw_slowdown"]), (1700.0, 1965.0, ["hw_slowdown", "sw_thermal_slowdown"])]
    s = _sampler(rows)
    assert s["reasons"] == ["hw_slowdown", "sw_thermal_slowdown"]
    assert s["sm_mhz"] == 1750.0


def test_clock_summary_without_samples():
    s = _sampler([])
    assert s["sm_mhz"] is None and s["reasons"] == ["clock sampling unavailable"]


def test_sampler_drops_idle_samples_taken_before_the_timed_region(monkeypatch):
    """__enter__ waits for the sampler to come up and discards what it saw while idle."""
    import threading
    sampled = threading.Event()
    c = bench.ClockSampler(0)

    def idle_sample():  # the sampler's first (idle) sample
        c.rows.append((1000.0, 1965.0, []))
        sampled.set()

    c._run = idle_sample
    monkeypatch.setattr(bench.time, "sleep", lambda s: sampled.wait(5))  # "sleep" until the sampler is up
    with c:
        pass
    assert c.rows == []


@pytest.mark.parametrize("impl_args", [["--impl", "reference", "--steps", "1", "--warmup", "0", "--seq", "2048"]])
def test_reference_arm_line(impl_args):
    """--impl reference runs the f64 oracle on host cores and prints one JSON line with the
    base contract's keys plus impl / cpu_baseline / e2e (no GPU needed)."""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + impl_args, capture_output=True, text=True,
                         timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "config",
                "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["value"] > 0 and d["dtype"] == "f64"
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
