"""bench.py host helpers on CPU: the clock sampler's per-job gating and its summary (the clocks
line the driver checks for throttling)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def test_clock_sampler_off_on_non_zero_local_ranks():
    c = bench.Clocks(None)
    with c:
        assert c.proc is None
    assert c.summary()["reasons"] == ["unsampled"]


def test_clock_summary_reads_every_gpu_and_reasons():
    c = bench.Clocks("0,1")
    # rows as nvidia-smi prints them for two GPUs: sm, max sm, hw, hw thermal, sw thermal, power cap
    c.samples = [["1965", "1965", "Not Active", "Not Active", "Not Active", "Active"],
                 ["1950", "1965", "Not Active", "Not Active", "Not Active", "Not Active"],
                 ["1965", "1965", "Not Active", "Not Active", "Not Active", "Not Active"]]
    s = c.summary()
    assert s["sm_mhz"] == 1965.0 and s["sm_max_mhz"] == 1965.0
    assert s["reasons"] == ["sw_power_cap"]
    assert s["samples"] == 3
