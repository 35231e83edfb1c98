"""Host-side logic of bench.py (no GPU): which workload the committed ncu traffic applies to, and
the clock sampler's output shape.  DESIGN.md §8."""
import importlib.util
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench():
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def test_ncu_traffic_only_for_the_captured_workload():
    b = _bench()
    t = b.ncu_traffic(True, "configs[3]", 1)
    assert t is not None and t["bytes_per_launch"] > 4e11  # one configs[3] sweep moves > 400 GB
    assert b.ncu_traffic(True, "configs[2]", 1) is None
    assert b.ncu_traffic(True, "configs[4]", 1) is None
    assert b.ncu_traffic(True, "configs[3]", 4) is None  # 4 overlapped sweeps: not captured


def test_clock_sampler_reports_without_a_gpu():
    c = _bench().Clocks(0).stop()
    assert set(c) >= {"sm_mhz", "sm_max_mhz", "reasons"}
    assert isinstance(c["reasons"], list)
