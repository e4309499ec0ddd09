"""Host-side logic of bench.py (no GPU): the algorithmic byte models
(SURVEY.md §8d), the combined HBM + NVLink roofline, the clock-sample
parser, and the CPU-baseline helpers' bookkeeping."""

import math
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402


def test_byte_models_match_survey():
    n = 1024
    R = 8.0 * n**3
    S = 16.0 * n * n * (n // 2 + 1)
    assert bench.spec_bytes(n) == S
    assert bench.fft_bytes(n) == 2 * (R + 5 * S)          # one forward + one inverse, R2C
    assert bench.pfc_bytes(n) == 10 * S                   # fused PFC step
    assert bench.multi_bytes(n) == 17 * R + 93 * S


def test_combined_roofline_single_gpu_is_hbm_only():
    r = bench.combined_roofline(bench.pfc_bytes(1024), 2 * bench.spec_bytes(1024), 1, 6535.1, 20.0)
    assert r["t_nvlink_ms"] == 0.0 and r["nvlink_bytes_per_gpu"] == 0.0
    assert r["t_roof_ms"] == pytest.approx(1e3 * bench.pfc_bytes(1024) / 6535.1e9, abs=1e-4)  # rounded to 4 places
    assert r["frac"] == pytest.approx(r["t_roof_ms"] / 20.0, abs=1e-4)


def test_combined_roofline_survey_2048_g8():
    """2048^3 on 8 GPUs at 8 TB/s / 900 GB/s = 10.75 + 16.72 ms."""
    S = bench.spec_bytes(2048)
    r = bench.combined_roofline(bench.pfc_bytes(2048), 2 * S, 8, 8000.0, 27.47)
    nv = 2 * S * 7 / 64
    assert r["nvlink_bytes_per_gpu"] == pytest.approx(nv)
    assert r["t_hbm_ms"] == pytest.approx(10.75, abs=0.01)
    t_nom = 1e3 * (bench.pfc_bytes(2048) / (8 * 8000e9) + nv / 900e9)
    assert t_nom == pytest.approx(27.47, abs=0.02)
    assert r["frac_nominal_nvlink_900"] == pytest.approx(t_nom / 27.47, abs=1e-3)


def test_clock_sampler_summary_parses_reasons():
    c = bench.ClockSampler(0)
    c.lines = ["1965, 1965, 900.1, 0x4, Not Active, Not Active, Not Active, Active",
               "1800, 1965, 995.0, 0x4, Not Active, Not Active, Not Active, Active",
               "garbage"]
    s = c.summary()
    assert s["sm_mhz"] == pytest.approx(1882.5) and s["sm_max_mhz"] == 1965.0
    assert s["reasons"] == ["sw_power_cap"] and s["samples"] == 2


def test_cpu_info_reports_cores_and_model():
    info = bench.cpu_info()
    assert info["usable_cpus"] >= 1 and info["logical_cpus"] >= 1
    assert bench.cpu_threads() == info["usable_cpus"]


def test_kernel_table_aggregates_launches():
    class Ev:
        def __init__(self, t):
            self.t = t

        def elapsed_time(self, other):
            return other.t - self.t

    trace = [("pfcs_rfft_x", (0, 0, 512, 512 * 512, 0), Ev(0.0), Ev(0.5)),
             ("pfcs_rfft_x", (0, 0, 512, 512 * 512, 0), Ev(1.0), Ev(1.3))]
    t = bench.kernel_table(trace, 2)
    row = t["rfft_x"]
    alg = 512 * 512 * 512 * 8.0 + 257 * 512 * 512 * 16.0
    assert row["launches_per_step"] == 1.0 and row["avg_ms"] == pytest.approx(0.4)
    assert row["alg_gb_per_launch"] == pytest.approx(alg / 1e9, rel=1e-4)
    assert row["gbs"] == pytest.approx(alg / 0.4e-3 / 1e9, rel=1e-3)
