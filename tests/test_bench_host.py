"""CPU checks of bench.py's roofline arithmetic (no GPU): the per-expert FFN roofline and
the HBM-kernel block with the router's tensor-side bound."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def test_per_expert_roofline_bounds():
    d, F, tf, hbm = 4096, 14336, 1000.0, 5000.0  # TFLOP/s, GB/s
    heavy, light = 4096, 16
    r = bench.per_expert_roofline([heavy, light, 0], d, F, tf, hbm, ffn_ms=10.0)
    t_heavy = 6.0 * d * F * heavy / (tf * 1e12)  # tensor-bound: 1.44 ms
    t_light = (3.0 * d * F * 2 + light * (4.0 * d + 4.0 * F)) / (hbm * 1e9)  # weight streaming
    assert t_heavy > (3.0 * d * F * 2 + heavy * (4.0 * d + 4.0 * F)) / (hbm * 1e9)
    assert r["ms"] == pytest.approx(1e3 * (t_heavy + t_light))
    assert r["frac"] == pytest.approx(r["ms"] / 10.0)
    assert r["hbm_bound_experts"] == 1 and r["experts_with_rows"] == 2 and r["rows_min_max"] == [0, heavy]


def test_hbm_block_router_tensor_side():
    nbytes = (100e6, 200e6, 300e6)
    before = (0.02, 0.04, 0.06)  # ms
    out = bench.hbm_block(before, before, nbytes, 6000.0, {}, router_flops=60e9, tf_burst=1650.0)
    assert out["permute"]["GB/s"] == pytest.approx(100e6 / 20e-6 / 1e9)
    rg = out["router_gate"]
    assert rg["us"] == pytest.approx(60.0)
    assert rg["tensor"]["TFLOP/s"] == pytest.approx(60e9 / 60e-6 / 1e12)
    t_hbm, t_tc = 300e6 / 6000.0 / 1e3, 60e9 / 1650.0 / 1e6  # µs at each peak
    assert rg["roofline_us"]["hbm"] == pytest.approx(t_hbm) and rg["roofline_us"]["tensor"] == pytest.approx(t_tc)
    assert rg["roofline_us"]["bound"] == "hbm" and rg["roofline_us"]["frac_of_bound"] == pytest.approx(t_hbm / 60.0)
