"""Host-side helpers of the measurement scripts: the alpha-B fit of scripts/sweep_bench.py
recovers a known latency / bandwidth exactly from noiseless points of t = alpha + x / B."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "scripts"))


def test_alpha_b_fit_recovers_model():
    from sweep_bench import fit_alpha_B
    W = 4
    alpha, B = 30.0, 650.0                  # us, GB/s (bus bytes)
    lines = []
    for lg in range(16, 31):
        ag = 1 << lg
        x_u = ag * (W - 1) / W
        x_r = 2 * ag * (W - 1) / W
        lines.append({"variant": "v", "ag_bytes": ag, "unshard_us": alpha + x_u / (B * 1e3),
                      "rs_us": 2 * alpha + x_r / (2 * B * 1e3)})
    fits = {f["op"]: f for f in fit_alpha_B(lines, W)}
    assert abs(fits["unshard"]["alpha_us"] - alpha) < 0.01
    assert abs(fits["unshard"]["B_GBps"] - B) < 0.1
    assert abs(fits["reduce_scatter"]["alpha_us"] - 2 * alpha) < 0.01
    assert abs(fits["reduce_scatter"]["B_GBps"] - 2 * B) < 0.2
    assert fit_alpha_B(lines, 1) == []      # W = 1 has no bus bytes
