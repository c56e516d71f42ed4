"""B200 profiler's model fit (paper §4.2 pivot rule; reference ModelProfile keys)."""
from paper_2503_13737_b200.profiler import fit


def test_fit_recovers_linear_model_and_pivot():
    t0, a = 0.006, 20e-6  # 6 ms fixed + 20 us/token
    sizes = [64, 128, 256, 512, 1024, 2048, 4096]
    pts = [{"s_f": s, "seconds": t0 + a * s, "tokens_per_s": s / (t0 + a * s)} for s in sizes]
    prof = fit(pts, hidden=5120, num_layers=40, kvc_tokens=1000)
    assert abs(prof["fixed_overhead_s"] - t0) < 1e-9
    assert abs(prof["pivot_time_s"] / prof["pivot_forward_size"] - a) < 1e-12
    # smallest size whose throughput is within 3% of the best measured
    best = max(p["tokens_per_s"] for p in pts)
    expect = min(p["s_f"] for p in pts if p["tokens_per_s"] >= 0.97 * best)
    assert prof["pivot_forward_size"] == expect
    assert set(prof) == {"hidden_size", "num_layers", "pivot_forward_size", "pivot_time_s", "bytes_per_element",
                         "fixed_overhead_s", "kvc_capacity_tokens"}
