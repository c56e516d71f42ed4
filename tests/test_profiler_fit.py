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


def test_fit_extended_recovers_kv_and_pair_terms():
    """The mixed-batch fit (profiler.fit_extended) recovers T_0 + a*S_f + b*kv + c*pairs on exact data, the
    pivot stays the prefill sweep's, and the result loads as a ModelProfile whose batch_time reproduces it."""
    import numpy as np

    from paper_2503_13737_b200 import cost_model as cm
    from paper_2503_13737_b200.profiler import fit_extended, mixed_cases

    t0, a, b, c = 0.005, 18e-6, 1.1e-7, 2e-10
    pts = []
    for seqs in mixed_cases(8192, 80000) + [[(512, 0)] * k for k in (1, 2, 4, 8)]:
        kv, pairs = cm.batch_features(seqs)
        s_f = sum(q for q, _ in seqs)
        pts.append({"s_f": s_f, "kv_tokens": kv, "pairs": pairs, "seconds": t0 + a * s_f + b * kv + c * pairs})
    base = {"hidden_size": 5120, "num_layers": 40, "pivot_forward_size": 1536, "pivot_time_s": 0.0,
            "bytes_per_element": 2, "fixed_overhead_s": 0.0, "kvc_capacity_tokens": 3200}
    prof, err = fit_extended(pts, base)
    assert err["max_rel_err"] < 1e-9
    assert np.isclose(prof["fixed_overhead_s"], t0) and np.isclose(prof["pivot_time_s"], a * 1536)
    assert np.isclose(prof["kv_read_s_per_token"], b) and np.isclose(prof["attn_s_per_pair"], c)
    mp = cm.ModelProfile(**prof)
    for p in pts[:5]:
        assert np.isclose(cm.batch_time(p["s_f"], p["kv_tokens"], p["pairs"], mp), p["seconds"])
