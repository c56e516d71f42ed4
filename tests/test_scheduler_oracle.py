"""Scheduler decisions of the product (policies.py + engine.py) vs the brute-force oracle
restatement (oracle/sched.py): chunk sizes, batch composition, preemptions and physical KV block
tables must be identical step for step under the virtual clock (north_star: bit-exact)."""
import pytest

from oracle.sched import OracleScheduler
from paper_2503_13737_b200 import configs, cost_model as cm, workload as wl
from paper_2503_13737_b200.engine import Engine
from paper_2503_13737_b200.policies import PolicyConfig


def _compare(trace, prof, kv_blocks=None, max_steps=None, kv_victim="resident_last", kv_watermark=0.0,
             retain_tg=False, live_only=False):
    eng = Engine(trace, prof, PolicyConfig(kv_victim=kv_victim, kv_watermark=kv_watermark, retain_tg=retain_tg,
                                           budget_live_only=live_only),
                 kv_blocks=kv_blocks, check_invariants=True)
    eng.keep_history = True
    eng.run(max_steps=max_steps)
    orc = OracleScheduler(trace, prof, kv_blocks=kv_blocks, kv_victim=kv_victim, kv_watermark=kv_watermark,
                          retain_tg=retain_tg, budget_live_only=live_only)
    log = orc.run(max_steps=max_steps)
    assert len(log) == len(eng.plans)
    for i, (plan, tables, ref) in enumerate(zip(eng.plans, eng.tables, log)):
        ours = [(s.request_id, s.chunk_len, s.is_final_chunk) for s in plan.selections]
        assert ours == [(r, c, f) for r, c, f, _ in ref["sel"]], f"step {i}"
        assert plan.token_budget == ref["s_b"], f"step {i}"
        assert plan.preempted == ref["preempted"], f"step {i}"
        assert {r: list(map(int, t)) for r, t in tables.items()} == ref["tables"], f"step {i}"
    return len(log)


def test_config1_decisions_match_oracle():
    c = configs.config1()
    n = _compare(wl.generate_trace(c.trace), c.trace.profile)
    assert n > 1000


@pytest.mark.parametrize("kv_victim,kv_watermark,retain_tg", [("resident_last", 0.0, False), ("max_tr", 0.0, False),
                                                              ("resident_last", 0.1, False),
                                                              ("resident_last", 0.1, True)])
def test_kv_pressure_with_preemption_matches_oracle(kv_victim, kv_watermark, retain_tg):
    """Small KV pool (paper-like capped regime): urgency, preemption (swap-out) and readmission, under
    both KV-deficit victim rules and with an admission watermark."""
    c = configs.config1()
    prof = cm.ModelProfile(hidden_size=256, num_layers=2, pivot_forward_size=256, pivot_time_s=0.002,
                           fixed_overhead_s=0.002, kvc_capacity_tokens=48 * 32)
    trace = wl.generate_trace(wl.TraceConfig(**{**c.trace.__dict__, "num_requests": 40, "profile": prof,
                                                "long_fraction": 0.0,
                                                "output_len_dist": wl.LengthDist("uniform", 100, 400)}))
    eng = Engine(trace, prof, PolicyConfig(kv_victim=kv_victim, kv_watermark=kv_watermark, retain_tg=retain_tg),
                 kv_blocks=48)
    assert eng.run().preemptions > 5  # the scenario really exercises preemption
    n = _compare(trace, prof, kv_blocks=48, kv_victim=kv_victim, kv_watermark=kv_watermark, retain_tg=retain_tg)
    assert n > 1000


def test_b200_like_profile_with_offline_matches_oracle():
    prof = cm.ModelProfile(hidden_size=5120, num_layers=40, pivot_forward_size=2048, pivot_time_s=0.05,
                           fixed_overhead_s=0.005, kvc_capacity_tokens=60000)
    cfg = configs.config5(profile=prof, num_requests=120, arrival_rate=12.0).trace
    _compare(wl.generate_trace(cfg), prof, max_steps=2000)


def test_extended_cost_model_matches_oracle():
    """The B200 extension of the cost model (K/V-read and attention-pair terms, cost_model.batch_time)
    drives the virtual clock of both sides with the same float expression: decisions stay bit-exact
    under KV pressure with preemptions, and the clock differs from the linear model's."""
    c = configs.config1()
    prof = cm.ModelProfile(hidden_size=256, num_layers=2, pivot_forward_size=256, pivot_time_s=0.002,
                           fixed_overhead_s=0.002, kvc_capacity_tokens=48 * 32, kv_read_s_per_token=2e-6,
                           attn_s_per_pair=3e-9)
    trace = wl.generate_trace(wl.TraceConfig(**{**c.trace.__dict__, "num_requests": 40, "profile": prof,
                                                "long_fraction": 0.0,
                                                "output_len_dist": wl.LengthDist("uniform", 100, 400)}))
    n = _compare(trace, prof, kv_blocks=48)
    assert n > 1000
    lin = cm.ModelProfile(**{**prof.__dict__, "kv_read_s_per_token": 0.0, "attn_s_per_pair": 0.0})
    e1, e2 = Engine(trace, prof, PolicyConfig(), kv_blocks=48), Engine(trace, lin, PolicyConfig(), kv_blocks=48)
    assert e1.run().makespan > e2.run().makespan


def test_batch_time_reduces_to_reference_linear_model():
    prof = cm.opt_13b_like()
    for s_f, kv, pairs in ((0, 0, 0), (768, 5000, 123456), (1, 2049, 2049)):
        assert cm.batch_time(s_f, kv, pairs, prof) == cm.iteration_time(s_f, prof)
    ext = cm.ModelProfile(**{**prof.__dict__, "kv_read_s_per_token": 1e-7, "attn_s_per_pair": 1e-9})
    assert cm.batch_features([(1, 2048), (512, 0)]) == (2049 + 512, 2049 + 512 * 513 // 2)
    assert cm.batch_time(768, 1000, 10, ext) == cm.iteration_time(768, prof) + 1e-7 * 1000 + 1e-9 * 10


def test_retain_tg_matches_oracle_b200_profile():
    """PAPER §4.4 TG retention on a B200-like profile with a large pool (decodes join B every step)."""
    prof = cm.ModelProfile(hidden_size=5120, num_layers=40, pivot_forward_size=1536, pivot_time_s=0.0367,
                           fixed_overhead_s=0.0037, kvc_capacity_tokens=40000, kv_read_s_per_token=1.4e-7,
                           attn_s_per_pair=7e-10)
    cfg = configs.config2(profile=prof, num_requests=150, arrival_rate=6.0).trace
    trace = wl.generate_trace(cfg)
    _compare(trace, prof, max_steps=1500, kv_watermark=0.1, retain_tg=True)
    _compare(trace, prof, max_steps=1500, kv_watermark=0.1, retain_tg=True, live_only=True)
