"""The reference-API mirror (cost_model, kvc, workload, sched_core) vs fixtures generated from the
reference itself (tests/golden/make_golden.py imports /root/reference/pkg/src/slosim), plus the
SPEC.md worked examples for those modules.  Bit-exact: integer and float results must be equal."""
import json
import math
from pathlib import Path

import pytest

from paper_2503_13737_b200 import cost_model as cm
from paper_2503_13737_b200 import kvc
from paper_2503_13737_b200 import sched_core as sc
from paper_2503_13737_b200 import workload as wl
from paper_2503_13737_b200.errors import AllocationError, ConfigError, StateError, TraceParseError, ValidationError

G = Path(__file__).resolve().parent / "golden"


def _trace_cfgs():
    L, S = wl.LengthDist, wl.ScaleRule
    tiny = cm.ModelProfile(hidden_size=256, num_layers=2, pivot_forward_size=256, pivot_time_s=0.002,
                           kvc_capacity_tokens=65536)
    return {
        "default": dict(num_requests=300),
        "config1": dict(num_requests=64, arrival_rate=8.0, long_fraction=0.1, short_len_dist=L("uniform", 8, 256),
                        long_len_dist=L("uniform", 4096, 8192), output_len_dist=L("uniform", 1, 64),
                        tbt_scale=S("choice", (0.5, 1.0, 2.0)), seed=0, profile=tiny),
        "config2": dict(num_requests=400, arrival_rate=8.0, long_fraction=0.1, short_len_dist=L("uniform", 10, 1024),
                        long_len_dist=L("log_uniform", 4096, 16384), output_len_dist=L("uniform", 1, 2048), seed=0),
        "paper_tbt_set": dict(num_requests=200, tbt_scale=S("choice", (0.25, 0.5, 1.0, 2.0)), seed=3),
        "offline_mix": dict(num_requests=200, offline_fraction=0.3, seed=5, profile=cm.opt_175b_like()),
        "choice_weights": dict(num_requests=150, short_len_dist=L("choice", values=(16, 64, 256), weights=(0.5, 0.3, 0.2)),
                               output_len_dist=L("choice", values=(1, 8, 32)), seed=11),
    }


@pytest.mark.parametrize("name", list(_trace_cfgs()))
def test_generate_trace_bit_identical_to_reference(name):
    golden = json.loads((G / "traces.json").read_text())[name]
    ours = wl.generate_trace(wl.TraceConfig(**_trace_cfgs()[name]))
    assert len(ours) == len(golden)
    for r, g in zip(ours, golden):
        slo = {"kind": r.slo.kind.value, "ttft": r.slo.ttft_slo, "tbt": r.slo.tbt_slo, "jct": r.slo.jct_slo}
        assert [r.id, r.arrival_time, r.prompt_len, r.output_len, r.predicted_output_len, slo] == g


def test_trace_roundtrip_and_errors(tmp_path):
    tr = wl.generate_trace(wl.TraceConfig(num_requests=20, seed=1))
    p = tmp_path / "t.jsonl"
    wl.save_trace(reversed(tr), p)
    back = wl.load_trace(p)
    assert [r.id for r in back] == [r.id for r in tr]  # re-sorted by arrival
    (tmp_path / "bad.jsonl").write_text('{"id": 1, "arrival": 0.0, "prompt": 0, "output": 1, '
                                        '"slo": {"kind": "online", "ttft": 0.5, "tbt": 0.1875}}\n')
    with pytest.raises(ValidationError):
        wl.load_trace(tmp_path / "bad.jsonl")
    (tmp_path / "bad2.jsonl").write_text("{not json\n")
    with pytest.raises(TraceParseError, match="line 1"):
        wl.load_trace(tmp_path / "bad2.jsonl")
    with pytest.raises(ConfigError):
        wl.TraceConfig(arrival_rate=0)


def test_trace_spec_examples():
    # SPEC.md:49-51
    tr = wl.generate_trace(wl.TraceConfig(num_requests=300, tbt_scale=wl.ScaleRule("choice", (0.25, 0.5, 1.0, 2.0))))
    assert {r.slo.tbt_slo for r in tr} <= {0.046875, 0.09375, 0.1875, 0.375}
    assert all(r.prompt_len < 4096 for r in wl.generate_trace(wl.TraceConfig(num_requests=300, long_fraction=0.0)))
    big = wl.generate_trace(wl.TraceConfig(num_requests=10000))
    s = wl.trace_summary(big)
    assert abs(s["empirical_rate"] - 8.0) / 8.0 < 0.05 and abs(s["long_fraction"] - 0.35) < 0.02


def test_cost_model_matches_reference():
    g = json.loads((G / "cost_model.json").read_text())
    for s, h, f, a, l in g["ops"]:
        assert (cm.fcl_ops(s, h), cm.attention_ops(s, h), cm.layer_ops(s, h)) == (f, a, l)
    p13, p175 = cm.opt_13b_like(), cm.opt_175b_like()
    for s, t13, t175 in g["iteration_time"]:
        assert cm.iteration_time(s, p13) == t13 and cm.iteration_time(s, p175) == t175
    assert [cm.kvc_bytes_per_token(p13), cm.kvc_bytes_per_token(p175)] == g["kvc_bytes"]
    gp = cm.GpuProfile(peak_flops=126.96e12)
    assert [cm.derive_pivot(5120, 40, gp), cm.derive_pivot_time(768, 5120, 40, gp)] == g["derive_pivot"]
    for n, v in g["base_ttft"]:
        assert wl.base_ttft(n, p13) == v


def test_cost_model_spec_examples(tmp_path):
    assert cm.fcl_ops(2, 3) == 432 and cm.attention_ops(3, 2) == 72 and cm.layer_ops(6, 1) == 288
    prof = cm.ModelProfile(hidden_size=3, num_layers=2, pivot_forward_size=768, pivot_time_s=0.08)
    assert cm.kvc_bytes_per_token(prof) == 24
    assert cm.iteration_time(384, prof) == 0.04 and cm.iteration_time(768, prof) == 0.08
    with pytest.raises(ValidationError):
        cm.ModelProfile(hidden_size=0, num_layers=1, pivot_forward_size=1, pivot_time_s=1)
    p = tmp_path / "prof.json"
    cm.save_profile(cm.opt_13b_like(), p)
    assert cm.load_profile(p) == cm.opt_13b_like()
    p.write_text('{"hidden_size": 1, "num_layers": 1, "pivot_forward_size": 1, "pivot_time_s": 1, "x": 2}')
    with pytest.raises(ConfigError):
        cm.load_profile(p)
    # acceptance 1: identity on random pairs
    import random
    rng = random.Random(0)
    for _ in range(10000):
        s, h = rng.randrange(0, 10 ** 6), rng.randrange(1, 8193)
        assert cm.layer_ops(s, h) == cm.fcl_ops(s, h) + cm.attention_ops(s, h)


def test_blockpool_replays_reference_sequence():
    ops = json.loads((G / "kvc_ops.json").read_text())
    pool = kvc.BlockPool(total_blocks=400, block_size=32)
    for step in ops:
        op = step["op"]
        kind, rid = op[0], op[1]
        if kind == "chunk":
            d = pool.demand_prompt_chunk(rid, op[2]) if rid not in pool.swapped_out else pool.demand_readmit(rid)
            assert [d.tokens_needed, d.blocks_needed] == op[3:5]
            pool.allocate(rid, d)
        elif kind == "chunk_nofit":
            d = pool.demand_prompt_chunk(rid, op[2]) if rid not in pool.swapped_out else pool.demand_readmit(rid)
            assert [d.tokens_needed, d.blocks_needed] == op[3:5]
        elif kind == "tg":
            d = pool.demand_tg(rid)
            assert [d.tokens_needed, d.blocks_needed] == op[2:4]
            if d.blocks_needed <= pool.free_blocks:
                pool.allocate(rid, d)
        elif kind == "preempt":
            assert pool.preempt(rid) == op[2]
        elif kind == "release":
            pool.release(rid)
        pool.check_conservation()
        assert pool.free_blocks == step["free"]
        assert {str(r): [pool.blocks_held(r), pool.tokens_stored(r)] for r in sorted(pool.resident_ids())} == step["held"]
        assert {str(k): v for k, v in sorted(pool.swapped_out.items())} == step["swapped"]


def test_blockpool_physical_ids_and_spec_examples():
    pool = kvc.BlockPool(8, 32)
    assert pool.demand_prompt_chunk(1, 33).blocks_needed == 2
    pool.allocate(1, pool.demand_prompt_chunk(1, 33))
    assert pool.block_table(1) == [0, 1] and pool.slots(1, 31, 3) == [31, 32, 33]
    pool.allocate(2, pool.demand_prompt_chunk(2, 10))
    assert pool.block_table(2) == [2]
    pool.release(1)
    pool.allocate(3, pool.demand_prompt_chunk(3, 70))
    assert pool.block_table(3) == [0, 1, 3]  # lowest free ids first
    assert pool.preempt(3) == 70 and pool.demand_readmit(3).blocks_needed == 3
    with pytest.raises(StateError):
        pool.preempt(3)
    with pytest.raises(AllocationError):
        pool.allocate(9, kvc.KvcDemand(320, 10))
    p128 = kvc.BlockPool(10, 128)  # 129 TG tokens at b=128 -> 2 blocks
    p128.allocate(5, p128.demand_prompt_chunk(5, 1))
    for _ in range(128):
        p128.allocate(5, p128.demand_tg(5))
    assert p128.blocks_held(5) == 2
    assert kvc.orca_reservation(8, 8192) == 65536


def test_blockpool_conservation_random():
    """Acceptance 2: 10k random ops never break conservation; tables stay disjoint."""
    import random
    rng = random.Random(5)
    pool = kvc.BlockPool(300, 32)
    for _ in range(10000):
        rid = rng.randrange(30)
        r = rng.random()
        if r < 0.5:
            d = pool.demand_readmit(rid) if rid in pool.swapped_out else pool.demand_prompt_chunk(rid, rng.randrange(1, 200))
            if d.blocks_needed <= pool.free_blocks:
                pool.allocate(rid, d)
        elif r < 0.7 and pool.is_resident(rid):
            d = pool.demand_tg(rid)
            if d.blocks_needed <= pool.free_blocks:
                pool.allocate(rid, d)
        elif r < 0.85 and pool.is_resident(rid):
            pool.preempt(rid)
        elif pool.is_resident(rid):
            pool.release(rid)
        pool.check_conservation()
        for q in pool.resident_ids():
            assert len(pool.block_table(q)) * 32 == math.ceil(pool.tokens_stored(q) / 32) * 32


def _entry(c):
    if c["online"]:
        slo = wl.SLOSpec(kind=wl.SLOKind.ONLINE, ttft_slo=c["ttft"], tbt_slo=c["tbt"])
    else:
        slo = wl.SLOSpec(kind=wl.SLOKind.OFFLINE, jct_slo=c["jct"])
    spec = wl.RequestSpec(id=c["id"], arrival_time=c["arrival"], prompt_len=c["prompt"], output_len=c["output"], slo=slo)
    return sc.QueueEntry(request=spec, phase=sc.Phase(c["phase"]), remaining_prompt_tokens=c["remaining"],
                         seq_len=c["seq_len"], enqueue_time=c["enqueue"], is_long=spec.is_long(), seq=c["seq"],
                         iter_allowance=c["allow"], debt=c["debt"])


def test_sched_core_matches_reference():
    g = json.loads((G / "sched_core.json").read_text())
    stats = sc.ChunkStats(avg_chunk_len=g["stats"][0], t_max=g["stats"][1])
    entries = [_entry(c) for c in g["cases"]]
    for e, c in zip(entries, g["cases"]):
        tr = sc.remaining_time(e, g["now"], stats)
        assert tr == c["t_r"] and sc.is_urgent(tr, stats) == c["urgent"]
        if not c["online"]:
            est = sc.jct_initial_estimate(e.request, stats)
            assert est == c["jct_est"] and sc.jct_allowance(e.request, est, stats) == c["jct_allow"]
    assert [e.request_id for e in sc.order_queue(entries, g["now"], stats)] == g["order"]
    cs = sc.ChunkStats(avg_chunk_len=768.0, t_max=0.156)
    for ev, avg, prob, pmax in g["chunk_stats"]:
        if ev[0] == "c":
            cs.observe_chunk(int(ev[1:]))
        elif ev == "t":
            cs.observe_tg_step()
        elif ev == "p":
            cs.observe_preemption()
        else:
            cs.observe_preemption_duration(float(ev[1:]))
        assert [cs.avg_chunk_len, cs.preempt_prob, cs.preempt_max_s] == [avg, prob, pmax]


def test_sched_core_spec_examples():
    stats = sc.ChunkStats(avg_chunk_len=512, t_max=0.08)
    assert sc.remaining_chunks(0, stats) == 1 and sc.remaining_chunks(1537, stats) == 4
    assert sc.remaining_chunks(512, stats) == 1
    spec = wl.RequestSpec(id=0, arrival_time=0, prompt_len=2048, output_len=10,
                          slo=wl.SLOSpec(kind=wl.SLOKind.OFFLINE, jct_slo=3.12))
    s2 = sc.ChunkStats(avg_chunk_len=512, t_max=0.08, preempt_prob=0.1, preempt_max_s=1.0)
    assert math.isclose(sc.jct_initial_estimate(spec, s2), 2.12)
    assert math.isclose(sc.jct_allowance(spec, 2.12, s2), 1.0 / 14)
    e = sc.QueueEntry(request=spec, phase=sc.Phase.PROMPT_PENDING, remaining_prompt_tokens=10, seq_len=0,
                      enqueue_time=0.0, is_long=False, iter_allowance=0.1)
    sc.propagate_debt(e, 0.15)
    assert math.isclose(e.effective_allowance(), 0.05)
    sc.propagate_debt(e, 0.05)  # under-wait d back: telescopes
    assert math.isclose(e.debt, 0.0, abs_tol=1e-12)
    assert sc.is_urgent(0.08, stats) and not sc.is_urgent(0.8, stats) and sc.is_urgent(-1.0, stats)
