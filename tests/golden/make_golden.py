"""Regenerate the golden fixtures in tests/golden/ (run HERE, where /root/reference exists).

  traces.json       reference slosim.workload.generate_trace on 6 TraceConfigs
  kvc_ops.json      a 3000-op random demand/allocate/release/preempt/readmit sequence on the
                    reference slosim.kvc.BlockPool with the state after every op
  sched_core.json   remaining_time / is_urgent / order_queue / JCT estimates / ChunkStats from
                    reference slosim.sched_core on random entries
  cost_model.json   reference cost-model values on sample points
  opt_tiny_hf.pt    transformers 5.5.0 OPTForCausalLM (fp32) logits for the tiny config with the
                    weights of paper_2503_13737_b200.model.init_weights(tiny, seed=0, init="test")

Usage:  python tests/golden/make_golden.py
The GPU box never reads /root/reference; it only reads these committed files.
"""
import json
import random
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(ROOT))

from slosim import cost_model as rcm, kvc as rkvc, sched_core as rsc, workload as rwl  # noqa: E402


def trace_cfgs():
    L, S = rwl.LengthDist, rwl.ScaleRule
    tiny_prof = rcm.ModelProfile(hidden_size=256, num_layers=2, pivot_forward_size=256, pivot_time_s=0.002,
                                 kvc_capacity_tokens=65536)
    return {
        "default": dict(num_requests=300),
        "config1": dict(num_requests=64, arrival_rate=8.0, long_fraction=0.1, short_len_dist=L("uniform", 8, 256),
                        long_len_dist=L("uniform", 4096, 8192), output_len_dist=L("uniform", 1, 64),
                        tbt_scale=S("choice", (0.5, 1.0, 2.0)), seed=0, profile=tiny_prof),
        "config2": dict(num_requests=400, arrival_rate=8.0, long_fraction=0.1, short_len_dist=L("uniform", 10, 1024),
                        long_len_dist=L("log_uniform", 4096, 16384), output_len_dist=L("uniform", 1, 2048), seed=0),
        "paper_tbt_set": dict(num_requests=200, tbt_scale=S("choice", (0.25, 0.5, 1.0, 2.0)), seed=3),
        "offline_mix": dict(num_requests=200, offline_fraction=0.3, seed=5,
                            profile=rcm.opt_175b_like()),
        "choice_weights": dict(num_requests=150, short_len_dist=L("choice", values=(16, 64, 256), weights=(0.5, 0.3, 0.2)),
                               output_len_dist=L("choice", values=(1, 8, 32)), seed=11),
    }


def slo_json(s):
    return {"kind": s.kind.value, "ttft": s.ttft_slo, "tbt": s.tbt_slo, "jct": s.jct_slo}


def make_traces():
    out = {}
    for name, kw in trace_cfgs().items():
        tr = rwl.generate_trace(rwl.TraceConfig(**kw))
        out[name] = [[r.id, r.arrival_time, r.prompt_len, r.output_len, r.predicted_output_len, slo_json(r.slo)]
                     for r in tr]
    (HERE / "traces.json").write_text(json.dumps(out))


def make_kvc():
    rng = random.Random(1234)
    pool = rkvc.BlockPool(total_blocks=400, block_size=32)
    ops = []
    live = set()
    for i in range(3000):
        r = rng.random()
        rid = rng.randrange(40)
        rec = None
        try:
            if r < 0.45:
                c = rng.choice([1, 5, 31, 32, 33, 64, 100, 250])
                d = pool.demand_prompt_chunk(rid, c) if rid not in pool.swapped_out else pool.demand_readmit(rid)
                if d.blocks_needed <= pool.free_blocks:
                    pool.allocate(rid, d)
                    rec = ["chunk", rid, c, d.tokens_needed, d.blocks_needed]
                else:
                    rec = ["chunk_nofit", rid, c, d.tokens_needed, d.blocks_needed]
            elif r < 0.75 and pool.is_resident(rid):
                d = pool.demand_tg(rid)
                if d.blocks_needed <= pool.free_blocks:
                    pool.allocate(rid, d)
                rec = ["tg", rid, d.tokens_needed, d.blocks_needed]
            elif r < 0.85 and pool.is_resident(rid):
                rec = ["preempt", rid, pool.preempt(rid)]
            elif r < 0.95 and pool.is_resident(rid):
                pool.release(rid)
                rec = ["release", rid]
            else:
                rec = ["noop", rid]
        except rkvc.StateError if hasattr(rkvc, "StateError") else Exception as exc:  # pragma: no cover
            rec = ["error", rid, type(exc).__name__]
        pool.check_conservation()
        held = {str(k): list(v) for k, v in sorted(pool._held.items())}
        ops.append({"op": rec, "free": pool.free_blocks, "held": held,
                    "swapped": {str(k): v for k, v in sorted(pool.swapped_out.items())}})
    (HERE / "kvc_ops.json").write_text(json.dumps(ops))


def make_sched_core():
    rng = np.random.default_rng(7)
    stats = rsc.ChunkStats(avg_chunk_len=512.0, t_max=0.08)
    cases = []
    entries = []
    for i in range(60):
        online = rng.random() < 0.8
        if online:
            slo = rwl.SLOSpec(kind=rwl.SLOKind.ONLINE, ttft_slo=float(rng.uniform(0.05, 2.0)),
                              tbt_slo=float(rng.uniform(0.05, 0.4)))
        else:
            slo = rwl.SLOSpec(kind=rwl.SLOKind.OFFLINE, jct_slo=float(rng.uniform(1.0, 50.0)))
        spec = rwl.RequestSpec(id=i, arrival_time=float(rng.uniform(0, 5)), prompt_len=int(rng.integers(1, 9000)),
                               output_len=int(rng.integers(1, 500)), slo=slo)
        phase = [rsc.Phase.PROMPT_PENDING, rsc.Phase.TG_READY, rsc.Phase.PREEMPTED][int(rng.integers(0, 3))]
        e = rsc.QueueEntry(request=spec, phase=phase,
                           remaining_prompt_tokens=int(rng.integers(1, spec.prompt_len + 1)) if phase is rsc.Phase.PROMPT_PENDING else 0,
                           seq_len=int(rng.integers(0, 100)), enqueue_time=float(rng.uniform(0, 5)),
                           is_long=spec.is_long(), seq=int(rng.integers(0, 5)),
                           iter_allowance=float(rng.uniform(-0.1, 0.5)), debt=float(rng.uniform(-0.2, 0.2)))
        entries.append(e)
        now = 6.0
        tr = rsc.remaining_time(e, now, stats)
        est = rsc.jct_initial_estimate(spec, stats) if not online else None
        cases.append({"id": i, "online": online, "ttft": slo.ttft_slo, "tbt": slo.tbt_slo, "jct": slo.jct_slo,
                      "arrival": spec.arrival_time, "prompt": spec.prompt_len, "output": spec.output_len,
                      "phase": phase.value, "remaining": e.remaining_prompt_tokens, "seq_len": e.seq_len,
                      "enqueue": e.enqueue_time, "seq": e.seq, "allow": e.iter_allowance, "debt": e.debt,
                      "t_r": tr, "urgent": rsc.is_urgent(tr, stats),
                      "jct_est": est, "jct_allow": rsc.jct_allowance(spec, est, stats) if est is not None else None})
    order = [e.request_id for e in rsc.order_queue(entries, 6.0, stats)]
    cs = rsc.ChunkStats(avg_chunk_len=768.0, t_max=0.156)
    trail = []
    for ev in ["c100", "t", "p", "t", "p", "p", "c2048", "t", "d0.5", "c1", "t", "d0.2"]:
        if ev[0] == "c":
            cs.observe_chunk(int(ev[1:]))
        elif ev == "t":
            cs.observe_tg_step()
        elif ev == "p":
            cs.observe_preemption()
        else:
            cs.observe_preemption_duration(float(ev[1:]))
        trail.append([ev, cs.avg_chunk_len, cs.preempt_prob, cs.preempt_max_s])
    (HERE / "sched_core.json").write_text(json.dumps({"stats": [512.0, 0.08], "now": 6.0, "cases": cases,
                                                      "order": order, "chunk_stats": trail}))


def make_cost_model():
    pts = [(0, 1), (1, 1), (2, 3), (6, 1), (768, 5120), (1280, 12288), (100000, 8192)]
    out = {"ops": [[s, h, rcm.fcl_ops(s, h), rcm.attention_ops(s, h), rcm.layer_ops(s, h)] for s, h in pts]}
    p13, p175 = rcm.opt_13b_like(), rcm.opt_175b_like()
    out["iteration_time"] = [[s, rcm.iteration_time(s, p13), rcm.iteration_time(s, p175)] for s in (0, 1, 384, 768, 5000)]
    out["kvc_bytes"] = [rcm.kvc_bytes_per_token(p13), rcm.kvc_bytes_per_token(p175)]
    g = rcm.GpuProfile(peak_flops=126.96e12)
    out["derive_pivot"] = [rcm.derive_pivot(5120, 40, g), rcm.derive_pivot_time(768, 5120, 40, g)]
    out["base_ttft"] = [[n, rwl.base_ttft(n, p13)] for n in (1, 511, 512, 513, 4096, 100000)]
    (HERE / "cost_model.json").write_text(json.dumps(out))


def make_hf():
    import torch
    from transformers import OPTConfig, OPTForCausalLM
    from paper_2503_13737_b200 import model as M
    cfg = M.tiny()
    w = M.init_weights(cfg, seed=0, init="test")
    hc = OPTConfig(vocab_size=cfg.vocab, hidden_size=cfg.hidden, num_hidden_layers=cfg.num_layers, ffn_dim=cfg.ffn,
                   num_attention_heads=cfg.num_heads, max_position_embeddings=cfg.max_positions,
                   do_layer_norm_before=True, word_embed_proj_dim=cfg.hidden, enable_bias=True,
                   layer_norm_elementwise_affine=True, activation_function="relu", dropout=0.0,
                   attention_dropout=0.0, pad_token_id=1)
    hf = OPTForCausalLM(hc).eval().float()
    f = lambda t: t.float()
    H = cfg.hidden
    sd = {"model.decoder.embed_tokens.weight": f(w["tok_emb"]), "model.decoder.embed_positions.weight": f(w["pos_emb"]),
          "model.decoder.final_layer_norm.weight": f(w["final_g"]), "model.decoder.final_layer_norm.bias": f(w["final_b"]),
          "lm_head.weight": f(w["tok_emb"])}
    for i, L in enumerate(w["layers"]):
        p = f"model.decoder.layers.{i}."
        for j, n in enumerate(("q_proj", "k_proj", "v_proj")):
            sd[p + f"self_attn.{n}.weight"] = f(L["qkv_w"][j * H:(j + 1) * H])
            sd[p + f"self_attn.{n}.bias"] = f(L["qkv_b"][j * H:(j + 1) * H])
        sd[p + "self_attn.out_proj.weight"], sd[p + "self_attn.out_proj.bias"] = f(L["out_w"]), f(L["out_b"])
        sd[p + "self_attn_layer_norm.weight"], sd[p + "self_attn_layer_norm.bias"] = f(L["ln1_g"]), f(L["ln1_b"])
        sd[p + "final_layer_norm.weight"], sd[p + "final_layer_norm.bias"] = f(L["ln2_g"]), f(L["ln2_b"])
        sd[p + "fc1.weight"], sd[p + "fc1.bias"] = f(L["fc1_w"]), f(L["fc1_b"])
        sd[p + "fc2.weight"], sd[p + "fc2.bias"] = f(L["fc2_w"]), f(L["fc2_b"])
    missing, unexpected = hf.load_state_dict(sd, strict=False)
    assert not unexpected, unexpected
    assert all("lm_head" in m or "embed_positions" in m for m in missing), missing
    g = torch.Generator().manual_seed(42)
    ids = torch.randint(4, cfg.vocab, (1, 77), generator=g)
    with torch.no_grad():
        logits = hf(input_ids=ids, attention_mask=torch.ones_like(ids)).logits[0]
    rows = [0, 40, 76]
    torch.save({"input_ids": ids[0].to(torch.int32), "rows": rows, "logits_head": logits[rows, :4096].clone(),
                "argmax": logits[rows].argmax(-1).to(torch.int32), "lse": torch.logsumexp(logits[rows], -1),
                "transformers": __import__("transformers").__version__}, HERE / "opt_tiny_hf.pt")


if __name__ == "__main__":
    make_traces()
    make_kvc()
    make_sched_core()
    make_cost_model()
    make_hf()
    print("golden fixtures written to", HERE)
