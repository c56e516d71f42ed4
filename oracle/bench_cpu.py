"""CPU timing of the oracle forward — TEST/BASELINE INFRASTRUCTURE ONLY (bench.py's cpu_baseline
and --impl reference legs).  The reference has no forward of its own (its GPU is the linear
iteration_time model, cost_model.py:101-109), so the "reference CPU path" is this repo's CPU
restatement: oracle.sched (policies + engine) producing the BatchPlans and oracle.forward
executing them, with all host threads.
"""
from __future__ import annotations

import os
import time

import numpy as np
import torch

from paper_2503_13737_b200 import model as M
from . import forward as orc


def _compact(batch):
    """Renumber the physical blocks a batch touches to 0..n-1 (keeps the CPU KV pool small)."""
    bt = np.asarray(batch.block_table)
    cu = np.asarray(batch.cu_q)
    ctx = np.asarray(batch.ctx_len)
    used = []
    for i in range(bt.shape[0]):
        n = (int(ctx[i]) + int(cu[i + 1] - cu[i]) + 31) // 32
        used.extend(int(x) for x in bt[i, :n])
    remap = {b: j for j, b in enumerate(dict.fromkeys(used))}
    bt2 = np.zeros_like(bt)
    for i in range(bt.shape[0]):
        n = (int(ctx[i]) + int(cu[i + 1] - cu[i]) + 31) // 32
        bt2[i, :n] = [remap[int(x)] for x in bt[i, :n]]
    slot = np.asarray(batch.slot_mapping)
    slot2 = np.array([remap[int(s) // 32] * 32 + int(s) % 32 for s in slot], dtype=np.int32)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.int32))
    return orc.StepInputs(t(batch.token_ids), t(batch.positions), t(cu), t(ctx), t(bt2), t(slot2),
                          t(batch.logit_rows)), max(1, len(remap))


def _one_layer(cfg):
    return M.OPTConfig(cfg.name + "-1layer", cfg.hidden, 1, cfg.num_heads, cfg.ffn, cfg.vocab, cfg.max_positions,
                       cfg.ln_eps)


_W_CACHE: dict = {}


def _weights(cfg1):
    key = (cfg1.hidden, cfg1.ffn, cfg1.vocab, cfg1.pos_rows)
    if key not in _W_CACHE:
        _W_CACHE[key] = M.init_weights(cfg1, seed=0, device="cpu", init="opt")
    return _W_CACHE[key]


def time_forward_sample(cfg, batch, budget_s: float = 20.0) -> dict:
    """One layer of cfg on `batch` (embed + 1 layer + final LN + LM head), scaled to cfg.num_layers."""
    threads = os.cpu_count() or 1
    torch.set_num_threads(threads)
    cfg1 = _one_layer(cfg)
    w = _weights(cfg1)
    st, nb = _compact(batch)
    o = orc.OracleOPT(cfg1, w, nb)
    t0 = time.perf_counter()
    o.forward(st)
    t1 = time.perf_counter() - t0
    # LM head alone (so it is not multiplied by the layer count)
    hl = torch.randn(len(batch.logit_rows), cfg.hidden)
    emb = orc.f32(w["tok_emb"])
    t0 = time.perf_counter()
    _ = hl @ emb.T
    t_head = time.perf_counter() - t0
    per_layer = max(t1 - t_head, 1e-9)
    total = t_head + cfg.num_layers * per_layer
    return {"tokens_per_s": batch.num_tokens / total, "seconds": t1 + t_head, "threads": threads,
            "est_forward_s": total}


def reference_arm(run_cfg, profile, steps: int, warmup: int, window_s: float = 1.0, tok_cap: int = 256) -> dict:
    """The reference's path on the CPU, measured like bench.py's GPU arm.  The oracle scheduler
    (oracle.sched, the restated AccelGen policy + engine) plans every iteration and its clock advances
    by the MEASURED CPU time of that iteration's forward (oracle.forward with all host threads; sampled:
    one of L layers on at most `tok_cap` of the batch's tokens (whole sequences), scaled linearly to all
    tokens and layers -- the bound that keeps the run to minutes).  Steps are `window_s` windows of that
    clock after `warmup` windows; SLO-meeting tokens are counted exactly as in bench.py (decode tokens
    that met TBT, a prompt's chunks iff its first token met TTFT).  At tens of CPU-seconds per forward no
    deadline is met, so value = 0; the forward tokens/s of the CPU path is reported beside it."""
    from paper_2503_13737_b200 import workload
    from paper_2503_13737_b200.engine import DeviceBatch, synthetic_tokens
    from .sched import OracleScheduler

    threads = os.cpu_count() or 1
    torch.set_num_threads(threads)
    cfg = run_cfg.model
    trace = workload.generate_trace(run_cfg.trace)
    kv_tok = cfg.kv_bytes_per_token()
    sch = OracleScheduler(trace, profile, kv_blocks=int(150e9 // (32 * kv_tok)))
    cfg1 = _one_layer(cfg)
    w = _weights(cfg1)

    def sample_batch(entry):
        ids, pos, slot, cu, ctx, tabs, lr = [], [], [], [0], [], [], []
        taken = 0
        for rid, c, final, before in entry["sel"]:
            if taken and taken + c > tok_cap:
                continue
            p = np.arange(before, before + c, dtype=np.int32)
            table = entry["tables"][rid]
            ids.append(synthetic_tokens(rid, p, cfg.vocab)); pos.append(p)
            slot.append(np.array([table[q // 32] * 32 + q % 32 for q in p], np.int32))
            ctx.append(before); cu.append(cu[-1] + c); tabs.append(table)
            if final:
                lr.append(cu[-1] - 1)
            taken += c
        bt = np.zeros((len(tabs), max(map(len, tabs))), np.int32)
        for i, t in enumerate(tabs):
            bt[i, :len(t)] = t
        return DeviceBatch(list(range(len(tabs))), np.concatenate(ids), np.concatenate(pos),
                           np.asarray(cu, np.int32), np.asarray(ctx, np.int32), bt, np.concatenate(slot),
                           np.asarray(lr, np.int32), [])

    stats = {"cpu_s": 0.0, "tokens": 0, "sampled": 0, "forwards": 0}

    def cpu_forward_time(entry):
        b = sample_batch(entry)
        st, nb = _compact(b)
        o = orc.OracleOPT(cfg1, w, nb)
        t0 = time.perf_counter()
        o.forward(st)
        dt = time.perf_counter() - t0
        full = sum(c for _, c, _, _ in entry["sel"])
        est = dt * cfg.num_layers * (full / b.num_tokens)
        stats["cpu_s"] += est
        stats["tokens"] += full
        stats["sampled"] += b.num_tokens
        stats["forwards"] += 1
        return est

    sch.clock_fn = cpu_forward_time
    t_w0, t_w1 = warmup * window_s, (warmup + steps) * window_s
    while sch.clock < t_w1:
        if sch.step() is None and sch.nxt >= len(sch.trace) and not sch.queue:
            break
    slo_tokens = 0
    for entry in sch.log:
        if not (t_w0 <= entry["end"] < t_w1):
            continue
        for rid, c, final, before in entry["sel"]:
            r = sch.reqs[rid]
            slo = r.spec.slo
            if before < r.spec.prompt_len:  # prompt chunk: iff the first token met TTFT
                ok = bool(r.emits) and r.emits[0] - r.spec.arrival_time <= slo.ttft_slo + 1e-12
            else:  # decode: this emission's gap to the previous one
                i = r.emits.index(entry["end"])
                ok = i > 0 and r.emits[i] - r.emits[i - 1] <= slo.tbt_slo + 1e-12
            slo_tokens += c if ok else 0
    span = (steps * window_s)
    return {"value": slo_tokens / span, "ms_per_step": 1e3 * window_s, "threads": threads,
            "forward_tokens_per_s": stats["tokens"] / stats["cpu_s"] if stats["cpu_s"] else 0.0,
            "forwards": stats["forwards"],
            "sample": f"{stats['forwards']} oracle-scheduled forwards over {t_w1:g} s of the CPU clock; each timed "
                      f"as 1 of {cfg.num_layers} OPT-13B layers on <= {tok_cap} tokens ({stats['sampled']} sampled "
                      f"of {stats['tokens']}), scaled linearly to all tokens and layers"}
