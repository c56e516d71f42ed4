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


def reference_arm(run_cfg, profile, steps: int, warmup: int, ramp_s: float = 6.0, tok_cap: int = 256) -> dict:
    """W + K steps of the reference path on the CPU.  Plans come from the oracle scheduler
    (virtual clock); each step executes one OPT-13B layer of that step's batch on the CPU
    oracle, on at most `tok_cap` of its tokens (whole sequences), scaled linearly to all tokens
    and all layers.  The value is forward tokens / CPU forward time: an upper bound on the
    reference's SLO-meeting tokens/s (at tens of seconds per iteration no TBT deadline is met)."""
    from paper_2503_13737_b200 import workload
    from paper_2503_13737_b200.engine import DeviceBatch, synthetic_tokens
    from .sched import OracleScheduler

    threads = os.cpu_count() or 1
    torch.set_num_threads(threads)
    cfg = run_cfg.model
    trace = workload.generate_trace(run_cfg.trace)
    kv_tok = cfg.kv_bytes_per_token()
    sch = OracleScheduler(trace, profile, kv_blocks=int(80e9 // (32 * kv_tok)))
    while sch.clock < ramp_s:
        sch.step()
    cfg1 = _one_layer(cfg)
    w = _weights(cfg1)

    def sample_batch(entry):
        ids, pos, slot, cu, ctx, tabs, lr = [], [], [], [0], [], [], []
        taken = 0
        full_tokens = sum(c for _, c, _, _ in entry["sel"])
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
        b = DeviceBatch(list(range(len(tabs))), np.concatenate(ids), np.concatenate(pos), np.asarray(cu, np.int32),
                        np.asarray(ctx, np.int32), bt, np.concatenate(slot), np.asarray(lr, np.int32), [])
        return b, full_tokens

    done_tokens, cpu_s, sampled = 0, 0.0, 0
    n = 0
    while n < warmup + steps:
        entry = sch.step()
        if entry is None:
            continue
        b, full = sample_batch(entry)
        st, nb = _compact(b)
        o = orc.OracleOPT(cfg1, w, nb)
        t0 = time.perf_counter()
        o.forward(st)
        dt = time.perf_counter() - t0
        if n >= warmup:
            est = dt * cfg.num_layers * (full / b.num_tokens)
            done_tokens += full
            cpu_s += est
            sampled += b.num_tokens
        n += 1
    return {"value": done_tokens / cpu_s, "ms_per_step": cpu_s / steps * 1e3, "threads": threads,
            "sample": f"{steps} oracle-scheduled steps; per step 1 of {cfg.num_layers} OPT-13B layers on <= {tok_cap} "
                      f"tokens ({sampled} sampled of {done_tokens}), scaled linearly to all tokens and layers"}
