"""Asynchronous steps on the B200 (ag_model_submit / ag_model_wait): two forwards in flight, decode
inputs fed on the device from the previous step's next-token ids, bitwise identical to the synchronous
ag_model_forward fed by the host; and the pipelined engine serving config 1 end to end through them."""
import os

import numpy as np
import pytest
import torch

from paper_2503_13737_b200 import configs, model as M, workload
from paper_2503_13737_b200.engine import DeviceBatch, Engine, synthetic_tokens
from paper_2503_13737_b200.kvc import BlockPool
from paper_2503_13737_b200.policies import PolicyConfig

pytestmark = pytest.mark.gpu


def _batch(pool, cfg, segs):
    ids, pos, slot, cu, ctx, tabs, lr, rids = [], [], [], [0], [], [], [], []
    for rid, start, n in segs:
        pool.allocate(rid, pool.demand_prompt_chunk(rid, n) if n > 1 or not pool.is_resident(rid)
                      else pool.demand_tg(rid))
        p = np.arange(start, start + n, dtype=np.int32)
        ids.append(synthetic_tokens(rid, p, cfg.vocab)); pos.append(p)
        slot.append(np.asarray(pool.slots(rid, start, n), np.int32)); ctx.append(start)
        cu.append(cu[-1] + n); tabs.append(pool.block_table(rid)); lr.append(cu[-1] - 1); rids.append(rid)
    bt = np.zeros((len(tabs), max(map(len, tabs))), np.int32)
    for i, t in enumerate(tabs):
        bt[i, :len(t)] = t
    return DeviceBatch(rids, np.concatenate(ids), np.concatenate(pos), np.asarray(cu, np.int32),
                       np.asarray(ctx, np.int32), bt, np.concatenate(slot), np.asarray(lr, np.int32), rids)


def test_submit_wait_feed_matches_synchronous_forward(monkeypatch):
    from paper_2503_13737_b200.executor import CudaExecutor
    monkeypatch.setenv("AG_DETERMINISTIC", "1")  # no fp32 atomics: both runs bitwise reproducible
    cfg = M.tiny()
    w = M.init_weights(cfg, seed=0, init="test")
    # step plans: prompts, then decodes of them (+ a new prompt), then decodes again
    steps = [[(0, 0, 150), (1, 0, 40)],
             [(0, 150, 1), (1, 40, 1), (2, 0, 77)],
             [(0, 151, 1), (1, 41, 1), (2, 77, 1)],
             [(2, 78, 1), (0, 152, 1)]]
    outs = {}
    for mode in ("sync", "async"):
        pool = BlockPool(256)
        ex = CudaExecutor(cfg, pool.total_blocks, max_tokens=512, max_seqs=16, weights=w, autotune=False)
        last = {}          # rid -> emitted token (host) / (step, row) of the step in flight
        got = []
        prev_rows = None
        for k, segs in enumerate(steps):
            b = _batch(pool, cfg, segs)
            if mode == "sync":
                for i, (rid, start, n) in enumerate(segs):
                    if n == 1 and rid in last:
                        b.token_ids[b.cu_q[i]] = last[rid]
                r = ex.execute(b)
                got.append(r.token_ids.tolist())
                last.update(zip(b.logit_request_ids, r.token_ids.tolist()))
            else:
                feed = [(int(b.cu_q[i]), prev_rows[rid]) for i, (rid, start, n) in enumerate(segs)
                        if n == 1 and prev_rows and rid in prev_rows]
                ex.submit(b, np.asarray(feed, np.int32).reshape(-1, 2) if feed else None)
                assert ex.inflight() <= 2
                if k > 0:
                    got.append(ex.wait().token_ids.tolist())
                prev_rows = {rid: j for j, rid in enumerate(b.logit_request_ids)}
        if mode == "async":
            r = ex.wait()
            got.append(r.token_ids.tolist())
            assert r.end_s is not None and r.device_s > 0
            assert ex.inflight() == 0
        outs[mode] = got
        ex.close()
    assert outs["sync"] == outs["async"]


def test_pipelined_engine_serves_config1():
    from paper_2503_13737_b200.executor import CudaExecutor
    c = configs.config1()
    trace = workload.generate_trace(c.trace)
    w = M.init_weights(c.model, seed=0, init="test")
    blocks = c.trace.profile.kvc_capacity_tokens // 32
    ex = CudaExecutor(c.model, blocks, max_tokens=512, max_seqs=128, weights=w, autotune=False)
    eng = Engine(trace, c.trace.profile, PolicyConfig(), ex, clock="wall", pipeline=True, check_invariants=True)
    rep = eng.run()
    assert rep.completed == len(trace)
    assert ex.inflight() == 0
    for rec in eng.metrics.requests.values():
        assert rec.generated == rec.spec.output_len and all(t >= 0 for t in rec.tokens_out)
        assert rec.emit_times == sorted(rec.emit_times)
    ex.close()
