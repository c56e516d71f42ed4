"""Shared test helper: build a DeviceBatch (the packed BatchPlan of ag_step) from segments.

A segment (rid, start, n) is request rid's tokens [start, start+n) on top of `start` cached tokens;
its blocks come from the BlockPool's demand rules (kvc.py:110-150) and the lowest-free-id policy,
exactly as the engine packs them, and its last row is a logit row."""
from __future__ import annotations

import numpy as np

from paper_2503_13737_b200.engine import DeviceBatch, synthetic_tokens


def make_batch(pool, cfg, segs, tok_rids=None) -> DeviceBatch:
    ids, pos, slot, cu, ctx, tabs, lrows, rids = [], [], [], [0], [], [], [], []
    for i, (rid, start, n) in enumerate(segs):
        d = pool.demand_prompt_chunk(rid, n) if (n > 1 or not pool.is_resident(rid)) else pool.demand_tg(rid)
        pool.allocate(rid, d)
        p = np.arange(start, start + n, dtype=np.int32)
        ids.append(synthetic_tokens(rid if tok_rids is None else tok_rids[i], p, cfg.vocab))
        pos.append(p)
        slot.append(np.asarray(pool.slots(rid, start, n), np.int32))
        ctx.append(start)
        cu.append(cu[-1] + n)
        tabs.append(pool.block_table(rid))
        lrows.append(cu[-1] - 1)
        rids.append(rid)
    bt = np.zeros((len(tabs), max(map(len, tabs))), np.int32)
    for i, t in enumerate(tabs):
        bt[i, :len(t)] = t
    return DeviceBatch(rids, np.concatenate(ids), np.concatenate(pos), np.asarray(cu, np.int32),
                       np.asarray(ctx, np.int32), bt, np.concatenate(slot), np.asarray(lrows, np.int32), rids)


def split_prefill(segs, cap):
    """Group fresh-prompt segments into forwards of at most `cap` tokens."""
    out, cur, used = [], [], 0
    for seg in segs:
        if cur and used + seg[2] > cap:
            out.append(cur)
            cur, used = [], 0
        cur.append(seg)
        used += seg[2]
    if cur:
        out.append(cur)
    return out
