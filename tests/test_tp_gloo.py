"""Tensor-parallel host logic on CPU with gloo, world_size 2: plan broadcast (tp.pack/unpack +
follower loop), Megatron sharding and the per-layer all-reduce composition, checked against the
unsharded oracle.  (The device path runs the same sharding with NCCL; one GPU is available here.)"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2503_13737_b200 import model as M
from paper_2503_13737_b200 import tp
from paper_2503_13737_b200.engine import DeviceBatch, synthetic_tokens
from paper_2503_13737_b200.kvc import BlockPool


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _batches(cfg):
    pool = BlockPool(256)
    out = []
    plan = [[(0, 0, 40), (1, 0, 7)], [(0, 40, 1), (1, 7, 20), (2, 0, 33)], [(0, 41, 1), (1, 27, 1), (2, 33, 1)]]
    for step in plan:
        ids, pos, slot, cu, ctx, tabs, lr, rids = [], [], [], [0], [], [], [], []
        for rid, start, n in step:
            pool.allocate(rid, pool.demand_prompt_chunk(rid, n) if n > 1 or not pool.is_resident(rid)
                          else pool.demand_tg(rid))
            p = np.arange(start, start + n, dtype=np.int32)
            ids.append(synthetic_tokens(rid, p, cfg.vocab)); pos.append(p)
            slot.append(np.asarray(pool.slots(rid, start, n), np.int32)); ctx.append(start)
            cu.append(cu[-1] + n); tabs.append(pool.block_table(rid)); lr.append(cu[-1] - 1); rids.append(rid)
        bt = np.zeros((len(tabs), max(map(len, tabs))), np.int32)
        for i, t in enumerate(tabs):
            bt[i, :len(t)] = t
        out.append(DeviceBatch(rids, np.concatenate(ids), np.concatenate(pos), np.asarray(cu, np.int32),
                               np.asarray(ctx, np.int32), bt, np.concatenate(slot), np.asarray(lr, np.int32), rids))
    return out


class _ShardExec:
    def __init__(self, cfg, rank, world):
        from oracle.executor import OracleExecutor
        w = M.init_weights(cfg, seed=0, tp_rank=rank, tp_size=world, init="test")

        def ar(x):
            y = x.clone()
            dist.all_reduce(y)
            return y

        self.inner = OracleExecutor(cfg, w, 256, tp_rank=rank, tp_size=world, allreduce=ar)
        self.vocab, self.max_tokens, self.max_seqs = cfg.vocab, 1 << 20, 1 << 20
        self.logits = []

    def execute(self, b):
        r = self.inner.execute(b)
        self.logits.append(r.logits)
        return r

    def swap_out(self, *a):
        self.inner.swap_out(*a)

    def swap_in(self, *a):
        self.inner.swap_in(*a)


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.set_num_threads(2)
    cfg = M.OPTConfig("tp-test", hidden=256, num_layers=2, num_heads=2, ffn=1024, max_positions=256)
    ex = _ShardExec(cfg, rank, world)
    if rank == 0:
        leader = tp.TPLeader(ex, dist.group.WORLD)
        for b in _batches(cfg):
            leader.execute(b)
        leader.stop()
        q.put([l.numpy() for l in ex.logits])
    else:
        n = tp.follower_loop(ex, dist.group.WORLD)
        assert n == 3
    dist.barrier()
    dist.destroy_process_group()


def test_tp2_matches_unsharded_oracle():
    from oracle.executor import OracleExecutor
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=300)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    cfg = M.OPTConfig("tp-test", hidden=256, num_layers=2, num_heads=2, ffn=1024, max_positions=256)
    w = M.init_weights(cfg, seed=0, init="test")
    full = OracleExecutor(cfg, w, 256)
    emu = OracleExecutor(cfg, w, 256, tp_emulate=2)  # unsharded weights, TP=2 rounding points
    for b, tl in zip(_batches(cfg), got):
        ref = full.execute(b).logits.numpy()
        assert np.abs(ref - tl).max() < 3e-2
        assert (ref.argmax(-1) == tl.argmax(-1)).mean() >= 0.99
        e = emu.execute(b).logits.numpy()
        print(f"sharded vs unsharded {np.abs(ref - tl).max():.3g}, vs tp_emulate=2 {np.abs(e - tl).max():.3g}")
        assert np.array_equal(e, tl)  # the emulation reproduces the sharded composition exactly


def test_pack_unpack_roundtrip():
    cfg = M.OPTConfig("x", hidden=256, num_layers=1, num_heads=2, ffn=1024, max_positions=256)
    for b in _batches(cfg):
        hdr, payload = tp.pack_batch(b)
        c = tp.unpack_batch(hdr, payload)
        for f in ("token_ids", "positions", "cu_q", "ctx_len", "block_table", "slot_mapping", "logit_rows"):
            assert np.array_equal(getattr(b, f), getattr(c, f))
        assert c.request_ids == b.request_ids and c.logit_request_ids == b.logit_request_ids


class _CountExec:
    vocab, max_tokens, max_seqs = 50272, 1 << 20, 1 << 20

    def __init__(self):
        self.n = 0

    def execute(self, b):
        self.n += 1


def _mark_worker(rank, world, port, q):
    """bench.py's timed-region protocol: the leader marks begin/end and joins a barrier; followers
    join it from the on_mark callback inside follower_loop, counting only the steps in between."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = M.OPTConfig("tp-test", hidden=256, num_layers=2, num_heads=2, ffn=1024, max_positions=256)
    bs = _batches(cfg)
    ex = _CountExec()
    if rank == 0:
        leader = tp.TPLeader(ex, dist.group.WORLD)
        leader.execute(bs[0])          # warm-up step (not counted)
        leader.mark(1)
        dist.barrier()
        leader.execute(bs[1])
        leader.execute(bs[2])          # 2 timed steps
        leader.mark(0)
        dist.barrier()
        leader.execute(bs[0])          # replay step (not counted)
        leader.stop()
    else:
        state = {"on": False, "timed": 0}

        class Counting(_CountExec):
            def execute(self, b):
                if state["on"]:
                    state["timed"] += 1

        def on_mark(tag):
            dist.barrier()
            state["on"] = tag == 1
        tp.follower_loop(Counting(), dist.group.WORLD, on_mark)
        q.put(state["timed"])
    dist.barrier()
    dist.destroy_process_group()


def test_timed_region_markers_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_mark_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    timed = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert timed == 2
