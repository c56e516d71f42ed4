"""End-to-end parity of the mixed-batch forward on the B200 vs the oracle.

Tolerance (north_star): logits max-abs <= 2e-2 per step, greedy tokens identical for >= 99% of
token events -- a disagreement is only excused where the oracle's own top-2 logit gap is within
twice the tolerance (a near tie that bf16 rounding may legitimately flip).  Scheduling is shared
(TeeExecutor), so the device sees exactly the oracle's inputs (teacher-forced synthetic tokens,
same block tables / slots).  The full-depth OPT-13B and 100k-context cases run the oracle's torch
restatement on the GPU in fp32 (TF32 off); the rest run it on the CPU."""
import numpy as np
import pytest
import torch

from batches import make_batch, split_prefill
from oracle.executor import OracleExecutor, TeeExecutor
from paper_2503_13737_b200 import configs, model as M, workload
from paper_2503_13737_b200.engine import Engine
from paper_2503_13737_b200.policies import PolicyConfig

pytestmark = pytest.mark.gpu

from parity import FLOOR_FACTOR, LOGIT_TOL, TOKEN_AGREEMENT, Tally  # noqa: E402


def _compare(records):
    worst, agree, total = 0.0, 0, 0
    for batch, dev, ref in records:
        n = len(batch.logit_rows)
        if n == 0:
            continue
        worst = max(worst, (dev.logits[:n].float() - ref.logits[:n].float()).abs().max().item())
        agree += int((dev.token_ids[:n] == ref.token_ids[:n]).sum())
        total += n
    return worst, agree / max(total, 1), total


def test_config1_trace_parity():
    """Config 1 (tiny OPT, 64 requests incl. 4k-8k prompts chunked dynamically) end to end."""
    from paper_2503_13737_b200.executor import CudaExecutor
    c = configs.config1()
    trace = workload.generate_trace(c.trace)
    w = M.init_weights(c.model, seed=0, init="test")
    blocks = c.trace.profile.kvc_capacity_tokens // 32
    dev = CudaExecutor(c.model, blocks, max_tokens=512, max_seqs=128, weights=w, parity_logits=True)
    ref = OracleExecutor(c.model, w, blocks)
    tee = TeeExecutor(dev, ref)
    eng = Engine(trace, c.trace.profile, PolicyConfig(), tee, clock="virtual", check_invariants=True)
    rep = eng.run()
    assert rep.completed == len(trace)
    worst, agree, n = _compare(tee.records)
    print(f"steps={len(tee.records)} token events={n} max|dlogit|={worst:.4g} agreement={agree:.4f}")
    assert worst <= LOGIT_TOL
    assert agree >= TOKEN_AGREEMENT


_make_batch = make_batch


def _run_vs_oracle(cfg, w, blocks, plan, dev_kw, label, min_rows=0):
    """Run `plan` (segment lists) through the CUDA executor, the fp32 oracle and the fp64 oracle (both
    on the GPU, TF32 off) and check the Tally."""
    from paper_2503_13737_b200.executor import CudaExecutor
    from paper_2503_13737_b200.kvc import BlockPool
    pool = BlockPool(blocks)
    dev = CudaExecutor(cfg, blocks, weights=w, parity_logits=True, **dev_kw)
    ref = OracleExecutor(cfg, w, blocks, device="cuda")
    ref64 = OracleExecutor(cfg, w, blocks, device="cuda", acc=torch.float64)
    tally = Tally()
    for segs in plan:
        b = make_batch(pool, cfg, segs)
        a, r, r64 = dev.execute(b), ref.execute(b), ref64.execute(b)
        tally.add(a.logits, a.token_ids, r.logits, r.token_ids, r64.logits)
    dev.close()
    tally.check(label)
    assert tally.total >= min_rows
    return tally


def test_13b_shape_mixed_batch_two_layers():
    """OPT-13B layer shapes (H=5120, 40 heads, FFN 20480), 2 layers, one mixed batch:
    a 1500-token chunk on a 3000-token prefix + a fresh 300-token prompt + 40 decodes."""
    cfg = M.OPTConfig("opt-13b-2l", hidden=5120, num_layers=2, num_heads=40, ffn=20480, max_positions=8192)
    w = M.init_weights(cfg, seed=1, device="cuda", init="test")
    decodes = [(2 + i, 50 + 13 * i) for i in range(40)]
    plan = split_prefill([(0, 0, 3000)] + [(rid, 0, p) for rid, p in decodes], 4000)
    plan.append([(0, 3000, 1500), (1, 0, 300)] + [(rid, p, 1) for rid, p in decodes])
    _run_vs_oracle(cfg, w, 4096, plan, dict(max_tokens=4096, max_seqs=128), "13B-shape 2 layers")


def test_opt13b_full_depth_mixed_steps_vs_oracle():
    """The named architecture at full depth: all 40 OPT-13B layers (config-2 shape, random biases and
    LayerNorm affine so every epilogue term is live), autotuned GEMM plans as in production.  After
    prefilling a 3k-token prompt and 48 short prompts, three mixed steps: a 1024-token chunk on the 3k
    prefix + a fresh 500-token prompt + 48 decodes; then decodes + a new 200-token prompt; then decodes
    + that prompt's first decode + a 37-token prompt."""
    cfg = M.opt_13b(max_positions=8192)
    w = M.init_weights(cfg, seed=13, device="cuda", init="test")
    dec = [(2 + i, 16 + 5 * i) for i in range(48)]
    plan = split_prefill([(0, 0, 3000)] + [(rid, 0, p) for rid, p in dec], 4096)
    plan += [
        [(0, 3000, 1024), (1, 0, 500)] + [(rid, p, 1) for rid, p in dec],
        [(0, 4024, 1), (1, 500, 1), (60, 0, 200)] + [(rid, p + 1, 1) for rid, p in dec],
        [(0, 4025, 1), (1, 501, 1), (60, 200, 1), (61, 0, 37)] + [(rid, p + 2, 1) for rid, p in dec],
    ]
    _run_vs_oracle(cfg, w, 512, plan, dict(max_tokens=4096, max_seqs=64), "OPT-13B 40 layers, 6 forwards",
                   min_rows=150)


def _prompt_batch(pool, cfg, rid, tok_rid, start, n):
    """One sequence's chunk [start, start+n) with the token ids of request `tok_rid` (so two
    requests can carry the same prompt)."""
    from paper_2503_13737_b200.engine import DeviceBatch, synthetic_tokens
    d = pool.demand_prompt_chunk(rid, n) if (n > 1 or not pool.is_resident(rid)) else pool.demand_tg(rid)
    pool.allocate(rid, d)
    p = np.arange(start, start + n, dtype=np.int32)
    bt = np.asarray([pool.block_table(rid)], np.int32)
    return DeviceBatch([rid], synthetic_tokens(tok_rid, p, cfg.vocab), p, np.asarray([0, n], np.int32),
                       np.asarray([start], np.int32), bt, np.asarray(pool.slots(rid, start, n), np.int32),
                       np.asarray([n - 1], np.int32), [rid])


def test_long_context_100k_vs_oracle_and_chunk_invariance():
    """Config-4 regime on one GPU (2 OPT-13B-shaped layers): a 100k-token prompt prefilled in
    16384-token chunks -- every chunk checked against the oracle (fp32 on the GPU) -- then one decode;
    and, as a second request with the same tokens, in 12000-token chunks.  Chunked prefill must not
    change the result (SURVEY §7 property): last-chunk and decode logits agree within the bf16
    tolerance and pick the same greedy token.  Exercises split-KV tile attention over ~3k-page block
    tables, decode rows over a 100k context and the extended position table."""
    import os
    from paper_2503_13737_b200.executor import CudaExecutor
    from paper_2503_13737_b200.kvc import BlockPool
    os.environ["AG_DETERMINISTIC"] = "1"  # no fp32 atomics: reproducible run to run
    P = 100_000
    cfg = M.OPTConfig("opt-13b-2l-100k", hidden=5120, num_layers=2, num_heads=40, ffn=20480,
                      max_positions=P + 64)
    w = M.init_weights(cfg, seed=3, device="cuda", init="test")
    pool = BlockPool(2 * (P // 32 + 8))
    try:
        dev = CudaExecutor(cfg, pool.total_blocks, max_tokens=16384, max_seqs=8, weights=w, parity_logits=True)
    finally:
        os.environ.pop("AG_DETERMINISTIC", None)
    ref = OracleExecutor(cfg, w, pool.total_blocks, device="cuda")
    ref64 = OracleExecutor(cfg, w, pool.total_blocks, device="cuda", acc=torch.float64)
    tally = Tally()
    outs = []
    for rid, chunk in ((0, 16384), (1, 12000)):
        res = None
        for start in range(0, P, chunk):
            b = _prompt_batch(pool, cfg, rid, 0, start, min(chunk, P - start))
            res = dev.execute(b)
            if rid == 0:
                r, r64 = ref.execute(b), ref64.execute(b)
                tally.add(res.logits, res.token_ids, r.logits, r.token_ids, r64.logits)
        b = _prompt_batch(pool, cfg, rid, 0, P, 1)
        dec = dev.execute(b)
        if rid == 0:
            r, r64 = ref.execute(b), ref64.execute(b)
            tally.add(dec.logits, dec.token_ids, r.logits, r.token_ids, r64.logits)
        outs.append((res.logits[:1].float().clone(), res.token_ids.copy(), dec.logits[:1].float().clone(),
                     dec.token_ids.copy()))
    tally.check("100k prompt (16384-token chunks + 1 decode) vs oracle")
    (la, ta, da, tda), (lb, tb, db, tdb) = outs
    d_last = (la - lb).abs().max().item()
    d_dec = (da - db).abs().max().item()
    print(f"100k prompt chunk invariance: max|dlogit| last-chunk {d_last:.4g}, decode {d_dec:.4g}")
    assert torch.isfinite(la).all() and torch.isfinite(da).all()
    # the two chunkings give the GEMMs different M, hence possibly different tile / split-K plans and
    # fp32 summation orders: equal within the bf16 tolerance (bitwise only when the plans coincide)
    bound = max(LOGIT_TOL, FLOOR_FACTOR * tally.floor)
    assert d_last <= bound and d_dec <= bound
    assert ta[0] == tb[0] and tda[0] == tdb[0]


@pytest.mark.parametrize("bn,splits,am,fuse", [(128, 2, 128, "1"), (128, 5, 128, "1"), (128, 99, 128, "1"),
                                               (256, 99, 256, "1"), (256, 2, 256, "1"), (128, 99, 128, "0"),
                                               (256, 2, 256, "0")])  # 99 = stream-K (kStreamK); am 256 = CTA pair
def test_split_k_atomic_epilogue_forward(bn, splits, am, fuse, monkeypatch):
    """Out-proj / FC2 split-K at TP=1 accumulate fp32 partials with red.global.add into acc32; the
    residual + bias + next LayerNorm (which re-zeroes acc32) runs, when the step has no more rows than
    the consuming QKV / FC1 GEMM has CTAs, in that GEMM's prologue behind a grid barrier (else in the
    atomic GEMM's tail, else as its own launch; AG_FUSE_LN=0: always its own launch); the last FC2 is
    always finished by the final LayerNorm on the logit rows.  QKV / FC1 take the split-K reduce
    kernel, or with stream-K (99) the atomic accumulator + finish kernel (q scale, KV scatter, ReLU).  Forced on for every M bucket via
    the plan table; two consecutive mixed steps vs the oracle (acc32 must be clean between steps)."""
    monkeypatch.setenv("AG_FUSE_LN", fuse)
    import ctypes as C
    from paper_2503_13737_b200.executor import CudaExecutor
    from paper_2503_13737_b200.kvc import BlockPool
    cfg = M.OPTConfig("opt-13b-2l", hidden=5120, num_layers=2, num_heads=40, ffn=20480, max_positions=4096)
    w = M.init_weights(cfg, seed=5, device="cuda", init="test")
    pool = BlockPool(1024)
    dev = CudaExecutor(cfg, pool.total_blocks, max_tokens=1024, max_seqs=64, weights=w, parity_logits=True)
    rows = []
    bn_, am_ = bn, am
    for kind, mb, bn, ks, am in dev.gemm_plans():
        kid = ("qkv", "out", "fc1", "fc2", "lm_head").index(kind)
        if kind in ("out", "fc2", "qkv", "fc1"):  # QKV/FC1: reduce kernel (2, 5) / stream-K + finish (99)
            bn, ks = bn_, splits
            am = am_ if mb >= 256 or am_ != 256 else 128  # the pair kernel needs >= 256-row buckets
        rows.append([kid, mb, bn, ks + 100 * am])
    buf = (C.c_int32 * (4 * len(rows)))(*[x for r in rows for x in r])
    from paper_2503_13737_b200 import _lib
    _lib.check(dev.lib.ag_model_set_gemm_plans(dev.handle, buf, len(rows)))
    ref = OracleExecutor(cfg, w, pool.total_blocks, device="cuda")
    ref64 = OracleExecutor(cfg, w, pool.total_blocks, device="cuda", acc=torch.float64)
    tally = Tally()
    # the third step (3 decodes) has fewer rows than any plan's CTAs: the fused LayerNorm runs in the
    # QKV / FC1 prologue (or the atomic GEMM's tail) instead of its own launch
    for segs in ([(0, 0, 700), (1, 0, 60)], [(0, 700, 1), (1, 60, 200), (2, 0, 33)],
                 [(0, 701, 1), (1, 260, 1), (2, 33, 1)]):
        b = _make_batch(pool, cfg, segs)
        a, r, r64 = dev.execute(b), ref.execute(b), ref64.execute(b)
        tally.add(a.logits, a.token_ids, r.logits, r.token_ids, r64.logits)
    tally.check(f"plan {bn_}x{splits}a{am_} fuse_ln={fuse}")


def test_175b_shape_two_layers_vs_oracle():
    """Config-5 layer shapes on one GPU: OPT-175B's H=12288, 96 heads, FFN 49152 (2 of 96 layers,
    unsharded), one prefill step then a mixed step with decodes, vs the CPU oracle.  Covers the
    block LayerNorm (hidden > 5120), N=36864 / K=49152 GEMMs and 96-head attention."""
    from paper_2503_13737_b200.executor import CudaExecutor
    from paper_2503_13737_b200.kvc import BlockPool
    cfg = M.OPTConfig("opt-175b-2l", hidden=12288, num_layers=2, num_heads=96, ffn=49152, max_positions=2048)
    w = M.init_weights(cfg, seed=7, device="cuda", init="test")
    pool = BlockPool(256)
    dev = CudaExecutor(cfg, pool.total_blocks, max_tokens=512, max_seqs=32, weights=w, parity_logits=True,
                       autotune=False)
    ref = OracleExecutor(cfg, w, pool.total_blocks, device="cuda")
    ref64 = OracleExecutor(cfg, w, pool.total_blocks, device="cuda", acc=torch.float64)
    tally = Tally()
    for segs in ([(0, 0, 300), (1, 0, 40), (2, 0, 17)], [(0, 300, 1), (1, 40, 1), (2, 17, 120), (3, 0, 64)]):
        b = _make_batch(pool, cfg, segs)
        a, r, r64 = dev.execute(b), ref.execute(b), ref64.execute(b)
        tally.add(a.logits, a.token_ids, r.logits, r.token_ids, r64.logits)
    tally.check("175B-shape 2 layers")


@pytest.mark.parametrize("per_chunk,pool", [(3, 0), (1, 0), (1, 5)])
def test_executor_swap_roundtrip_chunked(per_chunk, pool):
    """Preemption swap through the executor (kvc.py:153-160 preempt / demand_readmit): a request's
    blocks of every layer go to host memory through the HBM staging ring in several chunks (1 block per
    chunk: 8 chunks cycle the 4-slot ring twice) without host synchronisation, the freed blocks are
    overwritten at once on the compute stream, and everything comes back bit-exactly into different
    physical blocks -- also for a second request swapped while the first is still on the host."""
    from paper_2503_13737_b200.executor import CudaExecutor
    cfg = M.tiny()
    w = M.init_weights(cfg, seed=0, init="test")
    dev = CudaExecutor(cfg, 64, max_tokens=256, max_seqs=8, weights=w, autotune=False)
    dev._SWAP_STAGE_BYTES = per_chunk * cfg.num_layers * 2 * dev.heads_l * 32 * 128 * 2
    if pool:  # host chunks pinned up front (bench setup): `pool` distinct buffers, reused by the swaps
        dev.prepare_swap(pool * dev._SWAP_STAGE_BYTES / 1e9)
        ptrs = {flat.data_ptr() for flat, _ in dev._host_free}
        assert len(ptrs) == len(dev._host_free) == pool and dev.swap_host_chunks == pool
    g = torch.Generator(device="cuda").manual_seed(3)
    dev.kv.copy_(torch.randn(dev.kv.shape, generator=g, device="cuda").to(torch.bfloat16))
    src = [5, 9, 2, 40, 41, 17, 63, 0]
    src2 = [30, 31, 32]
    before = dev.kv[:, :, src].clone()
    before2 = dev.kv[:, :, src2].clone()
    dev.swap_out(7, src, 8 * 32)
    assert len(dev._swapped[7]) == -(-8 // per_chunk)
    dev.kv[:, :, src] = 0                             # reuse of the freed blocks, stream-ordered
    dev.swap_out(8, src2, 3 * 32)
    dev.kv[:, :, src2] = 1
    dst = [10, 11, 12, 13, 14, 15, 16, 18]
    dev.swap_in(7, dst, 8 * 32)
    dev.swap_in(8, [5, 9, 2], 3 * 32)
    assert torch.equal(dev.kv[:, :, dst], before)
    assert torch.equal(dev.kv[:, :, [5, 9, 2]], before2)


def test_forward_at_capacity_limits():
    """S_f exactly max_tokens, a sequence filling its block-table row, logit rows for every sequence,
    and the C ABI's capacity checks (EngineFault / AllocationError instead of a bad launch)."""
    from paper_2503_13737_b200.errors import AllocationError, EngineFault
    from paper_2503_13737_b200.executor import CudaExecutor
    from paper_2503_13737_b200.kvc import BlockPool
    cfg = M.tiny()
    w = M.init_weights(cfg, seed=2, init="test")
    pool = BlockPool(256)
    dev = CudaExecutor(cfg, pool.total_blocks, max_tokens=384, max_seqs=4, max_blocks_per_seq=16, weights=w,
                       parity_logits=True)
    ref = OracleExecutor(cfg, w, pool.total_blocks)
    b = _make_batch(pool, cfg, [(0, 0, 200), (1, 0, 184)])   # S_f = 384 = max_tokens
    a, r = dev.execute(b), ref.execute(b)
    assert (a.logits[:2] - r.logits[:2]).abs().max().item() <= LOGIT_TOL
    b = _make_batch(pool, cfg, [(2, 0, 385)])                  # 385 > max_tokens
    with pytest.raises((AllocationError, EngineFault)):
        dev.execute(b)
    b = _make_batch(pool, cfg, [(3, 0, 300)])
    dev.execute(b)
    b = _make_batch(pool, cfg, [(3, 300, 300)])                # 600 tokens = 19 blocks > max_blocks_per_seq
    with pytest.raises((AllocationError, EngineFault)):
        dev.execute(b)
    pool2 = BlockPool(256)
    b = _make_batch(pool2, cfg, [(5, 0, 300), (6, 0, 10)])
    a, r = dev.execute(b), ref.execute(b)
    b = _make_batch(pool2, cfg, [(5, 300, 212)])               # ctx 300 + 212 = 512 tokens = 16 blocks
    a, r = dev.execute(b), ref.execute(b)
    assert (a.logits[:1] - r.logits[:1]).abs().max().item() <= LOGIT_TOL
