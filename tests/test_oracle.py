"""Pin the CPU oracle before trusting it: against transformers' OPTForCausalLM (golden logits,
tests/golden/opt_tiny_hf.pt) and by the chunk-invariance property of the paged forward."""
from pathlib import Path

import numpy as np
import pytest
import torch

import oracle.forward as orc
from paper_2503_13737_b200 import model as M
from paper_2503_13737_b200.kvc import BlockPool

G = Path(__file__).resolve().parent / "golden"


def _run_chunks(cfg, w, ids, chunks, rid=0, num_blocks=64):
    """Feed one prompt through the oracle in the given chunk sizes; return last-token logits."""
    o = orc.OracleOPT(cfg, w, num_blocks)
    pool = BlockPool(num_blocks)
    done = 0
    logits = None
    for c in chunks:
        pool.allocate(rid, pool.demand_prompt_chunk(rid, c))
        pos = torch.arange(done, done + c, dtype=torch.int32)
        table = torch.tensor([pool.block_table(rid)], dtype=torch.int32)
        st = orc.StepInputs(ids[done:done + c], pos, torch.tensor([0, c], dtype=torch.int32),
                            torch.tensor([done], dtype=torch.int32), table,
                            torch.tensor(pool.slots(rid, done, c), dtype=torch.int32),
                            torch.arange(c, dtype=torch.int32))
        logits, _ = o.forward(st)
        done += c
    return logits


def test_oracle_matches_transformers_fp32():
    g = torch.load(G / "opt_tiny_hf.pt")
    cfg = M.tiny()
    w = M.init_weights(cfg, seed=0, init="test")
    orc.ROUND_BF16 = False
    try:
        logits = _run_chunks(cfg, w, g["input_ids"], [len(g["input_ids"])])
    finally:
        orc.ROUND_BF16 = True
    rows = g["rows"]
    assert torch.allclose(logits[rows, :4096], g["logits_head"], atol=2e-4, rtol=1e-4)
    assert torch.equal(logits[rows].argmax(-1).to(torch.int32), g["argmax"])
    assert torch.allclose(torch.logsumexp(logits[rows], -1), g["lse"], atol=2e-4)


def test_oracle_bf16_mode_close_to_transformers():
    g = torch.load(G / "opt_tiny_hf.pt")
    cfg = M.tiny()
    w = M.init_weights(cfg, seed=0, init="test")
    logits = _run_chunks(cfg, w, g["input_ids"], [len(g["input_ids"])])
    assert (logits[g["rows"], :4096] - g["logits_head"]).abs().max().item() < 2e-2


@pytest.mark.parametrize("chunks", [[77], [13, 20, 44], [1] * 10 + [67], [32, 32, 13]])
def test_chunk_invariance(chunks):
    """The last token's logits do not depend on how the prompt was chunked (paged prefix reuse)."""
    cfg = M.tiny()
    w = M.init_weights(cfg, seed=0, init="test")
    ids = torch.randint(4, cfg.vocab, (77,), generator=torch.Generator().manual_seed(1), dtype=torch.int32)
    whole = _run_chunks(cfg, w, ids, [77])[-1]
    part = _run_chunks(cfg, w, ids, chunks)[-1]
    assert (whole - part).abs().max().item() < 2e-2
    assert int(whole.argmax()) == int(part.argmax())


def test_tp_shards_reassemble():
    """Megatron sharding of init_weights: concatenating rank shards gives the full weights."""
    cfg = M.OPTConfig("t", hidden=256, num_layers=1, num_heads=2, ffn=1024, max_positions=64)
    full = M.init_weights(cfg, seed=3, init="test")["layers"][0]
    shards = [M.init_weights(cfg, seed=3, tp_rank=r, tp_size=2, init="test")["layers"][0] for r in range(2)]
    H = cfg.hidden
    q = torch.cat([s["qkv_w"][:H // 2] for s in shards])
    assert torch.equal(q, full["qkv_w"][:H])
    assert torch.equal(torch.cat([s["out_w"] for s in shards], dim=1), full["out_w"])
    assert torch.equal(torch.cat([s["fc1_w"] for s in shards]), full["fc1_w"])
    assert torch.equal(torch.cat([s["fc2_w"] for s in shards], dim=1), full["fc2_w"])
