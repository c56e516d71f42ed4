"""One tensor-parallel rank of the sharded CUDA forward, for tests/test_tp_gpu.py.

Several of these processes share ONE GPU; their per-layer all-reduces and the vocab-parallel argmax
all-gather go through the library's host collective backend (ag_model_init_tp_host) over a gloo
group, because NCCL refuses two ranks on one device.  Everything else is the production TP path:
Megatron shards (model.shard_layer), head-split paged attention, bias-after-reduce LayerNorm, the
vocab-parallel LM head (padded shard at TP=8) and the on-GPU argmax merge.

  python tests/tp_gpu_worker.py --rank R --world T --port P --case NAME --out FILE
"""
from __future__ import annotations

import argparse
import os
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
sys.path.insert(0, str(HERE))


def case(name: str):
    """(model config, weight seed, KV blocks, forwards as segment lists) -- shared with the test."""
    from paper_2503_13737_b200 import model as M
    if name == "13b2l":
        cfg = M.OPTConfig("opt-13b-2l", hidden=5120, num_layers=2, num_heads=40, ffn=20480, max_positions=4096)
        dec = [(10 + i, 20 + 7 * i) for i in range(24)]
        steps = [
            [(0, 0, 700), (1, 0, 300), (2, 0, 33)] + [(rid, 0, p) for rid, p in dec],
            [(0, 700, 256), (1, 300, 1), (2, 33, 1), (3, 0, 90)] + [(rid, p, 1) for rid, p in dec],
            [(0, 956, 1), (1, 301, 1), (2, 34, 1), (3, 90, 1)] + [(rid, p + 1, 1) for rid, p in dec],
        ]
        return cfg, 11, 1024, steps
    if name == "175b2l":  # config 5 shape: OPT-175B (H=12288, 96 heads, FFN 49152), 2 of 96 layers
        cfg = M.OPTConfig("opt-175b-2l", hidden=12288, num_layers=2, num_heads=96, ffn=49152, max_positions=4096)
        dec = [(10 + i, 30 + 11 * i) for i in range(16)]
        steps = [
            [(0, 0, 900), (1, 0, 257)] + [(rid, 0, p) for rid, p in dec],
            [(0, 900, 300), (1, 257, 1), (2, 0, 64)] + [(rid, p, 1) for rid, p in dec],
            [(0, 1200, 1), (1, 258, 1), (2, 64, 1)] + [(rid, p + 1, 1) for rid, p in dec],
        ]
        return cfg, 13, 1024, steps
    if name == "13b100k":  # config 4 regime: a 100k-token prompt chunked (8 chunks), a decode, + 2 short
        P, C = 100_000, 12_500
        cfg = M.OPTConfig("opt-13b-2l-100k", hidden=5120, num_layers=2, num_heads=40, ffn=20480, max_positions=P + 64)
        steps = [[(0, s, C)] for s in range(0, P - C, C)]
        steps.append([(0, P - C, C), (1, 0, 200)])
        steps.append([(0, P, 1), (1, 200, 1), (2, 0, 37)])
        return cfg, 17, P // 32 + 64, steps
    raise ValueError(name)


def checked_steps(name: str) -> set[int]:
    """Indices of the steps whose logits the test compares (all, except the long prefill chunks)."""
    cfg, _, _, steps = case(name)
    if name == "13b100k":
        return {len(steps) - 3, len(steps) - 2, len(steps) - 1}
    return set(range(len(steps)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rank", type=int, required=True)
    ap.add_argument("--world", type=int, required=True)
    ap.add_argument("--port", type=int, required=True)
    ap.add_argument("--case", default="13b2l")
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    import torch
    import torch.distributed as dist
    from batches import make_batch
    from paper_2503_13737_b200 import model as M
    from paper_2503_13737_b200.executor import CudaExecutor
    from paper_2503_13737_b200.kvc import BlockPool
    from paper_2503_13737_b200.tp import HostCollective

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{a.port}", rank=a.rank, world_size=a.world)
    cfg, seed, blocks, steps = case(a.case)
    w = M.init_weights(cfg, seed, device="cuda", tp_rank=a.rank, tp_size=a.world, init="test")
    hc = HostCollective(dist.group.WORLD, a.world)
    ex = CudaExecutor(cfg, blocks, max_tokens=max(4096, max(sum(n for *_, n in s) for s in steps)), max_seqs=64,
                      weights=w, tp_rank=a.rank, tp_size=a.world, parity_logits=True, autotune=False,
                      host_collective=hc, max_blocks_per_seq=(cfg.pos_rows + 31) // 32)
    pool = BlockPool(blocks)
    res = []
    for segs in steps:
        r = ex.execute(make_batch(pool, cfg, segs))
        res.append({"tokens": torch.from_numpy(r.token_ids.copy()), "logits": r.logits.clone()})
    torch.save({"res": res, "collective_calls": hc.calls, "launches": ex.launches}, a.out)
    ex.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
