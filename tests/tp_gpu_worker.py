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
    raise ValueError(name)


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
    ex = CudaExecutor(cfg, blocks, max_tokens=4096, max_seqs=64, weights=w, tp_rank=a.rank, tp_size=a.world,
                      parity_logits=True, autotune=False, host_collective=hc)
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
