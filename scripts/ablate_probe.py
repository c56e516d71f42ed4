"""Attribute the OPT-13B forward's device time to kernel classes inside the real (PDL-overlapped) launch
chain: the same batches are timed with AG_ABLATE=<class bits> skipping a class's launches (results are
garbage, timing only) and compared with the full forward.  Per-launch CUDA-event brackets cannot do this:
they serialise the chain and charge each short kernel its launch gap.

  AG_ABLATE=4 python scripts/ablate_probe.py TAG    -> one JSON line {tag, batch: median ms}
Classes (common.cuh PdlClass): 1 GEMM (+split-K reduce/finish), 2 attention (+combine), 4 LayerNorm,
8 embed/argmax/other."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2503_13737_b200 import model as Mo  # noqa: E402
from paper_2503_13737_b200.engine import DeviceBatch, synthetic_tokens  # noqa: E402
from paper_2503_13737_b200.executor import CudaExecutor  # noqa: E402

BS = 32


def build(segs, cfg, next_block):
    """segs: (cached tokens, new tokens) per sequence -> DeviceBatch with fresh, disjoint blocks."""
    ids, pos, slot, cu, ctx, tabs, lr = [], [], [], [0], [], [], []
    for i, (c, n) in enumerate(segs):
        nblk = (c + n + BS - 1) // BS
        tab = np.arange(next_block, next_block + nblk, dtype=np.int32)
        next_block += nblk
        p = np.arange(c, c + n, dtype=np.int32)
        ids.append(synthetic_tokens(i, p, cfg.vocab).astype(np.int32))
        pos.append(p)
        slot.append((tab[p // BS] * BS + p % BS).astype(np.int32))
        ctx.append(c)
        cu.append(cu[-1] + n)
        tabs.append(tab)
        lr.append(cu[-1] - 1)
    bt = np.zeros((len(tabs), max(map(len, tabs))), np.int32)
    for i, t in enumerate(tabs):
        bt[i, :len(t)] = t
    rids = list(range(len(segs)))
    return DeviceBatch(rids, np.concatenate(ids), np.concatenate(pos), np.asarray(cu, np.int32),
                       np.asarray(ctx, np.int32), bt, np.concatenate(slot), np.asarray(lr, np.int32), rids), next_block


rng = np.random.default_rng(0)
BATCHES = {
    # the bench's median step: ~60 decodes over 0.3-4k contexts + a short prompt chunk
    "decode60_chunk30": [(int(c), 1) for c in rng.integers(300, 4000, 60)] + [(0, 30)],
    # p90 step: 60 decodes + a 200-token chunk on a 1k prefix
    "decode60_chunk200": [(int(c), 1) for c in rng.integers(300, 4000, 60)] + [(1000, 200)],
    # pivot-sized prefill step: a 1536-token chunk on a 4k prefix + 16 decodes
    "pivot1536": [(4096, 1536)] + [(int(c), 1) for c in rng.integers(300, 4000, 16)],
}


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else os.environ.get("AG_ABLATE", "0")
    cfg = Mo.opt_13b(max_positions=8192)
    # timing only: every batch reuses block ids from 0 (its KV contents are whatever the last one wrote)
    need = max(sum((c + n + BS - 1) // BS for c, n in segs) for segs in BATCHES.values()) + 8
    ex = CudaExecutor(cfg, need, max_tokens=2048, max_seqs=256, autotune=True)
    out = {"tag": tag, "ablate": os.environ.get("AG_ABLATE", "0"), "pdl": os.environ.get("AG_PDL", "1")}
    for name, segs in BATCHES.items():
        b, _ = build(segs, cfg, 0)
        for _ in range(3):
            ex.execute(b)
        ts = sorted(ex.execute(b).device_s for _ in range(15))
        out[name] = round(ts[len(ts) // 2] * 1e3, 4)
    ex.close()
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
