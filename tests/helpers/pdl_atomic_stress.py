"""Helper for tests/test_pdl_gpu.py: the configuration that hung before atomic-epilogue GEMMs fenced
their red.global.add (profiles/r2/pdl_hang.md).  The full 40-layer OPT-13B shape, every kernel
class launched early (the caller sets AG_PDL_MASK=15), out-proj / FC2 forced to stream-K over their fp32 accumulator
(finished by the early-launched LayerNorm) in every M bucket, and the attention kernel in the chain:
30 decode-heavy forwards must complete.  Prints the forward times."""
import ctypes as C
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2503_13737_b200 import _lib, model as M  # noqa: E402
from paper_2503_13737_b200.engine import DeviceBatch, synthetic_tokens  # noqa: E402
from paper_2503_13737_b200.executor import CudaExecutor  # noqa: E402

cfg = M.opt_13b(max_positions=4096)
rng = np.random.default_rng(0)
segs = [(int(c), 1) for c in rng.integers(300, 4000, 60)] + [(0, 30)]
ids, pos, slot, cu, ctx, tabs, nb = [], [], [], [0], [], [], 0
for i, (c, n) in enumerate(segs):
    tab = np.arange(nb, nb + (c + n + 31) // 32, dtype=np.int32)
    nb += len(tab)
    p = np.arange(c, c + n, dtype=np.int32)
    ids.append(synthetic_tokens(i, p, cfg.vocab).astype(np.int32))
    pos.append(p)
    slot.append((tab[p // 32] * 32 + p % 32).astype(np.int32))
    ctx.append(c)
    cu.append(cu[-1] + n)
    tabs.append(tab)
bt = np.zeros((len(tabs), max(map(len, tabs))), np.int32)
for i, t in enumerate(tabs):
    bt[i, :len(t)] = t
rids = list(range(len(segs)))
b = DeviceBatch(rids, np.concatenate(ids), np.concatenate(pos), np.asarray(cu, np.int32), np.asarray(ctx, np.int32),
                bt, np.concatenate(slot), np.asarray(cu[1:], np.int32) - 1, rids)
ex = CudaExecutor(cfg, nb + 8, max_tokens=256, max_seqs=128, autotune=False)
kinds = ("qkv", "out", "fc1", "fc2", "lm_head")
rows = []
for mb in (16, 32, 64, 128, 192, 256):  # stream-K (99) with 128-row A tiles for out / FC2, 1 CTA elsewhere
    for k in kinds:
        rows.append([kinds.index(k), mb, 128, (99 if k in ("out", "fc2") else 1) + 100 * 128])
buf = (C.c_int32 * (4 * len(rows)))(*[x for r in rows for x in r])
_lib.check(ex.lib.ag_model_set_gemm_plans(ex.handle, buf, len(rows)))
ts = [ex.execute(b).device_s * 1e3 for _ in range(30)]
ex.close()
print(f"30 forwards ok, median {sorted(ts)[15]:.2f} ms")
