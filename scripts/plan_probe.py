"""Forward time of a decode-only OPT-13B step (M sequences x ctx tokens) under forced GEMM plans for
one GEMM kind: python scripts/plan_probe.py KIND M [ctx].  Prints one line per plan."""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2503_13737_b200 import _lib, model as Mo  # noqa: E402
from paper_2503_13737_b200.engine import DeviceBatch, synthetic_tokens  # noqa: E402
from paper_2503_13737_b200.executor import CudaExecutor  # noqa: E402

kind, M = sys.argv[1], int(sys.argv[2])
ctx = int(sys.argv[3]) if len(sys.argv) > 3 else 1500
cfg = Mo.opt_13b(max_positions=4096)
blocks_per = (ctx + 1 + 31) // 32
nb = M * blocks_per + 8
ex = CudaExecutor(cfg, nb, max_tokens=1536, max_seqs=256)
bt = np.arange(M * blocks_per, dtype=np.int32).reshape(M, blocks_per)
pos = np.full(M, ctx, np.int32)
rids = np.arange(M)
b = DeviceBatch(list(rids), synthetic_tokens(rids, pos, cfg.vocab).astype(np.int32), pos,
                np.arange(M + 1, dtype=np.int32), np.full(M, ctx, np.int32), bt,
                (bt[:, ctx // 32] * 32 + ctx % 32).astype(np.int32), np.arange(M, dtype=np.int32), list(rids))
base = ex.gemm_plans()
kinds = ("qkv", "out", "fc1", "fc2", "lm_head")


def install(bn, ks, am):
    rows = [[kinds.index(k), mb, (bn if k == kind else b_), (ks if k == kind else k_) + 100 * (am if k == kind else a_)]
            for k, mb, b_, k_, a_ in base]
    buf = (C.c_int32 * (4 * len(rows)))(*[x for r in rows for x in r])
    _lib.check(ex.lib.ag_model_set_gemm_plans(ex.handle, buf, len(rows)))


def timed():
    for _ in range(3):
        ex.execute(b)
    ts = sorted(ex.execute(b).device_s for _ in range(7))
    return ts[3] * 1e3


print("autotuned", [p for p in base if p[0] == kind], f"{timed():.3f} ms")
for bn, ks, am in [(256, 1, 64), (128, 1, 64), (256, 99, 64), (128, 99, 64), (64, 99, 64), (256, 2, 64),
                   (256, 4, 64), (256, 6, 64), (128, 2, 64), (256, 1, 128), (256, 99, 128)]:
    if am < 128 and M > am:
        am = 128
    try:
        install(bn, ks, am)
        print(f"{kind} {bn}x{ks}a{am}: {timed():.3f} ms", flush=True)
    except Exception as e:  # noqa: BLE001
        print(f"{kind} {bn}x{ks}a{am}: error {e}", flush=True)
