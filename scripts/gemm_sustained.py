"""Sustained GEMM throughput at pivot-sized M, as inside the forward: the four OPT-13B projections of
40 layers (distinct weights, 25 GB: every weight read is cold), random activations, back to back, so
the clock settles where a long prefill step runs it (power cap).  Our tcgen05 kernel per plan vs
cuBLAS (torch.mm).  python scripts/gemm_sustained.py [M] -> one JSON line per implementation."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2503_13737_b200 import kernels as K  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 1536
L = 40
H, F = 5120, 20480
SHAPES = [("qkv", 3 * H, H), ("out", H, H), ("fc1", F, H), ("fc2", H, F)]
torch.manual_seed(0)
W = [[torch.randn(n, k, device="cuda", dtype=torch.bfloat16) * 0.02 for _, n, k in SHAPES] for _ in range(L)]
A = {k: torch.randn(M, k, device="cuda", dtype=torch.bfloat16) for k in (H, F)}
OUT = {n: torch.empty(M, n, device="cuda", dtype=torch.bfloat16) for _, n, _ in SHAPES}
flops = 2.0 * M * sum(n * k for _, n, k in SHAPES) * L


def run(fn, reps=3):
    for _ in range(1):
        fn()
    torch.cuda.synchronize()
    best = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best.append(e0.elapsed_time(e1))
    return sorted(best)[len(best) // 2]


def per_kind(fn_one):
    """Per-projection time (all layers), for the breakdown."""
    res = {}
    for j, (name, n, k) in enumerate(SHAPES):
        def f():
            for l in range(L):
                fn_one(A[k], W[l][j], OUT[n])
        ms = run(f)
        res[name] = {"ms": round(ms, 3), "tflops": round(2.0 * M * n * k * L / ms / 1e9, 1)}
    return res


def whole(fn_one):
    def f():
        for l in range(L):
            for j, (_, n, k) in enumerate(SHAPES):
                fn_one(A[k], W[l][j], OUT[n])
    return run(f)


impls = {
    "cublas": lambda a, w, o: torch.mm(a, w.t(), out=o),
    "ours_auto": lambda a, w, o: K.gemm(a, w, out=o),
    "ours_pair256": lambda a, w, o: K.gemm(a, w, out=o, block_n=256, k_splits=1, a_rows=256),
    "ours_1cta256": lambda a, w, o: K.gemm(a, w, out=o, block_n=256, k_splits=1, a_rows=128),
    "ours_pair128": lambda a, w, o: K.gemm(a, w, out=o, block_n=128, k_splits=1, a_rows=256),
}
for name, fn in impls.items():
    try:
        ms = whole(fn)
        line = {"impl": name, "M": M, "ms_40_layers": round(ms, 3), "tflops": round(flops / ms / 1e9, 1),
                "per_kind": per_kind(fn)}
    except Exception as e:  # noqa: BLE001
        line = {"impl": name, "M": M, "error": str(e)[:200]}
    print(json.dumps(line), flush=True)
