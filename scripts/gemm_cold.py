"""GEMM timing with cold weights (8 rotating weight copies > L2), as inside the forward.
python scripts/gemm_cold.py [M,...]  -> one JSON line per (shape, M, plan)"""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2503_13737_b200 import kernels as K  # noqa: E402

SHAPES = {"qkv": (15360, 5120), "out": (5120, 5120), "fc1": (20480, 5120), "fc2": (5120, 20480)}
PLANS = [(128, 1, 0), (256, 1, 0), (128, 2, 0), (128, 4, 0), (256, 2, 0), (256, 1, 256), (128, 1, 256),
         (256, 2, 256), (256, 3, 256), (128, 2, 256), (64, 1, 0), (64, 2, 0), (64, 4, 0)]
Ms = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [64, 256, 384, 512]
torch.manual_seed(0)
for name, (N, Kd) in SHAPES.items():
    ws = [torch.randn(N, Kd, device="cuda", dtype=torch.bfloat16) * 0.02 for _ in range(8)]
    for M in Ms:
        a = torch.randn(M, Kd, device="cuda", dtype=torch.bfloat16)
        out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        row = {"shape": name, "M": M}
        for bn, ks, am in PLANS:
            if am == 256 and M < 256:
                continue
            try:
                for w in ws[:2]:
                    K.gemm(a, w, out=out, block_n=bn, k_splits=ks, a_rows=am)
            except Exception:
                continue
            # CUDA graph of 24 launches: device time only (host tensor-map encoding not in the loop)
            g = torch.cuda.CUDAGraph()
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                with torch.cuda.graph(g, stream=s):
                    for i in range(24):
                        K.gemm(a, ws[i % 8], out=out, block_n=bn, k_splits=ks, a_rows=am)
            torch.cuda.synchronize()
            g.replay()
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            torch.cuda.synchronize()
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            row[f"{bn}x{ks}" + ("p" if am == 256 else "")] = round(e0.elapsed_time(e1) / 24 * 1e3, 1)
        for w in ws[:2]:
            torch.matmul(a, w.T)
        e0.record()
        for i in range(24):
            torch.matmul(a, ws[i % 8].T)
        e1.record()
        torch.cuda.synchronize()
        row["cublas"] = round(e0.elapsed_time(e1) / 24 * 1e3, 1)
        row["hbm_floor_us"] = round(N * Kd * 2 / 6.5e12 * 1e6, 1)
        print(json.dumps(row), flush=True)
