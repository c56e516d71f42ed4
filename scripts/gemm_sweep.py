"""Time the tcgen05 GEMM over (M, shape) for candidate (BLOCK_N, k_splits) plans; CUDA events."""
import itertools, json, sys, torch
sys.path.insert(0, '.')
from paper_2503_13737_b200 import kernels as K

SHAPES = {"qkv": (15360, 5120), "out": (5120, 5120), "fc1": (20480, 5120), "fc2": (5120, 20480)}
res = []
torch.manual_seed(0)
for name, (N, Kd) in SHAPES.items():
    w = torch.randn(N, Kd, device='cuda', dtype=torch.bfloat16) * 0.02
    for M in [int(x) for x in (sys.argv[1].split(',') if len(sys.argv) > 1 else (16, 64, 128, 256, 512, 768, 1024, 2048, 3072))]:
        a = torch.randn(M, Kd, device='cuda', dtype=torch.bfloat16)
        out = torch.empty(M, N, device='cuda', dtype=torch.bfloat16)
        ref = (a.float() @ w.float().T)
        row = {"shape": name, "M": M}
        for bn, ks, am in [(0, 0, 0), (256, 1, 0), (128, 1, 0), (256, 2, 0), (256, 4, 0), (128, 2, 0), (128, 4, 0),
                           (64, 4, 0), (128, 8, 0), (256, 1, 256), (128, 1, 256), (256, 2, 256), (128, 2, 256),
                           (256, 4, 256), (128, 4, 256)]:
            if am == 256 and M < 256:
                continue
            try:
                K.gemm(a, w, out=out, block_n=bn, k_splits=ks, a_rows=am)
            except Exception as e:
                continue
            torch.cuda.synchronize()
            err = (out.float() - ref).abs().max().item() / ref.abs().max().item()
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            for _ in range(3): K.gemm(a, w, out=out, block_n=bn, k_splits=ks, a_rows=am)
            e0.record()
            for _ in range(20): K.gemm(a, w, out=out, block_n=bn, k_splits=ks, a_rows=am)
            e1.record(); torch.cuda.synchronize()
            us = e0.elapsed_time(e1) / 20 * 1e3
            row[f"{bn}x{ks}" + ("p" if am == 256 else "")] = [round(us, 1), round(2 * M * N * Kd / us / 1e6, 1), round(N * Kd * 2 / us / 1e3, 2), err < 2e-2]
        for _ in range(3): torch.matmul(a, w.T)
        e0.record()
        for _ in range(20): torch.matmul(a, w.T)
        e1.record(); torch.cuda.synchronize()
        row["cublas"] = round(e0.elapsed_time(e1) / 20 * 1e3, 1)
        print(json.dumps(row), flush=True)
