"""LayerNorm kernel time (CUDA graph of 20 launches, device time only)."""
import sys
import torch
sys.path.insert(0, '.')
from paper_2503_13737_b200 import kernels as K
for rows in (64, 334, 1536):
    x = torch.randn(rows, 5120, device='cuda', dtype=torch.bfloat16)
    d = torch.randn(rows, 5120, device='cuda', dtype=torch.bfloat16) * 0
    g = torch.ones(5120, device='cuda', dtype=torch.bfloat16); b = torch.zeros_like(g)
    for delta in (None, d):
        K.layernorm(x, g, b, delta=delta)
        gr = torch.cuda.CUDAGraph(); s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            with torch.cuda.graph(gr, stream=s):
                for _ in range(20): K.layernorm(x, g, b, delta=delta)
        gr.replay(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); gr.replay(); e1.record(); torch.cuda.synchronize()
        print(rows, delta is not None, round(e0.elapsed_time(e1) / 20 * 1e3, 2), 'us', flush=True)
