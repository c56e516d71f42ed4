import torch, time, sys
sys.path.insert(0, '.')
from paper_2503_13737_b200 import kernels as K
torch.manual_seed(0)
for (M,N,Kd) in [(2048,15360,5120),(2048,5120,5120),(2048,20480,5120),(2048,5120,20480),(8192,8192,8192),(4096,15360,5120)]:
    a=torch.randn(M,Kd,device='cuda',dtype=torch.bfloat16); w=torch.randn(N,Kd,device='cuda',dtype=torch.bfloat16)*0.02
    for bn in (128,256):
        out=torch.empty(M,N,device='cuda',dtype=torch.bfloat16)
        for _ in range(3): K.gemm(a,w,out=out,block_n=bn)
        torch.cuda.synchronize()
        e0=torch.cuda.Event(True); e1=torch.cuda.Event(True)
        e0.record()
        n=20
        for _ in range(n): K.gemm(a,w,out=out,block_n=bn)
        e1.record(); torch.cuda.synchronize()
        ms=e0.elapsed_time(e1)/n
        ref = torch.matmul(a,w.T)
        err=(out.float()-ref.float()).abs().max().item()
        print(f"M={M} N={N} K={Kd} bn={bn}: {ms*1e3:.1f} us  {2*M*N*Kd/ms/1e9:.1f} TFLOP/s  maxerr={err:.3g}", flush=True)
    # torch reference
    for _ in range(3): torch.matmul(a,w.T)
    torch.cuda.synchronize(); e0.record()
    for _ in range(20): torch.matmul(a,w.T)
    e1.record(); torch.cuda.synchronize(); ms=e0.elapsed_time(e1)/20
    print(f"   cublas: {ms*1e3:.1f} us {2*M*N*Kd/ms/1e9:.1f} TFLOP/s", flush=True)
