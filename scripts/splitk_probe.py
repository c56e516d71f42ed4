import sys, torch
sys.path.insert(0,'.')
from paper_2503_13737_b200 import kernels as K
for (N,Kd,M,bn,ks,am) in [(5120,5120,64,128,2,0),(5120,5120,64,128,1,0),(5120,20480,256,256,3,256),(5120,20480,256,256,1,256),(5120,20480,64,128,2,0),(5120,20480,64,256,4,64)]:
    ws=[torch.randn(N,Kd,device='cuda',dtype=torch.bfloat16)*0.02 for _ in range(4)]
    a=torch.randn(M,Kd,device='cuda',dtype=torch.bfloat16); out=torch.empty(M,N,device='cuda',dtype=torch.bfloat16)
    for i in range(8): K.gemm(a, ws[i%4], out=out, block_n=bn, k_splits=ks, a_rows=am)
    torch.cuda.synchronize()
