"""One profiled launch of each hot kernel at a representative shape, for ncu evidence
(run as: ncu --profile-from-start off --set full ... python scripts/kernel_evidence.py).
cudaProfilerStart/Stop brackets exactly one launch per op after warm-up."""
import math
import sys

import torch

sys.path.insert(0, ".")
from paper_2503_13737_b200 import kernels as K  # noqa: E402

prof = torch.cuda.cudart()
torch.manual_seed(0)


def once(fn, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    prof.cudaProfilerStart()
    fn()
    torch.cuda.synchronize()
    prof.cudaProfilerStop()


# 1) QKV GEMM at the old pivot (M=3072, N=15360, K=5120) on the CTA-pair kernel: tensor-pipe bound
a = torch.randn(3072, 5120, device="cuda", dtype=torch.bfloat16)
w = torch.randn(15360, 5120, device="cuda", dtype=torch.bfloat16) * 0.02
o = torch.empty(3072, 15360, device="cuda", dtype=torch.bfloat16)
once(lambda: K.gemm(a, w, out=o, block_n=256, k_splits=1, a_rows=256))
# 2) FC2 at a decode-heavy step (M=64, K=20480): weight streaming, split-K 4 + reduce
a2 = torch.randn(64, 20480, device="cuda", dtype=torch.bfloat16)
w2 = torch.randn(5120, 20480, device="cuda", dtype=torch.bfloat16) * 0.02
o2 = torch.empty(64, 5120, device="cuda", dtype=torch.bfloat16)
once(lambda: K.gemm(a2, w2, out=o2, block_n=256, k_splits=4, a_rows=64))


def attn_case(seqs, heads=40):
    pages = [math.ceil((c + q) / 32) for c, q in seqs]
    nb = sum(pages) + 1
    perm = torch.randperm(nb).to(torch.int32)
    bt = torch.zeros(len(seqs), max(pages), dtype=torch.int32)
    at = 0
    for i, n in enumerate(pages):
        bt[i, :n] = perm[at:at + n]
        at += n
    kp = torch.randn(nb, heads, 32, 128, device="cuda", dtype=torch.bfloat16)
    vp = torch.randn(nb, heads, 32, 128, device="cuda", dtype=torch.bfloat16)
    S = sum(q for _, q in seqs)
    q = torch.randn(S, heads * 128, device="cuda", dtype=torch.bfloat16) / math.sqrt(128)
    cu = torch.tensor([0] + list(torch.cumsum(torch.tensor([x for _, x in seqs]), 0)), dtype=torch.int32)
    ctx = torch.tensor([c for c, _ in seqs], dtype=torch.int32)
    out = torch.empty(S, heads * 128, device="cuda", dtype=torch.bfloat16)
    ws = torch.empty(256 << 20, device="cuda", dtype=torch.uint8)
    meta = (cu.cuda(), ctx.cuda())
    btd = bt.cuda()
    return lambda: K.paged_attention(q, kp, vp, btd, cu, ctx, out=out, workspace=ws, device_meta=meta)


# 3) prefill attention: a 2048-row chunk on an 8k prefix (tcgen05 tile path)
once(attn_case([(8192, 2048)]))
# 4) decode attention: 256 sequences x 2k context (TMA + mma.sync row path)
once(attn_case([(2000, 1)] * 256))
# 5) standalone paged KV append: 4096 tokens x 40 heads
kv_rows = 4096
k = torch.randn(kv_rows, 5120, device="cuda", dtype=torch.bfloat16)
v = torch.randn(kv_rows, 5120, device="cuda", dtype=torch.bfloat16)
kp = torch.zeros(kv_rows // 32 + 8, 40, 32, 128, device="cuda", dtype=torch.bfloat16)
vp = torch.zeros_like(kp)
slots = torch.randperm(kp.shape[0] * 32, device="cuda")[:kv_rows].to(torch.int32)
once(lambda: K.kv_append(k, v, slots, kp, vp))
# 6) LayerNorm, 1536 rows x 5120 (warp per row)
x = torch.randn(1536, 5120, device="cuda", dtype=torch.bfloat16)
g = torch.ones(5120, device="cuda", dtype=torch.bfloat16)
b = torch.zeros(5120, device="cuda", dtype=torch.bfloat16)
once(lambda: K.layernorm(x, g, b))
print("ok")
