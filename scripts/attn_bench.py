"""Time the mixed paged-attention kernel on representative OPT-13B (40 heads x 128) step shapes.

CUDA events around the C-ABI launch (work list built on the host per call, as in the forward);
algorithmic FLOPs/bytes per SURVEY §8d: FLOPs = sum 4*H*(q*p + q(q+1)/2), bytes = K+V read once
(4*H*(p+q)) + q read + out write (4*H*q).  Prints one JSON line per case.
"""
import json
import math
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2503_13737_b200 import kernels as K  # noqa: E402

HEADS = int(sys.argv[1]) if len(sys.argv) > 1 else 40

CASES = {
    "prefill_6x512": [(0, 512)] * 6,
    "prefill_3072": [(0, 3072)],
    "chunk2048_on_8k": [(8192, 2048)],
    "chunk1024_on_15k": [(15360, 1024)],
    "decode_256x2k": [(2000, 1)] * 256,
    "decode_64x8k": [(8000, 1)] * 64,
    "decode_1x100k": [(100000, 1)],
    "mixed": [(4096, 1024)] + [(1500, 1)] * 100 + [(0, 100)] * 10,
    "mixed_small_prompts": [(0, 37), (0, 300), (0, 900), (0, 17), (0, 650)] + [(700, 1)] * 40,
    "live_dec40": [(2200, 1)] * 40,
    "live_dec40_fresh300": [(2200, 1)] * 40 + [(0, 300)],
    "live_dec40_chunk280_on1200": [(2200, 1)] * 40 + [(1200, 280), (0, 20)],
    "live_dec60_chunk64_on510": [(2100, 1)] * 60 + [(510, 64)],
    "decode_var64": [(100 + (i * 977) % 4000, 1) for i in range(64)],
    "live_var48_chunk200": [(100 + (i * 977) % 4000, 1) for i in range(48)] + [(600, 200)],
}


def run(seqs, heads):
    g = torch.Generator().manual_seed(0)
    pages = [math.ceil((c + q) / 32) for c, q in seqs]
    nb = sum(pages) + 1
    perm = torch.randperm(nb, generator=g).to(torch.int32)
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
    btd = bt.cuda()
    out = torch.empty(S, heads * 128, device="cuda", dtype=torch.bfloat16)
    ws = torch.empty(256 << 20, device="cuda", dtype=torch.uint8)
    meta = (cu.cuda(), ctx.cuda())
    flush = torch.empty(256 << 20, device="cuda", dtype=torch.uint8)
    for _ in range(3):
        K.paged_attention(q, kp, vp, btd, cu, ctx, out=out, workspace=ws, device_meta=meta)
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        flush.zero_()  # L2 flush between timed launches
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        # keep the device busy while the host builds the work list, so the events bracket device
        # time only (as in the forward, where the list is built while earlier kernels run)
        torch.cuda._sleep(1_000_000)
        e0.record()
        K.paged_attention(q, kp, vp, btd, cu, ctx, out=out, workspace=ws, device_meta=meta)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / 1e3)
    t = sorted(ts)[len(ts) // 2]
    H = heads * 128
    fl = sum(4.0 * H * (qq * p + qq * (qq + 1) / 2) for p, qq in seqs)
    by = sum(4.0 * H * (p + qq) + 4.0 * H * qq for p, qq in seqs)
    return {"us": round(t * 1e6, 1), "tflops": round(fl / t / 1e12, 1), "gbs": round(by / t / 1e9, 1),
            "flops": fl, "bytes": by}


if __name__ == "__main__":
    if len(sys.argv) > 2:  # extra cases recorded from real batches (scripts/make_attn_cases.py)
        import json as _j
        CASES.update({k: [tuple(x) for x in v] for k, v in _j.load(open(sys.argv[2])).items()})
    only = os.environ.get("ATTN_CASES")  # comma-separated subset
    for name, seqs in CASES.items():
        if only and name not in only.split(","):
            continue
        r = run(seqs, HEADS)
        print(json.dumps({"case": name, "heads": HEADS, **r}), flush=True)
