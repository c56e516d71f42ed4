"""Per-kernel parity on the B200: each CUDA kernel (through the C-ABI) vs the CPU oracle
(bit-exact for integer/byte movement, stated tolerances for floating point)."""
import math

import pytest
import torch

from oracle import forward as orc

pytestmark = pytest.mark.gpu

DEV = "cuda"


@pytest.fixture(scope="module")
def K():
    from paper_2503_13737_b200 import kernels
    return kernels


def _bf(shape, seed, std=1.0):
    g = torch.Generator().manual_seed(seed)
    return (torch.randn(shape, generator=g) * std).to(torch.bfloat16)


@pytest.mark.parametrize("M,N,K_,bn", [
    (1, 256, 256, 0), (7, 768, 256, 0), (128, 256, 512, 256), (200, 1920, 640, 128), (777, 5120, 1024, 0),
    (1024, 3072, 5120, 256), (333, 50272, 256, 0), (2048, 2560, 5120, 0), (64, 1024, 4096, 128),
    (200, 1920, 640, 64), (5, 5120, 20480, 64), (64, 20480, 5120, 160), (300, 1600, 1024, 160),
])
@pytest.mark.parametrize("splits", [1, 3])
def test_gemm_matches_fp32(K, M, N, K_, bn, splits):
    a = _bf((M, K_), 1)
    w = _bf((N, K_), 2, 0.05)
    ref = a.float() @ w.float().T
    if splits > 1 and (K_ // 64) // splits < 2:
        pytest.skip("K too short for the split")
    out = K.gemm(a.to(DEV), w.to(DEV), block_n=bn if bn else 128, k_splits=splits)
    torch.cuda.synchronize()
    err = (out.float().cpu() - ref).abs().max().item()
    # bf16 output rounding (2^-8 relative) dominates; fp32 accumulation order is the rest
    assert err <= 2e-2 * ref.abs().max().item() + 1e-3, err


@pytest.mark.parametrize("M,N,K_,bn,splits,a_rows", [(1, 5120, 5120, 128, 1, 32), (32, 15360, 5120, 256, 2, 32),
                                                     (40, 20480, 5120, 160, 1, 64), (17, 3200, 2048, 160, 2, 32),
                                                     (60, 2048, 20480, 64, 4, 64), (64, 20480, 5120, 256, 1, 64)])
def test_gemm_small_m_variant(K, M, N, K_, bn, splits, a_rows):
    """Small-M path: only `a_rows` activation rows are staged; stale rows feed masked outputs only."""
    a, w = _bf((M, K_), 21), _bf((N, K_), 22, 0.05)
    bias, res = _bf((N,), 23), _bf((M, N), 24)
    ref = a.float() @ w.float().T + bias.float() + res.float()
    out = K.gemm(a.to(DEV), w.to(DEV), bias=bias.to(DEV), residual=res.to(DEV), block_n=bn, k_splits=splits,
                 a_rows=a_rows)
    torch.cuda.synchronize()
    assert torch.isfinite(out.float()).all()
    assert (out.float().cpu() - ref).abs().max().item() <= 2e-2 * ref.abs().max().item()


@pytest.mark.parametrize("M,N,K_,bn,splits", [(256, 512, 256, 256, 1), (300, 1920, 640, 128, 1), (1000, 5120, 1024, 256, 1),
                                              (777, 2560, 5120, 256, 2), (2048, 3072, 5120, 128, 1), (129, 768, 512, 256, 1),
                                              (192, 2560, 5120, 256, 1), (255, 1280, 2048, 128, 1)])
def test_gemm_cta_pair(K, M, N, K_, bn, splits):
    """CTA-pair (cta_group::2, 256-row tiles) kernel with bias + residual epilogue vs fp32."""
    a, w = _bf((M, K_), 31), _bf((N, K_), 32, 0.05)
    bias, res = _bf((N,), 33), _bf((M, N), 34)
    ref = a.float() @ w.float().T + bias.float() + res.float()
    out = K.gemm(a.to(DEV), w.to(DEV), bias=bias.to(DEV), residual=res.to(DEV), block_n=bn, k_splits=splits,
                 a_rows=256)
    torch.cuda.synchronize()
    assert (out.float().cpu() - ref).abs().max().item() <= 2e-2 * ref.abs().max().item()


@pytest.mark.parametrize("bn,splits", [(256, 1), (128, 4), (64, 2)])
def test_gemm_epilogue_bias_residual_relu_f32(K, bn, splits):
    M, N, K_ = 300, 1024, 768
    a, w = _bf((M, K_), 3), _bf((N, K_), 4, 0.05)
    bias, res = _bf((N,), 5), _bf((M, N), 6)
    ref = torch.relu(a.float() @ w.float().T + bias.float() + res.float())
    out = K.gemm(a.to(DEV), w.to(DEV), bias=bias.to(DEV), residual=res.to(DEV), relu=True, block_n=bn,
                 k_splits=splits)
    torch.cuda.synchronize()
    assert (out.float().cpu() - ref).abs().max().item() <= 2e-2 * ref.abs().max().item()
    ref32 = a.float() @ w.float().T + bias.float()
    out32 = K.gemm(a.to(DEV), w.to(DEV), bias=bias.to(DEV), out_f32=True)
    torch.cuda.synchronize()
    assert (out32.cpu() - ref32).abs().max().item() <= 1e-3 * ref32.abs().max().item() + 1e-4


@pytest.mark.parametrize("rows,H", [(37, 5120), (300, 256), (9, 12288)])  # warp-per-row / block kernels
def test_layernorm_plain_delta_gather(K, rows, H):
    x, d, db = _bf((rows, H), 7), _bf((rows, H), 8), _bf((H,), 9)
    g, b = (1 + 0.1 * _bf((H,), 10).float()).to(torch.bfloat16), _bf((H,), 11)
    out = K.layernorm(x.to(DEV), g.to(DEV), b.to(DEV))
    ref = orc.layernorm(x.float(), g, b)
    assert (out.float().cpu() - ref).abs().max().item() <= 3e-2
    xd = x.to(DEV)
    out2 = K.layernorm(xd, g.to(DEV), b.to(DEV), delta=d.to(DEV), delta_bias=db.to(DEV))
    xn = orc.rb(x.float() + (d.float() + db.float()))
    assert torch.equal(xd.float().cpu(), xn)  # residual stream update is exact
    assert (out2.float().cpu() - orc.layernorm(xn, g, b)).abs().max().item() <= 3e-2
    idx = torch.tensor([5 % rows, 0, rows - 1, 5 % rows], dtype=torch.int32)
    out3 = K.layernorm(x.to(DEV), g.to(DEV), b.to(DEV), row_index=idx.to(DEV))
    assert (out3.float().cpu() - orc.layernorm(x.float()[idx.long()], g, b)).abs().max().item() <= 3e-2


@pytest.mark.parametrize("rows,H", [(33, 5120), (7, 4096), (200, 256)])
def test_rmsnorm(K, rows, H):
    x, d = _bf((rows, H), 41), _bf((rows, H), 42)
    g = (1 + 0.1 * _bf((H,), 43).float()).to(torch.bfloat16)
    out = K.rmsnorm(x.to(DEV), g.to(DEV))
    assert (out.float().cpu() - orc.rmsnorm(x.float(), g)).abs().max().item() <= 3e-2
    xd = x.to(DEV)
    out2 = K.rmsnorm(xd, g.to(DEV), delta=d.to(DEV))
    xn = orc.rb(x.float() + d.float())
    assert torch.equal(xd.float().cpu(), xn)
    assert (out2.float().cpu() - orc.rmsnorm(xn, g)).abs().max().item() <= 3e-2


@pytest.mark.parametrize("rows,heads,rd", [(57, 4, 128), (5, 32, 64), (300, 2, 128)])
def test_rope(K, rows, heads, rd):
    x = _bf((rows, heads * 128), 44)
    pos = torch.randint(0, 16384, (rows,), dtype=torch.int32)
    out = K.rope(x.to(DEV).clone(), pos.to(DEV), heads, 128, rd)
    ref = orc.rope(x.float(), pos, heads, 128, rd)
    # fp32 angle (pos * inv_freq, as transformers computes it) vs the fp64 oracle: <= 4e-3 rad at
    # pos < 16384, then bf16 rounding of the output
    assert (out.float().cpu() - ref).abs().max().item() <= 3e-2


def test_embed_bit_exact(K):
    V, H, P = 1000, 256, 300
    te, pe = _bf((V, H), 12), _bf((P, H), 13)
    ids = torch.randint(0, V, (97,), dtype=torch.int32)
    pos = torch.randint(0, P - 2, (97,), dtype=torch.int32)
    out = K.embed_pos(ids.to(DEV), pos.to(DEV), te.to(DEV), pe.to(DEV))
    assert torch.equal(out.float().cpu(), orc.embed(ids, pos, te, pe))


def test_argmax_ties_lowest_index(K):
    logits = torch.randn(9, 50272)
    logits[3, 100] = 50.0
    logits[3, 7] = 50.0  # tie: lowest index wins
    logits[5, :] = 1.0
    val, idx = K.argmax(logits.to(DEV))
    ref = torch.argmax(logits, dim=-1)
    assert idx.cpu().tolist() == ref.tolist()
    assert idx[3].item() == 7 and idx[5].item() == 0


def test_kv_append_bit_exact(K):
    heads, nb, rows = 4, 64, 100
    kp = torch.zeros(nb, heads, 32, 128, dtype=torch.bfloat16)
    vp = torch.zeros_like(kp)
    k, v = _bf((rows, heads * 128), 14), _bf((rows, heads * 128), 15)
    slots = torch.randperm(nb * 32)[:rows].to(torch.int32)
    slots[3] = -1  # padding rows are skipped
    kd, vd = kp.to(DEV), vp.to(DEV)
    K.kv_append(k.to(DEV), v.to(DEV), slots.to(DEV), kd, vd)
    orc.kv_append(k, v, slots, kp, vp)
    assert torch.equal(kd.cpu(), kp) and torch.equal(vd.cpu(), vp)


def _attn_case(seqs, heads, seed):
    """seqs: list of (ctx_len, q_len).  Random pools, shuffled physical pages."""
    g = torch.Generator().manual_seed(seed)
    pages_per = [math.ceil((c + q) / 32) for c, q in seqs]
    nb = sum(pages_per) + 3
    perm = torch.randperm(nb, generator=g)
    stride = max(pages_per)
    bt = torch.zeros(len(seqs), stride, dtype=torch.int32)
    at = 0
    for i, n in enumerate(pages_per):
        bt[i, :n] = perm[at:at + n].to(torch.int32)
        at += n
    kp = (torch.randn(nb, heads, 32, 128, generator=g)).to(torch.bfloat16)
    vp = (torch.randn(nb, heads, 32, 128, generator=g)).to(torch.bfloat16)
    S = sum(q for _, q in seqs)
    q = (torch.randn(S, heads * 128, generator=g) / math.sqrt(128)).to(torch.bfloat16)
    cu = torch.tensor([0] + list(torch.cumsum(torch.tensor([q for _, q in seqs]), 0)), dtype=torch.int32)
    ctx = torch.tensor([c for c, _ in seqs], dtype=torch.int32)
    return q, kp, vp, bt, cu, ctx


ATTN_REL_TOL = 2e-2


def _attn_err(out, ref, heads):
    """Max over (query row, head) of max|out - ref| / max|ref| within that row-head's 128 dims.
    Normalised per row-head so long contexts -- whose outputs average ~N(0,1) values over up to
    100k keys and are ~1e-2 in magnitude -- cannot pass with a grossly wrong result."""
    d = (out.float().cpu() - ref.cpu()).abs().reshape(-1, heads, 128).amax(-1)
    scale = ref.cpu().abs().reshape(-1, heads, 128).amax(-1).clamp_min(1e-6)
    return (d / scale).max().item()


@pytest.mark.parametrize("seqs,heads", [
    ([(0, 100)], 2),
    ([(37, 1), (0, 5), (1000, 1), (0, 64), (5, 17)], 3),
    ([(300, 200), (5000, 64), (20000, 1), (0, 129), (63, 1), (64, 1), (65, 1)], 4),
    ([(16000, 2048)], 2),
    ([(100000, 1), (70000, 3)], 1),
    ([(c, 1) for c in range(0, 4000, 97)], 5),
])
def test_mixed_attention(K, seqs, heads):
    q, kp, vp, bt, cu, ctx = _attn_case(seqs, heads, seed=len(seqs) * 7 + heads)
    out = K.paged_attention(q.to(DEV), kp.to(DEV), vp.to(DEV), bt.to(DEV), cu, ctx)
    torch.cuda.synchronize()
    ref = orc.paged_attention(q.float(), kp, vp, bt, cu, ctx)
    err = _attn_err(out, ref, heads)
    assert err <= ATTN_REL_TOL, err


@pytest.mark.parametrize("seqs,heads", [
    # row path (q <= 16) vs tile path (q >= 17) boundary, at page (32) / KV-tile (128) boundaries
    ([(0, 16), (0, 17), (31, 16), (32, 17), (127, 1), (128, 1), (129, 17)], 3),
    ([(96, 31), (128, 128), (255, 129), (0, 257)], 2),
    # decode rows whose context straddles the split sizes (64-aligned row splits)
    ([(511, 1), (512, 1), (1023, 1), (1024, 1), (4095, 1), (4097, 1)], 4),
    # one long causal chunk over many tiles, heads of the 13B shard count
    ([(0, 1000)], 40),
    # chunk whose causal end is inside the first KV tile of a split
    ([(12000, 130), (7, 3)], 2),
    # many more (tile item, head) units than SMs: several waves of tile CTAs interleaved with the rows
    ([(0, 512)] * 6 + [(3000, 300), (9000, 1), (0, 40)], 24),
])
def test_mixed_attention_boundaries(K, seqs, heads):
    q, kp, vp, bt, cu, ctx = _attn_case(seqs, heads, seed=sum(c + n for c, n in seqs) % 997)
    out = K.paged_attention(q.to(DEV), kp.to(DEV), vp.to(DEV), bt.to(DEV), cu, ctx)
    torch.cuda.synchronize()
    ref = orc.paged_attention(q.float(), kp, vp, bt, cu, ctx)
    err = _attn_err(out, ref, heads)
    assert err <= ATTN_REL_TOL, err


def test_mixed_attention_back_to_back(K):
    """Consecutive launches of different shapes reuse the same host-built work-list buffers and
    split-KV partial workspace: each launch must cover exactly its own units (no stale items)."""
    cases = [([(0, 700)] * 3, 40), ([(2000, 129), (0, 5)], 40), ([(0, 700)] * 3, 40)]
    for seqs, heads in cases:
        q, kp, vp, bt, cu, ctx = _attn_case(seqs, heads, seed=11)
        out = K.paged_attention(q.to(DEV), kp.to(DEV), vp.to(DEV), bt.to(DEV), cu, ctx)
        torch.cuda.synchronize()
        ref = orc.paged_attention(q.float(), kp, vp, bt, cu, ctx)
        err = _attn_err(out, ref, heads)
        assert err <= ATTN_REL_TOL, (seqs[:2], err)


def test_kv_swap_roundtrip(K):
    pool = _bf((50, 2, 32, 128), 16).to(DEV)
    ids = torch.tensor([4, 9, 0, 31], dtype=torch.int32, device=DEV)
    staging = torch.empty(4, 2, 32, 128, dtype=torch.bfloat16, device=DEV)
    K.kv_swap_out(pool, ids, staging)
    assert torch.equal(staging, pool[ids.long()])
    new_ids = torch.tensor([40, 41, 42, 43], dtype=torch.int32, device=DEV)
    K.kv_swap_in(staging, new_ids, pool)
    assert torch.equal(pool[new_ids.long()], pool[ids.long()])


def test_kv_swap_planes_roundtrip(K):
    """All layers' K and V planes of a [P, blocks, ...] pool in one launch, into the first n slots of a
    larger staging ring slot and back into other blocks (byte-exact)."""
    pool = _bf((6, 50, 2, 32, 128), 17).to(DEV)
    ids = torch.tensor([4, 9, 0, 31, 7], dtype=torch.int32, device=DEV)
    staging = torch.zeros(6, 8, 2, 32, 128, dtype=torch.bfloat16, device=DEV)
    K.kv_swap_out_planes(pool, ids, staging, 5)
    assert torch.equal(staging[:, :5], pool[:, ids.long()])
    assert not staging[:, 5:].any()
    new_ids = torch.tensor([40, 41, 42, 43, 44], dtype=torch.int32, device=DEV)
    K.kv_swap_in_planes(staging, new_ids, pool, 5)
    assert torch.equal(pool[:, new_ids.long()], pool[:, ids.long()])
