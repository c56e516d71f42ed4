"""CPU ORACLE of the mixed-batch OPT forward — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg may
import this module.  The product path (paper_2503_13737_b200) never does.

What it restates
  The reference ships no forward pass: its "GPU" is the linear stand-in iteration_time
  (pkg/src/slosim/cost_model.py:101-109) and the paper's executor was vLLM + FlashAttention-2
  (PAPER.md:2002-2009), neither of which is under /root/reference.  Logit parity is therefore
  "parity unpinned" by the reference itself.  This oracle restates the OPT decoder the paper
  serves (per-layer QKV, attention, out-proj, FC1, FC2, residuals; the operation
  counts of Eq. 1-4 at PAPER.md:491-498) with the OPT details of transformers 5.5.0
  modeling_opt.py (learned positions offset 2, q*head_dim^-0.5, pre-LN, ReLU, tied LM head),
  executed over a PAGED KV cache driven by the same BatchPlan metadata as the GPU.  It is pinned
  against transformers' OPTForCausalLM by tests/golden/opt_tiny_hf.pt (tests/golden/make_golden.py).

Rounding points mirror the device kernels: activations are stored in bf16 between kernels
(q after scaling, K/V in the cache, attention output, residual stream, LN outputs, FC1 output);
every matmul accumulates in fp32; softmax and LN statistics are fp32; logits stay fp32.  In the
attention the unnormalised probabilities exp(s - max) are rounded to bf16 before P.V, while the
row sum l uses the fp32 values (attention.cu: pack_bf16x2 of p, l += p in fp32), then O = (P.V)/l.

Device: the restatement is plain torch.  It runs on the CPU by default; the large-shape tests
(40-layer OPT-13B, 100k-token contexts) run the SAME code on the GPU in fp32 with TF32 disabled
(``OracleOPT(..., device="cuda")``), where a CPU run would take hours.  It is still the checker,
never the product path.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import torch

POS_OFFSET = 2
HEAD_DIM = 128


ROUND_BF16 = True  # False = pure fp32 restatement (used to pin against transformers' fp32 OPT)
DEVICE = torch.device("cpu")  # where f32() materialises operands; OracleOPT switches it per forward
ACC = torch.float32           # accumulation dtype; float64 gives the same restatement with a different
                              # summation precision (tests use the fp32-vs-fp64 spread as bf16's noise floor)
ATTN_SCORE_ELEMS = 1 << 27     # heads x rows x kv_len fp32 scores held at once (query rows are chunked)


def rb(x: torch.Tensor) -> torch.Tensor:
    """Round to bf16 and return as fp32 (a storage point of the device pipeline)."""
    if not ROUND_BF16:
        return x
    return x.to(torch.bfloat16).to(ACC)


def f32(x: torch.Tensor) -> torch.Tensor:
    return x.detach().to(DEVICE, ACC)


def embed(ids, positions, tok_emb, pos_emb):
    return rb(f32(tok_emb)[ids.long()] + f32(pos_emb)[positions.long() + POS_OFFSET])


def layernorm(x, g, b, eps=1e-5):
    mean = x.mean(-1, keepdim=True)
    var = ((x - mean) ** 2).mean(-1, keepdim=True)
    return rb((x - mean) * torch.rsqrt(var + eps) * f32(g) + f32(b))


def rmsnorm(x, g, eps=1e-6):
    """Llama RMSNorm (transformers LlamaRMSNorm: fp32 statistics, weight applied after)."""
    return rb(x * torch.rsqrt((x * x).mean(-1, keepdim=True) + eps) * f32(g))


def rope(x, positions, heads, head_dim=128, rotary_dim=None, theta=10000.0):
    """Rotate-half rotary embedding (transformers apply_rotary_pos_emb with rotate_half) on
    x [rows, heads*head_dim] fp32; the first rotary_dim dims of each head rotate."""
    rd = rotary_dim or head_dim
    half = rd // 2
    inv_freq = theta ** (-torch.arange(0, half, dtype=torch.float64) * 2.0 / rd)
    ang = positions.double()[:, None] * inv_freq[None, :]
    cos, sin = torch.cos(ang).float()[:, None, :], torch.sin(ang).float()[:, None, :]
    y = x.clone().view(x.shape[0], heads, head_dim)
    x1, x2 = y[..., :half].clone(), y[..., half:rd].clone()
    y[..., :half] = x1 * cos - x2 * sin
    y[..., half:rd] = x2 * cos + x1 * sin
    return rb(y.view(x.shape[0], heads * head_dim))


def paged_attention(q, k_pool, v_pool, block_table, cu_q, ctx_len, block_size=32):
    """q [S, heads*128] (already scaled); pools [blocks, heads, bs, 128]; returns fp32 [S, heads*128].

    Sequence b's query row i sits at position ctx_len[b] + i and attends to kv positions
    0..ctx_len[b]+i of the sequence's pages (causal, prefix cache included)."""
    S = q.shape[0]
    heads = k_pool.shape[1]
    dev = q.device
    out = torch.zeros(S, heads * HEAD_DIM, dtype=ACC, device=dev)
    cu_q = [int(v) for v in cu_q]
    for b in range(len(cu_q) - 1):
        q0, q1 = cu_q[b], cu_q[b + 1]
        if q1 == q0:
            continue
        n_q = q1 - q0
        ctx = int(ctx_len[b])
        kv_len = ctx + n_q
        n_pages = (kv_len + block_size - 1) // block_size
        pages = block_table[b, :n_pages].long().to(k_pool.device)
        k = f32(k_pool[pages]).permute(1, 0, 2, 3).reshape(heads, n_pages * block_size, HEAD_DIM)[:, :kv_len]
        v = f32(v_pool[pages]).permute(1, 0, 2, 3).reshape(heads, n_pages * block_size, HEAD_DIM)[:, :kv_len]
        rows = max(1, ATTN_SCORE_ELEMS // (heads * kv_len))
        for r0 in range(0, n_q, rows):
            r1 = min(n_q, r0 + rows)
            qb = q[q0 + r0:q0 + r1].reshape(r1 - r0, heads, HEAD_DIM).permute(1, 0, 2)
            hi = ctx + r1  # keys past the chunk's last query row are masked for every row of it
            s = qb @ k[:, :hi].transpose(1, 2)  # [heads, rows, hi]
            qpos = ctx + torch.arange(r0, r1, device=dev).unsqueeze(1)
            kpos = torch.arange(hi, device=dev).unsqueeze(0)
            s = s.masked_fill(kpos > qpos, float("-inf"))
            p = torch.exp(s - s.amax(dim=-1, keepdim=True))
            l = p.sum(dim=-1, keepdim=True)
            o = (rb(p) @ v[:, :hi]) / l  # bf16 P into P.V, fp32 row sum (attention.cu)
            out[q0 + r0:q0 + r1] = o.permute(1, 0, 2).reshape(r1 - r0, heads * HEAD_DIM)
    return out


def kv_append(k_rows, v_rows, slot_mapping, k_pool, v_pool, block_size=32):
    """Write rows [S, heads*128] into their (block, offset) slots; slots < 0 are skipped."""
    heads = k_pool.shape[1]
    slots = slot_mapping.long().to(k_pool.device)
    keep = slots >= 0
    blk, off = slots[keep] // block_size, slots[keep] % block_size
    k_pool[blk, :, off, :] = k_rows[keep.to(k_rows.device)].reshape(-1, heads, HEAD_DIM).to(k_pool.device, k_pool.dtype)
    v_pool[blk, :, off, :] = v_rows[keep.to(v_rows.device)].reshape(-1, heads, HEAD_DIM).to(v_pool.device, v_pool.dtype)


@dataclass
class StepInputs:
    """The packed BatchPlan of one iteration (same fields as the C-ABI ag_step)."""
    token_ids: torch.Tensor
    positions: torch.Tensor
    cu_q: torch.Tensor
    ctx_len: torch.Tensor
    block_table: torch.Tensor
    slot_mapping: torch.Tensor
    logit_rows: torch.Tensor


class OracleOPT:
    """Paged-KV OPT forward on the CPU.  ``weights`` follows paper_2503_13737_b200.model.init_weights
    (full model, tp_size=1) or one TP shard when tp_size > 1 (then ``allreduce`` sums partials)."""

    def __init__(self, cfg, weights, num_blocks, block_size=32, tp_rank=0, tp_size=1, allreduce=None,
                 device="cpu", acc=torch.float32, tp_emulate=1):
        self.cfg = cfg
        self.acc = acc
        self.dev = torch.device(device)
        self.w = weights
        self.block_size = block_size
        self.tp_rank, self.tp_size = tp_rank, tp_size
        self.allreduce = allreduce
        # tp_emulate=t (unsharded weights): out-proj / FC2 as t column-shard partials, each rounded to bf16
        # as the sharded GEMM epilogue stores it, summed in fp32 and rounded once (the all-reduce), then
        # + bias + residual (the LayerNorm that follows the reduce) -- the TP=t device's rounding points
        self.tp_emulate = tp_emulate if tp_size == 1 else 1
        heads_l = cfg.num_heads // tp_size
        self.heads_l = heads_l
        pool_dtype = torch.bfloat16 if ROUND_BF16 else torch.float32
        self.k_pools = [torch.zeros(num_blocks, heads_l, block_size, HEAD_DIM, dtype=pool_dtype, device=self.dev)
                        for _ in range(cfg.num_layers)]
        self.v_pools = [torch.zeros_like(p) for p in self.k_pools]
        self.scale = 1.0 / math.sqrt(HEAD_DIM)

    def _reduce(self, partial):
        if self.tp_size == 1:
            return partial
        return self.allreduce(partial)

    def _row_parallel(self, a, w):
        """a @ w.T computed the way tp_emulate ranks do (Megatron row split of w by input columns)."""
        t = self.tp_emulate
        k = w.shape[1] // t
        parts = [rb(a[:, r * k:(r + 1) * k] @ f32(w[:, r * k:(r + 1) * k]).T) for r in range(t)]
        total = parts[0]
        for p in parts[1:]:
            total = total + p
        return rb(total)

    def forward(self, st: StepInputs):
        global DEVICE, ACC
        prev, DEVICE = DEVICE, self.dev
        prev_acc, ACC = ACC, self.acc
        tf32 = torch.backends.cuda.matmul.allow_tf32
        torch.backends.cuda.matmul.allow_tf32 = False  # true fp32 matmuls when run on the GPU
        try:
            return self._forward(st)
        finally:
            DEVICE, ACC = prev, prev_acc
            torch.backends.cuda.matmul.allow_tf32 = tf32

    def _forward(self, st: StepInputs):
        cfg, w = self.cfg, self.w
        dev = self.dev
        st = StepInputs(st.token_ids.to(dev), st.positions.to(dev), st.cu_q, st.ctx_len, st.block_table,
                        st.slot_mapping.to(dev), st.logit_rows.to(dev))
        hq = self.heads_l * HEAD_DIM
        x = embed(st.token_ids, st.positions, w["tok_emb"], w["pos_emb"])
        for l, L in enumerate(w["layers"]):
            h = layernorm(x, L["ln1_g"], L["ln1_b"], cfg.ln_eps)
            qkv = h @ f32(L["qkv_w"]).T + f32(L["qkv_b"])
            q = rb(qkv[:, :hq] * self.scale)
            k = rb(qkv[:, hq:2 * hq])
            v = rb(qkv[:, 2 * hq:])
            kv_append(k, v, st.slot_mapping, self.k_pools[l], self.v_pools[l], self.block_size)
            a = rb(paged_attention(q, self.k_pools[l], self.v_pools[l], st.block_table, st.cu_q, st.ctx_len,
                                   self.block_size))
            if self.tp_emulate > 1:
                x = rb(x + (self._row_parallel(a, L["out_w"]) + f32(L["out_b"])))
            elif self.tp_size == 1:
                x = rb(a @ f32(L["out_w"]).T + f32(L["out_b"]) + x)
            else:
                part = rb(self._reduce(rb(a @ f32(L["out_w"]).T)))  # bf16 all-reduce output
                x = rb(x + (part + f32(L["out_b"])))
            h = layernorm(x, L["ln2_g"], L["ln2_b"], cfg.ln_eps)
            f = rb(torch.relu(h @ f32(L["fc1_w"]).T + f32(L["fc1_b"])))
            if self.tp_emulate > 1:
                x = rb(x + (self._row_parallel(f, L["fc2_w"]) + f32(L["fc2_b"])))
            elif self.tp_size == 1:
                x = rb(f @ f32(L["fc2_w"]).T + f32(L["fc2_b"]) + x)
            else:
                part = rb(self._reduce(rb(f @ f32(L["fc2_w"]).T)))
                x = rb(x + (part + f32(L["fc2_b"])))
        rows = st.logit_rows.long()
        hl = layernorm(x[rows], w["final_g"], w["final_b"], cfg.ln_eps)
        logits = hl @ f32(w["tok_emb"]).T
        return logits.float().cpu(), torch.argmax(logits, dim=-1).to(torch.int32).cpu()
