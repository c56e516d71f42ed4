"""Thin torch-tensor front ends over the C-ABI kernels (device memory and streams from torch).

Each function validates shapes/dtypes, passes raw device pointers and the current CUDA stream
to libaccelgen_b200.so and raises the reference error classes on failure.  Used by the parity
tests, the B200 profiler and the swap path; the forward itself runs inside ``ag_model_forward``.
"""
from __future__ import annotations

import torch

from . import _lib
from .errors import EngineFault, ValidationError


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def _need_cuda(*ts: torch.Tensor | None) -> None:
    for t in ts:
        if t is not None and not t.is_cuda:
            raise EngineFault("libaccelgen_b200 kernels require CUDA tensors (no CPU fallback)")


_WS: dict = {}


def _workspace(device, nbytes: int) -> torch.Tensor:
    ws = _WS.get(device)
    if ws is None or ws.numel() < nbytes:
        ws = torch.empty(max(nbytes, 64 << 20), dtype=torch.uint8, device=device)
        _WS[device] = ws
    return ws


def gemm(a: torch.Tensor, w: torch.Tensor, bias: torch.Tensor | None = None, residual: torch.Tensor | None = None,
         relu: bool = False, out_f32: bool = False, out: torch.Tensor | None = None, block_n: int = 0,
         k_splits: int = 0, a_rows: int = 0) -> torch.Tensor:
    """D = a @ w.T (+bias) (+residual) (relu) on the tcgen05 GEMM; a [M,K], w [N,K] bf16.
    block_n / k_splits 0 = planned by the library (split-K partials in a cached workspace)."""
    _need_cuda(a, w, bias, residual, out)
    if a.dtype != torch.bfloat16 or w.dtype != torch.bfloat16:
        raise ValidationError("gemm operands must be bf16")
    M, K = a.shape
    N, K2 = w.shape
    if K != K2:
        raise ValidationError(f"K mismatch {K} vs {K2}")
    if out is None:
        out = torch.empty(M, N, device=a.device, dtype=torch.float32 if out_f32 else torch.bfloat16)
    ws = _workspace(a.device, 4 * max(1, k_splits, 16) * M * N)
    _lib.check(_lib.load().ag_gemm_bf16(
        a.data_ptr(), a.stride(0), w.data_ptr(), w.stride(0), _ptr(bias), _ptr(residual),
        residual.stride(0) if residual is not None else 0, int(relu), out.data_ptr(), out.stride(0), int(out_f32),
        M, N, K, block_n, k_splits, a_rows, ws.data_ptr(), ws.numel(), _stream()))
    return out


def kv_append(k: torch.Tensor, v: torch.Tensor, slot_mapping: torch.Tensor, k_pool: torch.Tensor,
              v_pool: torch.Tensor) -> None:
    """Scatter rows of k/v [rows, heads*128] into the paged pools [blocks, heads, 32, 128]."""
    _need_cuda(k, v, slot_mapping, k_pool, v_pool)
    heads, block_size = k_pool.shape[1], k_pool.shape[2]
    _lib.check(_lib.load().ag_kv_append(k.data_ptr(), v.data_ptr(), k.stride(0), slot_mapping.data_ptr(),
                                        k.shape[0], heads, block_size, k_pool.data_ptr(), v_pool.data_ptr(),
                                        _stream()))


def paged_attention(q: torch.Tensor, k_pool: torch.Tensor, v_pool: torch.Tensor, block_table: torch.Tensor,
                    cu_q: torch.Tensor, ctx_len: torch.Tensor, out: torch.Tensor | None = None,
                    workspace_bytes: int = 64 << 20, workspace: torch.Tensor | None = None,
                    device_meta: tuple[torch.Tensor, torch.Tensor] | None = None) -> torch.Tensor:
    """Mixed prefill/decode paged attention; q [S, heads*128] already scaled; cu_q/ctx_len int32 (CPU)."""
    _need_cuda(q, k_pool, v_pool, block_table)
    heads = k_pool.shape[1]
    cu_q_h = cu_q.to(torch.int32).cpu().contiguous()
    ctx_h = ctx_len.to(torch.int32).cpu().contiguous()
    cu_q_d, ctx_d = device_meta if device_meta is not None else (cu_q_h.to(q.device), ctx_h.to(q.device))
    if out is None:
        out = torch.zeros(q.shape[0], heads * 128, device=q.device, dtype=torch.bfloat16)
    ws = workspace if workspace is not None else torch.empty(workspace_bytes, device=q.device, dtype=torch.uint8)
    workspace_bytes = ws.numel()
    _lib.check(_lib.load().ag_paged_attention(
        q.data_ptr(), q.stride(0), k_pool.data_ptr(), v_pool.data_ptr(), k_pool.shape[0], block_table.data_ptr(),
        block_table.stride(0),
        cu_q_h.data_ptr(), ctx_h.data_ptr(), cu_q_d.data_ptr(), ctx_d.data_ptr(), ctx_h.numel(), heads,
        k_pool.shape[2], out.data_ptr(), out.stride(0), ws.data_ptr(), workspace_bytes, _stream()))
    return out


def layernorm(x: torch.Tensor, gamma: torch.Tensor, beta: torch.Tensor, eps: float = 1e-5,
              delta: torch.Tensor | None = None, delta_bias: torch.Tensor | None = None,
              row_index: torch.Tensor | None = None) -> torch.Tensor:
    """LN over rows (optionally of x[row_index]); with delta, x += delta (+bias) in place first."""
    _need_cuda(x, gamma, beta, delta, delta_bias, row_index)
    rows = row_index.numel() if row_index is not None else x.shape[0]
    out = torch.empty(rows, x.shape[1], device=x.device, dtype=torch.bfloat16)
    _lib.check(_lib.load().ag_layernorm(x.data_ptr(), _ptr(delta), _ptr(delta_bias), _ptr(row_index),
                                        gamma.data_ptr(), beta.data_ptr(), eps, rows, x.shape[1], out.data_ptr(),
                                        _stream()))
    return out


def rmsnorm(x: torch.Tensor, gamma: torch.Tensor, eps: float = 1e-6, delta: torch.Tensor | None = None) -> torch.Tensor:
    """RMSNorm over rows; with delta, x += delta in place first (residual stream)."""
    _need_cuda(x, gamma, delta)
    out = torch.empty_like(x)
    _lib.check(_lib.load().ag_rmsnorm(x.data_ptr(), _ptr(delta), gamma.data_ptr(), eps, x.shape[0], x.shape[1],
                                      out.data_ptr(), _stream()))
    return out


def rope(x: torch.Tensor, positions: torch.Tensor, heads: int, head_dim: int = 128, rotary_dim: int | None = None,
         theta: float = 10000.0) -> torch.Tensor:
    """Rotary embedding in place on x [rows, heads*head_dim] (rotate-half convention); returns x."""
    _need_cuda(x, positions)
    _lib.check(_lib.load().ag_rope(x.data_ptr(), x.stride(0), positions.data_ptr(), x.shape[0], heads, head_dim,
                                   rotary_dim or head_dim, theta, _stream()))
    return x


def embed_pos(ids: torch.Tensor, positions: torch.Tensor, tok_emb: torch.Tensor, pos_emb: torch.Tensor,
              pos_offset: int = 2) -> torch.Tensor:
    _need_cuda(ids, positions, tok_emb, pos_emb)
    out = torch.empty(ids.numel(), tok_emb.shape[1], device=ids.device, dtype=torch.bfloat16)
    _lib.check(_lib.load().ag_embed_pos(ids.data_ptr(), positions.data_ptr(), tok_emb.data_ptr(), pos_emb.data_ptr(),
                                        pos_offset, ids.numel(), tok_emb.shape[1], tok_emb.shape[0],
                                        pos_emb.shape[0], out.data_ptr(), _stream()))
    return out


def argmax(logits: torch.Tensor, index_offset: int = 0) -> tuple[torch.Tensor, torch.Tensor]:
    _need_cuda(logits)
    rows, cols = logits.shape
    val = torch.empty(rows, device=logits.device, dtype=torch.float32)
    idx = torch.empty(rows, device=logits.device, dtype=torch.int32)
    _lib.check(_lib.load().ag_argmax(logits.data_ptr(), rows, cols, logits.stride(0), index_offset, val.data_ptr(),
                                     idx.data_ptr(), _stream()))
    return val, idx


def kv_swap_out(pool: torch.Tensor, block_ids: torch.Tensor, staging: torch.Tensor) -> None:
    """staging[i] = pool[block_ids[i]] for whole blocks (pool [blocks, ...] bf16)."""
    _need_cuda(pool, block_ids, staging)
    block_elems = pool[0].numel()
    _lib.check(_lib.load().ag_kv_swap_out(pool.data_ptr(), block_ids.data_ptr(), block_ids.numel(), block_elems,
                                          staging.data_ptr(), _stream()))


def kv_swap_out_planes(pool: torch.Tensor, block_ids: torch.Tensor, staging: torch.Tensor, n: int) -> None:
    """staging[p, i] = pool[p, block_ids[i]] for every plane p (pool [P, blocks, ...], staging [P, slots, ...],
    both contiguous; i < n): all layers' K and V of a preempted request in one launch."""
    _need_cuda(pool, block_ids, staging)
    if not (pool.is_contiguous() and staging.is_contiguous()) or pool.shape[0] != staging.shape[0]:
        raise ValueError("kv_swap_out_planes: contiguous [planes, blocks, ...] pool and staging with equal planes")
    block_elems = pool[0, 0].numel()
    _lib.check(_lib.load().ag_kv_swap_out_planes(pool.data_ptr(), pool[0].numel(), block_ids.data_ptr(), n,
                                                 block_elems, staging.data_ptr(), staging[0].numel(),
                                                 pool.shape[0], _stream()))


def kv_swap_in_planes(staging: torch.Tensor, block_ids: torch.Tensor, pool: torch.Tensor, n: int) -> None:
    """pool[p, block_ids[i]] = staging[p, i] for every plane p and i < n."""
    _need_cuda(pool, block_ids, staging)
    if not (pool.is_contiguous() and staging.is_contiguous()) or pool.shape[0] != staging.shape[0]:
        raise ValueError("kv_swap_in_planes: contiguous [planes, blocks, ...] pool and staging with equal planes")
    block_elems = pool[0, 0].numel()
    _lib.check(_lib.load().ag_kv_swap_in_planes(staging.data_ptr(), staging[0].numel(), block_ids.data_ptr(), n,
                                                block_elems, pool.data_ptr(), pool[0].numel(), pool.shape[0],
                                                _stream()))


def kv_swap_in(staging: torch.Tensor, block_ids: torch.Tensor, pool: torch.Tensor) -> None:
    """pool[block_ids[i]] = staging[i]."""
    _need_cuda(pool, block_ids, staging)
    block_elems = pool[0].numel()
    _lib.check(_lib.load().ag_kv_swap_in(staging.data_ptr(), block_ids.data_ptr(), block_ids.numel(), block_elems,
                                         pool.data_ptr(), _stream()))
