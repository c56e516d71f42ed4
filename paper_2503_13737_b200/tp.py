"""Tensor-parallel plumbing: one process per GPU, rank 0 schedules, every rank executes.

Rank 0 runs the engine; each BatchPlan it packs is broadcast to the other ranks (a few KB of
int32 metadata over a gloo group on the host), then every rank launches the same forward on its
shard.  Inside the forward the per-layer out-proj/FC2 partial sums are all-reduced by NCCL over
NVLink (capi.cu), and the vocab-parallel argmax is merged with an NCCL all-gather.  Sharding:
model.shard_layer (QKV/FC1 by output rows, out-proj/FC2 by input columns, heads split evenly:
40/t for OPT-13B, 96/t for OPT-175B).
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from .engine import DeviceBatch, StepResult

OP_STOP, OP_STEP, OP_SWAP_OUT, OP_SWAP_IN, OP_MARK = 0, 1, 2, 3, 4
_HDR = 8


def pack_batch(b: DeviceBatch) -> tuple[torch.Tensor, torch.Tensor]:
    S, B, NL = b.num_tokens, int(b.ctx_len.shape[0]), int(b.logit_rows.shape[0])
    stride = int(b.block_table.shape[1]) if b.block_table.ndim == 2 else 0
    payload = np.concatenate([b.token_ids, b.positions, b.cu_q, b.ctx_len, b.block_table.reshape(-1), b.slot_mapping,
                              b.logit_rows, np.asarray(b.request_ids, np.int32),
                              np.asarray(b.logit_request_ids, np.int32)]).astype(np.int32)
    hdr = torch.tensor([OP_STEP, S, B, NL, stride, payload.size, 0, 0], dtype=torch.int64)
    return hdr, torch.from_numpy(payload)


def unpack_batch(hdr: torch.Tensor, payload: torch.Tensor) -> DeviceBatch:
    _, S, B, NL, stride, _, _, _ = [int(v) for v in hdr.tolist()]
    p = payload.numpy()
    o = 0

    def take(n):
        nonlocal o
        a = p[o:o + n]
        o += n
        return a

    ids, pos, cu, ctx = take(S), take(S), take(B + 1), take(B)
    bt = take(B * stride).reshape(B, stride)
    slot, lr = take(S), take(NL)
    rids, lids = take(B), take(NL)
    return DeviceBatch(rids.tolist(), ids, pos, cu, ctx, bt, slot, lr, lids.tolist())


def _bcast_msg(hdr: torch.Tensor, payload: torch.Tensor | None, group) -> None:
    dist.broadcast(hdr, src=0, group=group)
    if payload is not None and int(hdr[5]) > 0:
        dist.broadcast(payload, src=0, group=group)


class TPLeader:
    """Executor wrapper used on rank 0: broadcast, then run the local shard."""

    def __init__(self, local, group):
        self.local, self.group = local, group
        self.vocab, self.max_tokens, self.max_seqs = local.vocab, local.max_tokens, local.max_seqs

    def execute(self, batch: DeviceBatch) -> StepResult:
        hdr, payload = pack_batch(batch)
        _bcast_msg(hdr, payload, self.group)
        return self.local.execute(batch)

    def _swap(self, op, request_id, block_ids, tokens):
        ids = torch.tensor(list(block_ids), dtype=torch.int32)
        hdr = torch.tensor([op, request_id, tokens, 0, 0, ids.numel(), 0, 0], dtype=torch.int64)
        _bcast_msg(hdr, ids, self.group)

    def swap_out(self, request_id, block_ids, tokens):
        self._swap(OP_SWAP_OUT, request_id, block_ids, tokens)
        self.local.swap_out(request_id, block_ids, tokens)

    def swap_in(self, request_id, block_ids, tokens):
        self._swap(OP_SWAP_IN, request_id, block_ids, tokens)
        self.local.swap_in(request_id, block_ids, tokens)

    def mark(self, tag: int) -> None:
        """Forward a marker (e.g. timed-region begin / end) to the followers' on_mark callback."""
        _bcast_msg(torch.tensor([OP_MARK, tag, 0, 0, 0, 0, 0, 0], dtype=torch.int64), None, self.group)

    def stop(self) -> None:
        _bcast_msg(torch.zeros(_HDR, dtype=torch.int64), None, self.group)


def follower_loop(local, group, on_mark=None) -> int:
    """Ranks > 0: mirror rank 0's steps until OP_STOP; returns the number of steps executed."""
    steps = 0
    while True:
        hdr = torch.zeros(_HDR, dtype=torch.int64)
        dist.broadcast(hdr, src=0, group=group)
        op = int(hdr[0])
        if op == OP_STOP:
            return steps
        payload = torch.zeros(int(hdr[5]), dtype=torch.int32)
        if payload.numel():
            dist.broadcast(payload, src=0, group=group)
        if op == OP_STEP:
            local.execute(unpack_batch(hdr, payload))
            steps += 1
        elif op == OP_SWAP_OUT:
            local.swap_out(int(hdr[1]), payload.tolist(), int(hdr[2]))
        elif op == OP_SWAP_IN:
            local.swap_in(int(hdr[1]), payload.tolist(), int(hdr[2]))
        elif op == OP_MARK and on_mark is not None:
            on_mark(int(hdr[1]))


class HostCollective:
    """The library's host collective backend (ag_model_init_tp_host) over a torch.distributed group.

    Lets TP ranks run as processes that share ONE GPU (NCCL refuses two ranks on a device): the
    library stages each collective through pinned host memory and this callback completes it with
    the group (gloo).  bf16 all-reduces are summed in fp32 and rounded to bf16 once, as NCCL does
    for two ranks.  A correctness path for tests and bench smoke runs, not a performance path."""

    def __init__(self, group, tp_size: int):
        from . import _lib
        self.group, self.tp_size, self.calls = group, tp_size, 0
        self._L = _lib
        self.fn = _lib.HOST_COLLECTIVE_FN(self._call)  # keep a reference: the library holds the pointer

    def _call(self, ctx, op, ptr, count, dtype) -> int:
        import ctypes as C
        L = self._L
        try:
            self.calls += 1
            if op == L.COLL_ALLREDUCE_SUM:
                if dtype != L.DT_BF16:
                    return 2
                raw = np.ctypeslib.as_array((C.c_int16 * count).from_address(ptr))
                t = torch.from_numpy(raw).view(torch.bfloat16).float()
                dist.all_reduce(t, group=self.group)
                raw[:] = t.to(torch.bfloat16).view(torch.int16).numpy()
                return 0
            if op == L.COLL_ALLGATHER:
                ctype = {L.DT_F32: C.c_float, L.DT_I32: C.c_int32}.get(dtype)
                if ctype is None:
                    return 2
                buf = np.ctypeslib.as_array((ctype * (count * self.tp_size)).from_address(ptr))
                me = dist.get_rank(self.group)
                parts = [torch.empty(count, dtype=torch.float32 if dtype == L.DT_F32 else torch.int32)
                         for _ in range(self.tp_size)]
                dist.all_gather(parts, torch.from_numpy(buf[me * count:(me + 1) * count].copy()), group=self.group)
                for r, p in enumerate(parts):
                    buf[r * count:(r + 1) * count] = p.numpy()
                return 0
            return 3
        except Exception:  # pragma: no cover - surfaced to the library as a collective failure
            import traceback
            traceback.print_exc()
            return 1


def share_nccl_id(rank: int, group) -> bytes:
    """Rank 0 creates the library's NCCL unique id; everyone receives it over the host group."""
    from .executor import CudaExecutor
    buf = torch.zeros(128, dtype=torch.uint8)
    if rank == 0:
        buf = torch.frombuffer(bytearray(CudaExecutor.nccl_unique_id()), dtype=torch.uint8).clone()
    dist.broadcast(buf, src=0, group=group)
    return bytes(buf.tolist())
