"""CudaExecutor: runs each packed BatchPlan on the B200 through libaccelgen_b200.so.

Replaces the reference's "advance clock by iteration_time(S_f)" with a real
forward.  Ownership follows SURVEY §8b: weights and the KV pool are allocated once here (torch
is used only as the device allocator), the scheduler owns block-id assignment, metadata is
packed into pinned memory and copied H2D by the library each step, next-token ids come back
D2H.  There is no CPU fallback: without CUDA or the library this raises EngineFault.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import time
from pathlib import Path

import numpy as np
import torch

from . import _lib
from . import kernels as K
from .engine import DeviceBatch, StepResult
from .errors import EngineFault
from .model import HEAD_DIM, OPTConfig, init_weights


def _np_ptr(a: np.ndarray) -> int:
    return a.ctypes.data


class CudaExecutor:
    def __init__(self, cfg: OPTConfig, num_blocks: int, *, max_tokens: int = 4096, max_seqs: int = 512,
                 max_blocks_per_seq: int | None = None, tp_rank: int = 0, tp_size: int = 1, seed: int = 0,
                 init: str = "opt", weights: dict | None = None, device: int | None = None,
                 parity_logits: bool = False, nccl_uid: bytes | None = None, autotune: bool = True,
                 host_collective=None):
        if not torch.cuda.is_available():
            raise EngineFault("CudaExecutor needs a CUDA device (no CPU fallback)")
        self.lib = _lib.load()
        self.cfg = cfg
        self.tp_rank, self.tp_size = tp_rank, tp_size
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        self.vocab = cfg.vocab
        self.max_tokens, self.max_seqs = max_tokens, max_seqs
        self.block_size = 32
        self.num_blocks = num_blocks
        self.max_blocks_per_seq = max_blocks_per_seq or (cfg.pos_rows + self.block_size - 1) // self.block_size
        self.parity_logits = parity_logits
        heads_l = cfg.num_heads // tp_size
        self.heads_l = heads_l

        w = weights if weights is not None else init_weights(cfg, seed, self.device, tp_rank, tp_size, init)
        self.w = self._to_device(w)
        # one KV allocation for every layer: [L, 2, blocks, heads_l, 32, 128] bf16, zero-filled so
        # never-written slots hold finite values
        self.kv = torch.zeros(cfg.num_layers, 2, num_blocks, heads_l, self.block_size, HEAD_DIM,
                              dtype=torch.bfloat16, device=self.device)
        # weight init's fp32 temporaries stay in torch's cache; the library's own cudaMallocs (activations,
        # workspaces) need that HBM back -- with several ranks sharing one GPU (host TP backend) they failed
        torch.cuda.empty_cache()

        mc = _lib.ModelConfig(hidden=cfg.hidden, num_layers=cfg.num_layers, num_heads=cfg.num_heads, ffn=cfg.ffn,
                              vocab=cfg.vocab, pos_rows=cfg.pos_rows, tp_rank=tp_rank, tp_size=tp_size,
                              num_blocks=num_blocks, block_size=self.block_size, max_tokens=max_tokens,
                              max_seqs=max_seqs, max_blocks_per_seq=self.max_blocks_per_seq, ln_eps=cfg.ln_eps)
        handle = C.c_void_p()
        with torch.cuda.device(self.device):
            _lib.check(self.lib.ag_model_create(C.byref(mc), C.byref(handle)))
        self.handle = handle
        ww = self.w
        _lib.check(self.lib.ag_model_set_embeddings(handle, ww["tok_emb"].data_ptr(), ww["pos_emb"].data_ptr(),
                                                    ww["final_g"].data_ptr(), ww["final_b"].data_ptr()))
        for l, L in enumerate(ww["layers"]):
            lw = _lib.LayerWeights(*[L[name].data_ptr() for name, _ in _lib.LayerWeights._fields_])
            _lib.check(self.lib.ag_model_set_layer(handle, l, C.byref(lw)))
            _lib.check(self.lib.ag_model_set_kv_cache(handle, l, self.kv[l, 0].data_ptr(), self.kv[l, 1].data_ptr()))
        self.host_collective = host_collective
        if tp_size > 1:
            if host_collective is not None:  # tp.HostCollective: ranks sharing one GPU (tests)
                _lib.check(self.lib.ag_model_init_tp_host(handle, C.cast(host_collective.fn, C.c_void_p), None))
            elif nccl_uid is None:
                raise EngineFault("tp_size > 1 needs the NCCL unique id broadcast by rank 0 (or a host collective)")
            else:
                buf = C.create_string_buffer(bytes(nccl_uid), 128)
                _lib.check(self.lib.ag_model_init_tp(handle, buf))
        if autotune:
            self._autotune()
        self._dev_ms = C.c_float(0.0)
        self._swapped: dict[int, torch.Tensor] = {}
        self.logits_buf = torch.empty(max_seqs, cfg.vocab // tp_size, dtype=torch.float32, device=self.device) \
            if parity_logits else None
        self.steps = 0
        self.launches = 0       # our kernel launches summed over executed steps
        self.h2d_bytes = 0
        self.d2h_bytes = 0

    def set_profiling(self, on: bool) -> None:
        _lib.check(self.lib.ag_model_set_profiling(self.handle, int(on)))

    def set_roofline_peaks(self, tensor_tflops: float, hbm_gbs: float) -> None:
        _lib.check(self.lib.ag_model_set_roofline_peaks(self.handle, float(tensor_tflops), float(hbm_gbs)))

    def profile(self) -> dict:
        n = len(_lib.PROF_CLASSES)
        ms, fl, by, roof = (C.c_double * n)(), (C.c_double * n)(), (C.c_double * n)(), (C.c_double * n)()
        cnt = (C.c_int64 * n)()
        _lib.check(self.lib.ag_model_get_profile(self.handle, ms, fl, by, cnt, n))
        _lib.check(self.lib.ag_model_get_roofline_ms(self.handle, roof, n))
        return {name: {"ms": ms[i], "flops": fl[i], "bytes": by[i], "launches": cnt[i], "roofline_ms": roof[i]}
                for i, name in enumerate(_lib.PROF_CLASSES)}

    def _autotune(self) -> None:
        """Time the GEMM plan candidates on this GPU, or reuse a table cached by an earlier run of the
        same library on the same GPU model and shapes (AG_GEMM_PLAN_CACHE=<dir>, opt-in)."""
        cache_dir = os.environ.get("AG_GEMM_PLAN_CACHE")
        key = None
        if cache_dir:
            import hashlib
            lib_hash = hashlib.sha1(Path(_lib.LIB_PATH).read_bytes()).hexdigest()[:12]
            cfg = self.cfg
            key = Path(cache_dir) / (f"plans_{torch.cuda.get_device_name(self.device).replace(' ', '_')}_{lib_hash}_"
                                     f"h{cfg.hidden}_f{cfg.ffn}_v{cfg.vocab}_l{cfg.num_layers}_tp{self.tp_size}_"
                                     f"t{self.max_tokens}_s{self.max_seqs}.json")
            if key.exists():
                rows = json.loads(key.read_text())
                buf = (C.c_int32 * (4 * len(rows)))(*[x for r in rows for x in r])
                _lib.check(self.lib.ag_model_set_gemm_plans(self.handle, buf, len(rows)))
                return
        with torch.cuda.device(self.device):
            _lib.check(self.lib.ag_model_autotune(self.handle, torch.cuda.current_stream(self.device).cuda_stream))
        if key is not None:
            buf = (C.c_int32 * (4 * 512))()
            n = int(self.lib.ag_model_get_gemm_plans(self.handle, buf, 512))
            key.parent.mkdir(parents=True, exist_ok=True)
            key.write_text(json.dumps([[buf[4 * i + j] for j in range(4)] for i in range(min(n, 512))]))

    def gemm_plans(self) -> list[tuple[str, int, int, int]]:
        kinds = ("qkv", "out", "fc1", "fc2", "lm_head")
        buf = (C.c_int32 * (4 * 512))()
        n = int(self.lib.ag_model_get_gemm_plans(self.handle, buf, 512))
        # (kind, m_bucket, block_n, k_splits, a_rows)
        return [(kinds[buf[4 * i]], buf[4 * i + 1], buf[4 * i + 2], buf[4 * i + 3] % 100, buf[4 * i + 3] // 100)
                for i in range(min(n, 512))]

    @staticmethod
    def nccl_unique_id() -> bytes:
        lib = _lib.load()
        buf = C.create_string_buffer(128)
        _lib.check(lib.ag_nccl_get_unique_id(buf))
        return buf.raw

    def _to_device(self, w: dict) -> dict:
        def mv(t):
            return t.to(self.device, torch.bfloat16).contiguous()
        out = {k: mv(v) for k, v in w.items() if k != "layers"}
        out["layers"] = [{k: mv(v) for k, v in L.items()} for L in w["layers"]]
        return out

    def close(self) -> None:
        if getattr(self, "handle", None):
            self.lib.ag_model_destroy(self.handle)
            self.handle = None
        # the KV pool (sized from free HBM by the bench / CLI) and the weights go back to torch's
        # allocator even if a reference cycle keeps this object alive
        self.kv = self.w = self.logits_buf = None
        if getattr(self, "_swapped", None):
            self._swapped.clear()

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    # ---------------------------------------------------------------- step
    def make_step(self, b: DeviceBatch) -> tuple[_lib.Step, list[np.ndarray]]:
        arrs = [np.ascontiguousarray(a, dtype=np.int32) for a in
                (b.token_ids, b.positions, b.cu_q, b.ctx_len, b.block_table, b.slot_mapping, b.logit_rows)]
        ids, pos, cu, ctx, bt, slot, lr = arrs
        st = _lib.Step(num_tokens=ids.shape[0], num_seqs=ctx.shape[0], num_logits=lr.shape[0],
                       block_table_stride=bt.shape[1] if bt.ndim == 2 and bt.shape[1] > 0 else 1,
                       token_ids=_np_ptr(ids), positions=_np_ptr(pos), cu_q=_np_ptr(cu), ctx_len=_np_ptr(ctx),
                       block_table=_np_ptr(bt), slot_mapping=_np_ptr(slot), logit_rows=_np_ptr(lr))
        return st, arrs

    def execute(self, batch: DeviceBatch) -> StepResult:
        st, keep = self.make_step(batch)
        n = int(batch.logit_rows.shape[0])
        out = np.zeros(max(n, 1), dtype=np.int32)
        logits_ptr = self.logits_buf.data_ptr() if self.logits_buf is not None else None
        stream = torch.cuda.current_stream(self.device).cuda_stream
        t0 = time.perf_counter()
        _lib.check(self.lib.ag_model_forward(self.handle, C.byref(st), _np_ptr(out), logits_ptr,
                                             C.byref(self._dev_ms), stream))
        wall = time.perf_counter() - t0
        del keep
        self.steps += 1
        self.launches += int(self.lib.ag_model_last_launches(self.handle))
        self.h2d_bytes += int(self.lib.ag_model_last_h2d_bytes(self.handle))
        self.d2h_bytes += 4 * n
        logits = self.logits_buf[:n].cpu() if self.logits_buf is not None else None
        dev_s = self._dev_ms.value / 1e3
        return StepResult(token_ids=out[:n].copy(), elapsed_s=dev_s, device_s=dev_s, wall_s=wall, logits=logits)

    # ---------------------------------------------------------------- asynchronous steps
    def clock_ref(self) -> float:
        """Record the device reference event and return the host time it completed at; wait() maps each
        step's device completion onto this host clock (perf_counter seconds)."""
        _lib.check(self.lib.ag_model_clock_ref(self.handle, torch.cuda.current_stream(self.device).cuda_stream))
        self._ref_host = time.perf_counter()
        return self._ref_host

    def submit(self, batch: DeviceBatch, feed: np.ndarray | None = None) -> None:
        """Enqueue one forward and return (ag_model_submit); feed = int32 [n, 2] (token index, logit row of
        the previous submitted step) for decode inputs still on the device.  At most two in flight."""
        if getattr(self, "_ref_host", None) is None:
            self.clock_ref()
        st, keep = self.make_step(batch)
        n_feed = 0 if feed is None else int(feed.shape[0])
        fp = np.ascontiguousarray(feed, dtype=np.int32) if n_feed else None
        logits_ptr = self.logits_buf.data_ptr() if self.logits_buf is not None else None
        stream = torch.cuda.current_stream(self.device).cuda_stream
        t0 = time.perf_counter()
        _lib.check(self.lib.ag_model_submit(self.handle, C.byref(st), _np_ptr(fp) if n_feed else None, n_feed,
                                            logits_ptr, stream))
        wall = time.perf_counter() - t0
        del keep
        self.steps += 1
        self.launches += int(self.lib.ag_model_last_launches(self.handle))
        self.h2d_bytes += int(self.lib.ag_model_last_h2d_bytes(self.handle))
        n = int(batch.logit_rows.shape[0])
        self.d2h_bytes += 4 * n
        self._pending = getattr(self, "_pending", [])
        self._pending.append((n, wall))

    def wait(self) -> StepResult:
        """Complete the oldest submitted step: next-token ids, device time and completion time
        (StepResult.end_s, host perf_counter seconds)."""
        n, wall = self._pending.pop(0)
        out = np.zeros(max(n, 1), dtype=np.int32)
        end_ms = C.c_double(0.0)
        _lib.check(self.lib.ag_model_wait(self.handle, _np_ptr(out), max(n, 1), C.byref(self._dev_ms),
                                          C.byref(end_ms)))
        dev_s = self._dev_ms.value / 1e3
        res = StepResult(token_ids=out[:n].copy(), elapsed_s=dev_s, device_s=dev_s, wall_s=wall)
        res.end_s = self._ref_host + end_ms.value / 1e3
        return res

    def inflight(self) -> int:
        return int(self.lib.ag_model_inflight(self.handle))

    # ---------------------------------------------------------------- preemption swap (kvc.py:153-160)
    _SWAP_STAGE_BYTES = 512 << 20  # per staging slot (a request's KV can be tens of GB: moved slot by slot)
    _SWAP_SLOTS = 4

    def _swap_init(self) -> None:
        """Staging ring in HBM + a copy stream: a swap never blocks the host.  Swap-out gathers the
        victim's blocks into a slot on the compute stream (ordered after the forwards that wrote them;
        the freed blocks can be reallocated at once) and the copy stream drains the slot to pinned host
        memory while later forwards run.  Swap-in copies host -> slot on the copy stream and the compute
        stream waits for that copy only, then scatters into the newly allocated blocks."""
        if getattr(self, "_stage", None) is not None:
            return
        per_block = self.cfg.num_layers * 2 * self.heads_l * self.block_size * HEAD_DIM * 2
        self._stage_blocks = max(1, self._SWAP_STAGE_BYTES // per_block)
        self._stage = [torch.empty(self.cfg.num_layers, 2, self._stage_blocks, self.heads_l, self.block_size,
                                   HEAD_DIM, dtype=torch.bfloat16, device=self.device)
                       for _ in range(self._SWAP_SLOTS)]
        planes = self.cfg.num_layers * 2  # [L, 2, blocks, ...] viewed as [L*2, blocks, ...]
        self._kv_planes = self.kv.view(planes, *self.kv.shape[2:])
        self._stage_planes = [s.view(planes, *s.shape[2:]) for s in self._stage]
        self._slot_free = [None] * self._SWAP_SLOTS  # event after which the slot may be overwritten
        self._slot_keep = [[] for _ in range(self._SWAP_SLOTS)]  # host tensors the slot's copies still read
        self._next_slot = 0
        self._copy_stream = torch.cuda.Stream(self.device)
        self._host_free: list[tuple[torch.Tensor, torch.cuda.Event | None]] = []  # reusable host chunks
        self.swap_host_chunks = 0  # host chunks allocated (pinned unless the OS refused)
        self.swap_bytes = 0
        self.swap_wait_s, self.swap_waits = 0.0, 0  # host time blocked on a draining staging slot
        self.swap_host_s = 0.0  # host time inside swap_out / swap_in (launches, pinned allocation, waits)
        self.swap_section_s = {"acquire_slot": 0.0, "host_chunk": 0.0, "ids": 0.0, "enqueue": 0.0}

    def _acquire_slot(self) -> int:
        i = self._next_slot
        self._next_slot = (i + 1) % self._SWAP_SLOTS
        if self._slot_free[i] is not None:
            if not self._slot_free[i].query():  # only blocks when every slot is still draining
                t0 = time.perf_counter()
                self._slot_free[i].synchronize()
                self.swap_wait_s += time.perf_counter() - t0
                self.swap_waits += 1
            self._slot_free[i] = None
        self._slot_keep[i] = []
        return i

    def _ids_on_device(self, ids: list[int], keep: list) -> torch.Tensor:
        h = torch.tensor(ids, dtype=torch.int32).pin_memory()
        keep.append(h)  # the async H2D reads it later
        return h.to(self.device, non_blocking=True)

    def _host_chunk(self, n: int) -> tuple[torch.Tensor, torch.Tensor]:
        """A host chunk for n staged blocks: (the backing 1-D buffer, a contiguous [L, 2, n, heads, 32, 128]
        view of its head).  Every chunk is one full staging slot, so chunks are interchangeable: swap-in
        hands them back to a free list once their H2D copy is done and swap-out reuses them, instead of
        pinning fresh memory per swap (page-locking a multi-GB buffer blocked the host for seconds).
        Pageable memory when the OS refuses to lock more pages."""
        per_block = self._stage[0][:, :, 0].numel()
        shape = (self.cfg.num_layers, 2, n) + tuple(self._stage[0].shape[3:])
        # oldest first, and only a chunk whose H2D copy (swap-in) has finished; a fresh chunk otherwise --
        # waiting on a pending copy would block the host behind the copy stream's queue
        for i, (flat, ready) in enumerate(self._host_free):
            if ready is None or ready.query():
                del self._host_free[i]
                return flat, flat[: n * per_block].view(shape)
        flat = self._alloc_chunk()
        return flat, flat[: n * per_block].view(shape)

    def _alloc_chunk(self) -> torch.Tensor:
        """A fresh slot-sized host chunk: pinned, or pageable once the OS refuses to lock more pages."""
        per_block = self._stage[0][:, :, 0].numel()
        flat = None
        if not getattr(self, "_pin_failed", False):
            try:
                flat = torch.empty(self._stage_blocks * per_block, dtype=torch.bfloat16, pin_memory=True)
            except Exception:  # RuntimeError / torch.AcceleratorError: out of lockable memory
                self._pin_failed = True
        if flat is None:
            flat = torch.empty(self._stage_blocks * per_block, dtype=torch.bfloat16)
        self.swap_host_chunks += 1
        return flat

    def prepare_swap(self, host_gb: float) -> None:
        """Allocate the staging ring and pin ~host_gb of host chunks up front (bench setup), so the first
        preemptions do not page-lock memory on the serving path."""
        self._swap_init()
        n = int(host_gb * 1e9 // (self._stage_blocks * self._stage[0][:, :, 0].numel() * 2))
        # fresh chunks only: _host_chunk would hand back the chunk just added (the pool stayed at one
        # chunk and every preemption page-locked memory on the serving path)
        for _ in range(max(0, n)):
            chunk = self._alloc_chunk()
            if getattr(self, "_pin_failed", False):  # the OS refused: a pageable pool would only add sync copies
                break
            self._host_free.append((chunk, None))

    def swap_out(self, request_id: int, block_ids: list[int], tokens: int) -> None:
        """Preemption (reference BlockPool.preempt, kvc.py:153-160): the request's KV blocks of every
        layer go to host memory, asynchronously (see _swap_init)."""
        if not block_ids:
            return
        self._swap_init()
        t_host = time.perf_counter()
        comp = torch.cuda.current_stream(self.device)
        host_chunks = []
        sec = self.swap_section_s
        for c0 in range(0, len(block_ids), self._stage_blocks):
            t = time.perf_counter()
            slot = self._acquire_slot()
            sec["acquire_slot"] += time.perf_counter() - t
            stage = self._stage[slot]
            keep = self._slot_keep[slot]
            t = time.perf_counter()
            ids = self._ids_on_device(block_ids[c0:c0 + self._stage_blocks], keep)
            sec["ids"] += time.perf_counter() - t
            n = ids.numel()
            t = time.perf_counter()
            # every layer's K and V in one launch (80 per-plane launches cost ~2 ms of host time per slot)
            K.kv_swap_out_planes(self._kv_planes, ids, self._stage_planes[slot], n)
            gathered = torch.cuda.Event()
            gathered.record(comp)
            sec["enqueue"] += time.perf_counter() - t
            t = time.perf_counter()
            flat, host = self._host_chunk(n)
            sec["host_chunk"] += time.perf_counter() - t
            t = time.perf_counter()
            with torch.cuda.stream(self._copy_stream):
                self._copy_stream.wait_event(gathered)
                host.copy_(stage[:, :, :n], non_blocking=host.is_pinned())
                done = torch.cuda.Event()
                done.record(self._copy_stream)
            self._slot_free[slot] = done
            sec["enqueue"] += time.perf_counter() - t
            host_chunks.append((flat, host))
            self.swap_bytes += host.numel() * 2
        self._swapped[request_id] = host_chunks
        self.swap_host_s += time.perf_counter() - t_host

    def swap_in(self, request_id: int, block_ids: list[int], tokens: int) -> None:
        host_chunks = self._swapped.pop(request_id, None)
        if host_chunks is None:
            if tokens > 0:
                raise EngineFault(f"request {request_id} readmitted without swapped KV")
            return
        n_total = sum(h.shape[2] for _, h in host_chunks)
        if len(block_ids) < n_total:
            raise EngineFault("readmission allocated fewer blocks than were swapped out")
        self._swap_init()
        t_host = time.perf_counter()
        comp = torch.cuda.current_stream(self.device)
        at = 0
        sec = self.swap_section_s
        for flat, host in host_chunks:
            n = host.shape[2]
            t = time.perf_counter()
            slot = self._acquire_slot()
            sec["acquire_slot"] += time.perf_counter() - t
            stage = self._stage[slot]
            keep = self._slot_keep[slot]
            t = time.perf_counter()
            ids = self._ids_on_device(block_ids[at:at + n], keep)
            sec["ids"] += time.perf_counter() - t
            t = time.perf_counter()
            with torch.cuda.stream(self._copy_stream):  # same stream as the swap-out D2H: ordered after it
                stage[:, :, :n].copy_(host, non_blocking=host.is_pinned())
                loaded = torch.cuda.Event()
                loaded.record(self._copy_stream)
            self._host_free.append((flat, loaded))  # reusable once its H2D copy is done
            comp.wait_event(loaded)
            K.kv_swap_in_planes(self._stage_planes[slot], ids, self._kv_planes, n)
            scattered = torch.cuda.Event()
            scattered.record(comp)
            self._slot_free[slot] = scattered
            sec["enqueue"] += time.perf_counter() - t
            self.swap_bytes += host.numel() * 2
            at += n
        self.swap_host_s += time.perf_counter() - t_host
