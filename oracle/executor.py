"""Oracle executor — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Same interface as paper_2503_13737_b200.executor.CudaExecutor, computing each packed BatchPlan
with the CPU OracleOPT; ``TeeExecutor`` runs a device executor and the oracle on the very same
batch so a parity test compares logits and tokens step by step.
"""
from __future__ import annotations

import time

import numpy as np
import torch

from paper_2503_13737_b200.engine import StepResult
from .forward import OracleOPT, StepInputs


def step_inputs(batch) -> StepInputs:
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.int32))
    return StepInputs(t(batch.token_ids), t(batch.positions), t(batch.cu_q), t(batch.ctx_len), t(batch.block_table),
                      t(batch.slot_mapping), t(batch.logit_rows))


class OracleExecutor:
    def __init__(self, cfg, weights, num_blocks, max_tokens=1 << 20, max_seqs=1 << 20, **kw):
        self.cfg = cfg
        self.vocab = cfg.vocab
        self.max_tokens, self.max_seqs = max_tokens, max_seqs
        self.model = OracleOPT(cfg, weights, num_blocks, **kw)
        self._swapped = {}

    def execute(self, batch) -> StepResult:
        t0 = time.perf_counter()
        logits, toks = self.model.forward(step_inputs(batch))
        dt = time.perf_counter() - t0
        return StepResult(token_ids=toks.numpy(), elapsed_s=dt, device_s=dt, wall_s=dt, logits=logits)

    def swap_out(self, request_id, block_ids, tokens):
        ids = torch.tensor(block_ids, dtype=torch.long, device=self.model.dev)
        self._swapped[request_id] = [(k[ids].clone(), v[ids].clone())
                                     for k, v in zip(self.model.k_pools, self.model.v_pools)]

    def swap_in(self, request_id, block_ids, tokens):
        saved = self._swapped.pop(request_id, None)
        if saved is None:
            return
        n = saved[0][0].shape[0]
        ids = torch.tensor(block_ids[:n], dtype=torch.long, device=self.model.dev)
        for (k, v), kp, vp in zip(saved, self.model.k_pools, self.model.v_pools):
            kp[ids] = k
            vp[ids] = v


class TeeExecutor:
    """Runs `device` (the product) and `oracle` on each batch; records both outputs."""

    def __init__(self, device, oracle):
        self.device, self.oracle = device, oracle
        self.vocab = device.vocab
        self.max_tokens, self.max_seqs = device.max_tokens, device.max_seqs
        self.records = []

    def execute(self, batch):
        a = self.device.execute(batch)
        b = self.oracle.execute(batch)
        self.records.append((batch, a, b))
        return a

    def swap_out(self, request_id, block_ids, tokens):
        self.device.swap_out(request_id, block_ids, tokens)
        self.oracle.swap_out(request_id, block_ids, tokens)

    def swap_in(self, request_id, block_ids, tokens):
        self.device.swap_in(request_id, block_ids, tokens)
        self.oracle.swap_in(request_id, block_ids, tokens)
