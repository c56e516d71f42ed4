"""The pipelined wall-clock engine (host plans step k+1 while the device runs step k; engine.py
_step_pipelined) against an asynchronous fake executor: every request completes with exactly its
output length, prompts are chunked exactly, emissions are stamped at their step's completion time
in order, and every decode input that was still "on the device" is fed from the previous step's
output (the ag_model_submit feed contract)."""
import time

import numpy as np

from paper_2503_13737_b200 import configs, workload as wl
from paper_2503_13737_b200.engine import Engine, StepResult
from paper_2503_13737_b200.policies import PolicyConfig


class FakeAsyncExecutor:
    """submit()/wait() with at most two steps in flight; next token = f(request, position)."""
    vocab, max_tokens, max_seqs = 50272, 1 << 20, 1 << 20

    def __init__(self, step_s=0.0005):
        self.inflight, self.step_s = [], step_s
        self.prev_out = None
        self.inputs = {}   # (rid, position) -> token id the forward consumed
        self.outputs = {}  # (rid, position) -> token id emitted after consuming that position

    def submit(self, batch, feed=None):
        assert len(self.inflight) < 2
        ids = batch.token_ids.copy()
        if feed is not None:
            assert self.prev_out is not None
            for dst, src in feed:
                ids[dst] = self.prev_out[src]
        rids = np.repeat(np.asarray(batch.request_ids), np.diff(batch.cu_q))
        for r, p, t in zip(rids, batch.positions, ids):
            self.inputs[(int(r), int(p))] = int(t)
        out = np.asarray([(7919 * rid + 104729 * int(batch.positions[row])) % 50000 + 4
                          for rid, row in zip(batch.logit_request_ids, batch.logit_rows)], np.int32)
        for rid, row, t in zip(batch.logit_request_ids, batch.logit_rows, out):
            self.outputs[(int(rid), int(batch.positions[row]))] = int(t)
        self.prev_out = out
        self.inflight.append((out, time.perf_counter() + self.step_s))

    def wait(self):
        out, end = self.inflight.pop(0)
        while time.perf_counter() < end:
            pass
        return StepResult(token_ids=out, elapsed_s=self.step_s, device_s=self.step_s, end_s=end)

    def swap_out(self, *a):
        pass

    def swap_in(self, *a):
        pass


def test_pipelined_engine_completes_and_feeds_decodes():
    c = configs.config1()
    trace = wl.generate_trace(wl.TraceConfig(**{**c.trace.__dict__, "num_requests": 40, "arrival_rate": 200.0}))
    ex = FakeAsyncExecutor()
    eng = Engine(trace, c.trace.profile, PolicyConfig(), ex, clock="wall", pipeline=True, check_invariants=True)
    rep = eng.run()
    assert rep.completed == len(trace)
    assert not ex.inflight
    fed = 0
    for rid, rec in eng.metrics.requests.items():
        assert sum(rec.chunks) == rec.spec.prompt_len
        assert rec.generated == rec.spec.output_len == len(rec.emit_times) == len(rec.tokens_out)
        assert rec.emit_times == sorted(rec.emit_times)
        # decode input at position p = the token emitted after consuming position p-1
        for p in range(rec.spec.prompt_len, rec.spec.prompt_len + rec.spec.output_len - 1):
            assert ex.inputs[(rid, p)] == ex.outputs[(rid, p - 1)]
            fed += 1
        assert rec.tokens_out == [ex.outputs[(rid, p)] for p in
                                  range(rec.spec.prompt_len - 1, rec.spec.prompt_len + rec.spec.output_len - 1)]
    assert fed > 100
    its = eng.metrics.iterations
    assert all(b.start >= a.start for a, b in zip(its, its[1:]))


def test_pipelined_engine_with_kv_pressure():
    """Small pool: preemption / readmission interleave with in-flight steps."""
    from paper_2503_13737_b200 import cost_model as cm
    c = configs.config1()
    prof = cm.ModelProfile(hidden_size=256, num_layers=2, pivot_forward_size=256, pivot_time_s=0.002,
                           fixed_overhead_s=0.002, kvc_capacity_tokens=48 * 32)
    trace = wl.generate_trace(wl.TraceConfig(**{**c.trace.__dict__, "num_requests": 30, "profile": prof,
                                                "long_fraction": 0.0, "arrival_rate": 100.0,
                                                "output_len_dist": wl.LengthDist("uniform", 100, 300)}))
    ex = FakeAsyncExecutor(step_s=0.0002)
    eng = Engine(trace, prof, PolicyConfig(), ex, clock="wall", pipeline=True, kv_blocks=48, check_invariants=True)
    rep = eng.run()
    assert rep.completed == len(trace) and rep.preemptions > 0
    for rid, rec in eng.metrics.requests.items():
        for p in range(rec.spec.prompt_len, rec.spec.prompt_len + rec.spec.output_len - 1):
            assert ex.inputs[(rid, p)] == ex.outputs[(rid, p - 1)]
