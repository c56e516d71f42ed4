"""Iteration loop with the GPU forward behind an Executor.

step(): admit arrivals -> order_queue -> policy plan -> swap-out / KV allocation ->
``executor.execute(batch)`` -> advance the clock -> emit tokens -> release / re-enqueue.

The only departure from the reference engine is the clock advance.  SPEC.md:484 advances the
clock by ``iteration_time(S_f)``; here the clock source is selectable:

  clock="virtual"  iteration_time(S_f) from the cost model (bit-exact scheduler parity with the
                   CPU oracle run; the device still executes every plan) -- or, with a profile
                   carrying the B200 extension, batch_time(S_f, K/V rows read, attention pairs),
  clock="device"   CUDA-event time of the forward measured by the executor,
  clock="wall"     host wall time of executor.execute (packing + H2D + forward + D2H).

Pinned decisions: a prompt's final chunk emits the first output token (so a
request takes N_chunks + output_len - 1 iterations and output_len emissions, SPEC.md:429-437
and the token-conservation invariant :510); TTFT is taken at the end of that iteration
(:518); an empty plan advances the clock to min(next arrival, now + T_max) (:519).
"""
from __future__ import annotations

import math
import time
from dataclasses import asdict, dataclass, field
from typing import Protocol

import numpy as np

from .cost_model import ModelProfile, batch_time, iteration_time
from .errors import AllocationError, EngineFault, StateError
from .kvc import BlockPool
from .policies import BatchPlan, PlanContext, PolicyConfig, has_prompt_left, plan as make_plan
from .sched_core import (ChunkStats, Phase, QueueEntry, jct_allowance, jct_initial_estimate, order_queue,
                         propagate_debt)
from .workload import RequestSpec, SLOKind

CSV_COLUMNS = ("policy", "tokens_per_s", "reqs_per_s", "goodput", "slo_attainment", "jct_slo_attainment",
               "jct_mean", "jct_p5", "jct_p95", "gpu_util_mean", "kvc_util_mean", "preemptions", "truncated")


# ----------------------------------------------------------------------------- device batch
def synthetic_tokens(request_id, positions: np.ndarray, vocab: int) -> np.ndarray:
    """Deterministic token ids in [4, vocab) keyed by (request, position) (splitmix64);
    request_id may be a scalar or an array aligned with positions."""
    rid = np.asarray(request_id).astype(np.uint64)
    x = (rid << np.uint64(32)) ^ positions.astype(np.uint64)
    with np.errstate(over="ignore"):
        x = x + np.uint64(0x9E3779B97F4A7C15)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        x = x ^ (x >> np.uint64(31))
    return (np.uint64(4) + x % np.uint64(vocab - 4)).astype(np.int32)


@dataclass
class DeviceBatch:
    """Packed BatchPlan for one forward (the C-ABI ag_step)."""
    request_ids: list[int]
    token_ids: np.ndarray     # int32 [S_f]
    positions: np.ndarray     # int32 [S_f]
    cu_q: np.ndarray          # int32 [B+1]
    ctx_len: np.ndarray       # int32 [B]
    block_table: np.ndarray   # int32 [B, stride]
    slot_mapping: np.ndarray  # int32 [S_f]
    logit_rows: np.ndarray    # int32 [n_logit]
    logit_request_ids: list[int]

    @property
    def num_tokens(self) -> int:
        return int(self.token_ids.shape[0])

    def h2d_bytes(self) -> int:
        return sum(a.nbytes for a in (self.token_ids, self.positions, self.cu_q, self.ctx_len, self.block_table,
                                      self.slot_mapping, self.logit_rows))

    def seq_shapes(self) -> list[tuple[int, int]]:
        """(q_i, p_i) per sequence for roofline accounting."""
        q = np.diff(self.cu_q)
        return [(int(a), int(b)) for a, b in zip(q, self.ctx_len)]


@dataclass
class StepResult:
    token_ids: np.ndarray  # int32 [n_logit] greedy next tokens
    elapsed_s: float       # time charged to the clock by clock="device"
    device_s: float = 0.0
    wall_s: float = 0.0
    logits: object = None  # optional fp32 [n_logit, V] (parity mode)
    end_s: float | None = None  # host perf_counter time the forward completed at (asynchronous steps)


class Executor(Protocol):
    max_tokens: int
    max_seqs: int
    vocab: int

    def execute(self, batch: DeviceBatch) -> StepResult: ...

    def swap_out(self, request_id: int, block_ids: list[int], tokens: int) -> None: ...

    def swap_in(self, request_id: int, block_ids: list[int], tokens: int) -> None: ...


class VirtualExecutor:
    """No device: the reference simulator's behaviour (clock from the cost model only)."""

    def __init__(self, vocab: int = 50272, max_tokens: int = 1 << 30, max_seqs: int = 1 << 30):
        self.vocab, self.max_tokens, self.max_seqs = vocab, max_tokens, max_seqs

    def execute(self, batch: DeviceBatch) -> StepResult:
        return StepResult(token_ids=np.zeros(len(batch.logit_rows), np.int32), elapsed_s=0.0)

    def swap_out(self, request_id, block_ids, tokens):
        pass

    def swap_in(self, request_id, block_ids, tokens):
        pass


# ----------------------------------------------------------------------------- metrics
@dataclass
class RequestRecord:
    spec: RequestSpec
    prompt_done: int = 0
    generated: int = 0
    first_token_time: float | None = None
    emit_times: list[float] = field(default_factory=list)
    completion_time: float | None = None
    preempt_time: float | None = None
    tokens_out: list[int] = field(default_factory=list)
    chunks: list[int] = field(default_factory=list)

    def events_met(self) -> tuple[int, int]:
        """(met, total) iteration-level token events (TTFT + each TBT gap) of an online request."""
        slo = self.spec.slo
        if slo.kind is SLOKind.OFFLINE or not self.emit_times:
            return 0, 0
        met = int(self.emit_times[0] - self.spec.arrival_time <= slo.ttft_slo + 1e-12)
        for a, b in zip(self.emit_times, self.emit_times[1:]):
            met += int(b - a <= slo.tbt_slo + 1e-12)
        return met, len(self.emit_times)

    def good(self) -> bool:
        if self.completion_time is None:
            return False
        slo = self.spec.slo
        if slo.kind is SLOKind.OFFLINE:
            return self.completion_time - self.spec.arrival_time <= slo.jct_slo + 1e-12
        met, total = self.events_met()
        return met == total


@dataclass
class IterationRecord:
    index: int
    start: float
    elapsed: float
    forward_size: int
    token_budget: int
    num_seqs: int
    num_decode: int
    allocated_tokens: int
    preemptions: int
    device_s: float = 0.0
    wall_s: float = 0.0
    events: int = 0
    events_met: int = 0
    slo_tokens: int = 0   # tokens of this forward already known to meet their deadline (decodes, final chunks)
    # non-final prompt chunks (request id, tokens): they meet the SLO iff the request's first token (the
    # final chunk) meets TTFT, known only later -- resolve with Engine.prefill_met()
    pending_prefill: list = field(default_factory=list)
    host_pre_s: float = 0.0   # admit + order + plan + allocate + pack (before executor.execute)
    host_post_s: float = 0.0  # emission + re-enqueue (after executor.execute)


@dataclass
class MetricsReport:
    policy: str
    tokens_per_s: float
    reqs_per_s: float
    goodput: float
    slo_attainment: float
    jct_slo_attainment: float
    jct_mean: float
    jct_p5: float
    jct_p95: float
    gpu_util_mean: float
    kvc_util_mean: float
    preemptions: int
    truncated: bool
    goodput_windowed: float = 0.0
    slo_tokens_per_s: float = 0.0
    makespan: float = 0.0
    iterations: int = 0
    completed: int = 0

    def csv_row(self) -> str:
        vals = [getattr(self, c) for c in CSV_COLUMNS]
        return ",".join(str(v) if not isinstance(v, float) else repr(v) for v in vals)

    def to_dict(self) -> dict:
        return asdict(self)


class MetricsAccumulator:
    def __init__(self):
        self.requests: dict[int, RequestRecord] = {}
        self.iterations: list[IterationRecord] = []
        self.total_blocks_tokens = 1


def compute_metrics(acc: MetricsAccumulator, policy: str, truncated: bool, window_s: float = 1.0) -> MetricsReport:
    """SPEC.md:499-507 metric definitions over a finished (or truncated) run."""
    recs = list(acc.requests.values())
    done = [r for r in recs if r.completion_time is not None]
    if not recs or not acc.iterations:
        return MetricsReport(policy, 0.0, 0.0, 0.0, 1.0, 1.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0, truncated)
    t0 = min(r.spec.arrival_time for r in recs)
    t_end = max([r.completion_time for r in done] + [acc.iterations[-1].start + acc.iterations[-1].elapsed])
    makespan = max(t_end - t0, 1e-12)
    tokens = sum(r.prompt_done + r.generated for r in recs)
    met = tot = 0
    for r in recs:
        m, t = r.events_met()
        met += m
        tot += t
    good = [r for r in done if r.good()]
    offline = [r for r in done if r.spec.slo.kind is SLOKind.OFFLINE]
    jcts = np.array([r.completion_time - r.spec.arrival_time for r in done]) if done else np.zeros(1)
    n_win = max(1, math.ceil(makespan / window_s))
    per_win = np.zeros(n_win)
    for r in good:
        per_win[min(n_win - 1, int((r.completion_time - t0) / window_s))] += 1
    busy = [it for it in acc.iterations if it.forward_size > 0]
    return MetricsReport(
        policy=policy,
        tokens_per_s=tokens / makespan,
        reqs_per_s=len(done) / makespan,
        goodput=len(good) / makespan,
        slo_attainment=met / tot if tot else 1.0,
        jct_slo_attainment=(sum(r.good() for r in offline) / len(offline)) if offline else 1.0,
        jct_mean=float(jcts.mean()),
        jct_p5=float(np.percentile(jcts, 5)),
        jct_p95=float(np.percentile(jcts, 95)),
        gpu_util_mean=float(np.mean([it.forward_size / it.token_budget for it in busy])) if busy else 0.0,
        kvc_util_mean=float(np.mean([it.allocated_tokens / acc.total_blocks_tokens for it in busy])) if busy else 0.0,
        preemptions=sum(it.preemptions for it in acc.iterations),
        truncated=truncated,
        goodput_windowed=float(per_win.mean() / window_s),
        slo_tokens_per_s=sum(r.spec.prompt_len + r.spec.output_len for r in good) / makespan,
        makespan=makespan,
        iterations=len(acc.iterations),
        completed=len(done),
    )


# ----------------------------------------------------------------------------- engine
class Engine:
    """Deterministic single-threaded loop; the BlockPool is single-writer."""

    def __init__(self, trace: list[RequestSpec], profile: ModelProfile, policy: PolicyConfig | None = None,
                 executor: Executor | None = None, *, clock: str = "virtual", kv_blocks: int | None = None,
                 block_size: int = 32, horizon_s: float = math.inf, per_token_swap_cost_s: float = 0.0,
                 check_invariants: bool = False, autoregressive: bool = True, pipeline: bool = False):
        if clock not in ("virtual", "device", "wall"):
            raise ValueError(f"unknown clock {clock!r}")
        if pipeline and (clock != "wall" or not hasattr(executor, "submit")):
            raise ValueError("pipeline=True needs clock='wall' and an executor with submit()/wait()")
        self.trace = sorted(trace, key=lambda r: (r.arrival_time, r.id))
        self.profile = profile
        self.cfg = policy or PolicyConfig()
        self.executor = executor or VirtualExecutor()
        self.clock_mode = clock
        blocks = kv_blocks if kv_blocks is not None else profile.kvc_capacity_tokens // block_size
        self.pool = BlockPool(max(1, blocks), block_size)
        self.stats = ChunkStats(avg_chunk_len=float(profile.pivot_forward_size),
                                t_max=iteration_time(profile.pivot_forward_size, profile))
        self.clock = 0.0
        self.horizon = horizon_s
        self.swap_cost = per_token_swap_cost_s
        self.check = check_invariants
        # decode inputs: the token the executor emitted last for the request (real autoregressive
        # generation); prompt tokens -- and decodes of an executor that emits none -- are synthetic
        self.autoregressive = autoregressive
        self.queue: list[QueueEntry] = []
        self.long_active: set[int] = set()
        self.metrics = MetricsAccumulator()
        self.metrics.total_blocks_tokens = self.pool.total_blocks * block_size
        self._next_arrival = 0
        self._stamp = 0
        self.plans: list[BatchPlan] = []      # kept for parity tests (scheduler decisions)
        self.tables: list[dict] = []          # per-step block tables (physical ids)
        self.keep_history = False
        # pipelined wall clock: step k+1 is planned and submitted while the device runs step k
        self.pipeline = pipeline
        self.plan_host_s = 0.0              # host time in order_queue + make_plan (pipelined steps)
        self._inflight: dict | None = None
        self._origin: float | None = None   # perf_counter time of engine time 0 (minus idle jumps)
        self._offset = 0.0                  # idle jumps (empty queue: the clock skips to the next arrival)
        self._sched_emitted: dict[int, int] = {}
        self._pending_tok: dict[int, tuple[int, int]] = {}  # rid -> (step id, logit row) of a token in flight
        self._last_end = 0.0
        self._n_submitted = 0

    # -------------------------------------------------------------- helpers
    def _stamp_next(self) -> int:
        self._stamp += 1
        return self._stamp

    def _admit(self) -> None:
        while self._next_arrival < len(self.trace) and self.trace[self._next_arrival].arrival_time <= self.clock:
            spec = self.trace[self._next_arrival]
            self._next_arrival += 1
            e = QueueEntry(request=spec, phase=Phase.PROMPT_PENDING, remaining_prompt_tokens=spec.prompt_len,
                           seq_len=0, enqueue_time=spec.arrival_time, is_long=spec.is_long(), seq=self._stamp_next())
            if e.is_offline:
                e.iter_allowance = jct_allowance(spec, jct_initial_estimate(spec, self.stats), self.stats)
            self.queue.append(e)
            self.metrics.requests[spec.id] = RequestRecord(spec)

    def done(self) -> bool:
        return self._next_arrival >= len(self.trace) and not self.queue and self._inflight is None

    def prefill_met(self, request_id: int) -> bool | None:
        """Whether request_id's prompt tokens meet their SLO: TTFT of the first token (online) or the
        JCT deadline (offline, judged at the first token's time); None while the prompt is unfinished."""
        rec = self.metrics.requests[request_id]
        if rec.first_token_time is None:
            return None
        slo = rec.spec.slo
        limit = slo.jct_slo if slo.kind is SLOKind.OFFLINE else slo.ttft_slo
        return rec.first_token_time - rec.spec.arrival_time <= limit + 1e-12

    # -------------------------------------------------------------- one iteration
    def step(self) -> IterationRecord | None:
        if self.pipeline:
            return self._step_pipelined()
        t_step0 = time.perf_counter()
        self._admit()
        if not self.queue:
            if self._next_arrival < len(self.trace):
                self.clock = max(self.clock, self.trace[self._next_arrival].arrival_time)
            return None
        self.queue = order_queue(self.queue, self.clock, self.stats)
        ctx = PlanContext(self.pool, self.stats, self.profile, self.clock, set(self.long_active))
        plan = make_plan(self.queue, ctx, self.cfg)
        plan.check()
        if plan.forward_size > self.executor.max_tokens or len(plan.selections) > self.executor.max_seqs:
            raise EngineFault(f"plan of {plan.forward_size} tokens / {len(plan.selections)} sequences exceeds the "
                              f"executor capacity ({self.executor.max_tokens}/{self.executor.max_seqs})")
        start = self.clock
        by_id = {e.request_id: e for e in self.queue}

        # ---- preemptions (swap out) before allocation
        swap_tokens = 0
        for rid in plan.preempted:
            e = by_id[rid]
            tokens, table = self.pool.preempt_with_table(rid)
            self.executor.swap_out(rid, table, tokens)
            swap_tokens += tokens
            self.stats.observe_preemption()
            rec = self.metrics.requests[rid]
            rec.preempt_time = start
            e.phase = Phase.PREEMPTED
            e.enqueue_time = start
            e.seq = self._stamp_next()

        if not plan.selections:
            # empty plan: jump to min(next arrival, now + T_max), plus the swap time of a
            # plan that only preempts (PagedFcfs with the pool exhausted) -- whose swap-outs are real
            # work, so they are recorded as an iteration of forward size 0
            cost = swap_tokens * self.swap_cost
            if plan.preempted:
                self.metrics.iterations.append(IterationRecord(
                    index=len(self.metrics.iterations), start=start, elapsed=cost, forward_size=0,
                    token_budget=plan.token_budget, num_seqs=0, num_decode=0,
                    allocated_tokens=self.pool.allocated_tokens, preemptions=len(plan.preempted),
                    host_pre_s=time.perf_counter() - t_step0))
            nxt = self.trace[self._next_arrival].arrival_time if self._next_arrival < len(self.trace) else math.inf
            self.clock = min(nxt, self.clock + self.stats.t_max) + cost
            return None

        # ---- allocation + batch packing (vectorised: one numpy pass over all tokens)
        free_before = self.pool.free_blocks
        n_sel = len(plan.selections)
        chunk = np.empty(n_sel, np.int64)
        before_arr = np.empty(n_sel, np.int64)
        fed: list[tuple[int, int]] = []  # (selection index, token id) of decodes fed their last output
        tables: list[list[int]] = []
        for i, sel in enumerate(plan.selections):
            e = by_id[sel.request_id]
            rid = sel.request_id
            try:
                if rid in self.pool.swapped_out:
                    saved = self.pool.swapped_out[rid]
                    self.pool.allocate(rid, self.pool.demand_readmit(rid))
                    self.executor.swap_in(rid, self.pool.block_table(rid), saved)
                    swap_tokens += saved
                    rec = self.metrics.requests[rid]
                    if rec.preempt_time is not None:
                        self.stats.observe_preemption_duration(start - rec.preempt_time)
                before = self.pool.tokens_stored(rid)
                prompt_left = has_prompt_left(e)
                demand = (self.pool.demand_prompt_chunk(rid, sel.chunk_len) if prompt_left
                          else self.pool.demand_tg(rid))
                self.pool.allocate(rid, demand)
            except (AllocationError, StateError) as exc:
                raise EngineFault(f"plan infeasible against the pool: {exc}") from exc
            chunk[i] = sel.chunk_len
            before_arr[i] = before
            if self.autoregressive and not prompt_left:
                out = self.metrics.requests[rid].tokens_out
                if out and out[-1] >= 0:
                    fed.append((i, out[-1]))
            tables.append(self.pool.block_table(rid))
        if free_before - self.pool.free_blocks != plan.blocks_needed:
            raise EngineFault(f"allocated {free_before - self.pool.free_blocks} blocks, plan expected "
                              f"{plan.blocks_needed}")
        cu = np.zeros(n_sel + 1, np.int64)
        np.cumsum(chunk, out=cu[1:])
        S = int(cu[-1])
        seq_of_tok = np.repeat(np.arange(n_sel), chunk)
        positions = (np.arange(S) - cu[seq_of_tok] + before_arr[seq_of_tok]).astype(np.int32)
        rids_arr = np.asarray([s.request_id for s in plan.selections], np.int64)
        token_ids = synthetic_tokens(rids_arr[seq_of_tok], positions, self.executor.vocab)
        for i, tok in fed:
            token_ids[cu[i]] = tok
        stride = max(len(t) for t in tables)
        bt = np.zeros((n_sel, stride), dtype=np.int32)
        for i, t in enumerate(tables):
            bt[i, :len(t)] = t
        bs = self.pool.block_size
        slots = (bt[seq_of_tok, positions // bs] * bs + positions % bs).astype(np.int32)
        final = np.fromiter((s.is_final_chunk for s in plan.selections), bool, n_sel)
        logit_rows = (cu[1:][final] - 1).astype(np.int32)
        logit_ids = [int(r) for r in rids_arr[final]]
        batch = DeviceBatch(request_ids=[s.request_id for s in plan.selections], token_ids=token_ids,
                            positions=positions, cu_q=cu.astype(np.int32), ctx_len=before_arr.astype(np.int32),
                            block_table=bt, slot_mapping=slots, logit_rows=logit_rows, logit_request_ids=logit_ids)
        if self.check:
            self.pool.check_conservation()
        if self.keep_history:
            self.plans.append(plan)
            self.tables.append({rid: list(row[:len(t)]) for rid, row, t in zip(batch.request_ids, bt, tables)})

        # ---- execute and advance the clock
        t_host = time.perf_counter()
        pre_s = t_host - t_step0
        res = self.executor.execute(batch)
        wall = time.perf_counter() - t_host
        if self.clock_mode == "virtual":
            q_arr = chunk
            kv_tok = int(before_arr.sum() + q_arr.sum())
            pairs = int((q_arr * before_arr).sum() + (q_arr * (q_arr + 1) // 2).sum())
            elapsed = batch_time(plan.forward_size, kv_tok, pairs, self.profile)
        elif self.clock_mode == "device":
            elapsed = res.elapsed_s
        else:
            elapsed = time.perf_counter() - t_step0  # scheduling + packing + H2D + forward + D2H
        elapsed += swap_tokens * self.swap_cost
        self.clock = start + elapsed
        now = self.clock

        # ---- emission, statistics, re-enqueue
        it = IterationRecord(index=len(self.metrics.iterations), start=start, elapsed=elapsed,
                             forward_size=plan.forward_size, token_budget=plan.token_budget,
                             num_seqs=len(plan.selections), num_decode=0,
                             allocated_tokens=self.pool.allocated_tokens, preemptions=len(plan.preempted),
                             device_s=res.device_s, wall_s=wall, host_pre_s=pre_s)
        t_post = time.perf_counter()
        tok_by_id = dict(zip(logit_ids, res.token_ids.tolist()))
        selected = set()
        finished = []
        for sel in plan.selections:
            e = by_id[sel.request_id]
            rid = sel.request_id
            selected.add(rid)
            rec = self.metrics.requests[rid]
            spec = rec.spec
            if e.is_offline:
                propagate_debt(e, start - e.enqueue_time)
            prompt = has_prompt_left(e)
            if prompt:
                self.stats.observe_chunk(sel.chunk_len)
                rec.prompt_done += sel.chunk_len
                rec.chunks.append(sel.chunk_len)
                e.remaining_prompt_tokens -= sel.chunk_len
                e.seq_len += sel.chunk_len
                if e.is_long:
                    self.long_active.add(rid)
            else:
                self.stats.observe_tg_step()
                it.num_decode += 1
                e.seq_len += 1
            if not sel.is_final_chunk:
                # non-final chunk: same TTFT clock, back in the queue; its tokens count as SLO-meeting only
                # if the final chunk later meets TTFT (offline requests: JCT, resolved the same way)
                it.pending_prefill.append((rid, sel.chunk_len))
                e.phase = Phase.PROMPT_PENDING
                e.seq = self._stamp_next()
                continue
            if prompt and e.is_long:
                self.long_active.discard(rid)
            # token event
            prev = rec.emit_times[-1] if rec.emit_times else None
            rec.emit_times.append(now)
            rec.generated += 1
            rec.tokens_out.append(tok_by_id.get(rid, -1))
            if rec.first_token_time is None:
                rec.first_token_time = now
            if spec.slo.kind is SLOKind.ONLINE:
                it.events += 1
                ok = (now - spec.arrival_time <= spec.slo.ttft_slo + 1e-12) if prev is None else (
                    now - prev <= spec.slo.tbt_slo + 1e-12)
                it.events_met += int(ok)
                it.slo_tokens += sel.chunk_len if ok else 0
            else:
                it.slo_tokens += sel.chunk_len if now - spec.arrival_time <= spec.slo.jct_slo else 0
            if rec.generated >= spec.output_len:
                rec.completion_time = now
                self.pool.release(rid)
                finished.append(rid)
            else:
                e.phase = Phase.TG_READY
                e.remaining_prompt_tokens = 0
                e.enqueue_time = now
                e.seq = self._stamp_next()
        if finished:
            gone = set(finished)
            self.queue = [e for e in self.queue if e.request_id not in gone]
        it.host_post_s = time.perf_counter() - t_post
        self.metrics.iterations.append(it)
        return it

    # -------------------------------------------------------------- pipelined iteration (wall clock)
    def _now(self) -> float:
        return time.perf_counter() - self._origin + self._offset

    def flush(self) -> IterationRecord | None:
        """Complete the step still on the device (pipelined mode)."""
        if self._inflight is None:
            return None
        prev, self._inflight = self._inflight, None
        return self._complete(prev)

    def _step_pipelined(self) -> IterationRecord | None:
        """One iteration with the host one step ahead of the device (wall clock).

        Plan -> allocate -> pack -> ``executor.submit`` (returns at once) -> apply the step's state
        transitions optimistically (chunk progress, TG re-enqueue, KV release of finishing requests:
        none of them depends on the token values, the trace fixes output lengths) ->
        ``executor.wait`` for the PREVIOUS step, whose emissions are stamped with its device completion
        time.  Decode inputs whose token is still on the device are fed there (ag_model_submit feed
        pairs).  Scheduling decisions see the clock at planning time, one forward earlier than a
        synchronous engine would (as any asynchronous serving scheduler)."""
        t0 = time.perf_counter()
        if self._origin is None:
            self._origin = t0 - self.clock
        self.clock = max(self.clock, self._now())
        self._admit()
        if not self.queue:
            if self._inflight is not None:
                return self.flush()
            if self._next_arrival < len(self.trace):
                nxt = self.trace[self._next_arrival].arrival_time
                if nxt > self.clock:
                    self._offset += nxt - self.clock
                    self.clock = nxt
            return None
        t_plan = time.perf_counter()
        self.queue = order_queue(self.queue, self.clock, self.stats)
        ctx = PlanContext(self.pool, self.stats, self.profile, self.clock, set(self.long_active))
        plan = make_plan(self.queue, ctx, self.cfg)
        plan.check()
        self.plan_host_s += time.perf_counter() - t_plan
        if plan.forward_size > self.executor.max_tokens or len(plan.selections) > self.executor.max_seqs:
            raise EngineFault(f"plan of {plan.forward_size} tokens / {len(plan.selections)} sequences exceeds the "
                              f"executor capacity ({self.executor.max_tokens}/{self.executor.max_seqs})")
        start = self.clock
        by_id = {e.request_id: e for e in self.queue}
        for rid in plan.preempted:
            e = by_id[rid]
            tokens, table = self.pool.preempt_with_table(rid)
            self.executor.swap_out(rid, table, tokens)
            self.stats.observe_preemption()
            self.metrics.requests[rid].preempt_time = start
            e.phase = Phase.PREEMPTED
            e.enqueue_time = start
            e.seq = self._stamp_next()
        if not plan.selections:
            if plan.preempted:
                self.metrics.iterations.append(IterationRecord(
                    index=len(self.metrics.iterations), start=start, elapsed=0.0, forward_size=0,
                    token_budget=plan.token_budget, num_seqs=0, num_decode=0,
                    allocated_tokens=self.pool.allocated_tokens, preemptions=len(plan.preempted),
                    host_pre_s=time.perf_counter() - t0))
            if self._inflight is not None:
                return self.flush()  # its completion may release KV / return work
            nxt = self.trace[self._next_arrival].arrival_time if self._next_arrival < len(self.trace) else math.inf
            jump = min(nxt, self.clock + self.stats.t_max) - self.clock
            self._offset += max(0.0, jump)
            self.clock += max(0.0, jump)
            return None

        # ---- allocation + packing
        free_before = self.pool.free_blocks
        n_sel = len(plan.selections)
        chunk = np.empty(n_sel, np.int64)
        before_arr = np.empty(n_sel, np.int64)
        known: list[tuple[int, int]] = []   # (selection index, token id) decode inputs known on the host
        feed: list[tuple[int, int]] = []    # (selection index, logit row of the step in flight)
        tables: list[list[int]] = []
        inflight_id = self._inflight["id"] if self._inflight is not None else -1
        for i, sel in enumerate(plan.selections):
            e = by_id[sel.request_id]
            rid = sel.request_id
            try:
                if rid in self.pool.swapped_out:
                    saved = self.pool.swapped_out[rid]
                    self.pool.allocate(rid, self.pool.demand_readmit(rid))
                    self.executor.swap_in(rid, self.pool.block_table(rid), saved)
                    rec = self.metrics.requests[rid]
                    if rec.preempt_time is not None:
                        self.stats.observe_preemption_duration(start - rec.preempt_time)
                before = self.pool.tokens_stored(rid)
                prompt_left = has_prompt_left(e)
                demand = (self.pool.demand_prompt_chunk(rid, sel.chunk_len) if prompt_left
                          else self.pool.demand_tg(rid))
                self.pool.allocate(rid, demand)
            except (AllocationError, StateError) as exc:
                raise EngineFault(f"plan infeasible against the pool: {exc}") from exc
            chunk[i] = sel.chunk_len
            before_arr[i] = before
            if self.autoregressive and not prompt_left:
                pend = self._pending_tok.get(rid)
                if pend is not None and pend[0] == inflight_id:
                    feed.append((i, pend[1]))
                else:
                    out = self.metrics.requests[rid].tokens_out
                    if out and out[-1] >= 0:
                        known.append((i, out[-1]))
            tables.append(self.pool.block_table(rid))
        if free_before - self.pool.free_blocks != plan.blocks_needed:
            raise EngineFault(f"allocated {free_before - self.pool.free_blocks} blocks, plan expected "
                              f"{plan.blocks_needed}")
        cu = np.zeros(n_sel + 1, np.int64)
        np.cumsum(chunk, out=cu[1:])
        S = int(cu[-1])
        seq_of_tok = np.repeat(np.arange(n_sel), chunk)
        positions = (np.arange(S) - cu[seq_of_tok] + before_arr[seq_of_tok]).astype(np.int32)
        rids_arr = np.asarray([s.request_id for s in plan.selections], np.int64)
        token_ids = synthetic_tokens(rids_arr[seq_of_tok], positions, self.executor.vocab)
        for i, tok in known:
            token_ids[cu[i]] = tok
        stride = max(len(t) for t in tables)
        bt = np.zeros((n_sel, stride), dtype=np.int32)
        for i, t in enumerate(tables):
            bt[i, :len(t)] = t
        bs = self.pool.block_size
        slots = (bt[seq_of_tok, positions // bs] * bs + positions % bs).astype(np.int32)
        final = np.fromiter((s.is_final_chunk for s in plan.selections), bool, n_sel)
        logit_rows = (cu[1:][final] - 1).astype(np.int32)
        logit_ids = [int(r) for r in rids_arr[final]]
        batch = DeviceBatch(request_ids=[s.request_id for s in plan.selections], token_ids=token_ids,
                            positions=positions, cu_q=cu.astype(np.int32), ctx_len=before_arr.astype(np.int32),
                            block_table=bt, slot_mapping=slots, logit_rows=logit_rows, logit_request_ids=logit_ids)
        if self.check:
            self.pool.check_conservation()
        if self.keep_history:
            self.plans.append(plan)
            self.tables.append({rid: list(row[:len(t)]) for rid, row, t in zip(batch.request_ids, bt, tables)})
        fp = np.asarray([(int(cu[i]), r) for i, r in feed], np.int32).reshape(-1, 2) if feed else None
        t_sub = time.perf_counter()
        self.executor.submit(batch, fp)
        sid = self._n_submitted
        self._n_submitted += 1

        # ---- optimistic state transitions (no token values needed)
        step = {"id": sid, "start": start, "plan": plan, "logit_ids": logit_ids, "emit": [], "requeue": {},
                "pending_prefill": [], "num_decode": 0, "host_pre_s": t_sub - t0,
                "allocated_tokens": self.pool.allocated_tokens}
        finished = []
        row_of = {rid: j for j, rid in enumerate(logit_ids)}
        for sel in plan.selections:
            e = by_id[sel.request_id]
            rid = sel.request_id
            rec = self.metrics.requests[rid]
            if e.is_offline:
                propagate_debt(e, start - e.enqueue_time)
            prompt = has_prompt_left(e)
            if prompt:
                self.stats.observe_chunk(sel.chunk_len)
                rec.prompt_done += sel.chunk_len
                rec.chunks.append(sel.chunk_len)
                e.remaining_prompt_tokens -= sel.chunk_len
                e.seq_len += sel.chunk_len
                if e.is_long:
                    self.long_active.add(rid)
            else:
                self.stats.observe_tg_step()
                step["num_decode"] += 1
                e.seq_len += 1
            if not sel.is_final_chunk:
                step["pending_prefill"].append((rid, sel.chunk_len))
                e.phase = Phase.PROMPT_PENDING
                e.seq = self._stamp_next()
                continue
            if prompt and e.is_long:
                self.long_active.discard(rid)
            n_emit = self._sched_emitted.get(rid, 0) + 1
            self._sched_emitted[rid] = n_emit
            step["emit"].append((rid, sel.chunk_len, row_of[rid]))
            self._pending_tok[rid] = (sid, row_of[rid])
            if n_emit >= rec.spec.output_len:
                self.pool.release(rid)
                finished.append(rid)
                self._sched_emitted.pop(rid, None)
            else:
                e.phase = Phase.TG_READY
                e.remaining_prompt_tokens = 0
                e.enqueue_time = start  # provisional: set to the step's completion time when it completes
                e.seq = self._stamp_next()
                step["requeue"][rid] = (e, e.seq)
        if finished:
            gone = set(finished)
            self.queue = [e for e in self.queue if e.request_id not in gone]
        prev, self._inflight = self._inflight, step
        return self._complete(prev) if prev is not None else None

    def _complete(self, step: dict) -> IterationRecord:
        """Wait for a submitted step and record its emissions at its device completion time."""
        res = self.executor.wait()
        end = res.end_s - self._origin + self._offset if res.end_s is not None else self._now()
        start = max(step["start"], self._last_end)
        end = max(end, start)
        self._last_end = end
        plan = step["plan"]
        it = IterationRecord(index=len(self.metrics.iterations), start=start, elapsed=end - start,
                             forward_size=plan.forward_size, token_budget=plan.token_budget,
                             num_seqs=len(plan.selections), num_decode=step["num_decode"],
                             allocated_tokens=step["allocated_tokens"], preemptions=len(plan.preempted),
                             device_s=res.device_s, wall_s=res.wall_s, host_pre_s=step["host_pre_s"])
        it.pending_prefill = step["pending_prefill"]
        toks = res.token_ids.tolist()
        for rid, chunk_len, row in step["emit"]:
            rec = self.metrics.requests[rid]
            spec = rec.spec
            prev = rec.emit_times[-1] if rec.emit_times else None
            rec.emit_times.append(end)
            rec.generated += 1
            rec.tokens_out.append(toks[row] if row < len(toks) else -1)
            if rec.first_token_time is None:
                rec.first_token_time = end
            if spec.slo.kind is SLOKind.ONLINE:
                it.events += 1
                ok = (end - spec.arrival_time <= spec.slo.ttft_slo + 1e-12) if prev is None else (
                    end - prev <= spec.slo.tbt_slo + 1e-12)
                it.events_met += int(ok)
                it.slo_tokens += chunk_len if ok else 0
            else:
                it.slo_tokens += chunk_len if end - spec.arrival_time <= spec.slo.jct_slo else 0
            if rec.generated >= spec.output_len:
                rec.completion_time = end
            if self._pending_tok.get(rid, (None,))[0] == step["id"]:
                del self._pending_tok[rid]
            rq = step["requeue"].get(rid)
            if rq is not None and rq[0].seq == rq[1]:
                rq[0].enqueue_time = end  # T_w of a returned TG task starts at its emission
        self.metrics.iterations.append(it)
        return it

    def run(self, max_steps: int | None = None) -> MetricsReport:
        truncated = False
        steps = 0
        while not self.done():
            if self.clock > self.horizon:
                truncated = True
                break
            if max_steps is not None and steps >= max_steps:
                truncated = True
                break
            if self.step() is not None:
                steps += 1
        if self.pipeline:
            self.flush()
        return compute_metrics(self.metrics, self.cfg.policy, truncated)
