"""Batching policies (paper Algorithms 1-2).

The reference ships no ``policies`` module, so this is a restatement of the SPEC with every
ambiguity pinned once (SURVEY §8c'):

* Single waiting queue.  Every unfinished request returns to it after each iteration: a
  returned TG task with T_w = 0 (enqueue_time = now), a partially processed prompt with its
  original enqueue time (its TTFT clock keeps running), a preempted request with the preemption
  time.  ``running`` of the SPEC signature is therefore always empty.
* Token budget S_b = max(1, min(floor(S_pf * slo_min / T_pf), cap)), cap defaults to S_pf
  (SPEC.md:384-392).  slo_min is the smallest ONLINE iteration SLO among the urgent entries and
  the head of the queue; with no online entry S_b = cap.
* Algorithm 1: urgent entries join B in queue order; a TG or preempted TG task takes 1 token, a
  pending prompt takes min(remaining, max(1, S_b - S_f - R)) tokens where R counts the urgent
  TG tasks not yet placed (sequential token selection, PAPER §4.2, with the returned decodes
  "retained in the batch as much as possible", PAPER §4.4).  While S_f > S_b or B's block demand
  exceeds the free blocks, the member with max T_r (ties: later queue position) leaves B; only
  when the KV blocks are the deficit and it holds blocks is it preempted (swapped out, freeing
  them) -- a token-budget deficit merely defers it with its KV resident.  Under a KV deficit the
  default ``kv_victim="resident_last"`` first drops members holding no blocks (new prompts,
  swapped-out requests), so admitting work never evicts a resident request; ``"max_tr"`` is the
  paper-literal rule (evict/readmit churn once the pool is full).
* Algorithm 2 (select_requests): window = non-urgent entries with T_r <= T_r^1 + gamma.  Every
  pending prompt in the window (short or long, PAPER §4.2 "regardless of their associated
  requests") is offered as a chunk min(remaining, A_c, tokens fitting A_m); TG / preempted TG
  tasks are offered with D_c = 1.  D_m is blocks x b (block granularity).  The
  feasible candidate minimising (A_c-D_c)^2 + (A_m-D_m)^2 (exact integers; same order as the
  Euclidean distance) is taken (ties: earlier queue
  position), A_c/A_m shrink, candidates are re-sized, repeat.
* ERA: a long prompt that has not started prefill may not get a chunk while
  ``max_concurrent_long`` long prompts have started and not finished prefill.
"""
from __future__ import annotations

import math
from collections import deque
from dataclasses import dataclass, field
from typing import NamedTuple

from .cost_model import ModelProfile
from .errors import ConfigError
from .kvc import BlockPool, blocks_for
from .sched_core import DEFAULT_URGENCY_SLACK, ChunkStats, Phase, QueueEntry, is_urgent, iteration_slo, remaining_time
from .workload import SLOKind

POLICIES = ("accelgen", "paged_fcfs", "static_chunk", "orca_fcfs")


class Selection(NamedTuple):
    """(request_id, chunk_len, is_final_chunk) of SPEC.md:371; TG steps have chunk_len 1."""
    request_id: int
    chunk_len: int
    is_final_chunk: bool


@dataclass
class BatchPlan:
    selections: list[Selection] = field(default_factory=list)
    forward_size: int = 0
    token_budget: int = 0
    preempted: list[int] = field(default_factory=list)  # held blocks -> swapped out
    slo_min: float = 0.0
    deferred: list[int] = field(default_factory=list)   # urgent but dropped without holding blocks
    blocks_needed: int = 0

    def check(self, pool_free_blocks: int | None = None) -> None:
        from .errors import EngineFault
        if self.forward_size != sum(s.chunk_len for s in self.selections):
            raise EngineFault("BatchPlan: forward_size != sum of chunk lengths")
        if self.forward_size > self.token_budget:
            raise EngineFault("BatchPlan: S_f exceeds S_b")
        if any(s.chunk_len < 1 for s in self.selections):
            raise EngineFault("BatchPlan: empty chunk")
        if len({s.request_id for s in self.selections}) != len(self.selections):
            raise EngineFault("BatchPlan: request selected twice")


@dataclass(frozen=True)
class PolicyConfig:
    policy: str = "accelgen"
    static_chunk_len: int = 512
    gamma: float = 0.75
    max_concurrent_long: int = 1
    budget_cap: int | None = None     # None -> S_pf
    orca_batch_size: int = 8
    orca_max_seq: int = 8192
    urgency_slack: float = DEFAULT_URGENCY_SLACK
    era: bool = True
    fcfs_budget: int | None = None    # PagedFcfs / Orca forward cap (None -> max(S_pf, 16384))
    kv_victim: str = "resident_last"  # KV-deficit victim rule: "resident_last" or the paper-literal "max_tr"
    # admission watermark: work that holds no blocks (new prompts, readmissions) is admitted only while it
    # leaves this fraction of the pool free for the resident requests' decode growth (vLLM's watermark);
    # 0 = the SPEC's rule (admit up to the last free block, preempt when decodes then run out)
    kv_watermark: float = 0.0
    # PAPER §4.4 "the previous TG requests should be retained in the batch as much as possible": after
    # Algorithms 1-2, every resident TG task not yet in B joins it (queue order) while budget and free
    # blocks allow.  Off = the SPEC's restatement (TG tasks join only when urgent or in the gamma-window)
    retain_tg: bool = False
    # budget from live deadlines only: an entry whose current iteration deadline has already passed
    # (T_w > its iteration SLO) no longer constrains S_b -- shrinking the forward cannot make a missed
    # deadline, it only starves everyone else (with B200 TTFT SLOs of ~5-15 ms, below one decode-carrying
    # step, the SPEC rule holds S_b near 200 tokens and chunks resident prompts one token per step)
    budget_live_only: bool = False

    def __post_init__(self):
        if self.policy not in POLICIES:
            raise ConfigError(f"unknown policy {self.policy!r}; expected one of {POLICIES}")
        if self.gamma < 0:
            raise ConfigError("gamma must be >= 0")
        if self.budget_cap is not None and self.budget_cap < 1:
            raise ConfigError("budget_cap must be >= 1")
        if self.max_concurrent_long < 1:
            raise ConfigError("max_concurrent_long must be >= 1")
        if self.kv_victim not in ("resident_last", "max_tr"):
            raise ConfigError("kv_victim must be 'resident_last' or 'max_tr'")
        if not 0.0 <= self.kv_watermark < 1.0:
            raise ConfigError("kv_watermark must be in [0, 1)")


def token_budget(slo_min: float, profile: ModelProfile, cfg: PolicyConfig) -> int:
    cap = profile.pivot_forward_size if cfg.budget_cap is None else cfg.budget_cap
    raw = math.floor(profile.pivot_forward_size * slo_min / profile.pivot_time_s)
    return max(1, min(raw, cap))


def dynamic_chunks(prompt_remainder: int, room: int) -> int:
    """Sequential token selection: take as much of the prompt as the room allows."""
    return max(0, min(prompt_remainder, room))


def emit_token_on_final_chunk(selection: Selection) -> bool:
    return selection.is_final_chunk


# ----------------------------------------------------------------------------- demand helpers
def has_prompt_left(e: QueueEntry) -> bool:
    return e.remaining_prompt_tokens > 0 and e.phase in (Phase.PROMPT_PENDING, Phase.PREEMPTED)


def step_blocks(e: QueueEntry, n_tokens: int, pool: BlockPool) -> int:
    """Blocks this entry needs to run n_tokens this step (readmission included)."""
    rid = e.request_id
    if rid in pool.swapped_out:
        saved = pool.swapped_out[rid]
        held = blocks_for(saved, pool.block_size)
        room = held * pool.block_size - saved
        return held + blocks_for(max(0, n_tokens - room), pool.block_size)
    if has_prompt_left(e):
        return pool.demand_prompt_chunk(rid, n_tokens).blocks_needed
    return pool.demand_tg(rid).blocks_needed


def tokens_fitting(e: QueueEntry, free_blocks: int, pool: BlockPool) -> int:
    """Largest token count whose step_blocks() fits in free_blocks."""
    rid, b = e.request_id, pool.block_size
    if rid in pool.swapped_out:
        saved = pool.swapped_out[rid]
        held = blocks_for(saved, b)
        if held > free_blocks:
            return 0
        return held * b - saved + (free_blocks - held) * b
    return pool.headroom(rid) + free_blocks * b


@dataclass
class PlanContext:
    """State the planner reads besides the queue (all owned by the engine)."""
    pool: BlockPool
    stats: ChunkStats
    profile: ModelProfile
    now: float
    long_active: set[int] = field(default_factory=set)  # long prompts with prefill started, not finished


def watermark_blocks(pool: BlockPool, cfg: PolicyConfig) -> int:
    return int(cfg.kv_watermark * pool.total_blocks)


def _era_blocked(e: QueueEntry, cfg: PolicyConfig, long_active: set[int]) -> bool:
    if not (cfg.era and e.is_long and has_prompt_left(e)):
        return False
    return e.request_id not in long_active and len(long_active) >= cfg.max_concurrent_long


def _slo_min(entries, now: float | None = None) -> float | None:
    """Smallest online iteration SLO; with `now`, only over entries whose deadline is still ahead."""
    vals = [iteration_slo(e) for e in entries if e.request.slo.kind is SLOKind.ONLINE
            and (now is None or now - e.enqueue_time <= iteration_slo(e))]
    return min(vals) if vals else None


# ----------------------------------------------------------------------------- AccelGen
def select_requests(a_gpu: int, a_kv_tokens: int, window_src: list[QueueEntry], t_r: dict[int, float],
                    ctx: PlanContext, cfg: PolicyConfig, long_active: set[int]) -> list[tuple[QueueEntry, int, int]]:
    """Algorithm 2.  Returns [(entry, chunk_len, blocks)] in selection order; mutates long_active."""
    if not window_src or a_gpu <= 0:
        return []
    pool, b = ctx.pool, ctx.pool.block_size
    wm = watermark_blocks(pool, cfg) * b
    t1 = t_r[window_src[0].request_id]
    window = [e for e in window_src if t_r[e.request_id] <= t1 + cfg.gamma]
    a_c, a_m = a_gpu, a_kv_tokens
    taken: list[tuple[QueueEntry, int, int]] = []
    # Prompt candidates are re-sized every round; TG candidates (D_c = 1) have a fixed block
    # demand, and among equal demands only the earliest queue position can win the (distance,
    # position) comparison -- so they are kept as FIFO buckets and only bucket heads compete.
    prompts: list[tuple[int, QueueEntry]] = []
    tg_buckets: dict[int, deque] = {}
    for pos, e in enumerate(window):
        if has_prompt_left(e):
            prompts.append((pos, e))
        else:
            tg_buckets.setdefault(step_blocks(e, 1, pool), deque()).append((pos, e))
    prompt_used = [False] * len(prompts)
    while a_c > 0:
        best = None  # (distance, position, kind, index/bucket, entry, chunk, blocks)
        for i, (pos, e) in enumerate(prompts):
            if prompt_used[i] or _era_blocked(e, cfg, long_active):
                continue
            room = a_m if pool.is_resident(e.request_id) else a_m - wm
            c = min(e.remaining_prompt_tokens, a_c, tokens_fitting(e, max(0, room) // b, pool))
            if c < 1:
                continue
            blk = step_blocks(e, c, pool)
            if blk * b > room:
                continue
            key = ((a_c - c) ** 2 + (a_m - blk * b) ** 2, pos)
            if best is None or key < best[:2]:
                best = (key[0], pos, "p", i, e, c, blk)
        for blk, dq in tg_buckets.items():
            if not dq or blk * b > a_m:
                continue
            pos, e = dq[0]
            if wm and blk * b > a_m - wm and not pool.is_resident(e.request_id):
                # a swapped-out TG task under the watermark: the next resident one of this demand competes
                nxt = next(((p2, e2) for p2, e2 in dq if pool.is_resident(e2.request_id)), None)
                if nxt is None:
                    continue
                pos, e = nxt
            key = ((a_c - 1) ** 2 + (a_m - blk * b) ** 2, pos)
            if best is None or key < best[:2]:
                best = (key[0], pos, "t", blk, e, 1, blk)
        if best is None:
            break
        _, _, kind, idx, e, c, blk = best
        if kind == "p":
            prompt_used[idx] = True
        else:
            tg_buckets[idx].remove((best[1], e))
        taken.append((e, c, blk))
        a_c -= c
        a_m -= blk * b
        if e.is_long and has_prompt_left(e):
            long_active.add(e.request_id)
    return taken


def accelgen_plan(queue: list[QueueEntry], ctx: PlanContext, cfg: PolicyConfig) -> BatchPlan:
    """Algorithm 1 over an already ordered queue (order_queue)."""
    pool, stats, profile = ctx.pool, ctx.stats, ctx.profile
    if not queue:
        return BatchPlan(token_budget=token_budget(profile.pivot_time_s, profile, cfg))
    t_r = {e.request_id: remaining_time(e, ctx.now, stats) for e in queue}
    position = {e.request_id: i for i, e in enumerate(queue)}
    urgent = [e for e in queue if is_urgent(t_r[e.request_id], stats, cfg.urgency_slack)]
    slo_min = _slo_min(urgent + [queue[0]], ctx.now if cfg.budget_live_only else None)
    if slo_min is None:
        cap = profile.pivot_forward_size if cfg.budget_cap is None else cfg.budget_cap
        s_b, slo_min = cap, 0.0
    else:
        s_b = token_budget(slo_min, profile, cfg)

    long_active = set(ctx.long_active)
    started_here: set[int] = set()
    members: list[list] = []  # [entry, chunk, blocks]
    s_f = used = 0
    deferred: list[int] = []
    # every urgent TG / preempted-TG task needs exactly one token; reserve those before sizing the
    # urgent prompt chunks so a chunk never crowds the returned decodes out of B (PAPER §4.4:
    # "the previous TG requests should be retained in the batch as much as possible")
    reserved = sum(1 for e in urgent if not has_prompt_left(e))
    for e in urgent:
        if has_prompt_left(e):
            if _era_blocked(e, cfg, long_active):
                deferred.append(e.request_id)
                continue
            c = min(e.remaining_prompt_tokens, max(1, s_b - s_f - reserved))
            if e.is_long and e.request_id not in long_active:
                long_active.add(e.request_id)
                started_here.add(e.request_id)
        else:
            c = 1
            reserved -= 1
        blk = step_blocks(e, c, pool)
        members.append([e, c, blk])
        s_f += c
        used += blk

    free = pool.free_blocks
    preempted: list[int] = []
    wm = watermark_blocks(pool, cfg)
    used_new = sum(m[2] for m in members if not pool.is_resident(m[0].request_id))

    def wm_short():
        return wm > 0 and used_new > 0 and used > free - wm
    if members and (s_f > s_b or used > free or wm_short()):
        # repeatedly drop the member with max T_r (ties: later queue position) until B fits.  With
        # kv_victim="resident_last" a KV deficit first drops members that hold no blocks (prompts not yet
        # started, swapped-out requests awaiting readmission): admitting new work never evicts a resident
        # request's KV to host -- the evict/readmit churn the paper-literal rule ("max_tr") produces once
        # the pool is full
        # victims in descending (T_r, position) order; residency does not change inside this loop, so the
        # "max over the non-resident members, else over all" choice is two cursors over presorted lists
        order = sorted(range(len(members)), key=lambda i: (t_r[members[i][0].request_id],
                                                            position[members[i][0].request_id]), reverse=True)
        nonres = [i for i in order if not pool.is_resident(members[i][0].request_id)]
        p_all = p_nonres = 0
        dropped = set()
        while len(dropped) < len(members) and (s_f > s_b or used > free or wm_short()):
            kv_short = used > free
            under_wm = not kv_short and wm_short()
            while p_nonres < len(nonres) and nonres[p_nonres] in dropped:
                p_nonres += 1
            if under_wm and s_f <= s_b:
                i = nonres[p_nonres]  # only the admissions that cross the watermark leave B
            elif kv_short and cfg.kv_victim == "resident_last" and p_nonres < len(nonres):
                i = nonres[p_nonres]
            else:
                while order[p_all] in dropped:
                    p_all += 1
                i = order[p_all]
            e, c, blk = members[i]
            dropped.add(i)
            s_f -= c
            used -= blk
            rid = e.request_id
            if not pool.is_resident(rid):
                used_new -= blk
            if kv_short and pool.is_resident(rid):
                # KV deficit: swap the victim out to free its blocks (vLLM-style preemption)
                preempted.append(rid)
                free += pool.blocks_held(rid)
            else:
                # budget deficit only: the victim leaves B but keeps its KV resident
                deferred.append(rid)
            if rid in started_here:
                long_active.discard(rid)
                started_here.discard(rid)
        members = [m for i, m in enumerate(members) if i not in dropped]

    chosen = [(m[0], m[1], m[2]) for m in members]
    skip = {e.request_id for e in urgent} | set(preempted) | set(deferred)
    rest = [e for e in queue if e.request_id not in skip]
    chosen += select_requests(s_b - s_f, (free - used) * pool.block_size, rest, t_r, ctx, cfg, long_active)
    if cfg.retain_tg:
        a_c = s_b - sum(c for _, c, _ in chosen)
        a_blk = free - sum(blk for _, _, blk in chosen)
        taken = {e.request_id for e, _, _ in chosen}
        for e in rest:
            if a_c < 1:
                break
            if e.request_id in taken or has_prompt_left(e) or not pool.is_resident(e.request_id):
                continue
            blk = step_blocks(e, 1, pool)
            if blk > a_blk:
                continue
            chosen.append((e, 1, blk))
            a_c -= 1
            a_blk -= blk

    plan = BatchPlan(token_budget=s_b, preempted=preempted, slo_min=slo_min, deferred=deferred)
    for e, c, blk in chosen:
        final = (not has_prompt_left(e)) or c == e.remaining_prompt_tokens
        plan.selections.append(Selection(e.request_id, c, final))
        plan.forward_size += c
        plan.blocks_needed += blk
    return plan


# ----------------------------------------------------------------------------- baselines
def _fcfs_order(queue: list[QueueEntry]) -> list[QueueEntry]:
    return sorted(queue, key=lambda e: (e.request.arrival_time, e.request_id))


def _fcfs_budget(profile: ModelProfile, cfg: PolicyConfig) -> int:
    if cfg.fcfs_budget is not None:
        return cfg.fcfs_budget
    return max(profile.pivot_forward_size, 16384)


def baseline_plan(queue: list[QueueEntry], ctx: PlanContext, cfg: PolicyConfig) -> BatchPlan:
    pool, b = ctx.pool, ctx.pool.block_size
    order = _fcfs_order(queue)
    plan = BatchPlan()
    free = pool.free_blocks
    s_f = 0

    def add(e, c, blk):
        nonlocal s_f, free
        final = (not has_prompt_left(e)) or c == e.remaining_prompt_tokens
        plan.selections.append(Selection(e.request_id, c, final))
        s_f += c
        free -= blk
        plan.blocks_needed += blk

    tg = [e for e in order if not has_prompt_left(e)]
    prompts = [e for e in order if has_prompt_left(e)]

    if cfg.policy == "static_chunk":
        # Sarathi-Serve: decodes first, then fixed-size chunks FCFS until the budget is used
        s_b = profile_cap(ctx.profile, cfg)
        plan.token_budget = s_b
        for e in tg:
            blk = step_blocks(e, 1, pool)
            if s_f + 1 <= s_b and blk <= free:
                add(e, 1, blk)
        for e in prompts:
            room = s_b - s_f
            if room <= 0:
                break
            c = min(e.remaining_prompt_tokens, cfg.static_chunk_len, room)
            c = min(c, tokens_fitting(e, free, pool))
            if c < 1:
                break
            add(e, c, step_blocks(e, c, pool))
        if not plan.selections and tg:
            # pool exhausted by decodes that each need a new block: preempt the latest arrival, as vLLM /
            # Sarathi do (without it the baseline deadlocks once the KV pool is full)
            victim = max((e for e in tg if pool.is_resident(e.request_id)),
                         key=lambda e: (e.request.arrival_time, e.request_id), default=None)
            if victim is not None:
                plan.preempted.append(victim.request_id)
    elif cfg.policy == "paged_fcfs":
        # vLLM FCFS: running decodes, then whole prompts; stop at the first prompt that does not fit
        s_b = _fcfs_budget(ctx.profile, cfg)
        plan.token_budget = s_b
        for e in tg:
            blk = step_blocks(e, 1, pool)
            if s_f + 1 <= s_b and blk <= free:
                add(e, 1, blk)
        first = True
        for e in prompts:
            c = e.remaining_prompt_tokens
            blk = step_blocks(e, c, pool)
            # a prompt longer than the budget runs as the only prompt of its step (vLLM requires
            # max_num_batched_tokens >= max_model_len; without this the FCFS head blocks forever)
            over = s_f + c > s_b and not (first and c > s_b)
            if over or blk > free:
                break
            add(e, c, blk)
            first = False
            if c > s_b:
                break
        if not plan.selections and tg:
            # pool exhausted by decodes without headroom: preempt the latest arrival (vLLM policy)
            victim = max((e for e in tg if pool.is_resident(e.request_id)),
                         key=lambda e: (e.request.arrival_time, e.request_id), default=None)
            if victim is not None:
                plan.preempted.append(victim.request_id)
    else:  # orca_fcfs: <= orca_batch_size live requests, each reserving orca_max_seq tokens, no chunking
        s_b = _fcfs_budget(ctx.profile, cfg)
        plan.token_budget = s_b
        limit = min(cfg.orca_batch_size, max(1, pool.total_blocks // blocks_for(cfg.orca_max_seq, b)))
        live = [e for e in order if pool.is_resident(e.request_id) or e.request_id in pool.swapped_out]
        for e in live:
            c = e.remaining_prompt_tokens if has_prompt_left(e) else 1
            blk = step_blocks(e, c, pool)
            if s_f + c <= s_b and blk <= free:
                add(e, c, blk)
        n_live = len(live)
        live_ids = {e.request_id for e in live}
        for e in order:
            if n_live >= limit:
                break
            if e.request_id in live_ids:
                continue
            c = e.remaining_prompt_tokens
            blk = step_blocks(e, c, pool)
            if (s_f + c > s_b and not (s_f == 0 and c > s_b)) or blk > free:  # over-budget prompt: alone
                break
            add(e, c, blk)
            n_live += 1
    plan.forward_size = s_f
    plan.token_budget = max(plan.token_budget, s_f)  # an over-budget prompt alone stretches its step's budget
    return plan


def profile_cap(profile: ModelProfile, cfg: PolicyConfig) -> int:
    return profile.pivot_forward_size if cfg.budget_cap is None else cfg.budget_cap


def plan(queue: list[QueueEntry], ctx: PlanContext, cfg: PolicyConfig) -> BatchPlan:
    if cfg.policy == "accelgen":
        return accelgen_plan(queue, ctx, cfg)
    return baseline_plan(queue, ctx, cfg)
