"""Brute-force restatement of AccelGen's scheduler — TEST INFRASTRUCTURE ONLY.

An independent, deliberately naive re-derivation of the SPEC's policies + engine
(Algorithms 1-2 at PAPER.md:1868-1938) with the same pinned decisions as the
product, written without importing the product's scheduler.
The remaining-time arithmetic restates the reference's sched_core (pkg/src/slosim/
sched_core.py:89-146) in the same floating-point operation order, the block accounting restates
kvc.py:88-160 plus the lowest-free-id placement, and select_requests recomputes every
candidate's Euclidean distance from scratch each round (SPEC.md:410's "exhaustive greedy
oracle").  tests/test_scheduler_oracle.py checks the product's decisions (chunk sizes, batch
composition, preemptions, block tables) against this module bit for bit.

Inputs are the product's RequestSpec/ModelProfile values (plain data); nothing else is shared.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field


def _blocks(tokens, b):
    return -(-tokens // b)


@dataclass
class Req:
    spec: object
    phase: str = "prompt"          # prompt | tg | preempted
    remaining: int = 0
    enqueue: float = 0.0
    seq: int = 0
    allowance: float = 0.0
    debt: float = 0.0
    generated: int = 0
    emits: list = field(default_factory=list)

    @property
    def rid(self):
        return self.spec.id

    @property
    def online(self):
        return self.spec.slo.kind.value == "online"

    @property
    def long(self):
        return self.spec.prompt_len >= 4096


class Pool:
    def __init__(self, total, b=32):
        self.total, self.b, self.tables, self.stored, self.swapped = total, b, {}, {}, {}

    @property
    def free(self):
        return self.total - sum(len(t) for t in self.tables.values())

    def lowest(self, n):
        used = {i for t in self.tables.values() for i in t}
        out, i = [], 0
        while len(out) < n:
            if i not in used:
                out.append(i)
            i += 1
        return out

    def headroom(self, rid):
        return len(self.tables[rid]) * self.b - self.stored[rid] if rid in self.tables else 0

    def need(self, r, n):
        """Blocks to run n tokens of r this step (readmission included)."""
        if r.rid in self.swapped:
            s = self.swapped[r.rid]
            held = _blocks(s, self.b)
            return held + _blocks(max(0, n - (held * self.b - s)), self.b)
        if r.rid in self.tables:
            return _blocks(max(0, n - self.headroom(r.rid)), self.b)
        return _blocks(n, self.b)

    def fit(self, r, free_blocks):
        if r.rid in self.swapped:
            s = self.swapped[r.rid]
            held = _blocks(s, self.b)
            return 0 if held > free_blocks else held * self.b - s + (free_blocks - held) * self.b
        return self.headroom(r.rid) + free_blocks * self.b

    def grow(self, rid, n):
        if rid in self.swapped:
            s = self.swapped.pop(rid)
            self.tables[rid], self.stored[rid] = self.lowest(_blocks(s, self.b)), s
        if rid not in self.tables:
            self.tables[rid], self.stored[rid] = [], 0
        extra = _blocks(max(0, n - self.headroom(rid)), self.b)
        self.tables[rid] += self.lowest(extra)
        self.stored[rid] += n


class OracleScheduler:
    """Virtual-clock AccelGen simulation over a trace; records every plan."""

    def __init__(self, trace, profile, *, gamma=0.75, max_long=1, slack=0.1, kv_blocks=None, era=True,
                 kv_victim="resident_last", kv_watermark=0.0, retain_tg=False, budget_live_only=False):
        self.trace = sorted(trace, key=lambda r: (r.arrival_time, r.id))
        self.p = profile
        self.gamma, self.max_long, self.slack, self.era = gamma, max_long, slack, era
        self.kv_victim = kv_victim
        self.kv_watermark = kv_watermark
        self.retain_tg = retain_tg
        self.budget_live_only = budget_live_only
        self.pool = Pool(kv_blocks if kv_blocks is not None else profile.kvc_capacity_tokens // 32)
        self.t_max = profile.fixed_overhead_s + profile.pivot_time_s * profile.pivot_forward_size / profile.pivot_forward_size
        self.lc = float(profile.pivot_forward_size)
        self.tg_steps = self.preempts = 0
        self.p_prob = self.p_max = 0.0
        self.clock, self.nxt, self.stamp = 0.0, 0, 0
        self.queue, self.long_active, self.log = [], set(), []
        self.reqs = {}         # every admitted request (finished ones leave the queue, not this map)
        self.clock_fn = None   # optional entry -> elapsed seconds (the CPU-timed reference arm's clock)
        self.preempt_time = {}

    # ---- reference arithmetic (sched_core.py:89-146)
    def n_ck(self, tokens):
        return 1 if tokens <= 0 else math.ceil(tokens / self.lc)

    def slo(self, r):
        if not r.online:
            return r.allowance - r.debt
        return r.spec.slo.ttft_slo if r.phase == "prompt" else r.spec.slo.tbt_slo

    def t_r(self, r, now):
        pend = r.remaining if r.phase == "prompt" else 0
        return self.slo(r) - (now - r.enqueue) - self.n_ck(pend) * self.t_max

    def iter_time(self, s_f, shapes=()):
        """Reference linear model; plus the B200 extension's K/V-read and attention-pair terms when the
        profile carries them (shapes = [(q_i, p_i)]; same float expression as cost_model.batch_time)."""
        t = self.p.fixed_overhead_s + self.p.pivot_time_s * s_f / self.p.pivot_forward_size
        b, c = getattr(self.p, "kv_read_s_per_token", 0.0), getattr(self.p, "attn_s_per_pair", 0.0)
        if b or c:
            kv = sum(p + q for q, p in shapes)
            pairs = sum(q * p + q * (q + 1) // 2 for q, p in shapes)
            t = t + b * kv + c * pairs
        return t

    def budget(self, slo_min):
        return max(1, min(math.floor(self.p.pivot_forward_size * slo_min / self.p.pivot_time_s),
                          self.p.pivot_forward_size))

    def _stamp(self):
        self.stamp += 1
        return self.stamp

    def prompt_left(self, r):
        return r.remaining > 0 and r.phase in ("prompt", "preempted")

    def era_blocked(self, r, active):
        return (self.era and r.long and self.prompt_left(r) and r.rid not in active
                and len(active) >= self.max_long)

    # ---- one planning step (Algorithm 1 + 2)
    def plan(self):
        now, pool = self.clock, self.pool
        q = sorted(self.queue, key=lambda r: (self.t_r(r, now), r.seq))
        tr = {r.rid: self.t_r(r, now) for r in q}
        pos = {r.rid: i for i, r in enumerate(q)}
        urgent = [r for r in q if tr[r.rid] <= self.t_max * (1.0 + self.slack)]
        online = [self.slo(r) for r in urgent + q[:1]
                  if r.online and (not self.budget_live_only or now - r.enqueue <= self.slo(r))]
        s_b = self.budget(min(online)) if online else self.p.pivot_forward_size
        active = set(self.long_active)
        new_here = set()
        B, deferred = [], []
        s_f = used = 0
        tg_left = len([r for r in urgent if not self.prompt_left(r)])
        for r in urgent:
            if self.prompt_left(r):
                if self.era_blocked(r, active):
                    deferred.append(r.rid)
                    continue
                c = min(r.remaining, max(1, s_b - s_f - tg_left))
                if r.long and r.rid not in active:
                    active.add(r.rid)
                    new_here.add(r.rid)
            else:
                c = 1
                tg_left -= 1
            blk = pool.need(r, c)
            B.append([r, c, blk])
            s_f += c
            used += blk
        free = pool.free
        preempted = []
        wm = int(self.kv_watermark * pool.total)

        def used_new():  # blocks of members holding none (new prompts, readmissions)
            return sum(m[2] for m in B if m[0].rid not in pool.tables)

        def wm_short():
            return wm > 0 and used_new() > 0 and used > free - wm
        while B and (s_f > s_b or used > free or wm_short()):
            kv_short = used > free
            cand = B
            if not kv_short and wm_short() and s_f <= s_b:
                cand = [m for m in B if m[0].rid not in pool.tables]
            elif kv_short and self.kv_victim == "resident_last":
                # KV deficit: leave out work that holds no blocks (new / swapped-out) before preempting a
                # resident request -- brute force: scan the members that are not in the pool
                cand = [m for m in B if m[0].rid not in pool.tables] or B
            v = max(cand, key=lambda m: (tr[m[0].rid], pos[m[0].rid]))
            B.remove(v)
            s_f -= v[1]
            used -= v[2]
            if kv_short and v[0].rid in pool.tables:
                preempted.append(v[0].rid)
                free += len(pool.tables[v[0].rid])
            else:
                deferred.append(v[0].rid)
            if v[0].rid in new_here:
                active.discard(v[0].rid)
        chosen = [tuple(m) for m in B]
        skip = {r.rid for r in urgent} | set(preempted) | set(deferred)
        rest = [r for r in q if r.rid not in skip]
        a_c, a_m = s_b - s_f, (free - used) * pool.b
        if rest and a_c > 0:
            t1 = tr[rest[0].rid]
            win = [r for r in rest if tr[r.rid] <= t1 + self.gamma]
            taken = set()
            while a_c > 0:
                cands = []
                for i, r in enumerate(win):
                    if r.rid in taken:
                        continue
                    room = a_m if r.rid in pool.tables else a_m - wm * pool.b
                    if self.prompt_left(r):
                        if self.era_blocked(r, active):
                            continue
                        c = min(r.remaining, a_c, pool.fit(r, max(0, room) // pool.b))
                        if c < 1:
                            continue
                    else:
                        c = 1
                    blk = pool.need(r, c)
                    if c <= a_c and blk * pool.b <= room:
                        cands.append(((a_c - c) ** 2 + (a_m - blk * pool.b) ** 2, i, r, c, blk))
                if not cands:
                    break
                _, _, r, c, blk = min(cands, key=lambda x: (x[0], x[1]))
                taken.add(r.rid)
                chosen.append((r, c, blk))
                a_c -= c
                a_m -= blk * pool.b
                if r.long and self.prompt_left(r):
                    active.add(r.rid)
        if self.retain_tg:  # every resident TG task not in B joins it while budget and blocks allow
            a_c = s_b - sum(c for _, c, _ in chosen)
            a_blk = free - sum(blk for _, _, blk in chosen)
            taken = {r.rid for r, _, _ in chosen}
            for r in rest:
                if a_c < 1:
                    break
                if r.rid in taken or self.prompt_left(r) or r.rid not in pool.tables:
                    continue
                blk = pool.need(r, 1)
                if blk <= a_blk:
                    chosen.append((r, 1, blk))
                    a_c -= 1
                    a_blk -= blk
        return s_b, chosen, preempted, deferred

    # ---- engine step (SPEC.md:481-489 with the pinned decisions)
    def admit(self):
        while self.nxt < len(self.trace) and self.trace[self.nxt].arrival_time <= self.clock:
            s = self.trace[self.nxt]
            self.nxt += 1
            r = Req(spec=s, remaining=s.prompt_len, enqueue=s.arrival_time, seq=self._stamp())
            if not r.online:
                per_tok = self.t_max + self.p_max * self.p_prob
                est = self.n_ck(s.prompt_len) * self.t_max + s.predicted_output_len * per_tok
                r.allowance = (s.slo.jct_slo - est) / (self.n_ck(s.prompt_len) + s.predicted_output_len)
            self.queue.append(r)
            self.reqs[r.rid] = r

    def step(self):
        self.admit()
        if not self.queue:
            if self.nxt < len(self.trace):
                self.clock = max(self.clock, self.trace[self.nxt].arrival_time)
            return None
        s_b, chosen, preempted, deferred = self.plan()
        start = self.clock
        byid = {r.rid: r for r in self.queue}
        for rid in preempted:
            self.pool.swapped[rid] = self.pool.stored.pop(rid)
            self.pool.tables.pop(rid)
            self.preempts += 1
            if self.tg_steps:
                self.p_prob = min(1.0, self.preempts / self.tg_steps)
            self.preempt_time[rid] = start
            byid[rid].phase, byid[rid].enqueue, byid[rid].seq = "preempted", start, self._stamp()
        if not chosen:
            nxt = self.trace[self.nxt].arrival_time if self.nxt < len(self.trace) else math.inf
            self.clock = min(nxt, self.clock + self.t_max)
            return None
        entry = {"s_b": s_b, "sel": [], "preempted": list(preempted), "tables": {}}
        for r, c, blk in chosen:
            if r.rid in self.pool.swapped and r.rid in self.preempt_time:
                self.p_max = max(self.p_max, start - self.preempt_time[r.rid])
            before = self.pool.stored.get(r.rid, 0) if r.rid not in self.pool.swapped else self.pool.swapped[r.rid]
            self.pool.grow(r.rid, c)
            final = (not self.prompt_left(r)) or c == r.remaining
            entry["sel"].append((r.rid, c, final, before))
            entry["tables"][r.rid] = list(self.pool.tables[r.rid])
        s_f = sum(c for _, c, _ in chosen)
        if self.clock_fn is not None:
            self.clock = start + self.clock_fn(entry)
        else:
            self.clock = start + self.iter_time(s_f, [(c, before) for _, c, _, before in entry["sel"]])
        entry["start"], entry["end"] = start, self.clock
        now = self.clock
        done = set()
        for r, c, blk in chosen:
            if not r.online:
                r.debt += (start - r.enqueue) - r.allowance
            prompt = self.prompt_left(r)
            if prompt:
                self.lc += 0.1 * (c - self.lc)
                r.remaining -= c
                if r.long:
                    self.long_active.add(r.rid)
            else:
                self.tg_steps += 1
                self.p_prob = self.preempts / self.tg_steps
            final = (not prompt) or r.remaining == 0
            if not final:
                r.phase, r.seq = "prompt", self._stamp()
                continue
            if prompt and r.long:
                self.long_active.discard(r.rid)
            r.generated += 1
            r.emits.append(now)
            if r.generated >= r.spec.output_len:
                self.pool.tables.pop(r.rid)
                self.pool.stored.pop(r.rid)
                done.add(r.rid)
            else:
                r.phase, r.remaining, r.enqueue, r.seq = "tg", 0, now, self._stamp()
        self.queue = [r for r in self.queue if r.rid not in done]
        self.log.append(entry)
        return entry

    def run(self, max_steps=None):
        n = 0
        while self.nxt < len(self.trace) or self.queue:
            if max_steps is not None and n >= max_steps:
                break
            if self.step() is not None:
                n += 1
        return self.log
