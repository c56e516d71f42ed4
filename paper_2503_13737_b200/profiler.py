"""B200 profiler: measure the iteration-time cost model the chunker consumes.

The paper finds the pivot forward size S_pf by sweeping the forward size until throughput
saturates and records the batch time T_pf there (PAPER §4.2, "we measure the pivot forward size
(S_pf) by varying the forward size ... and measure the corresponding batch execution time";
the saturation criterion <3% marginal gain is in PAPER.md:726).  The reference's stand-in only
derives it from a peak FLOP/s (cost_model.py:112-127).  Here the sweep runs the real mixed
forward on the GPU (CUDA-event time of ag_model_forward), fits the reference's linear model
T(S_f) = T_0 + T_pf * S_f / S_pf by least squares, and writes a ModelProfile JSON
(PROFILE_KEYS, cost_model.py:23-31) that bench.py / the engine load with load_profile.

A second sweep runs MIXED batches -- decode tokens over 0.5k-16k cached contexts, prompt chunks
on cached prefixes, and both together -- and fits the extended model of cost_model.batch_time,
T = T_0 + a*S_f + b*(K/V rows read) + c*(attention query-key pairs), so the clock the scheduler
plans with (T_max, budgets, the virtual clock) also holds for the decode-heavy steps that make up
a serving trace (the linear model alone predicts a 64-decode step at 1.5k context at 7 ms; it
measures 17.6 ms).

  python -m paper_2503_13737_b200.profiler --out profiles/opt13b_b200_tp1.json
"""
from __future__ import annotations

import argparse
import json
from pathlib import Path

import numpy as np

SWEEP = (64, 128, 256, 512, 768, 1024, 1536, 2048, 3072, 4096, 6144, 8192)


def prefill_batch(pool, cfg, s_f: int, seq_len: int, rid0: int):
    """S_f tokens of fresh prompts (seq_len each, the last one shorter)."""
    from .engine import DeviceBatch, synthetic_tokens
    ids, pos, slot, cu, ctx, tabs, lr, rids = [], [], [], [0], [], [], [], []
    left, rid = s_f, rid0
    while left > 0:
        n = min(seq_len, left)
        pool.allocate(rid, pool.demand_prompt_chunk(rid, n))
        p = np.arange(0, n, dtype=np.int32)
        ids.append(synthetic_tokens(rid, p, cfg.vocab)); pos.append(p)
        slot.append(np.asarray(pool.slots(rid, 0, n), np.int32)); ctx.append(0)
        cu.append(cu[-1] + n); tabs.append(pool.block_table(rid)); lr.append(cu[-1] - 1); rids.append(rid)
        left -= n
        rid += 1
    bt = np.zeros((len(tabs), max(map(len, tabs))), np.int32)
    for i, t in enumerate(tabs):
        bt[i, :len(t)] = t
    return DeviceBatch(rids, np.concatenate(ids), np.concatenate(pos), np.asarray(cu, np.int32),
                       np.asarray(ctx, np.int32), bt, np.concatenate(slot), np.asarray(lr, np.int32), rids), rid


def sweep(cfg, tp: int = 1, sizes=SWEEP, seq_len: int = 512, reps: int = 5, executor=None) -> list[dict]:
    from .executor import CudaExecutor
    from .kvc import BlockPool
    max_t = max(sizes)
    n_blocks = 2 * (max_t // 32 + len(sizes) * 4)
    ex = executor or CudaExecutor(cfg, n_blocks, max_tokens=max_t, max_seqs=max_t // seq_len + 8, tp_size=tp)
    out = []
    rid = 0
    for s_f in sizes:
        times = []
        for r in range(reps + 2):
            pool = BlockPool(n_blocks)
            b, rid = prefill_batch(pool, cfg, s_f, seq_len, rid)
            res = ex.execute(b)
            if r >= 2:
                times.append(res.device_s)
        t = float(np.median(times))
        out.append({"s_f": s_f, "seconds": t, "tokens_per_s": s_f / t})
    return out


def mixed_batch(pool, cfg, seqs, rid0: int):
    """One forward of sequences (q_i new tokens on p_i cached tokens); the cached K/V are whatever the
    pool holds (timing only)."""
    from .engine import DeviceBatch, synthetic_tokens
    ids, pos, slot, cu, ctx, tabs, lr, rids = [], [], [], [0], [], [], [], []
    rid = rid0
    for q, p_len in seqs:
        pool.allocate(rid, pool.demand_prompt_chunk(rid, p_len + q))
        p = np.arange(p_len, p_len + q, dtype=np.int32)
        ids.append(synthetic_tokens(rid, p, cfg.vocab)); pos.append(p)
        slot.append(np.asarray(pool.slots(rid, p_len, q), np.int32)); ctx.append(p_len)
        cu.append(cu[-1] + q); tabs.append(pool.block_table(rid)); lr.append(cu[-1] - 1); rids.append(rid)
        rid += 1
    bt = np.zeros((len(tabs), max(map(len, tabs))), np.int32)
    for i, t in enumerate(tabs):
        bt[i, :len(t)] = t
    return DeviceBatch(rids, np.concatenate(ids), np.concatenate(pos), np.asarray(cu, np.int32),
                       np.asarray(ctx, np.int32), bt, np.concatenate(slot), np.asarray(lr, np.int32), rids), rid


def mixed_cases(max_tokens: int, max_kv: int) -> list[list[tuple[int, int]]]:
    """Decode-only, chunk-on-prefix and mixed batches spanning the serving regime (each within
    max_tokens forward tokens and max_kv cached tokens)."""
    cases = []
    for n in (16, 64, 128, 256, 512):
        for c in (512, 1536, 4096, 16384):
            if n * c <= max_kv and n <= max_tokens:
                cases.append([(1, c)] * n)
    for q in (256, 1024, 1536):
        for p in (2048, 8192, 16384, 65536):
            if q <= max_tokens and p + q <= max_kv:
                cases.append([(q, p)])
    for n, c, q, p in ((64, 1536, 512, 4096), (128, 1024, 1024, 8192), (256, 2048, 1024, 0), (32, 8192, 1280, 12288),
                       (200, 1500, 256, 0), (100, 3000, 1024, 2048)):
        if n + q <= max_tokens and n * c + p + q <= max_kv:
            cases.append([(1, c)] * n + [(q, p)])
    return cases


def mixed_sweep(cfg, executor, n_blocks: int, cases, reps: int = 3) -> list[dict]:
    from .cost_model import batch_features
    from .kvc import BlockPool
    out, rid = [], 1 << 20
    for seqs in cases:
        times = []
        for r in range(reps + 1):
            pool = BlockPool(n_blocks)
            b, rid = mixed_batch(pool, cfg, seqs, rid)
            res = executor.execute(b)
            if r >= 1:
                times.append(res.device_s)
        kv, pairs = batch_features(seqs)
        out.append({"s_f": sum(q for q, _ in seqs), "kv_tokens": kv, "pairs": pairs, "seqs": len(seqs),
                    "seconds": float(np.median(times))})
    return out


def fit_extended(points: list[dict], base: dict) -> dict:
    """Weighted (1/T) non-negative least squares of T = T_0 + a*S_f + b*kv + c*pairs over every measured
    batch; returns base with pivot_time_s / fixed_overhead_s re-fitted and kv_read_s_per_token /
    attn_s_per_pair added (coefficients that fit negative are dropped and the rest re-fitted)."""
    s = np.array([p["s_f"] for p in points], float)
    kv = np.array([p.get("kv_tokens", 0) for p in points], float)
    pr = np.array([p.get("pairs", 0) for p in points], float)
    t = np.array([p["seconds"] for p in points], float)
    cols = {"t0": np.ones_like(s), "a": s, "b": kv, "c": pr}
    keep = list(cols)
    while True:
        A = np.stack([cols[k] for k in keep], 1) / t[:, None]
        coef, *_ = np.linalg.lstsq(A, np.ones_like(t), rcond=None)
        neg = [k for k, v in zip(keep, coef) if v < 0 and k != "a"]
        if not neg:
            break
        keep.remove(neg[0])
    got = dict(zip(keep, coef))
    pred = sum(got[k] * cols[k] for k in keep)
    s_pf = base["pivot_forward_size"]
    out = dict(base)
    out.update({"pivot_time_s": float(got["a"] * s_pf), "fixed_overhead_s": float(got.get("t0", 0.0)),
                "kv_read_s_per_token": float(got.get("b", 0.0)), "attn_s_per_pair": float(got.get("c", 0.0))})
    return out, {"max_rel_err": float(np.max(np.abs(pred - t) / t)), "mean_rel_err": float(np.mean(np.abs(pred - t) / t))}


def fit(points: list[dict], hidden: int, num_layers: int, kvc_tokens: int, gain: float = 0.03) -> dict:
    """Least-squares T = T_0 + a*S_f over the sweep, weighted by 1/T (relative error, so the model
    is as accurate for a 64-token decode step as for a pivot-sized one: TTFT SLOs of short prompts
    come from the small end, workload.py base_ttft); S_pf = smallest size whose throughput is within
    `gain` of the best measured (the paper's <3% marginal-gain saturation rule)."""
    s = np.array([p["s_f"] for p in points], float)
    t = np.array([p["seconds"] for p in points], float)
    thr = s / t
    best = thr.max()
    s_pf = int(s[np.argmax(thr >= (1.0 - gain) * best)])
    a, t0 = np.polyfit(s, t, 1, w=1.0 / t)
    t0 = max(0.0, float(t0))
    return {"hidden_size": hidden, "num_layers": num_layers, "pivot_forward_size": s_pf,
            "pivot_time_s": float(a * s_pf), "bytes_per_element": 2, "fixed_overhead_s": t0,
            "kvc_capacity_tokens": int(kvc_tokens)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="opt-13b")
    ap.add_argument("--tp", type=int, default=1)
    ap.add_argument("--out", default=None)
    ap.add_argument("--kv-gb", type=float, default=80.0, help="KV pool size written into the profile")
    ap.add_argument("--sweep-kv-tokens", type=int, default=80000, help="cached tokens of the mixed sweep's pool")
    ap.add_argument("--linear-only", action="store_true", help="prefill sweep and the reference's linear fit only")
    args = ap.parse_args()
    from . import model as M
    from .cost_model import ModelProfile, save_profile
    from .executor import CudaExecutor
    try:  # positions for the 64k-prefix cases of the mixed sweep
        cfg = M.PRESETS[args.model](max_positions=70000)
    except TypeError:
        cfg = M.PRESETS[args.model]()
    max_t = max(SWEEP)
    n_blocks = max(2 * (max_t // 32 + len(SWEEP) * 4), args.sweep_kv_tokens // 32 + 64)
    ex = CudaExecutor(cfg, n_blocks, max_tokens=max_t, max_seqs=1024, max_blocks_per_seq=(cfg.pos_rows + 31) // 32,
                      tp_size=args.tp)
    pts = sweep(cfg, args.tp, executor=ex)
    kv_tokens = int(args.kv_gb * 1e9 // (32 * cfg.kv_bytes_per_token(args.tp))) * 32
    prof = fit(pts, cfg.hidden, cfg.num_layers, kv_tokens)
    mixed, err = [], None
    if not args.linear_only:
        from .cost_model import batch_features
        for p in pts:  # the prefill sweep's own features (512-token prompts)
            q, n = 512, p["s_f"]
            seqs = [(min(q, n - i), 0) for i in range(0, n, q)]
            p["kv_tokens"], p["pairs"] = batch_features(seqs)
        mixed = mixed_sweep(cfg, ex, n_blocks, mixed_cases(max_t, args.sweep_kv_tokens))
        prof, err = fit_extended(pts + mixed, prof)
    ex.close()
    out = Path(args.out or f"profiles/opt13b_b200_tp{args.tp}.json")
    out.parent.mkdir(parents=True, exist_ok=True)
    save_profile(ModelProfile(**prof), out)
    out.with_name(out.stem + "_sweep.json").write_text(json.dumps({"model": args.model, "tp": args.tp,
                                                                    "points": pts, "mixed": mixed, "fit": prof,
                                                                    "fit_error": err}, indent=1))
    print(json.dumps({"profile": prof, "fit_error": err, "points": pts, "mixed": mixed}))


if __name__ == "__main__":
    main()
