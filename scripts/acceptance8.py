"""SPEC acceptance 8, directional end to end, on the virtual clock: a generated mixed trace
(2,000 requests, 35% long from the reference's default log-uniform 4k-100k, rate 8/s, the paper's SLO
recipe) served by AccelGen, PagedFcfs, StaticChunk and OrcaFcfs with the B200-measured cost model, over a
fixed horizon (the trace overloads one B200 ~2x, so runs are truncated).  Prints one JSON line per
(seed, policy) and a summary of which orderings hold on how many seeds."""
import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2503_13737_b200 import cost_model as cm, workload as wl  # noqa: E402
from paper_2503_13737_b200.engine import Engine  # noqa: E402
from paper_2503_13737_b200.policies import PolicyConfig  # noqa: E402

POLICIES = ("accelgen", "paged_fcfs", "static_chunk", "orca_fcfs")


def run_seed(seed, prof, horizon, watermark, swap_cost, rate=8.0, long_fraction=0.35, n=2000):
    tr = wl.generate_trace(wl.TraceConfig(num_requests=n, arrival_rate=rate, long_fraction=long_fraction, seed=seed,
                                          profile=prof))
    out = {}
    for pol in POLICIES:
        t = time.time()
        eng = Engine(tr, prof, PolicyConfig(policy=pol, kv_watermark=watermark if pol == "accelgen" else 0.0),
                     horizon_s=horizon, per_token_swap_cost_s=swap_cost)
        r = eng.run()
        out[pol] = {"attain": r.slo_attainment, "goodput": r.goodput, "tokens_per_s": r.tokens_per_s,
                    "slo_tokens_per_s": sum(it.slo_tokens for it in eng.metrics.iterations) / r.makespan,
                    "completed": r.completed, "preemptions": r.preemptions, "sim_s": round(time.time() - t, 1)}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seeds", type=int, default=10)
    ap.add_argument("--horizon", type=float, default=300.0)
    ap.add_argument("--watermark", type=float, default=0.1)
    ap.add_argument("--swap-cost", type=float, default=819200 / 25e9)
    ap.add_argument("--profile", default="profiles/opt13b_b200_tp1.json")
    ap.add_argument("--kv-tokens", type=int, default=186720)
    a = ap.parse_args()
    prof = cm.load_profile(a.profile)
    prof = cm.ModelProfile(**{**prof.__dict__, "kvc_capacity_tokens": a.kv_tokens})
    holds = {"attain>paged,static": 0, "slo_tok>paged,static": 0, "goodput>paged,static": 0, "orca_lowest_tput": 0}
    for seed in range(a.seeds):
        r = run_seed(seed, prof, a.horizon, a.watermark, a.swap_cost)
        print(json.dumps({"seed": seed, **r}), flush=True)
        ag = r["accelgen"]
        holds["attain>paged,static"] += all(ag["attain"] > r[p]["attain"] for p in ("paged_fcfs", "static_chunk"))
        holds["slo_tok>paged,static"] += all(ag["slo_tokens_per_s"] > r[p]["slo_tokens_per_s"]
                                             for p in ("paged_fcfs", "static_chunk"))
        holds["goodput>paged,static"] += all(ag["goodput"] > r[p]["goodput"] for p in ("paged_fcfs", "static_chunk"))
        holds["orca_lowest_tput"] += r["orca_fcfs"]["tokens_per_s"] == min(v["tokens_per_s"] for v in r.values())
    print(json.dumps({"seeds": a.seeds, "horizon_s": a.horizon, "watermark": a.watermark, "holds": holds}))


if __name__ == "__main__":
    main()
