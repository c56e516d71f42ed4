"""Virtual-clock simulation of the config-2 trace with the extended cost model (no GPU): per-window
steady-state statistics for a policy and arrival rate.  Used to choose the bench operating point."""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2503_13737_b200 import configs, cost_model as cm, workload as wl  # noqa: E402
from paper_2503_13737_b200.engine import Engine  # noqa: E402
from paper_2503_13737_b200.policies import PolicyConfig  # noqa: E402


def run(rate, policy, horizon, t0, prof, n_req=6000, seed=0, watermark=0.0, swap_cost=0.0, retain_tg=False, live_only=False):
    cfg = configs.config2(profile=prof, arrival_rate=rate, num_requests=n_req, seed=seed)
    trace = wl.generate_trace(cfg.trace)
    eng = Engine(trace, prof, PolicyConfig(policy=policy, kv_watermark=watermark, retain_tg=retain_tg, budget_live_only=live_only), clock="virtual",
                 kv_blocks=prof.kvc_capacity_tokens // 32, per_token_swap_cost_s=swap_cost)
    w0 = time.time()
    while not eng.done() and eng.clock < horizon:
        eng.step()
    its = [it for it in eng.metrics.iterations if it.start >= t0]
    span = eng.clock - t0
    ev = sum(it.events for it in its)
    met = sum(it.events_met for it in its)
    toks = sum(it.forward_size for it in its)
    slo = sum(it.slo_tokens for it in its)
    dec = sum(it.num_decode for it in its)
    live = len(eng.queue)
    return {"rate": rate, "policy": policy, "wm": watermark, "retain_tg": retain_tg, "live_only": live_only, "iters": len(its), "ms_per_iter": 1e3 * span / max(1, len(its)),
            "attain": met / ev if ev else None, "fwd_tok_s": toks / span, "slo_tok_s": slo / span,
            "decode_tok_s": dec / span, "preempt": sum(it.preemptions for it in its),
            "S_f_p50": float(np.median([it.forward_size for it in its])) if its else 0,
            "kv_util": float(np.mean([it.allocated_tokens for it in its])) / prof.kvc_capacity_tokens if its else 0,
            "queue_end": live, "sim_s": round(time.time() - w0, 1)}


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--rates", default="2,3,4,6,8")
    ap.add_argument("--policies", default="accelgen,static_chunk")
    ap.add_argument("--horizon", type=float, default=300)
    ap.add_argument("--t0", type=float, default=120)
    ap.add_argument("--profile", default=None)
    ap.add_argument("--watermarks", default="0")
    ap.add_argument("--retain-tg", action="store_true")
    ap.add_argument("--live-only", action="store_true")
    ap.add_argument("--swap-cost", type=float, default=819200 / 25e9, help="s per swapped token (PCIe)")
    a = ap.parse_args()
    prof = cm.load_profile(a.profile) if a.profile else cm.ModelProfile(
        hidden_size=5120, num_layers=40, pivot_forward_size=1536, pivot_time_s=0.033, fixed_overhead_s=0.0045,
        kvc_capacity_tokens=186720, kv_read_s_per_token=1.3e-7, attn_s_per_pair=1.2e-9)
    for pol in a.policies.split(","):
        for r in a.rates.split(","):
            for wm in a.watermarks.split(","):
                print(json.dumps(run(float(r), pol, a.horizon, a.t0, prof, watermark=float(wm),
                                     swap_cost=a.swap_cost, retain_tg=a.retain_tg, live_only=a.live_only)), flush=True)
