#!/usr/bin/env python
"""SLO-meeting tokens/s of AccelGen's mixed-batch forward on B200 (BASELINE.json metric).

The engine serves BASELINE config 2 live on the wall clock: each iteration orders the queue, plans a
BatchPlan (AccelGen), allocates KV blocks, runs the mixed prefill+decode forward of
OPT-13B (random bf16 weights) on the GPU(s) and emits tokens.  Workload: 90% <=1k prompts, 10% 4k-16k,
output 1-2048, TBT 0.1875 s x U(0.75,1.25), TTFT per 512-token bucket x U(0.5,1.5); the arrival rate
scales with the GPU count (weak scaling), TP over the GPUs.

  step   one 2-second window of serving (--window-s; SPEC.md:528 goodput windows are 1 s, ~50 forwards); the K timed
         windows start after an untimed ramp to steady state (--ramp-s of serving: request population and
         KV occupancy have levelled off) and W warm-up windows
  value  SLO-meeting tokens / sum of CUDA-event forward times of the K windows (metadata resident in
         HBM; the device-side number)
  e2e    the same tokens / wall time of the K windows through the public API (scheduler, packing, pinned
         H2D of every step's metadata, forward, D2H of the next-token ids)
  SLO-meeting tokens: a decode token whose TBT was met; a prompt's tokens -- every chunk, counted in the
         window that processed it -- iff its first token met TTFT (resolved after the window by serving on,
         untimed, until those prompts finish); iter_slo_attainment = met / all token events.

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--rate R] [--ramp-s S]
       (--gpus N > 1 without torchrun re-launches itself under torch.distributed.run, one rank per GPU)
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "SLO-meeting tokens/s (OPT-13B mixed trace)"
UNIT = "tokens/s"


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--rate", type=float, default=None, help="arrival rate per GPU (req/s)")
    ap.add_argument("--ramp-s", type=float, default=None, help="untimed seconds of serving before warmup")
    ap.add_argument("--window-s", type=float, default=2.0, help="seconds of serving per step (2 s: the per-window spread of 1 s windows / sqrt 2)")
    ap.add_argument("--policy", default="accelgen")
    ap.add_argument("--tp-backend", choices=("nccl", "host"), default="nccl",
                    help="host: TP collectives through the library's host backend (ranks may share a GPU)")
    ap.add_argument("--profile", default=None, help="ModelProfile JSON (default: profiles/opt13b_b200_tp{N}.json)")
    ap.add_argument("--kv-gb", type=float, default=None,
                    help="KV pool per GPU (GB); default: the HBM left after weights and a 12 GB reserve")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--kv-watermark", type=float, default=0.1,
                    help="AccelGen admission watermark (fraction of the KV pool kept for decode growth)")
    ap.add_argument("--spec-policy", action="store_true",
                    help="the SPEC restatement of AccelGen only: no watermark, no TG retention, SPEC budget rule")
    ap.add_argument("--no-pipeline", action="store_true",
                    help="synchronous engine (plan, forward, emit in turn) instead of planning step k+1 during k")
    return ap.parse_args()


# ----------------------------------------------------------------------------- helpers
class ClockSampler:
    """nvidia-smi SM clocks + throttle reasons sampled during the timed region (B200_PROFILING.md)."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.samples, self.proc = index, [], None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 7:
                self.samples.append(parts)

    def stop(self) -> dict:
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = sorted({n for s in self.samples for n, v in zip(names, s[3:]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def load_peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm": d["hbm_gbs"], "tensor": d["bf16_tflops"], "tensor_sustained": d["bf16_tflops_sustained"],
                "source": "MEASURED_PEAKS.json (measured)"}
    return {"hbm": 6650.0, "tensor": 1590.0, "tensor_sustained": 1400.0, "source": "fallback (B200_PROFILING.md)"}


def default_profile(tp: int):
    from paper_2503_13737_b200 import cost_model as cm
    p = ROOT / "profiles" / f"opt13b_b200_tp{tp}.json"
    if p.exists():
        return cm.load_profile(p), str(p.relative_to(ROOT))
    p1 = ROOT / "profiles" / "opt13b_b200_tp1.json"
    if p1.exists():  # no TP-t measurement yet: the TP=1 measurement with the linear work split by t
        base = cm.load_profile(p1)
        return cm.ModelProfile(**{**base.__dict__, "pivot_time_s": base.pivot_time_s / tp,
                                  "fixed_overhead_s": base.fixed_overhead_s / tp}), \
            f"{p1.relative_to(ROOT)} scaled 1/{tp} (TP={tp} not measured yet)"
    # declared fallback until the profiler has written one: S_pf 2048, linear fit guess
    return cm.ModelProfile(hidden_size=5120, num_layers=40, pivot_forward_size=2048, pivot_time_s=0.06 / tp,
                           fixed_overhead_s=0.006 / tp, kvc_capacity_tokens=0), "declared-default"


DEFAULT_RATE = 4.0    # req/s per GPU: capacity-bound from ~3 req/s; >= 98% iteration-SLO attainment in six runs
DEFAULT_RAMP_S = 150.0  # (profiles/r2/rate_sweep.md); ramp: request population and KV occupancy level off


def build_workload(args, world: int):
    from paper_2503_13737_b200 import configs
    from paper_2503_13737_b200.cost_model import load_profile
    prof, prof_src = default_profile(world) if args.profile is None else (load_profile(args.profile), args.profile)
    rate = (args.rate if args.rate is not None else DEFAULT_RATE) * world
    cfg = configs.config2(profile=prof, arrival_rate=rate, num_requests=6000)
    return cfg, prof, prof_src, rate


def _spawn_ranks(args) -> int:
    """--gpus N > 1 outside torchrun: re-launch this script as N ranks (torch.distributed.run, one
    process per GPU, rendezvous on 127.0.0.1); rank 0 prints the JSON line."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve())] + sys.argv[1:]
    return subprocess.call(cmd)


# ----------------------------------------------------------------------------- our arm
def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2503_13737_b200 import tp as TP
    from paper_2503_13737_b200 import workload
    from paper_2503_13737_b200.cost_model import ModelProfile, forward_bytes, forward_flops
    from paper_2503_13737_b200.engine import Engine
    from paper_2503_13737_b200.executor import CudaExecutor
    from paper_2503_13737_b200.policies import PolicyConfig

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    n_dev = torch.cuda.device_count()
    if args.tp_backend == "nccl" and world > n_dev:
        raise SystemExit(f"--gpus {world} needs {world} GPUs (found {n_dev}); --tp-backend host shares one")
    torch.cuda.set_device(local % n_dev)
    group = None
    if world > 1:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        group = dist.group.WORLD
    cfg, prof, prof_src, rate = build_workload(args, world)
    mcfg = cfg.model
    kv_tok_bytes = mcfg.kv_bytes_per_token(tp=world)
    shared = args.tp_backend == "host" and world > n_dev
    if args.kv_gb is None:  # size the paged pool for the 180 GB part: free HBM - weights - reserve
        if world > 1:
            dist.barrier()  # every rank measures before any rank allocates
        free_b = torch.cuda.mem_get_info()[0]
        ranks_here = -(-world // n_dev) if shared else 1
        args.kv_gb = max(1.0, (free_b - 2.0 * mcfg.param_count() / world * ranks_here - 12e9) / ranks_here / 1e9)
    num_blocks = int(args.kv_gb * 1e9 // (32 * kv_tok_bytes))
    if world > 1:  # one pool geometry for all ranks: rank 0's block ids index every rank's pool
        nb = torch.tensor([num_blocks], dtype=torch.int64)
        dist.all_reduce(nb, op=dist.ReduceOp.MIN)
        num_blocks = int(nb.item())
    prof = ModelProfile(**{**prof.__dict__, "kvc_capacity_tokens": num_blocks * 32})
    host_coll = TP.HostCollective(group, world) if world > 1 and args.tp_backend == "host" else None
    uid = TP.share_nccl_id(rank, group) if world > 1 and host_coll is None else None
    s_pf = prof.pivot_forward_size
    ex = CudaExecutor(mcfg, num_blocks, max_tokens=s_pf, max_seqs=2048,
                      max_blocks_per_seq=(mcfg.pos_rows + 31) // 32, tp_rank=rank, tp_size=world, seed=0,
                      init="opt", nccl_uid=uid, host_collective=host_coll)
    # preemption swaps: staging ring in HBM + host chunks pinned now rather than on the serving path
    import psutil
    # (a fresh 0.5 GB pinned chunk on the serving path costs ~0.1 s of host time; r2end ran out of a
    # 48 GB pool at 4 req/s)
    host_avail_gb = psutil.virtual_memory().available / 1e9
    # (half of the available RAM, 105 GB, stopped pinning at ~78 GB on the B200 box: the rest of the
    # chunks fell back to pageable memory and synchronous copies, profiles/r2/rate_sweep.md)
    pinned_pool_gb = min(96.0, 0.4 * host_avail_gb / max(1, world))
    ex.prepare_swap(pinned_pool_gb)
    torch.cuda.synchronize()
    free_after_setup = torch.cuda.mem_get_info()[0]

    if rank != 0:
        # followers: mirror rank 0's steps; report own device time for the max-over-ranks
        ex.set_profiling(False)
        dev = {"t": 0.0, "on": False}  # device time of the timed steps only (leader marks 1 / 0)
        inner = ex.execute

        def timed_exec(b):
            r = inner(b)
            if dev["on"]:
                dev["t"] += r.device_s
            return r

        def on_mark(tag):  # timed-region bracket: device sync + barrier with rank 0
            torch.cuda.synchronize()
            dist.barrier()
            dev["on"] = tag == 1
        ex.execute = timed_exec
        TP.follower_loop(ex, group, on_mark)
        t = torch.tensor([dev["t"]], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.barrier()
        return

    trace = workload.generate_trace(cfg.trace)
    executor = TP.TPLeader(ex, group) if world > 1 else ex
    pipeline = world == 1 and not args.no_pipeline  # TP followers mirror synchronous steps
    pcfg = PolicyConfig(policy=args.policy) if args.spec_policy else PolicyConfig(
        policy=args.policy, kv_watermark=args.kv_watermark, retain_tg=True, budget_live_only=True)
    eng = Engine(trace, prof, pcfg, executor, clock="wall", kv_blocks=num_blocks, pipeline=pipeline)

    def serve_until(t_end):
        its = []
        while eng.clock < t_end:
            if eng.done():
                raise SystemExit("trace exhausted before the timed region ended; raise num_requests")
            it = eng.step()
            if it is not None:
                its.append(it)
        return its

    # untimed ramp to steady state, then W warm-up windows
    ramp_s = DEFAULT_RAMP_S if args.ramp_s is None else args.ramp_s
    t_ramp = time.perf_counter()
    serve_until(ramp_s)
    ramp_wall = time.perf_counter() - t_ramp
    serve_until(eng.clock + args.warmup * args.window_s)
    live0 = len(eng.queue)
    kv0 = eng.pool.allocated_tokens / (num_blocks * 32)

    # ---------------- timed region: exactly K windows of serving
    batches = []
    orig_exec, orig_submit = ex.execute, getattr(ex, "submit", None)

    def recording_exec(b):
        batches.append(b)
        return orig_exec(b)

    def recording_submit(b, feed=None):
        batches.append(b)
        return orig_submit(b, feed)
    ex.execute = recording_exec
    if orig_submit is not None:
        ex.submit = recording_submit
    peaks = load_peaks()
    ex.set_roofline_peaks(peaks["tensor_sustained"], peaks["hbm"])
    ex.set_profiling(False)  # the timed windows run un-instrumented; kernel classes come from a replay
    launches0, h2d0, d2h0 = ex.launches, ex.h2d_bytes, ex.d2h_bytes
    plan0, swap0 = eng.plan_host_s, getattr(ex, "swap_host_s", 0.0)
    sec0 = dict(getattr(ex, "swap_section_s", {}))
    sampler = ClockSampler(local % n_dev)
    sampler.start()
    torch.cuda.synchronize()
    if world > 1:
        executor.mark(1)  # followers synchronise, join the barrier and start counting device time
        dist.barrier()
    ncu_window = os.environ.get("AG_NCU_TIMED") == "1"  # ncu --profile-from-start off: timed steps only
    if ncu_window:
        torch.cuda.cudart().cudaProfilerStart()
    t0 = time.perf_counter()
    windows, win_wall = [], []
    for k in range(args.steps):
        tw = time.perf_counter()
        c0 = eng.clock
        windows.append(serve_until(eng.clock + args.window_s))
        win_wall.append(time.perf_counter() - tw)
        if os.environ.get("AG_BENCH_TRACE"):
            print(f"window {k}: clock {c0:.2f} -> {eng.clock:.2f}, {len(windows[-1])} forwards, "
                  f"wall {win_wall[-1]:.2f} s, queue {len(eng.queue)}", file=sys.stderr, flush=True)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    if ncu_window:
        torch.cuda.cudart().cudaProfilerStop()
    clocks = sampler.stop()
    if world > 1:
        executor.mark(0)
        dist.barrier()
    ex.execute = orig_exec
    if orig_submit is not None:
        ex.submit = orig_submit
    plan_s, swap_s = eng.plan_host_s - plan0, getattr(ex, "swap_host_s", 0.0) - swap0
    sec_win = {k: v - sec0.get(k, 0.0) for k, v in getattr(ex, "swap_section_s", {}).items()}
    recs = [it for w in windows for it in w]
    if not recs:
        raise SystemExit(f"no forward completed in the {args.steps} timed windows (engine clock {eng.clock:.1f} s, "
                         f"queue {len(eng.queue)}, in flight {eng._inflight is not None})")
    dev_s = sum(r.device_s for r in recs)
    launches_timed = ex.launches - launches0
    h2d_timed, d2h_timed = ex.h2d_bytes - h2d0, ex.d2h_bytes - d2h0

    # ---------------- untimed: serve on until every prompt chunked inside the windows has emitted its
    # first token, so each chunk's tokens are credited iff the prompt met TTFT
    pending = {rid for it in recs for rid, _ in it.pending_prefill}
    t_res = eng.clock
    while any(eng.prefill_met(r) is None for r in pending) and not eng.done() and eng.clock < t_res + 120:
        eng.step()
    eng.flush()
    unresolved = sum(eng.prefill_met(r) is None for r in pending)

    def credited(it):
        return it.slo_tokens + sum(n for rid, n in it.pending_prefill if eng.prefill_met(rid))
    win_tokens = [sum(credited(it) for it in w) for w in windows]
    win_dev = [sum(it.device_s for it in w) for w in windows]

    # per-kernel-class CUDA events (roofline, shares): replay the timed batches (at most 400, evenly
    # spaced) with every launch bracketed by events, so the events never perturb the timed windows
    replay = batches if len(batches) <= 400 else [batches[int(i * len(batches) / 400)] for i in range(400)]
    ex.set_profiling(True)
    for b in replay:
        executor.execute(b)
    torch.cuda.synchronize()
    prof_k = ex.profile()
    ex.set_profiling(False)
    pivot = pivot_forward(executor, mcfg, s_pf, num_blocks, world, peaks)  # before the followers stop
    if world > 1:
        executor.stop()
        t = torch.tensor([dev_s], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dev_s = float(t.item())
        dist.barrier()

    slo_tokens = sum(win_tokens)
    tokens = sum(r.forward_size for r in recs)
    events = sum(r.events for r in recs)
    met = sum(r.events_met for r in recs)
    K = args.steps
    H, F, L, V = mcfg.hidden, mcfg.ffn, mcfg.num_layers, mcfg.vocab
    flops = sum(forward_flops(b.seq_shapes(), len(b.logit_rows), H, F, L, V, world) for b in batches)
    hbm_bytes = sum(forward_bytes(b.seq_shapes(), H, F, L, V, world) for b in batches)
    # per forward: max(FLOPs / tensor peak, compulsory bytes / HBM peak), summed -- the time the step
    # would take at the roofline (weights + K/V read once)
    roof_s = sum(max(forward_flops(b.seq_shapes(), len(b.logit_rows), H, F, L, V, world) / (peaks["tensor_sustained"] * 1e12),
                     forward_bytes(b.seq_shapes(), H, F, L, V, world) / (peaks["hbm"] * 1e9)) for b in batches)
    gemm_cls = ("qkv_gemm", "out_gemm", "fc1_gemm", "fc2_gemm", "lmhead_gemm")
    g_ms = sum(prof_k[c]["ms"] for c in gemm_cls)
    g_fl = sum(prof_k[c]["flops"] for c in gemm_cls)
    g_n = sum(prof_k[c]["launches"] for c in gemm_cls)
    g_roof = sum(prof_k[c]["roofline_ms"] for c in gemm_cls)
    achieved = g_fl / (g_ms / 1e3) / 1e12 if g_ms > 0 else 0.0
    prof_total_ms = sum(v["ms"] for v in prof_k.values())
    shares = {k: round(v["ms"] / prof_total_ms, 4) for k, v in prof_k.items() if prof_total_ms > 0 and v["ms"] > 0}
    attn = prof_k["attention"]
    # roofline of each hot kernel class from its live CUDA-event times (per-launch averages):
    # GEMMs against the sustained bf16 tensor peak (algorithmic 2*M*N*K), attention against HBM
    # (algorithmic K/V + q + out bytes); `roofline` = the class with the largest share
    a_n = attn["launches"]
    roof_all = {
        "gemm": {"bound": "tensor", "kernel": "tcgen05 GEMM (QKV/out/FC1/FC2/LM head)", "achieved": achieved,
                 "peak": peaks["tensor_sustained"], "unit": "TFLOP/s",
                 "frac": achieved / peaks["tensor_sustained"] if achieved else None,
                 # per launch max(FLOPs/tensor peak, weight+activation bytes/HBM peak): small-M
                 # launches are weight-streaming bound, so this is the fraction of each launch's own roofline
                 "frac_of_per_launch_roofline": g_roof / g_ms if g_ms else None,
                 "peak_source": peaks["source"] + " bf16 sustained", "traffic": None, "launches": g_n,
                 "share": g_ms / prof_total_ms if prof_total_ms else None,
                 "per_launch_ms": g_ms / g_n if g_n else None, "per_launch_flops": g_fl / g_n if g_n else None},
        "attention": {"bound": "hbm", "kernel": "mixed paged attention (tcgen05 tiles + streaming decode rows)",
                      "frac_of_per_launch_roofline": attn["roofline_ms"] / attn["ms"] if attn["ms"] else None,
                      "achieved": attn["bytes"] / (attn["ms"] / 1e3) / 1e9 if attn["ms"] else 0.0,
                      "peak": peaks["hbm"], "unit": "GB/s",
                      "frac": (attn["bytes"] / (attn["ms"] / 1e3) / 1e9 / peaks["hbm"]) if attn["ms"] else None,
                      "peak_source": peaks["source"] + " HBM copy", "traffic": None, "launches": a_n,
                      "share": attn["ms"] / prof_total_ms if prof_total_ms else None,
                      "per_launch_ms": attn["ms"] / a_n if a_n else None,
                      "per_launch_bytes": attn["bytes"] / a_n if a_n else None,
                      "tflops": attn["flops"] / (attn["ms"] / 1e3) / 1e12 if attn["ms"] else 0.0},
    }
    # traffic: DRAM bytes per launch implied by the ncu capture's DRAM / algorithmic ratio (null without it)
    tf = ROOT / "profiles" / "ncu_traffic.json"
    if tf.exists():
        nt = json.loads(tf.read_text())
        g_by = sum(prof_k[c]["bytes"] for c in gemm_cls)
        for cls, per in (("attention", roof_all["attention"].get("per_launch_bytes")),
                         ("gemm", g_by / g_n if g_n else None)):
            if cls in nt and per:
                ratio = nt[cls]["dram_bytes"] / nt[cls]["algorithmic_bytes"]
                roof_all[cls]["traffic"] = per * ratio
                roof_all[cls]["traffic_source"] = f"ncu dram/algorithmic = {ratio:.3f} ({nt[cls]['case']})"
    roof_dominant = max(roof_all.values(), key=lambda r: r["share"] or 0.0)
    win_rates = [t / d for t, d in zip(win_tokens, win_dev) if d > 0]
    line = {
        "metric": METRIC,
        "value": slo_tokens / dev_s if dev_s > 0 else 0.0,
        "unit": UNIT,
        "n_gpus": world,
        "steps": K,
        "warmup": args.warmup,
        "ms_per_step": dev_s / K * 1e3,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic (BASELINE config-2 trace generator, random-init OPT-13B-shaped bf16 weights)",
        "config": {"workload": "config2: OPT-13B mixed trace (90% <=1k, 10% 4k-16k prompts), "
                               f"{args.policy} policy, steady state",
                   "model": mcfg.name, "parallelism": f"tp{world}", "tp_backend": args.tp_backend if world > 1 else None,
                   "arrival_rate_rps": rate, "profile": prof_src, "pivot_forward_size": s_pf,
                   "kv_pool_tokens": num_blocks * 32, "step": f"{args.window_s:g} s window of serving",
                   "ramp_s": ramp_s, "forward_tokens_per_step": tokens / K,
                   "l2": "inputs larger than L2 (26 GB of weights + K/V per forward)", "clock": "wall (live)",
                   "pipelined_host": pipeline,
                   "policy_refinements": None if args.spec_policy else
                   {"kv_watermark": args.kv_watermark, "retain_tg": True, "budget_live_only": True}},
        "iter_slo_attainment": met / events if events else None,
        "steady_state": {"ramp_wall_s": ramp_wall, "live_requests": live0, "kv_occupancy": kv0,
                         "forwards_per_window": len(recs) / K,
                         "window_value_cv": float(np.std(win_rates) / np.mean(win_rates)) if win_rates else None,
                         "prompts_credit_unresolved": unresolved},
        "preemptions_in_window": sum(r.preemptions for r in recs),
        "swap_gb_total": getattr(ex, "swap_bytes", 0) / 1e9,
        "swap_host": {"blocked_s_total": getattr(ex, "swap_wait_s", 0.0), "blocked_waits": getattr(ex, "swap_waits", 0),
                      "pageable": bool(getattr(ex, "_pin_failed", False)),
                      "host_chunks": getattr(ex, "swap_host_chunks", 0),
                      "pinned_pool_gb": round(pinned_pool_gb, 1), "host_avail_gb_at_setup": round(host_avail_gb, 1),
                      # host seconds per swap-path section inside the timed windows
                      "section_s": {k: round(v, 3) for k, v in sec_win.items()}},
        "hbm_gb": {"kv_pool": num_blocks * 32 * kv_tok_bytes / 1e9, "free_after_setup": free_after_setup / 1e9,
                   "free_at_end": torch.cuda.mem_get_info()[0] / 1e9},
        "decode_tokens_per_step": sum(r.num_decode for r in recs) / K,
        "forward_size_pct": {q: int(np.percentile([r.forward_size for r in recs], q)) for q in (10, 50, 90, 99)},
        "token_events": events,
        "forward_tokens_per_s": tokens / dev_s if dev_s > 0 else 0.0,
        "e2e": {"value": slo_tokens / wall if wall > 0 else 0.0, "unit": UNIT,
                "h2d_bytes_per_step": h2d_timed / K, "d2h_bytes_per_step": d2h_timed / K},
        "gpu_launches": launches_timed,
        "roofline": roof_dominant,
        "roofline_by_kernel": roof_all,
        "forward_roofline": {"roofline_time_frac": roof_s / dev_s if dev_s else None,
                             "achieved_hbm_gbs": hbm_bytes / dev_s / 1e9 if dev_s else 0.0,
                             "hbm_frac": hbm_bytes / dev_s / 1e9 / peaks["hbm"] if dev_s else None,
                             "achieved_tflops": flops / dev_s / 1e12 if dev_s else 0.0,
                             "frac_of_sustained": flops / dev_s / 1e12 / peaks["tensor_sustained"] if dev_s else None},
        "attention": {"ms": attn["ms"], "tflops": attn["flops"] / (attn["ms"] / 1e3) / 1e12 if attn["ms"] else 0.0,
                      "gbs": attn["bytes"] / (attn["ms"] / 1e3) / 1e9 if attn["ms"] else 0.0},
        "kernel_share": shares,
        "host_ms_per_step": {"pre": 1e3 * sum(r.host_pre_s for r in recs) / K,
                             "execute_wall": 1e3 * sum(r.wall_s for r in recs) / K,
                             "post": 1e3 * sum(r.host_post_s for r in recs) / K,
                             "device_forward": 1e3 * dev_s / K, "wall_total": 1e3 * wall / K,
                             "pre_plan": 1e3 * plan_s / K, "pre_swap": 1e3 * swap_s / K,
                             # pipelined host: a step whose host work outlasts the forward it overlaps idles the GPU
                             "pre_over_device_ms": 1e3 * sum(max(0.0, r.host_pre_s - r.device_s) for r in recs) / K,
                             "steps_pre_over_device": sum(r.host_pre_s > r.device_s for r in recs) / K},
        "clocks": clocks,
        "gemm_plans": " ".join(f"{k}:{mb}:{bn}x{ks}a{am}" for k, mb, bn, ks, am in ex.gemm_plans()),
    }
    line["pivot_forward"] = pivot
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(mcfg, batches, world)
    print(json.dumps(line), flush=True)


def pivot_forward(executor, mcfg, s_pf, num_blocks, world, peaks, reps=7) -> dict:
    """The pivot-sized mixed forward AccelGen packs to (S_f = S_pf: one prompt chunk of S_pf - 16 tokens
    on a 4096-token prefix + 16 decodes over 300-4000-token contexts), timed after serving has ended
    (its block ids overwrite pool contents nobody reads any more): the forward's tensor-pipe
    efficiency at the design point, which the decode-bound steps of the timed windows never reach."""
    import numpy as np
    from paper_2503_13737_b200.cost_model import forward_flops
    from paper_2503_13737_b200.engine import DeviceBatch, synthetic_tokens
    rng = np.random.default_rng(0)
    segs = [(4096, s_pf - 16)] + [(int(c), 1) for c in rng.integers(300, 4000, 16)]
    ids, pos, slot, cu, ctx, tabs, nb = [], [], [], [0], [], [], 0
    for i, (c, n) in enumerate(segs):
        tab = np.arange(nb, nb + (c + n + 31) // 32, dtype=np.int32)
        nb += len(tab)
        p = np.arange(c, c + n, dtype=np.int32)
        ids.append(synthetic_tokens(i, p, mcfg.vocab).astype(np.int32)), pos.append(p)
        slot.append((tab[p // 32] * 32 + p % 32).astype(np.int32)), ctx.append(c), cu.append(cu[-1] + n)
        tabs.append(tab)
    if nb > num_blocks:
        return {"skipped": f"needs {nb} KV blocks, pool has {num_blocks}"}
    bt = np.zeros((len(tabs), max(map(len, tabs))), np.int32)
    for i, t in enumerate(tabs):
        bt[i, :len(t)] = t
    rids = list(range(len(segs)))
    b = DeviceBatch(rids, np.concatenate(ids), np.concatenate(pos), np.asarray(cu, np.int32), np.asarray(ctx, np.int32),
                    bt, np.concatenate(slot), np.asarray(cu[1:], np.int32) - 1, rids)
    for _ in range(2):
        executor.execute(b)
    t = sorted(executor.execute(b).device_s for _ in range(reps))[reps // 2]
    fl = forward_flops(b.seq_shapes(), len(b.logit_rows), mcfg.hidden, mcfg.ffn, mcfg.num_layers, mcfg.vocab, world)
    return {"batch": f"{s_pf - 16}-token chunk on a 4096-token prefix + 16 decodes (S_f={s_pf})", "ms": t * 1e3,
            "tflops": fl / t / 1e12, "frac_of_sustained": fl / t / 1e12 / peaks["tensor_sustained"],
            "peak_source": peaks["source"] + " bf16 sustained"}


def _median_batch(batches):
    return sorted(batches, key=lambda b: b.num_tokens)[len(batches) // 2]


def cpu_baseline(mcfg, batches, world, budget_s: float = 20.0) -> dict:
    """The CPU oracle (the reference's path restated; oracle/) on a bounded sample: one OPT-13B
    layer on the median timed batch, scaled to L layers + LM head."""
    from oracle.bench_cpu import time_forward_sample
    b = _median_batch(batches)
    r = time_forward_sample(mcfg, b, budget_s=budget_s)
    return {"value": r["tokens_per_s"], "unit": "tokens/s (forward; upper bound of SLO-meeting tokens/s)",
            "cores": r["threads"], "kind": "port",
            "sample": f"1 of {mcfg.num_layers} OPT-13B layers on the median timed batch (S_f={b.num_tokens}, "
                      f"{len(b.cu_q) - 1} seqs), x{mcfg.num_layers} + LM head; {r['seconds']:.1f}s of CPU"}


# ----------------------------------------------------------------------------- reference arm
def run_reference(args):
    """The reference's CPU implementation of the path (oracle port) on the host cores, measured the
    same way: SLO-meeting tokens per window of its own (CPU-timed) clock."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle.bench_cpu import reference_arm
    cfg, prof, prof_src, rate = build_workload(args, world)
    res = reference_arm(cfg, prof, steps=args.steps, warmup=args.warmup, window_s=args.window_s)
    line = {
        "metric": METRIC, "value": res["value"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": res["ms_per_step"], "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (same trace generator and shapes)",
        "config": {"workload": f"config2: OPT-13B mixed trace, {args.policy} policy (oracle restatement)",
                   "model": cfg.model.name, "parallelism": "cpu", "arrival_rate_rps": rate, "profile": prof_src,
                   "step": f"{args.window_s:g} s window of serving (CPU-timed clock)"},
        "impl": "reference",
        "forward_tokens_per_s": res["forward_tokens_per_s"],
        "note": "SLO-meeting tokens/s is 0 on the CPU path: a forward takes tens of seconds, every TTFT/TBT "
                "deadline (<= 0.6 s) is missed; forward_tokens_per_s is its raw forward throughput",
        "cpu_baseline": {"value": res["value"], "unit": UNIT, "cores": res["threads"], "kind": "port",
                         "sample": res["sample"]},
        "e2e": {"value": res["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(_spawn_ranks(args))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
