"""The five BASELINE.json configurations as (model, trace, profile, parallelism) bundles.

Config 1 is CPU-runnable (the oracle executes every iteration); configs 2-5 are the B200 runs.
Trace recipes follow SURVEY §8d (paper settings PAPER.md:652, 758, 2081).
"""
from __future__ import annotations

from dataclasses import dataclass, replace

from . import model as M
from .cost_model import ModelProfile, opt_13b_like
from .workload import LengthDist, ScaleRule, TraceConfig


@dataclass(frozen=True)
class RunConfig:
    name: str
    model: M.OPTConfig
    trace: TraceConfig
    tp: int
    description: str


def tiny_profile(kvc_capacity_tokens: int = 65536) -> ModelProfile:
    """Declared (not measured) cost model of the tiny model: S_pf=256 tokens in 2 ms."""
    return ModelProfile(hidden_size=256, num_layers=2, pivot_forward_size=256, pivot_time_s=0.002,
                        kvc_capacity_tokens=kvc_capacity_tokens)


def config1(seed: int = 0) -> RunConfig:
    tr = TraceConfig(num_requests=64, arrival_rate=8.0, long_fraction=0.1,
                     short_len_dist=LengthDist(kind="uniform", lo=8, hi=256),
                     long_len_dist=LengthDist(kind="uniform", lo=4096, hi=8192),
                     output_len_dist=LengthDist(kind="uniform", lo=1, hi=64),
                     tbt_scale=ScaleRule(kind="choice", values=(0.5, 1.0, 2.0)), seed=seed, profile=tiny_profile())
    return RunConfig("config1-tiny", M.tiny(), tr, 1, "tiny OPT (2 layers, d=256), 64 requests, 3 SLO classes")


def config2(profile: ModelProfile | None = None, arrival_rate: float = 8.0, num_requests: int = 2000,
            seed: int = 0) -> RunConfig:
    tr = TraceConfig(num_requests=num_requests, arrival_rate=arrival_rate, long_fraction=0.10,
                     short_len_dist=LengthDist(kind="uniform", lo=10, hi=1024),
                     long_len_dist=LengthDist(kind="log_uniform", lo=4096, hi=16384),
                     output_len_dist=LengthDist(kind="uniform", lo=1, hi=2048),
                     tbt_scale=ScaleRule(kind="range", values=(0.75, 1.25)), ttft_scale_range=(0.5, 1.5),
                     seed=seed, profile=profile or opt_13b_like())
    return RunConfig("config2-opt13b", M.opt_13b(max_positions=16384 + 2048 + 64), tr, 1,
                     "OPT-13B shape, 1xB200, 90% <=1k prompts + 10% 4k-16k, heterogeneous TBT")


def config3(tp: int, **kw) -> RunConfig:
    c = config2(**kw)
    return replace(c, name=f"config3-opt13b-tp{tp}", tp=tp, description=f"config 2 at TP={tp}")


def config4(profile: ModelProfile | None = None, arrival_rate: float = 8.0, num_requests: int = 1000,
            seed: int = 0) -> RunConfig:
    tr = TraceConfig(num_requests=num_requests, arrival_rate=arrival_rate, long_fraction=0.35, seed=seed,
                     profile=profile or opt_13b_like())
    return RunConfig("config4-longctx-tp8", M.opt_13b(max_positions=100000 + 2048 + 64), tr, 8,
                     "prompts up to 100k (log-uniform 4k-100k, 35% long), OPT-13B, TP=8")


def config5(profile: ModelProfile | None = None, arrival_rate: float = 8.0, num_requests: int = 1000,
            seed: int = 0) -> RunConfig:
    tr = TraceConfig(num_requests=num_requests, arrival_rate=arrival_rate, long_fraction=0.10,
                     short_len_dist=LengthDist(kind="uniform", lo=10, hi=1024),
                     long_len_dist=LengthDist(kind="log_uniform", lo=4096, hi=16384),
                     output_len_dist=LengthDist(kind="uniform", lo=1, hi=2048),
                     tbt_scale=ScaleRule(kind="choice", values=(0.25, 0.5, 1.0, 2.0)), offline_fraction=0.2,
                     seed=seed, profile=profile or opt_13b_like())
    return RunConfig("config5-opt175b-tp8", M.opt_175b(max_positions=16384 + 2048 + 64), tr, 8,
                     "OPT-175B shape, TP=8, tight/loose TBT mix + 20% offline (JCT SLO)")
