"""OPT decoder shapes, deterministic random-init weights and tensor-parallel sharding.

Architecture (pre-LN OPT, as in transformers ``modeling_opt.py`` OPTDecoderLayer): learned
positions with offset 2, q scaled by head_dim^-0.5, LayerNorm before attention and before the
MLP, ReLU FC1, biases everywhere, final LayerNorm, LM head tied to the token embedding.  The
paper serves OPT-13B and OPT-175B; the reference folds the model into
``hidden_size``/``num_layers`` of ModelProfile (pkg/src/slosim/cost_model.py:34-58).

Weights are generated per (layer, tensor) from a keyed seed so every rank can materialise
exactly its own shard of the same global model (no checkpoint exists offline).
"""
from __future__ import annotations

import hashlib
from dataclasses import dataclass

import torch

POS_OFFSET = 2  # OPTLearnedPositionalEmbedding offset
HEAD_DIM = 128


@dataclass(frozen=True)
class OPTConfig:
    name: str
    hidden: int
    num_layers: int
    num_heads: int
    ffn: int
    vocab: int = 50272
    max_positions: int = 2048  # positions the table covers (rows = max_positions + 2)
    ln_eps: float = 1e-5

    @property
    def head_dim(self) -> int:
        return self.hidden // self.num_heads

    @property
    def pos_rows(self) -> int:
        return self.max_positions + POS_OFFSET

    def with_positions(self, n: int) -> "OPTConfig":
        """OPT's table stops at 2048; 16k/100k-token prompts need a longer (random-init) table."""
        return OPTConfig(self.name, self.hidden, self.num_layers, self.num_heads, self.ffn, self.vocab, n, self.ln_eps)

    def param_count(self) -> int:
        H, F, L = self.hidden, self.ffn, self.num_layers
        per_layer = 4 * H * H + 2 * H * F + 4 * H + F + H + 4 * H
        return L * per_layer + self.vocab * H + self.pos_rows * H + 2 * H

    def kv_bytes_per_token(self, tp: int = 1, bytes_per_element: int = 2) -> int:
        """2 * bytes * L * H / tp  (reference kvc_bytes_per_token, cost_model.py:96-98)."""
        return 2 * bytes_per_element * self.num_layers * self.hidden // tp


def tiny() -> OPTConfig:
    """Config 1 of BASELINE.json: 2 layers, d=256, 2 heads of 128 (head_dim kept at 13B's 128)."""
    return OPTConfig("opt-tiny", hidden=256, num_layers=2, num_heads=2, ffn=1024, max_positions=16384)


def opt_13b(max_positions: int = 2048) -> OPTConfig:
    return OPTConfig("opt-13b", hidden=5120, num_layers=40, num_heads=40, ffn=20480, max_positions=max_positions)


def opt_175b(max_positions: int = 2048) -> OPTConfig:
    return OPTConfig("opt-175b", hidden=12288, num_layers=96, num_heads=96, ffn=49152, max_positions=max_positions)


PRESETS = {"opt-tiny": tiny, "opt-13b": opt_13b, "opt-175b": opt_175b}

LAYER_KEYS = ("ln1_g", "ln1_b", "qkv_w", "qkv_b", "out_w", "out_b", "ln2_g", "ln2_b", "fc1_w", "fc1_b", "fc2_w",
              "fc2_b")


def _seed(base: int, *key) -> int:
    h = hashlib.sha256(repr((base,) + key).encode()).digest()
    return int.from_bytes(h[:8], "little") & ((1 << 63) - 1)


def _randn(shape, seed: int, device, std: float) -> torch.Tensor:
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    return (torch.randn(shape, generator=g, device=device, dtype=torch.float32) * std).to(torch.bfloat16)


def _layer_full(cfg: OPTConfig, seed: int, layer: int, device, init: str) -> dict[str, torch.Tensor]:
    """Full (unsharded) layer tensors, bf16.  init="opt": N(0,.02) weights, zero biases, LN (1,0)
    (SURVEY §8d); init="test": additionally random biases and LN affine so every fused
    epilogue term is exercised by the parity tests."""
    H, F = cfg.hidden, cfg.ffn
    t = {
        "qkv_w": _randn((3 * H, H), _seed(seed, layer, "qkv_w"), device, 0.02),
        "out_w": _randn((H, H), _seed(seed, layer, "out_w"), device, 0.02),
        "fc1_w": _randn((F, H), _seed(seed, layer, "fc1_w"), device, 0.02),
        "fc2_w": _randn((H, F), _seed(seed, layer, "fc2_w"), device, 0.02),
    }
    if init == "test":
        t["qkv_b"] = _randn((3 * H,), _seed(seed, layer, "qkv_b"), device, 0.1)
        t["out_b"] = _randn((H,), _seed(seed, layer, "out_b"), device, 0.1)
        t["fc1_b"] = _randn((F,), _seed(seed, layer, "fc1_b"), device, 0.1)
        t["fc2_b"] = _randn((H,), _seed(seed, layer, "fc2_b"), device, 0.1)
        for k in ("ln1", "ln2"):
            t[k + "_g"] = (1.0 + _randn((H,), _seed(seed, layer, k + "_g"), device, 0.1).float()).to(torch.bfloat16)
            t[k + "_b"] = _randn((H,), _seed(seed, layer, k + "_b"), device, 0.1)
    else:
        for k, n in (("qkv_b", 3 * H), ("out_b", H), ("fc1_b", F), ("fc2_b", H)):
            t[k] = torch.zeros(n, device=device, dtype=torch.bfloat16)
        for k in ("ln1", "ln2"):
            t[k + "_g"] = torch.ones(H, device=device, dtype=torch.bfloat16)
            t[k + "_b"] = torch.zeros(H, device=device, dtype=torch.bfloat16)
    return t


def shard_layer(cfg: OPTConfig, full: dict[str, torch.Tensor], tp_rank: int, tp_size: int) -> dict[str, torch.Tensor]:
    """Megatron-style split: QKV/FC1 by output rows (heads / ffn), out-proj/FC2 by input columns.
    out_b/fc2_b stay whole (added once after the all-reduce)."""
    if tp_size == 1:
        return dict(full)
    H, F = cfg.hidden, cfg.ffn
    hl, fl = H // tp_size, F // tp_size
    r0 = tp_rank * hl
    q, k, v = full["qkv_w"][:H], full["qkv_w"][H:2 * H], full["qkv_w"][2 * H:]
    qb, kb, vb = full["qkv_b"][:H], full["qkv_b"][H:2 * H], full["qkv_b"][2 * H:]
    s = dict(full)
    s["qkv_w"] = torch.cat([q[r0:r0 + hl], k[r0:r0 + hl], v[r0:r0 + hl]]).contiguous()
    s["qkv_b"] = torch.cat([qb[r0:r0 + hl], kb[r0:r0 + hl], vb[r0:r0 + hl]]).contiguous()
    s["out_w"] = full["out_w"][:, r0:r0 + hl].contiguous()
    f0 = tp_rank * fl
    s["fc1_w"] = full["fc1_w"][f0:f0 + fl].contiguous()
    s["fc1_b"] = full["fc1_b"][f0:f0 + fl].contiguous()
    s["fc2_w"] = full["fc2_w"][:, f0:f0 + fl].contiguous()
    return s


def init_weights(cfg: OPTConfig, seed: int = 0, device="cpu", tp_rank: int = 0, tp_size: int = 1,
                 init: str = "opt") -> dict:
    """{"tok_emb", "pos_emb", "final_g", "final_b", "layers": [dict per layer]} for one TP rank.

    The embedding is replicated on every rank (lookup needs all rows; the LM head uses the
    rank's vocab slice of it)."""
    if cfg.head_dim != HEAD_DIM:
        raise ValueError("head_dim must be 128")
    if cfg.num_heads % tp_size or cfg.ffn % tp_size or cfg.vocab % tp_size:
        raise ValueError("tp_size must divide heads, ffn and vocab")
    w = {
        "tok_emb": _randn((cfg.vocab, cfg.hidden), _seed(seed, "tok_emb"), device, 0.02),
        "pos_emb": _randn((cfg.pos_rows, cfg.hidden), _seed(seed, "pos_emb"), device, 0.02),
    }
    if init == "test":
        w["final_g"] = (1.0 + _randn((cfg.hidden,), _seed(seed, "final_g"), device, 0.1).float()).to(torch.bfloat16)
        w["final_b"] = _randn((cfg.hidden,), _seed(seed, "final_b"), device, 0.1)
    else:
        w["final_g"] = torch.ones(cfg.hidden, device=device, dtype=torch.bfloat16)
        w["final_b"] = torch.zeros(cfg.hidden, device=device, dtype=torch.bfloat16)
    w["layers"] = [shard_layer(cfg, _layer_full(cfg, seed, l, device, init), tp_rank, tp_size)
                   for l in range(cfg.num_layers)]
    return w
