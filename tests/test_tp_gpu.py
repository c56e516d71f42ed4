"""Tensor-parallel CUDA forward on the B200: TP=2/4/8 shards of an OPT-13B-shaped model vs the
UNSHARDED oracle (BASELINE configs 3-5).

The ranks are processes sharing the one GPU this suite gets; collectives go through the library's
host backend (ag_model_init_tp_host, gloo), everything else is the production sharded path:
QKV / FC1 column shards by heads / FFN, out-proj / FC2 row shards with the bf16 partial sums
all-reduced and bias + residual + LayerNorm applied after the reduce, the vocab-parallel LM head
(TP=8: 6284-column shards of OPT's 50272, padded to 32 columns on the device) and the merge of the
per-rank (max, index) candidates.  Tolerance as tests/test_forward_gpu.py (tests/parity.py): max|dlogit|
<= 2e-2 or 1.5x the oracle's own fp32-vs-fp64 noise floor, >= 99% identical greedy tokens.  The oracle
mirrors the TP=t rounding points (tp_emulate: bf16 per-shard partials of out-proj / FC2, one bf16 rounding
after the fp32 reduce) on the unsharded weights."""
import socket
import subprocess
import sys
from pathlib import Path

import pytest
import torch

pytestmark = pytest.mark.gpu

HERE = Path(__file__).resolve().parent


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("tp,name", [(2, "13b2l"), (4, "13b2l"), (8, "13b2l"), (8, "175b2l"), (8, "13b100k")])
def test_tp_sharded_forward_vs_unsharded_oracle(tp, name, tmp_path):
    """13b2l: OPT-13B shape (config 3); 175b2l: OPT-175B shape at TP=8 (config 5, 12 heads per rank);
    13b100k: a 100k-token prompt in 12.5k-token chunks, then a decode over it, at TP=8 (config 4, 5 heads
    per rank; the long prefill chunks build the KV cache, the last chunk and the decode are compared)."""
    sys.path.insert(0, str(HERE))
    from batches import make_batch
    from tp_gpu_worker import case, checked_steps
    from oracle.executor import OracleExecutor
    from parity import Tally
    from paper_2503_13737_b200 import model as M
    from paper_2503_13737_b200.kvc import BlockPool

    # the workers share this GPU: hand back what earlier tests in this process left in torch's cache
    import gc
    gc.collect()
    torch.cuda.empty_cache()
    port = _free_port()
    procs = [subprocess.Popen([sys.executable, str(HERE / "tp_gpu_worker.py"), "--rank", str(r), "--world", str(tp),
                               "--port", str(port), "--case", name, "--out", str(tmp_path / f"rank{r}.pt")])
             for r in range(tp)]
    try:
        codes = [p.wait(timeout=900) for p in procs]
    finally:
        for p in procs:
            if p.poll() is None:
                p.kill()
    assert codes == [0] * tp, f"worker exit codes {codes}"
    ranks = [torch.load(tmp_path / f"rank{r}.pt") for r in range(tp)]

    cfg, seed, blocks, steps = case(name)
    check = checked_steps(name)
    w = M.init_weights(cfg, seed, device="cuda", init="test")  # the same global model, unsharded
    # unsharded weights, TP=tp rounding points (bf16 partials, one rounding after the reduce)
    ref = OracleExecutor(cfg, w, blocks, device="cuda", tp_emulate=tp)
    ref64 = OracleExecutor(cfg, w, blocks, device="cuda", acc=torch.float64, tp_emulate=tp)
    pool = BlockPool(blocks)
    tally = Tally()
    for i, segs in enumerate(steps):
        b = make_batch(pool, cfg, segs)
        r, r64 = ref.execute(b), ref64.execute(b)
        if i not in check:
            continue
        n = r.logits.shape[0]
        full = torch.cat([rk["res"][i]["logits"][:n] for rk in ranks], dim=1)  # vocab shards in rank order
        assert full.shape == r.logits.shape
        toks = [rk["res"][i]["tokens"][:n] for rk in ranks]
        for t in toks[1:]:
            assert torch.equal(t, toks[0]), "ranks disagree on the merged argmax"
        tally.add(full, toks[0].numpy(), r.logits, r.token_ids, r64.logits)
    calls = ranks[0]["collective_calls"]
    assert calls == len(steps) * (2 * cfg.num_layers + 2)  # 2 all-reduces per layer + 2 argmax all-gathers
    tally.check(f"TP={tp} {name} sharded CUDA forward vs unsharded oracle ({calls} host collectives per rank)")
