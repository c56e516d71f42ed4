"""Helper for tests/test_pdl_gpu.py: one mixed forward (prefill chunk on a prefix + fresh prompt +
decodes) of a 2-layer OPT-shaped model; writes the parity logits to argv[1] (.npy).  The
environment (AG_PDL, AG_DETERMINISTIC, AG_GEMM_PLAN_CACHE) is set by the caller."""
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from paper_2503_13737_b200 import model as M  # noqa: E402
from paper_2503_13737_b200.executor import CudaExecutor  # noqa: E402
from paper_2503_13737_b200.kvc import BlockPool  # noqa: E402
from test_forward_gpu import _make_batch  # noqa: E402

cfg = M.OPTConfig("opt-2k-2l", hidden=2048, num_layers=2, num_heads=16, ffn=8192, max_positions=4096)
w = M.init_weights(cfg, seed=5, init="test")
pool = BlockPool(2048)
dev = CudaExecutor(cfg, pool.total_blocks, max_tokens=4096, max_seqs=64, weights=w, parity_logits=True)
decodes = [(2 + i, 40 + 13 * i) for i in range(16)]
dev.execute(_make_batch(pool, cfg, [(0, 0, 1200)]))
dev.execute(_make_batch(pool, cfg, [(rid, 0, p) for rid, p in decodes]))
res = dev.execute(_make_batch(pool, cfg, [(0, 1200, 700), (1, 0, 260)] + [(rid, p, 1) for rid, p in decodes]))
np.save(sys.argv[1], res.logits.float().cpu().numpy())
