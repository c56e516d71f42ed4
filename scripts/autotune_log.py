"""Print the autotuner's best time per (GEMM kind, M bucket) for OPT-13B at TP=1 against the
per-launch roofline max(2MNK / tensor peak, 2(NK + MK + MN) / HBM peak).
  AG_AUTOTUNE_LOG=1 python scripts/autotune_log.py 2> gpurun_out/autotune.log"""
import json
import os
import subprocess
import sys

if os.environ.get("AG_AUTOTUNE_LOG") is None:
    env = dict(os.environ, AG_AUTOTUNE_LOG="1")
    r = subprocess.run([sys.executable, __file__], env=env, capture_output=True, text=True)
    peaks = json.load(open("MEASURED_PEAKS.json")) if os.path.exists("MEASURED_PEAKS.json") else {}
    hbm = 6542.4e9
    ten = 1368.2e12
    kinds = ("qkv", "out", "fc1", "fc2", "lm_head")
    tot_us = tot_roof = 0.0
    for line in r.stderr.splitlines():
        if not line.startswith('{"autotune"'):
            continue
        d = json.loads(line)
        M, N, K = d["M"], d["N"], d["K"]
        roof = max(2.0 * M * N * K / ten, 2.0 * (N * K + M * K + M * N) / hbm) * 1e6
        print(f"{kinds[d['autotune']]:8s} M={M:5d} {d['us']:8.1f} us  roof {roof:7.1f}  frac {roof / d['us']:.2f}  "
              f"plan {d['bn']}x{d['ks']}a{d['am']}")
    sys.exit(r.returncode)

import torch  # noqa: E402

sys.path.insert(0, ".")
from paper_2503_13737_b200 import model as Mo  # noqa: E402
from paper_2503_13737_b200.executor import CudaExecutor  # noqa: E402

cfg = Mo.opt_13b(max_positions=4096)
ex = CudaExecutor(cfg, 4096, max_tokens=1536, max_seqs=256)
torch.cuda.synchronize()
