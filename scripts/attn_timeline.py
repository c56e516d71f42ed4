"""Per-CTA timeline of the attention tile path (build with NVCC_EXTRA=-DAG_ATTN_TIMELINE).

Runs one case of scripts/attn_bench.py, then reads the globaltimer stamps of every tile CTA and
prints: setup / loop / epilogue durations, per-tile loop time, and gaps between consecutive CTAs on
one SM (launch + teardown cost)."""
import ctypes
import statistics as st
import sys

import torch

case = sys.argv[1] if len(sys.argv) > 1 else "chunk2048_on_8k"
sys.argv = sys.argv[:1]  # attn_bench reads argv at import
sys.path.insert(0, ".")
sys.path.insert(0, "scripts")
import attn_bench  # noqa: E402
from paper_2503_13737_b200 import _lib  # noqa: E402

seqs = attn_bench.CASES[case]
r = attn_bench.run(seqs, 40)
lib = _lib.load()
fn = lib.ag_debug_attn_timeline
n = 16384
buf = (ctypes.c_ulonglong * (16 * n))()
torch.cuda.synchronize()
assert fn(ctypes.cast(buf, ctypes.c_void_p), n) == 0
rows = [tuple(buf[16 * i:16 * i + 16]) for i in range(n)]
rows = [x for x in rows if x[0] and x[3] >= x[0]]
t0 = min(x[0] for x in rows)
last = max(x[3] for x in rows)
setup = [(x[1] - x[0]) / 1e3 for x in rows]
loop = [(x[2] - x[1]) / 1e3 for x in rows]
epi = [(x[3] - x[2]) / 1e3 for x in rows]
per_tile = [(x[2] - x[1]) / 1e3 / x[4] for x in rows if x[4] > 0]
by_sm = {}
for x in rows:
    by_sm.setdefault(x[5], []).append(x)
gaps = []
for sm, xs in by_sm.items():
    xs.sort()
    gaps += [(b[0] - a[3]) / 1e3 for a, b in zip(xs, xs[1:])]
starts = sorted((x[0] - t0) / 1e3 for x in rows)
q = lambda v: f"med {st.median(v):.2f} min {min(v):.2f} max {max(v):.2f}"  # noqa: E731
print(f"case {case}: kernel-timed {r['us']} us; tile CTAs {len(rows)} on {len(by_sm)} SMs; span {(last - t0) / 1e3:.1f} us")
print("setup us", q(setup))
print("loop us", q(loop))
print("epilogue us", q(epi))
print("per-tile us", q(per_tile), "tiles/CTA", q([x[4] for x in rows]))
if gaps:
    print("gap between CTAs on an SM us", q(gaps))
print("first-wave start spread us", f"{starts[min(len(starts) - 1, 147)]:.2f}")
tiles = sum(x[4] for x in rows)
names = {6: "softmax wait S", 7: "softmax load S", 8: "softmax max/rescale", 9: "softmax exp/store P",
         10: "mma wait P", 11: "mma wait K/V", 12: "mma wait S-empty", 13: "producer wait stage"}
for k, nm in names.items():
    print(f"{nm:22s} {sum(x[k] for x in rows) / max(tiles, 1):8.0f} cycles/tile")
