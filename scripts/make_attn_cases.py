"""Record the (ctx_len, q_len) mix of real AccelGen batches (virtual clock, bench trace) for
scripts/attn_bench.py: python scripts/make_attn_cases.py RATE T0 N > cases.json"""
import json
import sys

sys.path.insert(0, ".")
from paper_2503_13737_b200 import configs, workload  # noqa: E402
from paper_2503_13737_b200.cost_model import load_profile  # noqa: E402
from paper_2503_13737_b200.engine import Engine  # noqa: E402
from paper_2503_13737_b200.policies import PolicyConfig  # noqa: E402

rate, t0, n = float(sys.argv[1]), float(sys.argv[2]), int(sys.argv[3])
t1 = t0 + 4.0  # sample n steps spread evenly over [t0, t0 + 4 s] of trace time
prof = load_profile("profiles/opt13b_b200_tp1.json")
cfg = configs.config2(profile=prof, arrival_rate=rate, num_requests=4000)
eng = Engine(workload.generate_trace(cfg.trace), prof, PolicyConfig(), None, clock="virtual",
             kv_blocks=186720 // 32)
eng.executor.max_tokens, eng.executor.max_seqs = prof.pivot_forward_size, 2048
eng.keep_history = True
allc = []
while eng.clock < t1:
    it = eng.step()
    if it is None or eng.clock < t0:
        continue
    plan = eng.plans[-1]
    seqs = []
    for sel in plan.selections:
        rec = eng.metrics.requests[sel.request_id]
        # tokens cached before this step = tokens of the request now in the pool minus this step's
        seqs.append((eng.pool.tokens_stored(sel.request_id) - sel.chunk_len, sel.chunk_len))
    allc.append((f"r{rate:g}_t{eng.clock:.2f}_S{plan.forward_size}", seqs))
cases = dict(allc[i * len(allc) // n] for i in range(n))
print(json.dumps(cases))
