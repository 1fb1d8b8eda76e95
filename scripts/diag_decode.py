import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2604_13327_b200.decode import CONFIGS, DecodeModel, TINY
name = sys.argv[1] if len(sys.argv) > 1 else "llama3-8b"
nw = int(sys.argv[2]) if len(sys.argv) > 2 else 0
cfg = CONFIGS[name]
m = DecodeModel(cfg, samples=(1024,), num_workers=nw or None, record_trace=True)
m.fill_cache(1024)
m.set_token(1)
for i in range(3):
    t0 = time.perf_counter()
    st = m.executor.run({"s": 1024})
    print("stats", st, "wall ms", (time.perf_counter() - t0) * 1e3)
print("logits", m.logits[0, :8], m.logits.abs().max())
print("h_a", m.h_a[0, :4], "q", m.q[:4])
t = m.executor.trace()
recs = t.records
import collections
per_call = collections.defaultdict(list)
for r in recs:
    per_call[r["call"]].append(r["exec"][1] - r["exec"][0])
fns = m.graph.call_functions
for c in list(per_call)[:8] + [len(fns) - 1]:
    v = per_call[c]
    print(fns[c], len(v), "exec ns median", sorted(v)[len(v) // 2], "max", max(v))
print("makespan ns", t.makespan)
