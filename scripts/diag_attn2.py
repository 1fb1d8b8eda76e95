"""Per-group attention split/merge timing of one layer (fused merge; timing experiment)."""
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_13327_b200.decode import CONFIGS, DecodeModel  # noqa: E402

m = DecodeModel(CONFIGS["llama3-8b"], samples=(1024,), record_trace=True)
m.fill_cache(1024)
m.set_token(1)
for _ in range(3):
    m.executor.run({"s": 1024})
t = m.executor.trace()
calls = m.graph.call_functions
c = calls.index("L1.attn")
rs = [r for r in t.records if r["call"] == c]
base = min(r["exec"][0] for r in rs)
by = collections.defaultdict(list)
for r in rs:
    by[r["coord"][0]].append(r)
for g in sorted(by):
    ends = sorted((r["exec"][1] - base) / 1e3 for r in by[g])
    starts = sorted((r["exec"][0] - base) / 1e3 for r in by[g])
    ex = sorted((r["exec"][1] - r["exec"][0]) / 1e3 for r in by[g])
    print(f"group {g}: start {starts[0]:.2f}..{starts[-1]:.2f}  end {ends[0]:.2f} med {ends[len(ends)//2]:.2f} "
          f"2nd-last {ends[-2]:.2f} last {ends[-1]:.2f}  exec med {ex[len(ex)//2]:.2f} max {ex[-1]:.2f}")
