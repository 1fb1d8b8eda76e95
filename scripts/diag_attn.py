"""Attention stage timing with phases switched off (ET_DEBUG bits; timing experiment only)."""
import collections
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_13327_b200.decode import CONFIGS, DecodeModel  # noqa: E402

cfg = CONFIGS["llama3-8b"]
m = DecodeModel(cfg, samples=(1024,), record_trace=True)
m.fill_cache(1024)
m.set_token(1)
calls = m.graph.call_functions
for name, f in [("all", 0), ("no-scores", 128), ("no-pv", 256), ("no-merge", 512), ("no-qload", 1024),
                ("none", 128 + 256 + 512 + 1024)]:
    os.environ["ET_DEBUG"] = str(f)
    ts = [m.executor.run({"s": 1024})["kernel_ms"] for _ in range(4)]
    t = m.executor.trace()
    by = collections.defaultdict(list)
    for r in t.records:
        by[r["call"]].append(r)
    ex, span = [], []
    for c in range(len(calls)):
        if ".attn" in calls[c]:
            rs = by[c]
            ex += [r["exec"][1] - r["exec"][0] for r in rs]
            span.append(max(r["exec"][1] for r in rs) - min(r["exec"][0] for r in rs))
    ex.sort()
    print(f"{name:10s} step {statistics.median(ts[1:]):.4f} ms  attn exec med {ex[len(ex)//2]} p90 {ex[len(ex)*9//10]} "
          f"max {ex[-1]}  stage span med {statistics.median(span):.0f} ns", flush=True)
