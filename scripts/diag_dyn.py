"""Dynamic-scheduler timeline of one decode layer (timing experiment): per call,
push -> pop -> wait end -> exec end spans."""
import collections
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_13327_b200.moe import MOE_CONFIGS, MoEDecodeModel  # noqa: E402

cfg = MOE_CONFIGS["qwen3-30b-a3b"]
m = MoEDecodeModel(cfg, samples=(1024,), record_trace=True, scheduler="dynamic")
m.fill_cache(1024)
m.set_token(1)
for _ in range(3):
    st = m.executor.run({"s": 1024})
print("kernel_ms", st["kernel_ms"])
raw = m.executor.raw_trace()
calls = m.graph.call_functions
t = m.executor.trace()
by = collections.defaultdict(list)
for rec, tr in zip(raw, t.records):
    by[tr["call"]].append(rec)
cs = [c for c in range(len(calls)) if calls[c].startswith("L5.")]
base = min(r[1] for c in cs for r in by[c] if r[1] > 0)
for c in cs:
    rs = [r for r in by[c] if r[1] > 0]
    if not rs:
        continue
    push = sorted((r[0] - base) / 1e3 for r in rs if r[0] > 0)
    pop = sorted((r[1] - base) / 1e3 for r in rs)
    we = sorted((r[2] - base) / 1e3 for r in rs)
    ee = sorted((r[4] - base) / 1e3 for r in rs)
    ex = sorted((r[4] - r[2]) / 1e3 for r in rs)
    print(f"{calls[c]:10s} n={len(rs):4d} push[{push[0] if push else 0:7.2f}..{push[-1] if push else 0:7.2f}] "
          f"pop[{pop[0]:7.2f}..{pop[-1]:7.2f}] waitend[{we[0]:7.2f}..{we[-1]:7.2f}] end[{ee[0]:7.2f}..{ee[-1]:7.2f}] "
          f"exec med {statistics.median(ex):5.2f}")
